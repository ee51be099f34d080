"""paper_1505_03851_b200 -- B200-native (sm_100a) butterfly sampler and LDA z-step.

Drop-in for the hot path of the reference package `warpdraw`
(arXiv 1505.03851, Steele & Tristan): the kernel registry (KERNELS, draw_z),
the stop providers, the standalone SAMPLERS and the uncollapsed-LDA driver
keep the reference's names and signatures; the draws run in hand-written CUDA
kernels behind the C ABI in include/warpdraw_b200.h.
"""

from .kernels import (
    KERNELS,
    DeviceCorpus,
    InjectedStops,
    PhiloxStops,
    SeededStops,
    StopOutOfRangeError,
    draw_z,
    draw_z_basic,
    draw_z_butterfly,
    draw_z_device,
    draw_z_transposed,
)
from .lda import (
    Corpus,
    CorpusParseError,
    ModelParams,
    WordIdOutOfRangeError,
    gibbs_iterate,
    init_assignments,
    load_corpus,
    load_corpus_npz,
    log_likelihood,
    modal_topics,
    resample_params,
    run_gibbs,
    save_corpus,
    save_corpus_npz,
    topic_counts,
)
from .rng import derive_seed, mix64, unit_for, units_for
from .samplers import (
    SAMPLERS,
    alias_table,
    chi_square,
    chi_square_critical,
    sample_alias,
    sample_binary,
    sample_butterfly,
    sample_prefix,
    sample_rows,
)
from .sampling import AllZeroError, EmptyWeightsError
from .tables import ButterflyTable, build_block_tables, butterfly_search, table_snapshot
from .warp import OutOfBoundsError, Trace, WarpConfig

__version__ = "0.1.0"
