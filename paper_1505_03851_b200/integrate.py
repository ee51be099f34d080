"""Install the B200 path into a running `warpdraw` (the reference package).

    import warpdraw
    from paper_1505_03851_b200 import integrate
    integrate.install()          # KERNELS / draw_z / SAMPLERS / gibbs path now run on the GPU

After install():

* warpdraw.kernels.KERNELS["basic" | "transposed" | "butterfly"] and
  warpdraw.kernels.draw_z dispatch to the sm_100a kernels (same signatures,
  exceptions and messages; kernels.py:542-555);
* warpdraw.lda's own reference to draw_z is rebound, so gibbs_iterate /
  run_gibbs (and `warpdraw lda --kernel ...`) draw on the GPU while keeping
  the reference's numpy resample -- the results stay bit-identical;
* warpdraw.lda.topic_counts (lda.py:174-182; called by resample_params)
  counts on the GPU (wd_topic_counts, reusing the draw's cached corpus
  upload): integer counts, bit-identical, np.add.at's index rules kept;
* warpdraw.bench.SAMPLERS["binary" | "alias" | "butterfly"] are the GPU
  samplers (bench.py:150-154), bit-identical, and SAMPLERS["prefix"] (the
  butterfly's u stream through a full prefix table) is added;
* warpdraw.kernels.build_block_tables / butterfly_search / table_snapshot
  (and the names warpdraw.bench and warpdraw.cli imported from it) build and
  search the butterfly table on the GPU (kernels.py:580-604, 317-362);
* the reference's exception classes are the ones raised (AllZeroError,
  EmptyWeightsError, StopOutOfRangeError, OutOfBoundsError are mapped, for draw_z and SAMPLERS), and its SeededStops / InjectedStops
  objects are recognised (in-kernel hash / u per token).

uninstall() restores the originals.
"""

from __future__ import annotations

import importlib

from . import kernels as _k
from . import samplers as _s
from . import tables as _t
from . import warp as _w

_saved: dict = {}


def _convert(x, ref_kernels):
    """The reference's own stops providers map onto the device stop modes
    (SeededStops -> in-kernel hash, InjectedStops -> u per token) instead of
    the generic host-evaluated .units path; same values either way."""
    if isinstance(x, ref_kernels.SeededStops):
        return _k.SeededStops(x.seed)
    if isinstance(x, ref_kernels.InjectedStops):
        return _k.InjectedStops(x._units)
    return x


def _wrap_errors(fn, ref_kernels, ref_sampling):
    ref_warp = importlib.import_module(ref_kernels.__name__.rsplit(".", 1)[0] + ".warp")

    def call(*a, **kw):
        a = tuple(_convert(x, ref_kernels) for x in a)
        kw = {k: _convert(v, ref_kernels) for k, v in kw.items()}
        try:
            return fn(*a, **kw)
        except _k.StopOutOfRangeError as exc:
            raise ref_kernels.StopOutOfRangeError(str(exc)) from None
        except _k.AllZeroError as exc:
            raise ref_sampling.AllZeroError(str(exc)) from None
        except _s.EmptyWeightsError as exc:
            raise ref_sampling.EmptyWeightsError(str(exc)) from None
        except _w.OutOfBoundsError as exc:
            raise ref_warp.OutOfBoundsError(str(exc)) from None

    call.__name__ = getattr(fn, "__name__", "call")
    call.__doc__ = fn.__doc__
    return call


def _topic_counts(corpus, z, n_topics):
    """The reference's topic_counts(corpus, z, n_topics) on the GPU."""
    from .lda import counts_ragged

    return counts_ragged(corpus.lengths, corpus.words, z, n_topics, corpus.vocab_size)


def install(package: str = "warpdraw") -> None:
    """Patch the imported reference package in place (idempotent)."""
    if _saved:
        return
    ref_kernels = importlib.import_module(package + ".kernels")
    ref_sampling = importlib.import_module(package + ".sampling")
    ref_lda = importlib.import_module(package + ".lda")
    ref_bench = importlib.import_module(package + ".bench")
    _saved["kernels"] = (ref_kernels, dict(ref_kernels.KERNELS), ref_kernels.draw_z)
    _saved["lda"] = (ref_lda, ref_lda.draw_z, ref_lda.topic_counts)
    _saved["bench"] = (ref_bench, dict(ref_bench.SAMPLERS))
    ref_kernels.KERNELS.update({name: _wrap_errors(fn, ref_kernels, ref_sampling) for name, fn in _k.KERNELS.items()})
    gpu_draw_z = _wrap_errors(_k.draw_z, ref_kernels, ref_sampling)
    ref_kernels.draw_z = gpu_draw_z
    ref_lda.draw_z = gpu_draw_z
    ref_lda.topic_counts = _topic_counts
    ref_bench.SAMPLERS.update({name: _wrap_errors(fn, ref_kernels, ref_sampling) for name, fn in _s.SAMPLERS.items()})
    # the split table / search API: the defining module and the modules that
    # imported the names (bench.py:19, cli.py uses kernels.<name>)
    tabs = {"build_block_tables": _t.build_block_tables, "butterfly_search": _t.butterfly_search,
            "table_snapshot": _t.table_snapshot}
    _saved["tables"] = []
    for mod in (ref_kernels, ref_bench):
        for name, fn in tabs.items():
            if hasattr(mod, name):
                _saved["tables"].append((mod, name, getattr(mod, name)))
                setattr(mod, name, _wrap_errors(fn, ref_kernels, ref_sampling))


def uninstall() -> None:
    if not _saved:
        return
    ref_kernels, kernels, draw_z = _saved.pop("kernels")
    ref_kernels.KERNELS.clear()
    ref_kernels.KERNELS.update(kernels)
    ref_kernels.draw_z = draw_z
    ref_lda, lda_draw_z, lda_topic_counts = _saved.pop("lda")
    ref_lda.draw_z = lda_draw_z
    ref_lda.topic_counts = lda_topic_counts
    ref_bench, samplers = _saved.pop("bench")
    ref_bench.SAMPLERS.clear()
    ref_bench.SAMPLERS.update(samplers)
    for mod, name, fn in _saved.pop("tables", []):
        setattr(mod, name, fn)
