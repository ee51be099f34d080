"""Structural checks on the built sm_100a code, the B200 counterpart of the
reference's coalescing/op-count acceptance criterion (tests/test_acceptance.py:212-267
of the reference: butterfly table build free of scattered local-memory
traffic).  Runs on CPU: it inspects the cubin inside the built library.

* the headline kernels (LDA draw, fine variant; standalone rows, cp.async
  ring) use no local memory at all (no spills, no stack, no LDL/STL);
* their block loops use 128-bit vector loads and the shuffle butterfly
  (SHFL.BFLY), never the per-lane table of the prefix baseline.
"""

import os
import re
import shutil
import subprocess

import pytest

from paper_1505_03851_b200 import _lib

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
HOT = {
    "lda_fine": "_ZN2wd11bfly_kernelIfLi32ELb1ELi0ELi1ELi0EEEvNS_10DrawParamsIT_EE",
    "rows_ring": "_ZN2wd11bfly_kernelIfLi32ELb1ELi1ELi5ELi0EEEvNS_10DrawParamsIT_EE",
}


def _need():
    if not os.path.exists(CUOBJDUMP):
        pytest.skip("cuobjdump not available")
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")


def test_hot_kernels_use_no_local_memory():
    _need()
    out = subprocess.run([CUOBJDUMP, "--dump-resource-usage", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for tag, sym in HOT.items():
        m = re.search(re.escape(sym) + r":\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:\d+ LOCAL:(\d+)", out)
        assert m, f"{tag}: {sym} not found in the library"
        reg, stack, local = map(int, m.groups())
        assert stack == 0 and local == 0, f"{tag}: stack {stack} local {local}"
        assert reg <= 128, f"{tag}: {reg} registers"


@pytest.mark.parametrize("tag", sorted(HOT))
def test_hot_kernels_vector_loads_and_shuffle_butterfly(tag):
    _need()
    sass = subprocess.run([CUOBJDUMP, "-sass", "-fun", HOT[tag], _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "Function" in sass
    assert not re.search(r"\b(LDL|STL)\b", sass), f"{tag}: local memory traffic"
    assert "LDG.E.128" in sass or "LDGSTS.E.BYPASS.128" in sass, f"{tag}: no 128-bit loads"
    assert sass.count("SHFL.BFLY") >= 7, f"{tag}: no shuffle butterfly"
