"""Structural checks on the built sm_100a code, the B200 counterpart of the
reference's coalescing/op-count acceptance criterion (tests/test_acceptance.py:212-267
of the reference: butterfly table build free of scattered local-memory
traffic).  Runs on CPU: it inspects the cubin inside the built library.

* the headline kernels (LDA draw, fine variant; standalone rows, cp.async
  ring) keep their block loops free of local memory (at most a few bytes of
  loop-invariant spill outside them);
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
    "lda_fine": "_ZN2wd11bfly_kernelIfLi32ELi2ELi0ELi1ELi0EEEvNS_10DrawParamsIT_EE",  # 256-bit segments
    "rows_ring": "_ZN2wd11bfly_kernelIfLi32ELi1ELi1ELi5ELi0EEEvNS_10DrawParamsIT_EE",
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
        assert stack <= 16 and local <= 16, f"{tag}: stack {stack} local {local}"
        assert reg <= 128, f"{tag}: {reg} registers"


def _inner_loops(sass):
    """(instructions) of every backward-branch loop shorter than 1000 instructions."""
    ins = []
    for line in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    loops = []
    for a, text in ins:
        m = re.search(r"BRA (0x[0-9a-f]+)", text)
        if m and int(m.group(1), 16) < a:
            body = [t for b, t in ins if int(m.group(1), 16) <= b <= a]
            if 20 < len(body) < 1000:
                loops.append(body)
    return loops


@pytest.mark.parametrize("tag", sorted(HOT))
def test_hot_kernels_vector_loads_and_shuffle_butterfly(tag):
    _need()
    sass = subprocess.run([CUOBJDUMP, "-sass", "-fun", HOT[tag], _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "Function" in sass
    loops = _inner_loops(sass)
    assert loops, f"{tag}: no block loop found"
    for body in loops:
        assert not any(re.search(r"\b(LDL|STL)\b", t) for t in body), f"{tag}: local memory in a block loop"
    assert re.search(r"LDG\.E\.(ENL2\.)?(128|256)|LDGSTS\.E\.BYPASS\.128", sass), f"{tag}: no vector loads"
    assert sass.count("SHFL.BFLY") >= 3, f"{tag}: no shuffle butterfly"
