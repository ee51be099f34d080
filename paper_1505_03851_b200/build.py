"""Build the in-tree CUDA library libwarpdraw_b200.so for sm_100a.

    python -m paper_1505_03851_b200.build [--force] [--ptxas-verbose]

The .so lands in paper_1505_03851_b200/_lib/ (git-ignored, but it travels to
the GPU box with the gpurun snapshot).  Flags: no fast-math, no FMA
contraction (-fmad=false), so the kernels keep the reference's IEEE
operations bit for bit.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.environ.get("WD_LIB_OUT") or os.path.join(OUT_DIR, "libwarpdraw_b200.so")
SOURCES = ["wd_draw_f32.cu", "wd_draw_f64.cu", "wd_capi.cu", "wd_resample.cu", "wd_stream.cu", "wd_probe.cu",
           "wd_table.cu", "wd_mixed.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# sources whose results are statistical (device resample, log-likelihood)
STATISTICAL_SOURCES = {"wd_resample.cu"}


HOST_SRC = os.path.join(CSRC, "wd_host.c")
IO_SRC = os.path.join(CSRC, "wd_io.c")
IO_LIB = os.path.join(OUT_DIR, "libwdio.so")


def build_io(force: bool = False) -> str:
    """libwdio.so: the native corpus / stop-file parsers and CSV writers
    (csrc/wd_io.c, plain C over pthreads, loaded with ctypes by corpus_io)."""
    if not force and os.path.exists(IO_LIB) and os.path.getmtime(IO_LIB) >= os.path.getmtime(IO_SRC):
        return IO_LIB
    cc = os.environ.get("CC") or shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        raise RuntimeError("no C compiler for libwdio")
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = IO_LIB + ".tmp"
    # no fast-math: strtod / printf must stay correctly rounded
    cmd = [cc, "-O2", "-shared", "-fPIC", "-std=c11", "-Wall", "-pthread", IO_SRC, "-o", tmp, "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"libwdio build failed:\n{r.stderr}")
    os.replace(tmp, IO_LIB)
    return IO_LIB


def host_ext_path() -> str:
    import sysconfig

    return os.path.join(PKG, "_wdhost" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_host(force: bool = False) -> str:
    """The CPython host helper (_wdhost: ragged <-> CSR loops of the drop-in
    boundary), compiled with the system C compiler against this interpreter's
    and numpy's headers."""
    import sysconfig

    import numpy as np

    out = host_ext_path()
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(HOST_SRC):
        return out
    cc = os.environ.get("CC") or shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        raise RuntimeError("no C compiler for the host helper")
    tmp = out + ".tmp"
    cmd = [cc, "-O2", "-shared", "-fPIC", "-std=gnu11", "-Wall", "-pthread", f"-I{sysconfig.get_paths()['include']}",
           f"-I{np.get_include()}", HOST_SRC, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"host helper build failed:\n{r.stderr}")
    os.replace(tmp, out)
    return out


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _flags(ptxas_verbose: bool):
    f = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC,-O2",
         f"-I{INCLUDE}", f"-I{CSRC}", "--expt-relaxed-constexpr"]
    if ptxas_verbose:
        f += ["-Xptxas", "-v"]
    f += os.environ.get("WD_EXTRA_FLAGS", "").split()  # experiments only
    return f


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f not in ("wd_host.c", "wd_io.c")] + \
        [os.path.join(INCLUDE, "warpdraw_b200.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, ptxas_verbose: bool = False, verbose: bool = True) -> str:
    build_host(force)
    build_io(force)
    if not force and up_to_date():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    obj_dir = os.path.join(os.path.dirname(LIB), "obj_" + os.path.basename(LIB).replace(".so", ""))
    os.makedirs(obj_dir, exist_ok=True)
    cc = nvcc()
    flags = _flags(ptxas_verbose)

    def compile_one(src):
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        f = list(flags)
        if src in STATISTICAL_SOURCES:  # no bitwise contract: FMA contraction, flush-to-zero
            f[f.index("-fmad=false")] = "-fmad=true"
            f.append("-ftz=true")
        cmd = [cc, *f, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for _, log in results:
        if verbose and log.strip():
            print(log, file=sys.stderr)
    tmp = LIB + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *[o for o, _ in results]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--ptxas-verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, ptxas_verbose=a.ptxas_verbose))
