"""Build the sm_100a shared library libnsf_mpm.so in-tree with nvcc.

    python -m paper_2310_17790_b200.build [--force]

Every .cu under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -Xptxas -v
and linked into paper_2310_17790_b200/libnsf_mpm.so (C ABI: include/nsf_mpm.h).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# NSF_BUILD_DIR / NSF_LIB_OUT: experiment variants built side by side (tools/ab_build.sh)
BUILD = os.environ.get("NSF_BUILD_DIR") or os.path.join(PKG, "_build")
LIB = os.environ.get("NSF_LIB_OUT") or os.path.join(PKG, "libnsf_mpm.so")
LIB_CHECKED = os.path.join(PKG, "libnsf_mpm_checked.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                     "--expt-relaxed-constexpr", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]
# tuning knobs for experiments, e.g. NSF_DEFINES="NSF_P2G_ROWS=8 NSF_FUSED_MIN_BLOCKS=4"
NVCC_FLAGS += [f"-D{d}" for d in os.environ.get("NSF_DEFINES", "").split()]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + [os.path.join(ROOT, "include", "nsf_mpm.h")])


def _compile(src: str, force: bool, log: list) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    newest_dep = max([os.path.getmtime(d) for d in _deps()] + [os.path.getmtime(src)])
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [nvcc(), *NVCC_FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.append((src, r.stdout + r.stderr))
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """checked=True: the bounds-checked variant libnsf_mpm_checked.so (-DNSF_CHECKED=1,
    csrc/params.cuh NSF_CHECK), used by tests/test_gpu_checked.py only."""
    global BUILD, LIB, NVCC_FLAGS
    if checked:
        saved = (BUILD, LIB, NVCC_FLAGS)
        BUILD, LIB = BUILD + "_checked", LIB_CHECKED
        NVCC_FLAGS = NVCC_FLAGS + ["-DNSF_CHECKED=1"]
        try:
            return build(force, verbose)
        finally:
            BUILD, LIB, NVCC_FLAGS = saved
    os.makedirs(BUILD, exist_ok=True)
    stamp = os.path.join(BUILD, "flags.txt")     # a change of flags (NSF_DEFINES) forces a rebuild
    flags = " ".join(NVCC_FLAGS)
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True
        if os.path.exists(stamp):
            os.remove(stamp)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    log: list = []
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, log), srcs))   # raises on any nvcc error
    if force or not os.path.exists(LIB) or max(os.path.getmtime(o) for o in objs) > os.path.getmtime(LIB):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    with open(stamp, "w") as f:
        f.write(flags)
    with open(os.path.join(BUILD, "ptxas.log"), "w" if log else "a") as f:
        for src, out in log:
            f.write(f"==== {src}\n{out}\n")
    if verbose:
        for src, out in log:
            print(f"==== {src}\n{out}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
