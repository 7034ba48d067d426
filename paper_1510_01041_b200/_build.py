"""Build the sm_100a C-ABI library in-tree (``_lib/liblmsb200.so``).

nvcc cross-compiles for B200 without a GPU; the resulting ``.so`` travels to
the GPU box with the repo snapshot.  The library links the CUDA runtime
statically, so loading it needs only the driver.
"""

from __future__ import annotations

import os
import shutil
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_DIR = os.path.join(PKG_DIR, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "liblmsb200.so")

SOURCES = ["lms_engine.cu", "lms_band.cu", "lms_sweep.cu", "lms_segsort.cu", "lms_samplesort.cu", "lms_nccl.cu", "lms_detect.cu", "lms_sets.cu", "lms_band_small.cu", "lms_exact.cu", "lms_filter32m.cu", "lms_order.cu", "lms_plan.cu",
           "lms_hough.cu", "lms_primal.cu", "lms_probe.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build the engine")
    return cand


def build(verbose: bool = False, extra: list[str] | None = None, out: str | None = None) -> str:
    out = out or LIB_PATH
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objs = []
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp",
              "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]
    if verbose:
        common += ["-Xptxas", "-v"]
    if extra:
        common += extra
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src: str) -> str:
        obj = os.path.join(os.path.dirname(out), src.replace(".cu", ".o"))
        subprocess.run([*common, "-c", os.path.join(CSRC, src), "-o", obj], check=True)
        return obj

    objs = [os.path.join(os.path.dirname(out), s.replace(".cu", ".o")) for s in SOURCES]
    try:
        with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as pool:
            list(pool.map(compile_one, SOURCES))
        tmp = out + ".tmp"
        # --no-undefined: a symbol missing from the objects fails the link here
        # instead of the load on the GPU box
        subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-lgomp", "-ldl",
                        "-Xlinker", "--no-undefined"], check=True)
        os.replace(tmp, out)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return out


if __name__ == "__main__":
    import sys

    print(build(verbose="-v" in sys.argv))
