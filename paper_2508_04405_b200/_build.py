"""Build recipe for libflexq_sm100a.so (in-tree, sm_100a only).

    python -m paper_2508_04405_b200._build        # or __graft_entry__.build()

The library is a plain C-ABI shared object (include/flexq.h) compiled with
nvcc for `-gencode arch=compute_100a,code=sm_100a`; CUDA runtime linked
statically so the .so only needs the driver on the GPU box.
"""
from __future__ import annotations

import concurrent.futures
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libflexq_sm100a.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=default",
    "-Xptxas", "-v",
    "-cudart", "static",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the sm_100a library cannot be built")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_rebuild() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "flexq.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, obj: str) -> subprocess.CompletedProcess:
    return subprocess.run([nvcc(), *NVCC_FLAGS, "-c", "-o", obj, src], capture_output=True,
                          text=True)


def build(verbose: bool = False, force: bool = False) -> str:
    """Compile every csrc/*.cu to an object in parallel (one nvcc per translation unit),
    then link the shared library."""
    if not force and not needs_rebuild():
        return LIB
    obj_dir = os.path.join(OUT_DIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sources()
    objs = [os.path.join(obj_dir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    with concurrent.futures.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(_compile, srcs, objs))
    failed = False
    for src, res in zip(srcs, results):
        if res.returncode != 0:
            sys.stderr.write(f"--- {os.path.basename(src)}\n" + res.stdout + res.stderr)
            failed = True
        elif verbose:
            sys.stderr.write(res.stderr)
    if failed:
        raise RuntimeError("nvcc failed building libflexq_sm100a.so")
    tmp = LIB + ".tmp"
    res = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                          "-cudart", "static", "-o", tmp, *objs], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libflexq_sm100a.so")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
