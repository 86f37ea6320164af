"""Build libnalar.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnalar.so")
SOURCES = ["nalar_ctx.cu", "k_validate.cu", "k_sweep.cu", "k_assign.cu", "k_delta.cu", "k_io.cu", "k_migrate.cu", "k_batch.cu",
           "k_peer.cu", "k1_kernels.cu"]
# k1_kernels.cu holds the nine ~500 KB K1 builds: one object per build
# (-DNALAR_K1_PART=k), all objects compiled in parallel
K1_PARTS = 9
HEADERS = ["internal.h", "k1_body.cuh", "k4_body.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
          f"-I{os.path.join(ROOT, 'include')}"]
OBJDIR = os.path.join(ROOT, "build", "obj")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "nalar.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _units():
    for src in SOURCES:
        if src == "k1_kernels.cu":
            for k in range(K1_PARTS):
                yield src, [f"-DNALAR_K1_PART={k}"], f"k1_kernels_{k}.o"
        else:
            yield src, [], src[:-3] + ".o"


def build_lib(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    jobs = [([NVCC, *ARCH, *CFLAGS, *defs, "-c", os.path.join(CSRC, src), "-o", os.path.join(OBJDIR, obj)], obj)
            for src, defs, obj in _units()]
    workers = max(1, min(len(jobs), os.cpu_count() or 1))
    with concurrent.futures.ThreadPoolExecutor(workers) as ex:
        results = list(ex.map(lambda j: (j[1], subprocess.run(j[0], capture_output=True, text=True)), jobs))
    log = []
    for obj, r in results:
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed building {obj}")
    link = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *[os.path.join(OBJDIR, o) for _, _, o in _units()], "-ldl"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libnalar.so")
    if verbose:
        sys.stderr.write("".join(log))
    os.replace(LIB + ".tmp", LIB)
    return LIB

if __name__ == "__main__":
    build_lib(force="--force" in sys.argv, verbose=True)
    print(LIB)
