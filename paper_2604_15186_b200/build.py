"""Build the in-tree C-ABI library libscepsy_alp.so for sm_100a (nvcc; no torch JIT cache).

    python -m paper_2604_15186_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libscepsy_alp.so")
SOURCES = ["alp_api.cu", "alp_kernels.cu", "alp_search_t8.cu", "alp_search_t12.cu", "alp_search_t16.cu",
           "alp_search_u.cu", "alp_levels.cu"]
# every file under csrc/ (sources and headers) plus the public header is a dependency
HEADERS = [os.path.join("..", "..", "include", "alp.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# IEEE semantics: no fast-math, no FTZ; explicit __d*_rn intrinsics in the FP64 option terms.
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-ftz=false", "-prec-div=true",
         "-prec-sqrt=true", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in os.listdir(CSRC)] + [os.path.join(CSRC, h) for h in HEADERS]
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: tuple = (),
          extra: tuple = ()) -> str:
    """Build the library (out/defines/extra: tuning variants, e.g. defines=("ALP_A_UNROLL=2",),
    extra=("-Xptxas", "-O2"))."""
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)

    def compile_one(src):
        obj = os.path.join(os.path.dirname(lib), src.replace(".cu", ".o") if out is None else
                           os.path.basename(lib) + "." + src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *extra, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {src}")
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with concurrent.futures.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
