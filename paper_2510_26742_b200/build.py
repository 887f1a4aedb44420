"""In-tree build of libpi0b.so (sm_100a) with nvcc; no JIT cache, so the built library
travels with the repository snapshot to the GPU box."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libpi0b.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr"] + os.environ.get("PI0B_NVCC_EXTRA", "").split()
SOURCES = ["gemm.cu", "skinny.cu", "fattn.cu", "aemk.cu", "kernels_misc.cu", "engine.cu", "capi.cu", "naive.cu"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, lib: str = LIB, defines: list[str] | None = None) -> str:
    """Build `lib` (default libpi0b.so); `defines` (-DNAME=V) select an experimental variant,
    built in its own object directory."""
    obj = OBJ if not defines else OBJ + "_" + os.path.basename(lib).replace(".so", "")
    os.makedirs(obj, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(os.path.dirname(PKG), "include", "pi0b.h"))
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj, src.replace(".cu", ".o"))
        if force or _newer(o, [s] + headers):
            jobs.append([NVCC, *ARCH, *FLAGS, *(defines or []), "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose:
            sys.stdout.write(r.stdout + r.stderr)

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(obj, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _newer(lib, objs):
        run([NVCC, *ARCH, "-shared", "-o", lib, *objs])
    return lib


if __name__ == "__main__":
    # python build.py [-v] [-f] [out.so -DNAME=V ...]
    args = [a for a in sys.argv[1:] if a not in ("-v", "-f")]
    if args:
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, lib=os.path.abspath(args[0]), defines=args[1:]))
    else:
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
