"""Build libslq_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

The shared library is a plain C ABI (include/slq_b200.h); Python binds it with ctypes.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libslq_b200.so")
SOURCES = ["capi.cu", "graph.cu", "lanczos.cu", "spmm_f32.cu", "spmm_f64.cu", "spmm_flat.cu", "step_f32_wide.cu", "step_f32_narrow.cu",
           "step_f64_wide.cu", "step_f64_narrow.cu", "rules.cu", "batched.cu", "rmat.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "slq_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit in parallel (nvcc -c), then link the shared library."""
    import concurrent.futures
    import tempfile

    if not force and not needs_build():
        return LIB
    flags = [nvcc(), "-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"),
             *os.environ.get("SLQ_NVCC_FLAGS", "").split()]
    with tempfile.TemporaryDirectory() as tmp:
        objs = [os.path.join(tmp, s.replace(".cu", ".o")) for s in SOURCES]

        def compile_one(k):
            return subprocess.run(flags + ["-c", os.path.join(CSRC, SOURCES[k]), "-o", objs[k]],
                                  capture_output=True, text=True)

        with concurrent.futures.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
            results = list(ex.map(compile_one, range(len(SOURCES))))
        for r in results:
            if r.returncode != 0:
                raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
            if verbose:
                sys.stderr.write(r.stderr)
        r = subprocess.run([nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp"] + objs, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
