"""Build libtsf.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2604_16590_b200.build [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libtsf.so")
SOURCES = [os.path.join(HERE, "csrc", "tsf.cu")]
HEADERS = [os.path.join(HERE, "csrc", f) for f in ("sm100.cuh", "attn_common.cuh", "attn_packed.cuh",
                                                   "attn_flash.cuh", "layout.cuh", "attn_stream.cuh", "attn_smallt.cuh", "attn_flash3.cuh", "gemm.cuh", "attn_bwd.cuh")] + \
    [os.path.join(ROOT, "include", "tsf.h")]


def nccl_paths():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl-cu12 wheel (nccl.h, libnccl.so.2) not found")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(verbose: bool = False, force: bool = False, trace: bool = False) -> str:
    """trace=True builds libtsf_trace.so with -DTSF_TRACE (clock64 stamps, diagnostics)."""
    out = LIB.replace("libtsf.so", "libtsf_trace.so") if trace else LIB
    if not force and not trace and not needs_build():
        return LIB
    inc, lib = nccl_paths()
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2", "-shared", "-cudart", "shared",
           "-I", os.path.join(ROOT, "include"), "-I", inc,
           *(["-DTSF_TRACE"] if trace else []),
           "-o", out + ".tmp", *SOURCES,
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(r.stdout, r.stderr, flush=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True, trace="--trace" in sys.argv))
