"""Builds the in-tree CUDA library liblongflow.so for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "liblongflow.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in
           ("lf_runtime.cu", "lf_decode_simt.cu", "lf_decode_tc.cu", "lf_snapkv.cu", "lf_diag.cu")]
HEADERS = [os.path.join(HERE, "csrc", f) for f in ("lf_internal.h", "lf_tc_ptx.cuh", "lf_common.cuh")] + [
           os.path.join(ROOT, "include", "longflow.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.exists(f) and os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or _stale():
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *FLAGS, "-o", tmp, *SOURCES]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stderr[-6000:]}")
        if verbose:
            print(r.stderr)
        os.replace(tmp, LIB)
    return LIB


def build_variant(out: str, defines=()) -> str:
    """Debug builds (e.g. -DLF_TRACE) to a separate path, loaded with LF_LIB=<out>."""
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stderr[-6000:]}")
    return out


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
