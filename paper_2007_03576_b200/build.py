"""Build libhqr_b200.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with gpurun)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhqr_b200.so")
SOURCES = ["hqr_api.cu", "chase.cu", "update.cu", "step.cu", "qz.cu", "qriter.cu"]
HEADERS = ["plan.hpp", "kernels.hpp", "dist.hpp", "device_common.cuh", "gemm_tile.cuh", "step.hpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "hqr.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def nccl_dirs():
    """NCCL headers / library bundled with the image's torch (nvidia-nccl wheel)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("NCCL (nvidia.nccl) not found: the multi-GPU path needs it")
    root = list(spec.submodule_search_locations)[0]
    return os.path.join(root, "include"), os.path.join(root, "lib")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    inc, lib = nccl_dirs()
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-cudart", "shared", "--expt-relaxed-constexpr",
           "-I", inc, "-o", LIB] + os.environ.get("HQR_NVCC_EXTRA", "").split() + [os.path.join(CSRC, f) for f in SOURCES] + [
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
