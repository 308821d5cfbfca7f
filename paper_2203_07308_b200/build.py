"""Build libms2g.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

NCCL headers and library come from the torch-bundled nvidia-nccl wheel; the
library path is baked in with an rpath so the same .so loads on the GPU box.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libms2g.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl as nn
    base = list(nn.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "ms2g.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Build libms2g.so (or, for kernel-variant experiments, `out` with extra -D defines)."""
    target = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    inc, lib = nccl_dirs()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
           "-Xptxas", "-v" if verbose else "-O3",
           *[f"-D{d}" for d in defines],
           f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}", *sources(),
           f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}", "-o", target + ".tmp"]
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    # --debug: device bounds checks (MS2G_DASSERT) into the default library path
    print(build(force=True, verbose="-v" in sys.argv, defines=("MS2G_DEBUG=1",) if "--debug" in sys.argv else ()))
