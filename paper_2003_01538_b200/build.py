"""Build the native library (sm_100a) in-tree: paper_2003_01538_b200/libensemble_b200.so.

Plain nvcc, no torch extension machinery: the library exposes only the C ABI in
include/ensemble_b200.h and is loaded with ctypes.  The CUDA runtime is linked
statically so the .so has no runtime-library search dependencies on the GPU box.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libensemble_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I", str(ROOT / "include"), "-I", str(CSRC)]

# EB_BUILD_TRACE=1: build the EB_TRACE timing probes into a separate library
# (tools/_ab/libtrace.so, loaded with EB_LIB_PATH); the production build has none.
if os.environ.get("EB_BUILD_TRACE"):
    FLAGS = FLAGS + ["-DEB_ENABLE_TRACE"]
    BUILD = ROOT / "build_trace"
    LIB = ROOT / "tools" / "_ab" / "libtrace.so"

SOURCES = ["conv_umma.cu", "block1.cu", "stem_pool.cu", "pointwise.cu", "combine.cu", "ref32.cu", "runtime.cu", "tmap.cpp",
           "wire_decode.cpp"]


def _needs(obj: Path, deps) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, verbose: bool) -> Path:
    obj = BUILD / (src.name + ".o")
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    if not _needs(obj, [src] + headers):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    if src.suffix == ".cpp":
        cmd = [NVCC, *FLAGS, "-x", "cu", *ARCH, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    LIB.parent.mkdir(exist_ok=True)
    srcs = [CSRC / s for s in SOURCES]
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if _needs(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
