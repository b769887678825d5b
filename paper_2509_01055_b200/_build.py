"""Build the C-ABI library `libtoolloop_b200.so` in-tree with nvcc (sm_100a).

Each csrc/*.cu is compiled to an object in parallel (cached by mtime against
the sources and headers), then linked with the static CUDA runtime.  The
library has no torch dependency: it is the drop-in boundary, and Python binds
it with ctypes (paper_2509_01055_b200/_lib.py).
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_objs"
LIB = PKG / "libtoolloop_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", "-Xptxas", "-v"]
if os.environ.get("TL_GEMM_STATS") == "1":  # profiling build: GEMM stall counters
    FLAGS.append("-DTL_GEMM_STATS=1")
if os.environ.get("TL_STAGES256"):  # tuning build: smem ring depth of 256-wide tiles
    FLAGS.append(f"-DTL_STAGES256={int(os.environ['TL_STAGES256'])}")
FLAGS += os.environ.get("TL_EXTRA_NVCC_FLAGS", "").split()  # A/B builds on the GPU box


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted((ROOT / "include").glob("*.h"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, verbose: bool, build_dir: Path = BUILD, extra=()) -> Path:
    obj = build_dir / (src.stem + ".o")
    deps = [src] + _headers()
    if not _stale(obj, deps):
        return obj
    if src.suffix == ".cpp":  # host-only C++ (ingest)
        cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++17", "-fPIC", "-pthread", "-Wall",
               f"-I{ROOT / 'include'}", "-c", str(src), "-o", str(obj)]
    else:
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    (build_dir / (src.stem + ".ptxas.txt")).write_text(res.stderr)
    if verbose:
        print(f"[build] {src.name}", file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = True, variant: str | None = None,
          extra_flags=()) -> Path:
    """Build the library.  variant="name" + extra_flags: an A/B build of the
    same sources into _objs/<name>/libtoolloop_b200.so (selected at run time
    with TOOLLOOP_B200_LIB=<path>); the product library is untouched."""
    build_dir = BUILD / variant if variant else BUILD
    lib = build_dir / LIB.name if variant else LIB
    build_dir.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    if force:
        for o in build_dir.glob("*.o"):
            o.unlink()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, build_dir, tuple(extra_flags)), srcs))
    if force or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs),
               "-lpthread", "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
        if verbose:
            print(f"[build] linked {lib}", file=sys.stderr)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv)
