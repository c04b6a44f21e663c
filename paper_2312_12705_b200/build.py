"""Builds the in-tree native library ``lib/libtrainplan_b200.so`` with nvcc for sm_100a.

The library holds every CUDA kernel (K1-K12), the C++ host runtime (train step, 1F1B
executor, NCCL communicators) and the C-ABI declared in ``include/trainplan/capi.h``.
Incremental: an object is rebuilt when its source or any header under ``csrc``/``include``
is newer than it.
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
BUILD = PKG / "build"
LIB = PKG / "lib" / "libtrainplan_b200.so"
# Debug variant (experiments only; loaded with GPTB200_LIB=<path>): GPTB200_NVCC_EXTRA="-DGPTB200_DEBUG_HANG"
# turns every mbarrier wait of the attention kernels into a bounded wait that prints the stuck
# barrier and traps instead of hanging.
_EXTRA = os.environ.get("GPTB200_NVCC_EXTRA", "").split()
if _EXTRA:
    _DBG = os.environ.get("GPTB200_DEBUG_DIR", "lib_debug")
    BUILD = PKG / f"build_{_DBG}"
    LIB = PKG / _DBG / "libtrainplan_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp",
          f"-I{ROOT / 'include'}", f"-I{CSRC}", "-I/usr/local/cuda/include"]
# NCCL: link the libnccl.so.2 that the image's PyTorch bundles (rpath'd), so a process that loads
# both this library and torch — in either order — holds exactly one NCCL (same SONAME).
# Fallback: the system libnccl.so.2.
_TORCH_NCCL = Path(sys.prefix) / "lib" / f"python{sys.version_info.major}.{sys.version_info.minor}" / \
    "site-packages" / "nvidia" / "nccl" / "lib"
NCCL_DIR = _TORCH_NCCL if (_TORCH_NCCL / "libnccl.so.2").exists() else Path("/usr/lib/x86_64-linux-gnu")
# headers of the same NCCL (2.28: symmetric windows + device API used by the NVLS TP kernels)
if (NCCL_DIR.parent / "include" / "nccl_device.h").exists():
    COMMON.insert(COMMON.index("-I/usr/local/cuda/include"), f"-I{NCCL_DIR.parent / 'include'}")
LINK = ["-shared", "-lcudart", f"-L{NCCL_DIR}", "-l:libnccl.so.2", "-lgomp",
        "-Xlinker", f"-rpath={NCCL_DIR}", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]


def _sources() -> list[Path]:
    return sorted(p for p in CSRC.rglob("*") if p.suffix in (".cu", ".cpp"))


def _headers_mtime() -> float:
    hs = [p for d in (CSRC, ROOT / "include") for p in d.rglob("*") if p.suffix in (".h", ".cuh", ".hpp")]
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, hdr_mtime: float) -> Path:
    obj = BUILD / (src.relative_to(CSRC).as_posix().replace("/", "__") + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, *_EXTRA, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cpp":
        cmd[1:1] = ["-x", "cu"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    LIB.parent.mkdir(exist_ok=True)
    hdr = _headers_mtime()
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [NVCC, *ARCH, *[str(o) for o in objs], "-o", str(LIB), *LINK]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
