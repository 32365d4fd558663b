"""In-tree build of libpec.so (sm_100a kernels + host CRC) with nvcc.

The shared object lands in ``paper_2408_04307_b200/_lib/`` so that it travels
to the GPU box with the repo snapshot (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB_PATH = LIB_DIR / "libpec.so"
DEBUG_LIB_PATH = LIB_DIR / "libpec_debug.so"
SOURCES = [CSRC / "pec_kernels.cu", CSRC / "pec_crc.cu", CSRC / "pec_host.cpp"]
HEADERS = [ROOT / "include" / "pec.h", CSRC / "pec_device.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-pthread",
    "-Xptxas", "-v",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    return any(p.stat().st_mtime > built for p in SOURCES + HEADERS)


def _compile(out: Path, extra=(), log: str = "ptxas.log", verbose: bool = False) -> Path:
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    tmp = out.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-I", str(CSRC),
           *map(str, SOURCES), "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}) building {out}")
    if verbose:
        sys.stderr.write(res.stderr)
    (LIB_DIR / log).write_text(res.stderr)
    os.replace(tmp, out)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB_PATH
    return _compile(LIB_PATH, verbose=verbose)


def build_debug(force: bool = False) -> Path:
    """libpec_debug.so: the same sources with the device-side invariant
    checks (PEC_DCHECK) compiled in; selected with PEC_LIB=debug.  Test
    tooling only (tools/guard_kernels.py)."""
    if not force and DEBUG_LIB_PATH.exists() and \
            DEBUG_LIB_PATH.stat().st_mtime > max(p.stat().st_mtime for p in SOURCES + HEADERS):
        return DEBUG_LIB_PATH
    return _compile(DEBUG_LIB_PATH, extra=("-DPEC_DEBUG",), log="ptxas_debug.log")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
