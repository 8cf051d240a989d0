"""Build libogm_b200.so in-tree with nvcc for sm_100a (no JIT cache).

``python -m paper_2209_03526_b200.build`` or ``__graft_entry__.build()``.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libogm_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
         "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{CSRC}"]
SOURCES = [CSRC / "ogm_lib.cu"]


def sources_newer_than_lib() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not sources_newer_than_lib():
        return LIB
    cmd = [NVCC, *ARCH, *FLAGS, "-o", str(LIB), *map(str, SOURCES), "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}) building {LIB.name}")
    if verbose:
        sys.stderr.write(res.stderr)
    (PKG / "ptxas_info.txt").write_text(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
