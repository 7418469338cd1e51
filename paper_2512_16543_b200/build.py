"""Build the sm_100a library in-tree: paper_2512_16543_b200/_lib/libleorzf_b200.so.

    python -m paper_2512_16543_b200.build [--force]

nvcc cross-compiles without a GPU.  The .so is git-ignored but travels to
the GPU box with the gpurun snapshot (it is not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libleorzf_b200.so"
HEADER = PKG.parent / "include" / "leorzf_b200.h"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = sources() + sorted(CSRC.glob("*.cuh")) + [HEADER]
    return any(p.stat().st_mtime > t for p in deps)


GEN = CSRC / "_gen" / "ziggurat_tables.h"


def build(force: bool = False, verbose: bool = True) -> Path:
    if not GEN.exists():
        # numpy's ziggurat tables, read from the installed numpy (rng/tables.py)
        from .rng import tables
        tables.write_header(GEN)
    if not force and not _stale():
        return LIB
    OUT_DIR.mkdir(exist_ok=True)
    obj_dir = OUT_DIR / "obj"
    obj_dir.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    # one nvcc per translation unit, in parallel (no relocatable device code:
    # every .cu is self-contained), then one link
    cflags = [f for f in FLAGS if f != "-shared"]

    def compile_one(src: Path) -> Path:
        obj = obj_dir / (src.stem + ".o")
        cmd = [_nvcc(), *ARCH, *cflags, "-I", str(PKG.parent / "include"), "-c", str(src),
               "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(sources()), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    cmd = [_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(tmp),
           *map(str, objs), "-lcudart"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    tmp.replace(LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
