"""Build libgazecut_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1803_01516_b200.build
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
# gz_solver.cu: host side, C ABI, small kernels; gz_k*.cu: the v4 solve-kernel
# instances (the long compiles), built in parallel and linked into one library
SOURCES = [PKG / "csrc" / n for n in ("gz_solver.cu", "gz_k16.cu", "gz_k32.cu", "gz_k32w.cu")]
HEADERS = sorted((PKG / "csrc").glob("*.cuh")) + [ROOT / "include" / "gazecut_b200.h"]
OUT = PKG / "libgazecut_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False) -> Path:
    # rebuild when the sources' content differs from what the library was built
    # from (a content digest, not mtimes: an edit during a running build counts)
    digest = hashlib.sha256(b"".join(p.read_bytes() for p in SOURCES + HEADERS)).hexdigest()
    stamp = OUT.with_suffix(".so.src")
    if not force and OUT.exists() and stamp.exists() and stamp.read_text() == digest:
        return OUT
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    common = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}"]
    if verbose:
        common.insert(0, "-Xptxas=-v")
    procs = []
    for src in SOURCES:
        obj = objdir / (src.stem + ".o")
        procs.append((src, subprocess.Popen([nvcc(), *common, "-c", "-o", str(obj), str(src)])))
    failed = [str(src) for src, pr in procs if pr.wait() != 0]
    if failed:
        raise RuntimeError(f"nvcc failed on {failed}")
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", str(OUT), *(str(objdir / (s_.stem + ".o")) for s_ in SOURCES),
                    "-lcudart"], check=True)
    stamp.write_text(digest)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
