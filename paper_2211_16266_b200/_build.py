"""In-tree build of libd360.so (nvcc, sm_100a).  Cross-compiles without a GPU."""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libd360.so"
SOURCES = ["d360_common.cu", "d360_aux.cu", "d360_patchmatch.cu", "d360_fast.cu", "d360_fast_eval.cu",
           "d360_fast_rb.cu", "d360_fast_refine.cu", "d360_io.cu"]
HEADERS = [CSRC / "d360_device.cuh", CSRC / "d360_fast.cuh", PKG.parent / "include" / "d360.h"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build libd360.so")


STAMP = PKG / "build" / "libd360.stamp"


def source_digest() -> str:
    """Content hash of every source, header and flag the library is built from.  (A time-stamp
    comparison would reuse a stale prebuilt library whose file happens to be newer than the sources.)"""
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for dep in [CSRC / s for s in SOURCES] + HEADERS:
        h.update(dep.name.encode())
        h.update(dep.read_bytes())
    return h.hexdigest()


def needs_build() -> bool:
    if not LIB.exists() or not STAMP.exists():
        return True
    return STAMP.read_text().strip() != source_digest()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every CUDA source into paper_2211_16266_b200/libd360.so."""
    if not force and not needs_build():
        return LIB
    nvcc = _nvcc()
    objs = []
    procs = []
    build_dir = PKG / "build"
    build_dir.mkdir(exist_ok=True)
    flags = list(NVCC_FLAGS)
    for src in SOURCES:
        obj = build_dir / (src + ".o")
        objs.append(str(obj))
        cmd = [nvcc, *flags, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
        if verbose:
            print(out)
    link = [nvcc, "-shared", "-o", str(LIB), *objs, "-gencode", "arch=compute_100a,code=sm_100a"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    STAMP.write_text(source_digest() + "\n")
    return LIB


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
