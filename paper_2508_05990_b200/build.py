"""Build libbmc_b200.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels with the repo snapshot to the GPU box).

Each .cu is compiled to an object in parallel (the stage-kernel
instantiation units dominate the build), then linked into one shared library.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = PKG / "lib" / "libbmc_b200.so"
SOURCES = ["bmc_api.cu", "bmc_fme.cu", "bmc_fme_k_u8c4.cu", "bmc_fme_k_u8c2.cu", "bmc_fme_k_u16.cu", "bmc_fme_small.cu",
           "bmc_ops.cu"]
HEADERS = ["bmc_internal.cuh", "bmc_launch.cuh", "bmc_fme_impl.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _deps():
    return [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "bmc.h", Path(__file__)]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(d.stat().st_mtime > t for d in _deps())


def _compile(src: str, obj: Path, verbose: bool):
    cmd = [nvcc(), *ARCH, *FLAGS, "-Xptxas", "-v" if verbose else "-O3", "-I", str(ROOT / "include"),
           "-c", str(CSRC / src), "-o", str(obj)]
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    objdir = PKG / "lib" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    objs = [objdir / (Path(s).stem + ".o") for s in SOURCES]
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda so: _compile(so[0], so[1], verbose), zip(SOURCES, objs)))
    for src, res in zip(SOURCES, results):
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed compiling {src}")
        if verbose:
            sys.stderr.write(res.stderr)
    tmp = LIB.with_suffix(".so.tmp")
    res = subprocess.run([nvcc(), *ARCH, "--shared", "-o", str(tmp), *map(str, objs)],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libbmc_b200.so")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
