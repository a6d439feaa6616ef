"""Build libbmc_b200.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels with the repo snapshot to the GPU box).

Each .cu is compiled to an object in parallel (the stage-kernel
instantiation units dominate the build), then linked into one shared library;
an object is recompiled only when its source or a header it includes changed.
Builds are serialised across processes with an fcntl lock (torchrun ranks that
all find a stale library build it once), objects and the library are written
under per-process temporary names and renamed into place.
"""

from __future__ import annotations

import fcntl
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = PKG / "lib" / "libbmc_b200.so"
LOCK = PKG / "lib" / ".build.lock"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def sources():
    return sorted(p.name for p in CSRC.glob("*.cu"))


def sources_present() -> bool:
    return CSRC.is_dir() and any(CSRC.glob("*.cu"))


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _deps():
    return ([CSRC / s for s in sources()] + sorted(CSRC.glob("*.cuh")) + sorted((ROOT / "include").glob("*.h"))
            + [Path(__file__)])


_INC = re.compile(r'^\s*#\s*include\s+"([^"]+)"', re.M)


def _includes(path: Path, seen=None) -> set:
    """Local (quoted) headers a source pulls in, transitively."""
    seen = set() if seen is None else seen
    for name in _INC.findall(path.read_text()):
        for cand in (path.parent / name, ROOT / "include" / name):
            cand = cand.resolve()
            if cand.exists() and cand not in seen:
                seen.add(cand)
                _includes(cand, seen)
                break
    return seen


def _obj_stale(src: str, obj: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    deps = [CSRC / src, Path(__file__), *_includes(CSRC / src)]
    return any(d.stat().st_mtime > t for d in deps)


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(d.stat().st_mtime > t for d in _deps())


def _compile(src: str, obj: Path, verbose: bool, extra=()):
    tmp = obj.with_name(f"{obj.name}.{os.getpid()}.tmp")
    cmd = [nvcc(), *ARCH, *FLAGS, *extra, "-Xptxas", "-v" if verbose else "-O3", "-I", str(ROOT / "include"),
           "-c", str(CSRC / src), "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode == 0:
        os.replace(tmp, obj)
    return res


def build(force: bool = False, verbose: bool = False, out: Path | None = None, extra=()) -> Path:
    """Compile every csrc/*.cu and link the library.  ``extra`` nvcc flags and
    ``out`` are for measurement builds (tools/), which go to their own path."""
    target = Path(out) if out else LIB
    target.parent.mkdir(parents=True, exist_ok=True)
    LOCK.parent.mkdir(parents=True, exist_ok=True)
    with open(LOCK, "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if not force and out is None and not _stale():
                return LIB
            objdir = target.parent / ("obj" if out is None else f"obj_{target.stem}")
            objdir.mkdir(parents=True, exist_ok=True)
            srcs = sources()
            objs = [objdir / (Path(s).stem + ".o") for s in srcs]
            # per-object staleness (source + transitively included headers); a forced
            # or measurement build recompiles everything
            todo = [(s, o) for s, o in zip(srcs, objs) if force or out is not None or _obj_stale(s, o)]
            with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
                results = list(ex.map(lambda so: _compile(so[0], so[1], verbose, extra), todo))
            for (src, _), res in zip(todo, results):
                if res.returncode != 0:
                    sys.stderr.write(res.stdout + res.stderr)
                    raise RuntimeError(f"nvcc failed compiling {src}")
                if verbose:
                    sys.stderr.write(res.stderr)
            tmp = target.with_name(f"{target.name}.{os.getpid()}.tmp")
            res = subprocess.run([nvcc(), *ARCH, "--shared", "-o", str(tmp), *map(str, objs)],
                                 capture_output=True, text=True)
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError("nvcc failed linking libbmc_b200.so")
            os.replace(tmp, target)
            return target
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
