"""Build the C-ABI library in-tree: csrc/*.cu -> _native/libb2ddp.so (sm_100a only).

Each source compiles to its own object (in parallel, rebuilt only when the
source or a header changed), then one link step writes the shared library.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SOURCES = ["capi.cu", "bucket_clip.cu", "fused_allreduce.cu", "comm.cu", "strata.cu", "presort.cu", "radix.cu",
           "mc.cu", "draws.cpp"]
OUT = PKG / "_native" / "libb2ddp.so"
OBJ_DIR = PKG / "_native" / "obj"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
LINK_FLAGS = [*ARCH, "-shared", "-ldl", "-lpthread"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _headers() -> list:
    return list((PKG / "csrc").glob("*.cuh")) + list((PKG / "csrc").glob("*.h")) + [ROOT / "include" / "b2ddp.h"]


def _compile(src: Path, obj: Path, verbose: bool) -> None:
    tmp = obj.with_suffix(".o.tmp")
    cmd = [nvcc(), *COMPILE_FLAGS, f"-I{ROOT / 'include'}", "-c", "-o", str(tmp), str(src)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, obj)


def build(verbose: bool = False) -> Path:
    srcs = [PKG / "csrc" / s for s in SOURCES]
    hdr_mtime = max(h.stat().st_mtime for h in _headers())
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    objs, todo = [], []
    for s in srcs:
        o = OBJ_DIR / (s.name + ".o")
        objs.append(o)
        if not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, hdr_mtime):
            todo.append((s, o))
    if todo:
        with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
            for f in [ex.submit(_compile, s, o, verbose) for s, o in todo]:
                f.result()
    if OUT.exists() and not todo and all(OUT.stat().st_mtime >= o.stat().st_mtime for o in objs):
        return OUT
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [nvcc(), *LINK_FLAGS, "-o", str(tmp), *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True))
