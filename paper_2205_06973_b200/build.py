"""In-tree build of libhisvsim.so (nvcc, sm_100a only)."""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
SRC = PKG / "csrc"
OUT = PKG / "_lib" / "libhisvsim.so"
SOURCES = ("hs_api.cu", "hs_kernels.cu", "hs_planner.cpp", "hs_jit.cpp", "hs_dagp.cpp")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
    "-lnvrtc", "-Xlinker", "-rpath=/usr/local/cuda/lib64",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [SRC / s for s in SOURCES] + [SRC / "hs_common.h", PKG.parent / "include" / "hisvsim.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [nvcc(), *FLAGS, "-o", str(tmp), *[str(SRC / s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    (OUT.parent / "ptxas.log").write_text(res.stdout + res.stderr)
    os.replace(tmp, OUT)
    if verbose:
        print(res.stderr)
    return OUT


if __name__ == "__main__":
    print(build_native(force=True))
