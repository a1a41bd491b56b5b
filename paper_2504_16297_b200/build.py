"""Build libptsbe.so in-tree with nvcc for sm_100a (no torch, no JIT cache)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libptsbe.so"
SOURCES = [CSRC / "engine.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [PKG.parent / "include" / "ptsbe.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS if p.exists())


def write_prelude_inc() -> None:
    """Embed gen_prelude.cuh as a C++ raw string for NVRTC (codegen.h)."""
    text = (CSRC / "gen_prelude.cuh").read_text()
    inc = CSRC / "gen_prelude.inc"
    body = 'static const char* kGenPrelude = R"PTSBE_PRELUDE(' + text + ')PTSBE_PRELUDE";\n'
    if not inc.exists() or inc.read_text() != body:
        inc.write_text(body)


def build(force: bool = False, verbose: bool = False) -> Path:
    write_prelude_inc()
    if not force and up_to_date():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(OUT), *map(str, SOURCES)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
