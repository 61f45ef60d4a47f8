"""Build recipe for the C oracle (test infrastructure only)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "resoct_oracle.c")
OUT_DIR = os.path.join(HERE, "_build")


def lib_path() -> str:
    return os.path.join(OUT_DIR, "libresoct_oracle.so")


def build(force: bool = False) -> str:
    """Compile resoct_oracle.c with gcc (no FMA contraction, OpenMP bands)."""
    out = lib_path()
    if (not force and os.path.exists(out)
            and os.path.getmtime(out) >= os.path.getmtime(SRC)):
        return out
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = out + ".tmp"
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-fPIC", "-shared", "-o", tmp, SRC, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out
