"""Build libresoct.so in-tree with nvcc for sm_100a (no JIT, no torch ext)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libresoct.so")
SOURCES = ["raycast.cu", "feedback.cu", "residency.cu", "ingest.cu", "metadata.cu", "pack.cu",
           "api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # the decision path must round exactly like the reference's unfused fp64
    "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "--expt-relaxed-constexpr",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(INCLUDE, "resoct.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out=None) -> str:
    """Compile csrc/*.cu into libresoct.so (or `out` with extra -D defines)."""
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    tag = "_".join(d.replace("=", "") for d in defines) or "default"
    objdir = os.path.join(HERE, "_obj", tag)
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-c",
               os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = lib + ".tmp"
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-o", tmp, *objs, "-lcudart"], check=True)
    os.replace(tmp, lib)
    return lib


def build_variant(name: str, defines) -> str:
    """Experiment builds (kernel variants) next to the package."""
    return build(force=True, defines=tuple(defines),
                 out=os.path.join(HERE, "_variants", f"libresoct_{name}.so"))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
