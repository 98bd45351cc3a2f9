"""Build libreax.so in-tree for sm_100a (B200).  No JIT cache: the .so lives
next to this file so it travels with the repo snapshot."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "reax.cu")
DEPS = [SRC, os.path.join(HERE, "csrc", "kernels.cuh"), os.path.join(HERE, "csrc", "common.cuh"),
        os.path.join(ROOT, "include", "reax.h")]
OUT = os.path.join(HERE, "libreax.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177"]


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    newest = max(os.path.getmtime(p) for p in DEPS)
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    cmd = [NVCC] + FLAGS + [f"-D{d}" for d in defines] + (["-Xptxas", "-v"] if verbose else []) + ["-o", out, SRC]
    subprocess.check_call(cmd, cwd=ROOT)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose="-v" in sys.argv,
                out=outs[0] if outs else OUT, defines=defs))
