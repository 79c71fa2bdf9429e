"""Build libbcgs.so (the C-ABI library of include/bcgs.h) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib", "libbcgs.so")
SRC = os.path.join(PKG, "csrc", "bcgs_api.cu")


def nccl_dir() -> str:
    import nvidia.nccl  # the NCCL that ships with torch (2.28); a namespace package
    return list(nvidia.nccl.__path__)[0]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*")) +
                  [os.path.join(ROOT, "include", "bcgs.h")])


def nvcc_cmd(out: str) -> list[str]:
    nccl = nccl_dir()
    return ["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
            # R17: no FMA contraction anywhere (bitwise parity with the oracle)
            "--fmad=false", "-std=c++17",
            "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v", "-shared",
            "-o", out, SRC,
            "-I", os.path.join(nccl, "include"), "-L", os.path.join(nccl, "lib"),
            "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nccl, "lib")]


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    newest = max(os.path.getmtime(p) for p in sources())
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = nvcc_cmd(tmp)
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "lib", "ptxas.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libbcgs.so (see %s)" % log)
    if verbose:
        sys.stdout.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
