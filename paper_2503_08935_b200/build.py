"""Build libbcgs.so (the C-ABI library of include/bcgs.h) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# BCGS_BUILD_OUT / BCGS_NVCC_EXTRA: build a variant elsewhere (A/B timing with BCGS_LIB)
LIB = os.environ.get("BCGS_BUILD_OUT") or os.path.join(PKG, "lib", "libbcgs.so")
SRC = os.path.join(PKG, "csrc", "bcgs_api.cu")


def nccl_dir() -> str:
    import nvidia.nccl  # the NCCL that ships with torch (2.28); a namespace package
    return list(nvidia.nccl.__path__)[0]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*")) +
                  [os.path.join(ROOT, "include", "bcgs.h")])


CU_SOURCES = ["bcgs_api.cu", "tb_multi.cu", "tb_multi_c.cu", "st_tma.cu"] + [f"tb_k{k}.cu" for k in range(1, 9)]
NVCC_FLAGS = ["-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              # R17: no FMA contraction except the contract's explicit fma()
              "--fmad=false", "-std=c++17",
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v"]


def build(force: bool = False, verbose: bool = False, jobs: int = 0) -> str:
    """Compile the translation units in parallel, link libbcgs.so (in-tree)."""
    import concurrent.futures as cf
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    newest = max(os.path.getmtime(p) for p in sources())
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    nccl = nccl_dir()
    objdir = os.path.join(os.path.dirname(LIB), "obj")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(nccl, "include")]

    # headers are shared by every unit: an object is reused only if it is newer than its own
    # .cu, every header and this script (and not force)
    hdr = max(os.path.getmtime(p) for p in sources() + [os.path.abspath(__file__)]
              if not p.endswith(".cu"))

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        extra = os.environ.get("BCGS_NVCC_EXTRA", "").split()
        cmd = ["nvcc", *NVCC_FLAGS, *extra, *inc, "-c", "-o", obj, os.path.join(PKG, "csrc", src)]
        cu = os.path.join(PKG, "csrc", src)
        if (not force and not extra and os.path.exists(obj) and
                os.path.getmtime(obj) >= max(hdr, os.path.getmtime(cu))):
            return src, obj, cmd, subprocess.CompletedProcess(cmd, 0, "(up to date)\n", "")
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, r

    jobs = jobs or min(len(CU_SOURCES), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(compile_one, CU_SOURCES))
    log = os.path.join(os.path.dirname(LIB), "ptxas.log")
    with open(log, "w") as f:
        for src, obj, cmd, r in results:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    bad = [r for r in results if r[3].returncode != 0]
    if bad:
        for src, obj, cmd, r in bad:
            sys.stderr.write(f"--- {src}\n" + r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libbcgs.so (see %s)" % log)
    tmp = LIB + f".tmp{os.getpid()}"
    link = ["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp,
            *[r[1] for r in results], "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + os.path.join(nccl, "lib")]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libbcgs.so failed")
    if verbose:
        sys.stdout.write(open(log).read())
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
