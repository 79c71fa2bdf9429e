"""Run a few outer iterations of the solver (for ncu captures / quick timing).

  python tools/run_iters.py --n 512 --iters 3 --kernels 1 [--pc gnocomm --degree 4]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--kernels", type=int, default=1)
ap.add_argument("--pc", default="gnocomm")
ap.add_argument("--degree", type=int, default=4)
ap.add_argument("--bpr", type=int, default=1)
a = ap.parse_args()
s = bcgs.Solver(a.n, si.unit_cube_h(a.n))
s.set_option(bcgs.OPT_KERNELS, a.kernels)
s.set_preconditioner(a.pc, a.degree, blocks_per_rank=a.bpr)
s.set_rhs_random(si.SEED)
t0 = time.perf_counter()
rep = s.solve(fixed_iters=a.iters)
torch.cuda.synchronize()
print(rep, f"{time.perf_counter() - t0:.3f}s")
