"""Per-kernel times of one outer iteration at n^3 for each stencil+dot launch configuration
(BCGS_OPT_STENCIL_CFG).  python tools/stencil_cfg_bench.py --n 512"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
s = bcgs.Solver(a.n, si.unit_cube_h(a.n))
s.set_preconditioner("gnocomm", 4)
s.set_rhs_random(si.SEED)
for cfg in [0, 1, 2, 3, 4, 0]:
    s.set_option(bcgs.OPT_STENCIL_CFG, cfg)
    s.set_option(bcgs.OPT_PROFILE, 1)
    s.begin(fixed_iters=a.iters + 3)
    s.iterate(3)
    s.kernel_times_reset()
    s.iterate(a.iters)
    kt = s.kernel_times()
    s.finish()
    print(cfg, {k: round(v["ms"] / a.iters, 3) for k, v in kt.items() if "stencil" in k}, flush=True)
