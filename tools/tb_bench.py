"""Time the temporally blocked preconditioner variants (apply_preconditioner, MODE_PLAIN)
and one full iteration per variant; check that all variants agree bitwise (and with the
oracle once).  python tools/tb_bench.py --n 512 --degree 4"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--degree", type=int, default=4)
ap.add_argument("--variants", default="2,7")
ap.add_argument("--oracle", action="store_true")
a = ap.parse_args()
n, k = a.n, a.degree
h = si.unit_cube_h(n)
s = bcgs.Solver(n, h)
s.set_preconditioner("gnocomm", k)
q = torch.randn((n, n, n), dtype=torch.float64, device="cuda")
outs = {}
for v in [int(x) for x in a.variants.split(",")]:
    s.set_option(bcgs.OPT_TB_VARIANT, v)
    s.set_option(bcgs.OPT_KERNELS, 1)
    s.set_option(bcgs.OPT_PROFILE, 1)
    s.kernel_times_reset()
    for _ in range(3):
        o = s.apply_preconditioner(q)
    torch.cuda.synchronize()
    s.kernel_times_reset()
    for _ in range(10):
        o = s.apply_preconditioner(q)
    kt = s.kernel_times()
    ms = kt["fused_p_cheb"]["ms"] / kt["fused_p_cheb"]["calls"]
    outs[v] = o.clone()
    s.set_rhs_random(si.SEED)
    s.kernel_times_reset()
    s.begin(fixed_iters=20)
    s.iterate(20)
    s.finish()
    kt2 = s.kernel_times()
    it = {kk: round(vv["ms"] / 20, 3) for kk, vv in kt2.items()}
    print(f"variant {v}: precond {ms:.3f} ms ({16 * n**3 / ms / 1e6:.0f} GB/s alg); "
          f"per-iteration {it}", flush=True)
vs = list(outs)
for v in vs[1:]:
    print(f"variant {v} == variant {vs[0]}:", bool(torch.equal(outs[v], outs[vs[0]])))
if a.oracle:
    import oracle
    ivl, _, _ = bcgs.chebyshev_constants(n, h, 1, "gnocomm", k)
    ref = oracle.apply_cheb(q.cpu().numpy(), h, 1, k, ivl[0], ivl[1])
    print("oracle equal:", np.array_equal(outs[vs[0]].cpu().numpy(), ref))
