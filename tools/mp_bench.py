"""Time one preconditioner application (M^-1 q) at n^3 for several degrees, with the
multi-pass temporally blocked path (default) and with one sweep per launch (reference
kernels).  python tools/mp_bench.py --n 512 --degrees 4,8,12,16,24"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--degrees", default="4,8,12,16,24")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
n = a.n
h = si.unit_cube_h(n)
q = torch.randn((n, n, n), dtype=torch.float64, device="cuda")
for k in [int(x) for x in a.degrees.split(",")]:
    res = {}
    for label, kern, mp in (("blocked", 1, 8), ("blocked_mp4", 1, 4), ("ref", 0, 64)):
        if label == "blocked_mp4" and k <= 4:
            continue
        s = bcgs.Solver(n, h)
        s.set_option(bcgs.OPT_KERNELS, kern)
        s.set_option(bcgs.OPT_MULTIPASS, mp)
        s.set_preconditioner("gnocomm", k)
        o = s.apply_preconditioner(q)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            o = s.apply_preconditioner(q)
        e1.record()
        torch.cuda.synchronize()
        # includes 2 device copies of 8 B/pt each (in/out staging of the API call)
        res[label] = (e0.elapsed_time(e1) / a.reps, o.clone())
        s.close()
    base = res["ref"][1]
    line = ", ".join(f"{kk} {v[0]:.3f} ms" + ("" if torch.equal(v[1], base) else " MISMATCH")
                     for kk, v in res.items())
    print(f"k={k}: {line}", flush=True)
