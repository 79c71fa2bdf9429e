"""How often does the R19 certification refuse a compensated dot?  Solves to 1e-8 and prints
the number of refusals (= exact-path recomputations) and the last refused certification
(stage, dot, D, r, offset, bound E, gaps, Σ|ab|).  python tools/cert_diag.py 128,512"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402

for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128,512").split(",")]:
    for pc, k, bpr in (("gnocomm", 4, 1), ("gnocomm", 4, 8), ("none", 0, 1)):
        s = bcgs.Solver(n, si.unit_cube_h(n))
        s.set_preconditioner(pc, k, blocks_per_rank=bpr)
        s.set_rhs_random(si.SEED)
        t = time.perf_counter()
        rep = s.solve(tol=1e-8, max_iter=5000)
        dt = time.perf_counter() - t
        ci = s.certification_info()
        print(f"{n}^3 {pc} k={k} P={bpr}: {rep['iterations']} it {rep['status_name']} "
              f"{dt:.2f}s exact={s.exact_dots()} refused={ci['refused']:.0f} last={ci}", flush=True)
        s.close()
