"""Small solves through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402

for n3, pc, k, bpr, kern, var in [((64, 48, 32), "gnocomm", 4, 2, 1, 7), ((64, 48, 32), "bj", 3, 1, 1, 5),
                                  ((40, 24, 32), "gnocomm", 2, 1, 1, 7), ((33, 20, 16), "gnocomm", 4, 1, 1, 7),
                                  ((32, 32, 32), "gnocomm", 4, 1, 0, 7)]:
    s = bcgs.Solver(n3, si.unit_cube_h(n3[0]))
    s.set_option(bcgs.OPT_KERNELS, kern)
    s.set_option(bcgs.OPT_TB_VARIANT, var)
    s.set_preconditioner(pc, k, blocks_per_rank=bpr)
    s.set_rhs_random(si.SEED)
    rep = s.solve(fixed_iters=3)
    q = torch.randn((n3[2], n3[1], n3[0]), dtype=torch.float64, device="cuda")
    s.apply_preconditioner(q)
    s.apply_operator(q)
    torch.cuda.synchronize()
    print(n3, pc, k, bpr, kern, var, rep["status_name"], flush=True)
    s.close()
