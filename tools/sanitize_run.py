"""Small solves through every kernel family (incl. multi-pass blocking and the inner-Krylov
preconditioners), for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402

for n3, pc, k, bpr, kern, var in [((64, 48, 32), "gnocomm", 4, 2, 1, 7), ((64, 48, 32), "bj", 3, 1, 1, 2),
                                  ((40, 24, 32), "gnocomm", 2, 1, 1, 7), ((33, 20, 16), "gnocomm", 4, 1, 1, 7),
                                  ((32, 32, 32), "gnocomm", 4, 1, 0, 7),
                                  # multi-pass (k = 5: passes 3 + 2, k = 11: 4 + 4 + 3)
                                  ((48, 40, 32), "gnocomm", 5, 2, 1, 7),
                                  ((40, 36, 24), "gnocomm", 11, 1, 1, 7),
                                  # inner-Krylov preconditioners (private block contexts)
                                  ((32, 24, 16), "bj_bicgs", 0, 2, 1, 7),
                                  ((24, 24, 24), "g_bicgs", 0, 1, 1, 7)]:
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

# mirror-ghost (Neumann) pass kernels: the paper's faces, k = 24
f, hp, faces = si.paper_problem(32)
s = bcgs.Solver((32, 32, 32), hp, bc=faces)
s.set_preconditioner("gnocomm", 24, blocks_per_rank=2)
s.set_rhs(torch.from_numpy(f).cuda())
rep = s.solve(fixed_iters=2)
torch.cuda.synchronize()
print("paper problem k=24", rep["status_name"], flush=True)
s.close()
