"""Config C3 solved to convergence on the GPU and by the oracle: 512^3,
GNoComm(CI) k = 4, RANDOM RHS, tol 1e-8 -- iteration count, every residual, every scalar
and the converged x compared; the oracle runs on the host cores (~20-25 min).

    python tools/converged_512.py [--n 512] [--out gpurun_out/converged_512.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--pc", default="gnocomm")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--bpr", type=int, default=1)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--out", default="gpurun_out/converged_512.json")
    a = ap.parse_args()
    n, h = a.n, si.unit_cube_h(a.n)
    s = bcgs.Solver(n, h)
    s.set_preconditioner(a.pc, a.k, blocks_per_rank=a.bpr)
    s.set_rhs_random(si.SEED)
    t0 = time.perf_counter()
    rep = s.solve(tol=a.tol)
    t_gpu = time.perf_counter() - t0
    g_hist, g_scal = s.residual_history(), s.scalar_history()
    g_x = s.solution().cpu().numpy()
    n_exact = s.exact_dots()
    s.close()
    del s
    torch.cuda.empty_cache()
    b = oracle.rhs_random((n, n, n), si.SEED)
    t0 = time.perf_counter()
    o = oracle.bicgstab(b, h, pc=a.pc, k=a.k, nslab=a.bpr, tol=a.tol)
    t_orc = time.perf_counter() - t0
    m = min(len(g_hist), len(o.history))
    out = {
        "config": f"{n}^3 {a.pc} k={a.k} P={a.bpr} tol={a.tol} RANDOM seed {si.SEED}",
        "gpu": {"iterations": rep["iterations"], "status": rep["status_name"],
                "rel_residual": rep["rel_residual"], "true_rel_residual": rep["true_rel_residual"],
                "seconds": t_gpu, "exact_dots": n_exact},
        "oracle": {"iterations": o.iterations, "status": o.status, "true_rel": o.true_rel,
                   "seconds": t_orc, "threads": oracle.threads()},
        "history_bitwise": bool(np.array_equal(g_hist, o.history)),
        "history_max_rel_diff": float(np.max(np.abs(g_hist[:m] - o.history[:m]) /
                                             np.abs(o.history[:m]))),
        "scalars_bitwise": bool(np.array_equal(g_scal, o.scalars)),
        "x_bitwise": bool(np.array_equal(g_x, o.x)),
        "x_rel_l2_diff": float(np.linalg.norm(g_x - o.x) / np.linalg.norm(o.x)),
    }
    print(json.dumps(out), flush=True)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
