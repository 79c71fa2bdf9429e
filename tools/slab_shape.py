"""Per-GPU shape of the strong-scaling runs, measured on ONE GPU.

On P GPUs each rank owns a 512 x 512 x (512/P) z-slab of the 512^3 problem.
This times one outer iteration of that slab with zero ghost planes (GNoComm k = 4: the
preconditioner is slab-local, so the compute is exactly a rank's; only the two face halos
and the cross-rank reductions are missing) and reports

    T_compute(P)   ms per iteration of the 512 x 512 x L slab, L = 512 / P
    E_P            = T_1 / (P * T_compute(P))   -- the compute-only strong-scaling bound
    GB/s, frac     200 B/pt x points / T (the HBM roofline fraction of the slab)
    kernel ms      per kernel class (CUDA events, profiled pass)

    python tools/slab_shape.py [--L 512,256,128,64] [--steps 50] [--out profiles/x.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth_inputs as si  # noqa: E402
from paper_2503_08935_b200 import bcgs  # noqa: E402


def time_iters(s, k, profile):
    s.set_option(bcgs.OPT_PROFILE, profile)
    s.kernel_times_reset()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    s.iterate(k)
    s.join_stream()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--L", default="512,256,128,64")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--degree", type=int, default=4)
    ap.add_argument("--stencil", default="1",
                    help="BCGS_OPT_STENCIL values to compare (1 = auto chunk, >= 2 planes per CTA)")
    ap.add_argument("--schedule", default="0",
                    help="BCGS_OPT_TB_SCHEDULE values (0 auto, 1 chunk grid, 2 segments)")
    ap.add_argument("--pdl", default="0", help="BCGS_OPT_PDL values (library default 0)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    n = a.n
    h = si.unit_cube_h(n)
    rows = []
    t1 = None
    combos = [(int(x), int(v), int(g), int(q)) for x in a.L.split(",")
              for v in a.stencil.split(",") for g in a.schedule.split(",")
              for q in a.pdl.split(",")]
    for L, sv, sched, pdl in combos:
        P = n // L
        s = bcgs.Solver((n, n, L), h)
        s.set_option(bcgs.OPT_STENCIL, sv)
        s.set_option(bcgs.OPT_TB_SCHEDULE, sched)
        s.set_option(bcgs.OPT_PDL, pdl)
        s.set_preconditioner("gnocomm", a.degree)
        s.set_rhs_random(si.SEED)
        s.begin(fixed_iters=a.warmup + 2 * a.steps)
        s.iterate(a.warmup)
        ms = time_iters(s, a.steps, 0)
        time_iters(s, a.steps, 1)
        kt = s.kernel_times()
        rep = s.finish()
        assert rep["iterations"] == a.warmup + 2 * a.steps, rep
        if t1 is None and P == 1 and sv == 1 and sched == 0 and pdl == 0:
            t1 = ms
        pts = n * n * L
        gbs = 200.0 * pts / (ms * 1e-3) / 1e9
        row = {"L": L, "P": P, "stencil_opt": sv, "schedule": sched, "pdl": pdl, "ms_per_iter": ms, "alg_gbs": gbs, "frac": gbs / peak,
               "E_P_compute_bound": (t1 / (P * ms)) if t1 else None,
               "kernel_ms": {k: v["ms"] / a.steps for k, v in kt.items()}}
        rows.append(row)
        print(json.dumps(row), flush=True)
        s.close()
        del s
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"n": n, "degree": a.degree, "peak_gbs": peak, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
