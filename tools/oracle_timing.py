"""The CPU oracle timed on this host (SURVEY §8(d) "Oracle timing"): seconds per outer
iteration at 512^3 (fixed iterations, GNoComm(CI) k = 4) and full solves to 1e-8 at 32^3
(C1: MMS_POLYEXP, no preconditioner), 64^3 and 256^3 (GNoComm k = 4), with all host threads
and with one thread (OMP_NUM_THREADS=1, run in a child process; the 256^3 single-thread solve
is skipped -- ~25 min).  The paper's CPU baselines (LUMI-C) are context only.

    python tools/oracle_timing.py [--out gpurun_out/oracle_timing.json]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_cases(cases):
    import oracle
    import synth_inputs as si
    out = {"threads": oracle.threads()}
    for name, n, pc, k, fixed in cases:
        h = si.unit_cube_h(n)
        if name == "C1":
            b, _, h = si.mms_polyexp(n)
        else:
            b = oracle.rhs_random((n, n, n), si.SEED)
        t0 = time.perf_counter()
        r = oracle.bicgstab(b, h, pc=pc, k=k, tol=1e-8, fixed_it=fixed)
        dt = time.perf_counter() - t0
        out[name] = {"n": n, "pc": pc, "k": k, "iterations": r.iterations, "status": r.status,
                     "seconds": dt, "s_per_iteration": dt / max(r.iterations, 1),
                     "mode": f"fixed {fixed}" if fixed else "to 1e-8"}
        print(name, out[name], flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/oracle_timing.json")
    ap.add_argument("--child", default="")
    a = ap.parse_args()
    all_cases = [("C1", 32, "none", 0, 0), ("64", 64, "gnocomm", 4, 0),
                 ("256", 256, "gnocomm", 4, 0), ("512x3", 512, "gnocomm", 4, 3)]
    if a.child == "single":
        cases = [c for c in all_cases if c[0] in ("C1", "64")] + [("512x1", 512, "gnocomm", 4, 1)]
        print(json.dumps(run_cases(cases)))
        return
    res = {"all_threads": run_cases(all_cases)}
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run([sys.executable, __file__, "--child", "single"], env=env,
                       capture_output=True, text=True, timeout=3000)
    try:
        res["one_thread"] = json.loads(p.stdout.strip().splitlines()[-1])
    except Exception:  # noqa: BLE001
        res["one_thread"] = {"error": p.stderr[-500:]}
    try:
        res["host_cpu"] = [l for l in subprocess.run(["lscpu"], capture_output=True,
                                                     text=True).stdout.splitlines()
                           if "Model name" in l][0].split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    print(json.dumps(res))
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
