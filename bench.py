#!/usr/bin/env python3
"""Benchmark of the B200-native preconditioned Bi-CGSTAB hot path (arXiv 2503.08935).

Metric (BASELINE.json): fp64 Bi-CGSTAB iters/s & GDoF/s at 512³, % of HBM roofline.
A "step" = one outer iteration of Alg. 3 (all §8(a) rows a2-a14) on the 512³ grid
(config C3: GNoComm(CI) k = 4, slab decomposition over N GPUs, strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 Bi-CGSTAB iters/s & GDoF/s at 512^3; % of HBM roofline"
ALG_BYTES_PER_PT = 200.0   # compulsory bytes per point per outer iteration
ALG_BYTES_NONE = 168.0     # M = I: the same rows without the preconditioner


def workload(n: int, pc: str, k: int) -> str:
    """BASELINE.json config names: C2 = 256^3, C3 = 512^3, C5 = 1024^3 (here on one GPU)."""
    tag = {256: "C2 ", 512: "C3 ", 1024: "C5 "}.get(n, "")
    name = {"gnocomm": "GNoComm(CI)", "bj": "BJ(CI)", "g": "G(CI)", "none": "BiCGS (M = I)"}.get(pc, pc)
    return f"{tag}{n}^3 {name} k={k}"

# FP64 flops per point of one launch of the fused Chebyshev kernels at degree k:
# sweep 1: 12, sweep 2: 16, sweeps 3..k: 15 each; + the fused vector update (p: 4, s: 2)
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def _cheb_flops(k):
    return 0 if k == 0 else 12 + (16 if k >= 2 else 0) + 15 * max(0, k - 2)


FLOPS_PER_PT = {"fused_p_cheb": lambda k: _cheb_flops(k) + 4,
                "fused_s_cheb": lambda k: _cheb_flops(k) + 2}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--pc", default="gnocomm", choices=["gnocomm", "bj", "none"])
    ap.add_argument("--degree", type=int, default=4)
    ap.add_argument("--kernels", type=int, default=1, help="0 = reference kernels, 1 = fused")
    ap.add_argument("--sync2", action="store_true",
                    help="2-sync rewrite (R31): 2 reductions per iteration instead of 3")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1: NCCL, or the peer-memory transport (p2p.cuh: one-shot "
                         "reductions, graph replay)")
    ap.add_argument("--pipelined", action="store_true",
                    help="pipelined Bi-CGSTAB (R32): 2 reductions per iteration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while running."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def ncu_bytes_per_pt(n, world, k, args):
    """Measured DRAM bytes per grid point per iteration: the committed ncu
    capture's dram read + write of the iteration's five kernels at 512^3 (one rank, the
    default fused GNoComm k = 4 path), divided by the points; None for other workloads."""
    if (n, world, k, args.pc, args.kernels) != (512, 1, 4, "gnocomm", 1) or args.sync2 or \
            args.pipelined:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        keys = ["fused_p_cheb", "stencil_dot1", "fused_s_cheb", "stencil_dot2", "fused_xr"]
        return sum(tr[f"{kk}@512"] for kk in keys) / float(512 ** 3)
    except Exception:
        return None


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank float over all ranks (timings are reported as the slowest rank)."""
    if dist is None or not dist.is_available() or not dist.is_initialized() \
            or dist.get_world_size() == 1:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(n, pc, k, seed, iters=5):
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload:
    `iters` outer iterations of the same 512³ problem in one fixed-iteration solve (the setup
    dots, the allocations and the final true-residual evaluation are included and amortised
    over the iterations, ~10-15 s on 16 cores)."""
    import oracle
    import synth_inputs as si
    h = si.unit_cube_h(n)
    b = oracle.rhs_random((n, n, n), seed)
    t0 = time.perf_counter()
    oracle.bicgstab(b, h, pc=pc, k=k, fixed_it=iters)
    dt = time.perf_counter() - t0
    return {"value": iters / dt, "unit": "iters/s", "cores": oracle.threads(), "kind": "oracle",
            "sample": f"{iters} outer iterations of {n}^3 {pc} k={k} in one solve (incl. setup "
                      f"+ true residual), {dt:.2f} s"}


def reference_sample_planes(n: int, steps: int, warmup: int) -> int:
    """z-planes of the reference arm's sample: the full grid for the driver's short runs
    (steps + warmup <= 30 oracle iterations, ~4.4 s each at 512^3 on 16 host cores), else a
    slab sized so that the whole run stays within a few minutes."""
    if steps + warmup <= 30:
        return n
    return max(8, (n * 30 // (steps + warmup)) // 8 * 8)


def reference_arm(args, rank, world):
    """--impl reference: the oracle as it stands (the CPU program of oracle/, never tuned),
    on this host's cores, on the same workload: W untimed outer iterations, then K timed
    outer iterations of Alg. 3 in ONE oracle solve (fixed_it = K; the timed call also does
    the setup dots and the final true-residual evaluation, i.e. it is slightly pessimistic
    for the oracle).  For the driver's K + W <= 30 the sample is the full n^3 grid (same
    config as our arm); for longer runs a 512x512xLs slab, scaled by the point ratio."""
    if rank != 0:
        return
    import oracle
    import synth_inputs as si
    n = args.n
    ls = reference_sample_planes(n, args.steps, args.warmup)
    h = si.unit_cube_h(n)
    b = si.rhs_random(n, n, n, si.SEED, z0=0, nzl=ls)
    if args.warmup:
        oracle.bicgstab(b, h, pc=args.pc, k=args.degree, fixed_it=args.warmup)
    t0 = time.perf_counter()
    res = oracle.bicgstab(b, h, pc=args.pc, k=args.degree, fixed_it=max(args.steps, 1))
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    scale = n / ls
    v = 1.0 / (dt * scale)
    if ls == n:
        sample = (f"{args.steps} timed oracle outer iterations (one fixed-iteration solve incl. "
                  f"setup and true residual) of the full {n}^3 problem after {args.warmup} "
                  f"untimed ones")
    else:
        sample = (f"{args.steps} timed oracle outer iterations on a {n}x{n}x{ls} slab of the "
                  f"{n}^3 problem, scaled x{scale:g} to {n}^3")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * scale * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_keys(args, n, args.degree, world),
            "gdof_s": n ** 3 * v / 1e9,
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": oracle.threads(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "report": {"iterations": res.iterations, "status": res.status}}
    print(json.dumps(line), flush=True)


def config_keys(args, n, k, world):
    return {"workload": workload(n, args.pc, k),
            "grid": n, "preconditioner": args.pc, "degree": k,
            "c_min": 10.0, "c_max": 1 - 1e-4, "decomposition": f"z-slab x{world}",
            "kernels": "fused" if args.kernels else "reference",
            "reductions_per_iteration": 2 if (args.sync2 or args.pipelined) else 3,
            "transport": args.transport if world > 1 else None,
            "algorithm": "pipelined (R32)" if args.pipelined else "Alg. 3",
            "l2": "inputs larger than L2 (each field 8*N^3/P bytes >> 126 MB)",
            "rhs": "splitmix64 uniform[-1,1), seed 20250311"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import synth_inputs as si
    from paper_2503_08935_b200 import bcgs

    assert world == args.gpus, f"WORLD_SIZE {world} != --gpus {args.gpus}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        if args.transport == "nccl":
            idt = torch.zeros(128, dtype=torch.uint8, device=dev)
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(bcgs.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, 0)
            nccl_id = bytes(idt.cpu().numpy().tobytes())

    n, k = args.n, args.degree
    h = si.unit_cube_h(n)
    s = bcgs.Solver(n, h, rank=rank, nranks=world, nccl_id=nccl_id, device=local,
                    transport=args.transport)
    if world > 1 and args.transport == "p2p":
        bcgs.connect_p2p(s)
    s.set_option(bcgs.OPT_KERNELS, args.kernels)
    if args.pipelined:
        s.set_option(bcgs.OPT_PIPELINED, 1)
    s.set_option(bcgs.OPT_SYNC2, 1 if args.sync2 else 0)
    s.set_preconditioner(args.pc, k)
    s.set_rhs_random(si.SEED)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    total = args.warmup + 2 * args.steps
    clocks = ClockSampler(local)
    clocks.start()
    s.begin(fixed_iters=total)
    s.iterate(args.warmup)
    barrier()
    stream = torch.cuda.current_stream(dev)

    def timed(k, profile):
        s.set_option(bcgs.OPT_PROFILE, profile)
        s.kernel_times_reset()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        s.iterate(k)                 # enqueued on the library stream (CUDA graph replays)
        s.join_stream()              # caller stream waits for the library stream
        e1.record(stream)
        barrier()
        return e0.elapsed_time(e1) / k

    # pass A (headline): K iterations replayed from the captured CUDA graph, no inner events.
    ms_iter = timed(args.steps, 0)
    # pass B: K more iterations with CUDA events around every kernel on its launching stream
    # (per-kernel durations for the roofline; events disable graph replay).
    ms_iter_prof = timed(args.steps, 1)
    clk = clocks.stop()
    ktimes = s.kernel_times()
    phases = s.phase_times()     # SPEC S:382 phase keys, pass B
    s.set_option(bcgs.OPT_PROFILE, 0)
    rep = s.finish()
    # every enqueued iteration must have run: after a breakdown the remaining iterations are
    # device no-ops and the timing would be meaningless
    short = 0.0 if rep["iterations"] == total else 1.0
    valid = max_over_ranks(short, dist, dev) == 0.0
    # a reduction parked for the exact path (R19) turns the rest of the enqueued iterations
    # into no-ops until the host resolves it: the timed passes must not contain one
    n_exact = s.exact_dots()
    valid = valid and max_over_ranks(float(n_exact), dist, dev) == 0.0
    comm = None
    if world > 1:
        # exposed halo / reduction share by ablation: K_a iterations of a fresh
        # solve with the face halos (bit 0) and / or the cross-rank reductions (bit 1) skipped.
        # The maths is wrong while ablated, the timing right; a pass that stopped early (the
        # wrong scalars hit a breakdown) is reported as null.  Max over ranks like the headline.
        ka = min(args.steps, 20)
        abl = {}
        for bits in (1, 2, 3):
            s.set_option(bcgs.OPT_ABLATE, bits)
            s.begin(fixed_iters=args.warmup + ka)
            s.iterate(args.warmup)
            t_abl = max_over_ranks(timed(ka, 0), dist, dev)
            ok = s.finish()["iterations"] == args.warmup + ka
            ok = max_over_ranks(0.0 if ok else 1.0, dist, dev) == 0.0
            abl[bits] = t_abl if ok else None
        s.set_option(bcgs.OPT_ABLATE, 0)
    ms_iter = max_over_ranks(ms_iter, dist, dev)
    ms_iter_prof = max_over_ranks(ms_iter_prof, dist, dev)
    if world > 1:
        def share(v):
            return None if v is None else 1.0 - v / ms_iter
        comm = {"ms_full": ms_iter, "ms_no_halo": abl[1], "ms_no_reductions": abl[2],
                "ms_no_comm": abl[3], "halo_share": share(abl[1]),
                "reduction_share": share(abl[2]), "comm_share": share(abl[3]),
                "ablated_iterations": ka,
                "method": "ablation: BCGS_OPT_ABLATE skips the face halos (1) / the cross-rank "
                          "Dot2 all-gathers (2) / both (3); share = 1 - T_ablated / T_full"}

    its = 1000.0 / ms_iter
    gdof = n ** 3 * its / 1e9
    peak, peak_src = peaks()
    pts_local = n * n * (n // world)
    alg_bpp = ALG_BYTES_NONE if args.pc == "none" else ALG_BYTES_PER_PT
    iter_gbs = alg_bpp * pts_local / (ms_iter * 1e-3) / 1e9

    # dominant kernel of the timed region (largest total device time)
    ours = {kname: v for kname, v in ktimes.items() if kname not in ("halo", "allgather")}
    dom_name = max(ours, key=lambda kk: ours[kk]["ms"]) if ours else None
    roof = None
    if dom_name:
        d = ours[dom_name]
        per_launch_ms = d["ms"] / d["calls"]
        achieved = d["bytes_per_call"] / (per_launch_ms * 1e-3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                tr = json.load(f)
            traffic = tr.get(f"{dom_name}@{n}")
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": peak_src,
                "share_of_step": d["ms"] / (ms_iter_prof * args.steps),
                "timing": "average launch duration from CUDA events on the launching stream over "
                          "a second timed pass of K iterations (pass B)"}
        if dom_name in ("fused_p_cheb", "fused_s_cheb"):
            roof["limiter"] = ("L1/shared-memory throughput and FP64 dependency latency per "
                               "z-step (ncu l1tex 80 % / 75 % of peak for the p / s kernels, "
                               "issue slots 54 %, FP64 pipe 42 %, 24 warps per SM at the "
                               "80-register cap: profiles/round2b_ncu_full.txt; a layout with "
                               "26 % fewer shared wavefronts but 12 warps was slower: "
                               "profiles/round2b_ncu_xpair_512.txt, DESIGN.md §4, §8); the HBM "
                               "fraction is reported against the kernel's compulsory bytes")
        if dom_name in FLOPS_PER_PT:
            # the temporally blocked Chebyshev kernels are FP64-ALU heavy: report that roof too
            fl = FLOPS_PER_PT[dom_name](k) * pts_local
            roof["alu"] = {"bound": "alu", "achieved": fl / (per_launch_ms * 1e-3) / 1e12,
                           "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                           "frac": fl / (per_launch_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                           "flops_per_pt": FLOPS_PER_PT[dom_name](k),
                           "peak_source": "148 SMs x 64 FP64 lanes x 2 (FMA) x 1.965 GHz "
                                          "(DESIGN.md §5)"}
    launches = sum(v["calls"] for kname, v in ktimes.items() if kname not in ("halo", "allgather"))

    # e2e through the public API with host buffers: set_rhs(host) + solve(K) + x -> host
    e2e = None
    if not args.no_e2e:
        f_host = torch.from_numpy(si.rhs_random(n, n, n, si.SEED, z0=rank * (n // world),
                                                nzl=n // world)).pin_memory()
        x_host = torch.empty_like(f_host).pin_memory()
        barrier()
        t0 = time.perf_counter()
        s.set_rhs(f_host)
        s.solve(fixed_iters=args.steps)
        s.lib.bcgs_get_solution(s.ctx, x_host.data_ptr(), bcgs.MEM_HOST)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        dt = max_over_ranks(dt, dist, dev)
        e2e = {"value": args.steps / dt, "unit": "iters/s",
               "h2d_bytes_per_step": f_host.numel() * 8 / args.steps,
               "d2h_bytes_per_step": x_host.numel() * 8 / args.steps,
               "note": "set_rhs(host pinned) + solve(fixed K) + get_solution(host); per-step "
                       "bytes = one RHS in and one solution out amortised over K"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(n, args.pc, k, si.SEED)
        except Exception as ex:  # report, do not fail the bench
            cpu = {"error": repr(ex)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": its, "unit": "iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_iter,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": config_keys(args, n, k, world),
            "gdof_s": gdof,
            "iteration_roofline": {"alg_bytes_per_pt": alg_bpp,
                                   "achieved_gbs": iter_gbs, "peak_gbs": peak,
                                   "frac": iter_gbs / peak,
                                   "ncu_bytes_per_pt": ncu_bytes_per_pt(n, world, k, args)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "comm": comm,
            "kernel_ms_per_step": {kk: v["ms"] / args.steps for kk, v in ktimes.items()},
            "phase_ms_per_step": {kk: v / args.steps for kk, v in phases.items()},
            "ms_per_step_profiled_pass": ms_iter_prof,
            "clocks": clk, "report": {kk: rep[kk] for kk in ("iterations", "rel_residual",
                                                             "true_rel_residual")},
        }
        if not valid:
            line["valid"] = False
            line["invalid_reason"] = (f"the solve ran {rep['iterations']} of {total} enqueued "
                                      f"iterations ({rep['status_name']}); {n_exact} dots took "
                                      f"the exact path")
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
