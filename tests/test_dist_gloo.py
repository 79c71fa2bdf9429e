"""Multi-process (world_size 2, gloo, CPU) checks of the host-side logic of the z-slab
decomposition that the NCCL path relies on:
  * each rank's slab of the RANDOM right-hand side is the global field's slice (R16);
  * every rank derives bit-identical Chebyshev constants for nslab = nranks*blocks (R9/R10),
    equal to the oracle's;
  * per-rank Dot2 (hi, lo) partials combined in ascending rank order (R19, the all-gather
    reduction of the library) give the oracle's global dot exactly;
  * bench.py's max-over-ranks timing.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth_inputs as si

NX, NY, NZ = 12, 10, 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def two_sum(a, b):
    s = a + b
    z = s - a
    return s, (a - (s - z)) + (b - z)


def _worker(rank, world, port, out):
    import torch
    import oracle
    from paper_2503_08935_b200 import bcgs
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    L = NZ // world
    h = 1.0 / (NX + 1)
    # 1) slab of the RHS
    b_slab = si.rhs_random(NX, NY, NZ, si.SEED, z0=rank * L, nzl=L)
    gathered = [torch.zeros((L, NY, NX), dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(b_slab))
    # 2) host constants
    ivl, cst, rho = bcgs.chebyshev_constants((NX, NY, NZ), h, world * 2, "bj", 4)
    consts = torch.from_numpy(np.concatenate([ivl, cst, rho]))
    allc = [torch.zeros_like(consts) for _ in range(world)]
    dist.all_gather(allc, consts)
    # 3) rank-ordered Dot2 combination of per-rank partials
    pair = torch.tensor(oracle.dot_pair(b_slab, b_slab), dtype=torch.float64)
    pairs = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(pairs, pair)
    # 4) max over ranks
    import bench
    mx = bench.max_over_ranks(float(rank + 1) * 1.5, dist, "cpu")
    if rank == 0:
        out.put({"gathered": torch.cat(gathered).numpy(), "consts": [c.numpy() for c in allc],
                 "pairs": [tuple(p.tolist()) for p in pairs], "max": mx})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slab_decomposition_gloo(orc, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    b = orc.rhs_random((NZ, NY, NX), si.SEED)
    assert np.array_equal(res["gathered"], b)
    for c in res["consts"][1:]:
        assert np.array_equal(c, res["consts"][0])
    lo, hi = orc.bounds(NX, NY, NZ // (world * 2), 1.0 / (NX + 1))
    assert tuple(res["consts"][0][:2]) == (lo, hi)
    P, S = 0.0, 0.0
    for hi_, lo_ in res["pairs"]:          # ascending rank order (R19)
        P, q_ = two_sum(P, hi_)
        S = S + (q_ + lo_)
    assert P + S == orc.dot(b, b)
    assert res["max"] == 1.5 * world
