"""Peer-memory transport (p2p.cuh; SURVEY §8(e), NEXT-4 one-shot reductions): halos and
reductions as device kernels storing into the peers' memory with sequence-numbered flags.

* in one process: bcgs_create_local_p2p, one host thread per rank, multi-rank iterations
  replayed as CUDA graphs;
* across processes: two OS processes on the SAME GPU, mailboxes mapped through CUDA IPC
  (bcgs_p2p_handle / bcgs_p2p_connect) -- the code path of one process per GPU; on one GPU
  the two contexts time-slice, so the spin waits are slow but the protocol is the same.

Every case is compared bitwise with the oracle's P-slab emulation (R19: correctly rounded
dots make the rank count invisible in the reductions)."""
import os
import threading

import numpy as np
import pytest

import synth_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_08935_b200 import bcgs
    bcgs.load()
    return bcgs


def host(t):
    return t.cpu().numpy()


def run_local(bc, n3, h, P, pc, k, kernels=1, exact=0, tol=1e-8, fixed=0, graph=1):
    grp = bc.local_group(n3, h, P, transport="p2p")
    reps, errs = [None] * P, []

    def work(r):
        try:
            s = grp[r]
            s.set_option(bc.OPT_KERNELS, kernels)
            s.set_option(bc.OPT_EXACT_DOT, exact)
            s.set_option(bc.OPT_GRAPH, graph)
            s.set_preconditioner(pc, k)
            s.set_rhs_random(si.SEED)
            reps[r] = s.solve(tol=tol, fixed_iters=fixed)
        except Exception as ex:  # surface thread errors
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    x = np.concatenate([host(s.solution()) for s in grp])
    hists = [s.residual_history() for s in grp]
    scals = [s.scalar_history() for s in grp]
    for s in grp:
        s.close()
    return reps, x, hists, scals


@pytest.mark.parametrize("P,n3,pc,k,kernels", [(2, (48, 40, 64), "gnocomm", 4, 1),
                                               (4, (64, 64, 64), "gnocomm", 4, 1),
                                               (2, (40, 36, 48), "bj", 3, 1),
                                               (4, (32, 32, 64), "none", 0, 1),
                                               (2, (48, 40, 64), "g", 4, 1),
                                               (4, (40, 32, 32), "g", 8, 0),
                                               (8, (32, 32, 64), "gnocomm", 4, 0)])
def test_p2p_local_group_matches_oracle(bc, orc, P, n3, pc, k, kernels):
    h = si.unit_cube_h(n3[0])
    reps, x, hists, scals = run_local(bc, n3, h, P, pc, k, kernels)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc=pc, k=k, nslab=P, tol=1e-8)
    for rep, hist, scal in zip(reps, hists, scals):
        assert rep["iterations"] == o.iterations
        assert np.array_equal(hist, o.history)
        assert np.array_equal(scal, o.scalars)
    assert np.array_equal(x, o.x)


def test_p2p_forced_exact_and_direct_launches(bc, orc):
    """The exact path's superaccumulators travel through the mailboxes too (k_limbs_p2p);
    without graphs (direct launches) the same iterates."""
    n3, P = (32, 32, 64), 2
    h = si.unit_cube_h(32)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=4, nslab=P, tol=1e-8)
    for exact, graph in ((1, 1), (0, 0)):
        reps, x, hists, _ = run_local(bc, n3, h, P, "gnocomm", 4, exact=exact, graph=graph)
        assert reps[0]["iterations"] == o.iterations
        assert np.array_equal(hists[0], o.history)
        assert np.array_equal(x, o.x)


def test_p2p_timeout_instead_of_hang(bc):
    """A rank whose peer never answers gets BCGS_E_COMM after the configured timeout."""
    n3 = (16, 16, 32)
    grp = bc.local_group(n3, 1.0 / 17, 2, transport="p2p")
    s = grp[0]
    s.set_option(bc.OPT_COMM_TIMEOUT, 2)
    s.set_preconditioner("gnocomm", 2)
    s.set_rhs_random(1)
    with pytest.raises(bc.BcgsError) as ei:
        s.solve(tol=1e-8)          # rank 1 never runs: the first reduction times out
    assert ei.value.status == bc.E_COMM
    for g in grp:
        g.close()


# ------------------------------------------------------------------ two processes (CUDA IPC)

def _proc(rank, world, port, n3, pc, k, q):
    import torch
    import torch.distributed as dist
    from paper_2503_08935_b200 import bcgs
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        h = si.unit_cube_h(n3[0])
        s = bcgs.Solver(n3, h, rank=rank, nranks=world, transport="p2p", device=0)
        bcgs.connect_p2p(s)
        s.set_option(bcgs.OPT_COMM_TIMEOUT, 60)
        s.set_preconditioner(pc, k)
        s.set_rhs_random(si.SEED)
        rep = s.solve(tol=1e-8)
        q.put((rank, rep, s.residual_history(), s.solution().cpu().numpy()))
        dist.barrier()
        s.close()
    except Exception as ex:  # noqa: BLE001
        q.put((rank, repr(ex), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("pc,k", [("gnocomm", 4), ("g", 4)])
def test_p2p_two_processes_one_gpu(bc, orc, pc, k):
    import socket
    import torch.multiprocessing as mp
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    n3, P = (32, 24, 32), 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc, args=(r, P, port, n3, pc, k, q)) for r in range(P)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(P):
        r, rep, hist, x = q.get(timeout=600)
        out[r] = (rep, hist, x)
    for p in procs:
        p.join(timeout=120)
    for r in range(P):
        assert isinstance(out[r][0], dict), out[r][0]
    h = si.unit_cube_h(n3[0])
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc=pc, k=k, nslab=P, tol=1e-8)
    x = np.concatenate([out[r][2] for r in range(P)])
    for r in range(P):
        assert out[r][0]["iterations"] == o.iterations
        assert np.array_equal(out[r][1], o.history)
    assert np.array_equal(x, o.x)
