"""Multi-process runner for the transport tests (p2p: P OS processes on ONE GPU; NCCL: one
GPU per rank, tests/test_gpu_nccl_multi.py).  p2p: P OS processes on ONE GPU, each a rank
with its own CUDA context (one process per rank -- the deployment shape), mailboxes mapped
through CUDA IPC (bcgs_p2p_handle / bcgs_p2p_connect), records exchanged over gloo.  The
contexts time-slice on the shared GPU, so the device-side waits are slow but the protocol
is exactly the multi-GPU one."""
import socket

import synth_inputs as si


def _worker(rank, world, port, job, q):
    import torch
    import torch.distributed as dist
    from paper_2503_08935_b200 import bcgs
    # job["transport"] == "nccl": one GPU per rank (NCCL refuses two ranks on one device)
    nccl = job.get("transport", "p2p") == "nccl"
    dev = rank if nccl else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        n3 = job["n3"]
        h = si.unit_cube_h(n3[0])
        if nccl:
            uid = [bcgs.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            s = bcgs.Solver(n3, h, rank=rank, nranks=world, nccl_id=uid[0], device=dev)
        else:
            s = bcgs.Solver(n3, h, rank=rank, nranks=world, transport="p2p", device=0)
            bcgs.connect_p2p(s)
        s.set_option(bcgs.OPT_COMM_TIMEOUT, 120)
        for opt, val in job.get("options", {}).items():
            s.set_option(getattr(bcgs, opt), val)
        s.set_preconditioner(job["pc"], job.get("k", 0))
        s.set_rhs_random(si.SEED)
        rep = s.solve(tol=job.get("tol", 1e-8), max_iter=job.get("max_iter", 5000),
                      fixed_iters=job.get("fixed", 0))
        q.put((rank, rep, s.residual_history(), s.scalar_history(),
               s.solution().cpu().numpy(), s.inner_iterations(), s.exact_dots()))
        dist.barrier()
        s.close()
    except Exception as ex:  # noqa: BLE001  (reported to the parent)
        q.put((rank, repr(ex), None, None, None, None, None))
    finally:
        dist.destroy_process_group()


def run(P, job, timeout=900):
    """Run `job` on P processes; returns {rank: (report, history, scalars, x, inner, exact)}."""
    import torch.multiprocessing as mp
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, P, port, job, q)) for r in range(P)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(P):
            r, *rest = q.get(timeout=timeout)
            out[r] = rest
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    return out
