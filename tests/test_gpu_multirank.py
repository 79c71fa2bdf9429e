"""Multi-rank z-slab path on ONE GPU: P contexts of an in-process group (bcgs_create_local)
exchange face halos and Dot2 pairs by device copies -- the same driver sequence, layout,
ghost-plane indexing and rank-ordered reduction as the NCCL path, which needs >= 2 GPUs.
Each rank is driven by its own host thread.  Compared bitwise with the oracle's P-slab
emulation and with the single-context blocks_per_rank = P emulation."""
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


def run_group(bc, n3, h, P, pc, k, kernels, tol=1e-8, fixed=0, rhs=None, options=None):
    grp = bc.local_group(n3, h, P)
    L = n3[2] // P
    reps = [None] * P
    errs = []

    def work(r):
        try:
            s = grp[r]
            s.set_option(bc.OPT_KERNELS, kernels)
            for opt, val in (options or {}).items():
                s.set_option(getattr(bc, opt), val)
            s.set_preconditioner(pc, k)
            if rhs is None:
                s.set_rhs_random(si.SEED)
            else:
                s.set_rhs(torch.from_numpy(np.ascontiguousarray(rhs[r * L:(r + 1) * L])).cuda())
            reps[r] = s.solve(tol=tol, fixed_iters=fixed)
        except Exception as ex:  # surface thread errors
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    x = np.concatenate([s.solution().cpu().numpy() for s in grp])
    hists = [s.residual_history() for s in grp]
    for s in grp:
        s.close()
    return reps, x, hists


@pytest.mark.parametrize("kernels", [0, 1])
@pytest.mark.parametrize("P,n3,pc,k", [(2, (48, 40, 64), "gnocomm", 4), (4, (64, 64, 64), "gnocomm", 4),
                                       (2, (40, 36, 48), "bj", 3), (4, (32, 32, 64), "none", 0),
                                       (2, (48, 40, 64), "g", 4), (4, (64, 64, 64), "g", 4),
                                       (4, (40, 32, 32), "g", 8), (8, (32, 32, 64), "g", 2)])
def test_local_group_matches_oracle(bc, orc, P, n3, pc, k, kernels):
    h = si.unit_cube_h(n3[0])
    reps, x, hists = run_group(bc, n3, h, P, pc, k, kernels)
    b = orc.rhs_random(n3[::-1], si.SEED)
    o = orc.bicgstab(b, h, pc=pc, k=k, nslab=P, tol=1e-8)
    for rep, hist in zip(reps, hists):
        assert rep["iterations"] == o.iterations
        assert np.array_equal(hist, o.history)        # identical scalars on every rank
    assert np.array_equal(x, o.x)


@pytest.mark.parametrize("options", [{"OPT_TB_SCHEDULE": 2}, {"OPT_STENCIL": 5},
                                     {"OPT_STENCIL": 4, "OPT_TB_SCHEDULE": 2}])
def test_local_group_schedules_match_oracle(bc, orc, options):
    """Ranks running the segment schedule of the Chebyshev kernel and short stencil chunks
    (the interior launch of the halo-overlapped stencil, planes 1..L-2, in 4- / 5-plane
    chunks) -- bitwise the oracle's P-slab iterates."""
    n3, P = (70, 52, 48), 2
    h = si.unit_cube_h(n3[0])
    reps, x, hists = run_group(bc, n3, h, P, "gnocomm", 4, 1, options=options)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=4, nslab=P, tol=1e-8)
    for rep, hist in zip(reps, hists):
        assert rep["iterations"] == o.iterations
        assert np.array_equal(hist, o.history)
    assert np.array_equal(x, o.x)


def test_local_group_equals_blocks_per_rank(bc):
    """P ranks x 1 block == 1 rank x P blocks (same math, bitwise)."""
    n3 = (64, 48, 64)
    h = si.unit_cube_h(64)
    reps, x, hists = run_group(bc, n3, h, 4, "gnocomm", 4, 1, fixed=15)
    s = bc.Solver(n3, h)
    s.set_preconditioner("gnocomm", 4, blocks_per_rank=4)
    s.set_rhs_random(si.SEED)
    s.solve(fixed_iters=15)
    assert np.array_equal(hists[0], s.residual_history())
    assert np.array_equal(x, s.solution().cpu().numpy())


def test_local_group_dot_and_operator(bc, orc):
    n3 = (24, 20, 32)
    h = si.unit_cube_h(24)
    P, L = 2, 16
    grp = bc.local_group(n3, h, P)
    r = np.random.default_rng(5)
    a = r.standard_normal(n3[::-1])
    v = r.standard_normal(n3[::-1])
    out = [None] * P
    dots = [None] * P

    def work(k):
        sl = slice(k * L, (k + 1) * L)
        av = torch.from_numpy(np.ascontiguousarray(a[sl])).cuda()
        vv = torch.from_numpy(np.ascontiguousarray(v[sl])).cuda()
        dots[k] = grp[k].dot(av, av)
        out[k] = grp[k].apply_operator(vv).cpu().numpy()

    th = [threading.Thread(target=work, args=(k,)) for k in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert dots[0] == dots[1] == orc.dot(a, a)
    assert np.array_equal(np.concatenate(out), orc.apply_A(v, h, 1))   # halo-exchanged operator
    for s in grp:
        s.close()


def test_gci_multirank_equals_single_gpu(bc):
    """G(CI) on P ranks with one k-deep halo exchange per application reproduces the
    single-GPU global Chebyshev bitwise (decomposition-independent preconditioner)."""
    n3 = (64, 48, 64)
    h = si.unit_cube_h(64)
    reps, x, hists = run_group(bc, n3, h, 4, "g", 4, 1)
    s = bc.Solver(n3, h)
    s.set_preconditioner("gnocomm", 4)
    s.set_rhs_random(si.SEED)
    rep = s.solve(tol=1e-8)
    assert reps[0]["iterations"] == rep["iterations"]
    assert np.array_equal(hists[0], s.residual_history())
    assert np.array_equal(x, s.solution().cpu().numpy())


def test_comm_ablation_runs_and_is_inert_when_off(bc, orc):
    """BCGS_OPT_ABLATE (bench.py's exposed halo / reduction share): with halos and
    cross-rank reductions skipped a fixed-iteration run still completes (finite scalars) and
    differs from the real one; switching it off restores the bitwise oracle result."""
    n3, h, P = (32, 32, 32), 1.0 / 33, 2
    results = {}
    for abl in (3, 0):
        grp = bc.local_group(n3, h, P)
        reps, errs = [None] * P, []

        def work(r):
            try:
                grp[r].set_option(bc.OPT_ABLATE, abl)
                grp[r].set_preconditioner("gnocomm", 4)
                grp[r].set_rhs_random(si.SEED)
                reps[r] = grp[r].solve(fixed_iters=25 if abl else 5)
            except Exception as ex:
                errs.append(ex)

        th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
        assert not errs, errs
        results[abl] = np.concatenate([s.solution().cpu().numpy() for s in grp])
        # bench.py times 20 ablated iterations after warm-up: the wrong scalars must not stop
        assert all(r["iterations"] == (25 if abl else 5) for r in reps)
        for s in grp:
            s.close()
    assert np.all(np.isfinite(results[3])) and not np.array_equal(results[3], results[0])
    b = orc.rhs_random(n3[::-1], si.SEED)
    o = orc.bicgstab(b, h, pc="gnocomm", k=4, nslab=P, fixed_it=5)
    assert np.array_equal(results[0], o.x)
