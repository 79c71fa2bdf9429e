"""GPU-vs-oracle parity of the inner-Krylov preconditioners FBiCGS-BJ(BiCGS) and
FBiCGS-G(BiCGS) (Eq. 15; inner settings P:393-394; R29).
The inner solves run the library's own unpreconditioned Bi-CGSTAB on private block contexts;
every dot is Dot2, so the GPU reproduces the oracle's outer AND inner iterate sequences:
compared bitwise (histories, scalars, solution, total inner iterations)."""
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("bpr", [1, 2, 4])
@pytest.mark.parametrize("faces", [None, si.PAPER_BC])
def test_inner_apply_bitwise(bc, orc, bpr, faces):
    n3, h, tol = (34, 18, 24), 0.2, 1e-6
    s = bc.Solver(n3, h, bc=faces) if faces else bc.Solver(n3, h)
    s.set_preconditioner("bj_bicgs", 0, blocks_per_rank=bpr)
    q = np.random.default_rng(11).standard_normal(n3[::-1])
    out = host(s.apply_preconditioner(dev(q)))
    ref, its = orc.apply_inner(q, h, bpr, tol, 500, bc=faces)
    assert np.array_equal(out, ref)
    s.close()


@pytest.mark.parametrize("n3,pc,bpr,faces,inner", [
    ((32, 32, 32), "bj_bicgs", 2, None, None),
    ((24, 20, 32), "bj_bicgs", 4, None, (1e-3, 20)),
    ((32, 32, 32), "g_bicgs", 1, None, None),
    ((34, 18, 20), "bj_bicgs", 2, si.PAPER_BC, None),
    ((34, 18, 20), "g_bicgs", 1, si.PAPER_BC, (1e-4, 50)),
])
def test_inner_solve_bitwise(bc, orc, n3, pc, bpr, faces, inner):
    h = si.unit_cube_h(n3[0]) if faces is None else 0.2
    s = bc.Solver(n3, h, bc=faces) if faces else bc.Solver(n3, h)
    s.set_preconditioner(pc, 0, blocks_per_rank=bpr)
    kw = {}
    if inner:
        s.set_inner_solver(*inner)
        kw = {"inner_tol": inner[0], "inner_max": inner[1]}
    b = orc.rhs_random(n3[::-1], si.SEED)
    s.set_rhs(dev(b))
    rep = s.solve(tol=1e-8, max_iter=500)
    o = orc.bicgstab(b, h, pc=pc, nslab=bpr, tol=1e-8, max_it=500, bc=faces, **kw)
    assert rep["status_name"] == o.status == "ok"
    assert rep["iterations"] == o.iterations
    assert s.inner_iterations() == o.extra["inner_iterations"] > 0
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(s.scalar_history(), o.scalars)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


def test_inner_group_two_ranks(bc, orc):
    """BJ(BiCGS) on two in-process ranks: each rank solves its own block (no inner
    communication) -> bitwise the single-context 2-block run AND the oracle: with
    correctly rounded dot products (R19) no inner stopping decision depends on the summation
    order any more (round 1 saw a last-bit Dot2 difference change an inner solve at outer
    iteration 8)."""
    n3, P = (32, 24, 32), 2
    h = si.unit_cube_h(32)
    grp = bc.local_group(n3, h, P)
    reps, errs = [None] * P, []

    def work(r):
        try:
            grp[r].set_preconditioner("bj_bicgs", 0)
            grp[r].set_rhs_random(si.SEED)
            reps[r] = grp[r].solve(tol=1e-8, max_iter=500)
        except Exception as ex:
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    x = np.concatenate([host(s.solution()) for s in grp])
    hist = grp[0].residual_history()
    scal = grp[0].scalar_history()
    inner = [s.inner_iterations() for s in grp]
    for s in grp:
        s.close()
    one = bc.Solver(n3, h)
    one.set_preconditioner("bj_bicgs", 0, blocks_per_rank=P)
    one.set_rhs_random(si.SEED)
    rep1 = one.solve(tol=1e-8, max_iter=500)
    assert all(r["iterations"] == rep1["iterations"] for r in reps)
    assert np.array_equal(hist, one.residual_history())
    assert np.array_equal(x, host(one.solution()))
    one.close()
    b = orc.rhs_random(n3[::-1], si.SEED)
    o = orc.bicgstab(b, h, pc="bj_bicgs", nslab=P, tol=1e-8, max_it=500)
    assert o.status == "ok" and reps[0]["converged"]
    assert reps[0]["iterations"] == o.iterations
    assert np.array_equal(hist, o.history)
    assert np.array_equal(scal, o.scalars)
    assert np.array_equal(x, o.x)
    assert sum(inner) == o.extra["inner_iterations"]


def test_g_bicgs_copy_transport_rejected(bc):
    """G(BiCGS) across ranks runs its global inner solve on the outer context's transport
    (NCCL or p2p; tested across processes in test_gpu_p2p.py); the in-process copy transport
    (a host-barrier test twin of NCCL) has no second group for it."""
    grp = bc.local_group((16, 16, 16), 1.0 / 17, 2)
    with pytest.raises(bc.BcgsError):
        grp[0].set_preconditioner("g_bicgs", 0)
    for s in grp:
        s.close()
