"""GPU-vs-oracle parity of the 2-sync rewrite (DESIGN.md §3 R31): the a9
stencil+dot reduces five Dot2 pairs (tᵀs, tᵀt, r~ᵀs, r~ᵀt, sᵀs), ρ_new and ||r||² follow from
the identities for r = s - ω t, the a12 update carries no dot -> 2 reductions per iteration.
Same flag on both sides -> bitwise."""
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


@pytest.mark.parametrize("n3,pc,k,bpr,fixed", [((64, 64, 64), "gnocomm", 4, 1, 0),
                                               ((48, 40, 64), "gnocomm", 4, 2, 0),
                                               ((64, 48, 32), "bj", 3, 2, 0),
                                               ((64, 64, 64), "gnocomm", 24, 1, 0),
                                               ((64, 64, 64), "gnocomm", 4, 1, 7),
                                               ((32, 32, 32), "g", 4, 1, 0)])
def test_sync2_solve_bitwise(bc, orc, n3, pc, k, bpr, fixed):
    h = si.unit_cube_h(n3[0])
    s = bc.Solver(n3, h)
    s.set_option(bc.OPT_SYNC2, 1)
    s.set_preconditioner(pc, k, blocks_per_rank=bpr)
    s.set_rhs_random(si.SEED)
    rep = s.solve(tol=1e-8, fixed_iters=fixed)
    b = orc.rhs_random(n3[::-1], si.SEED)
    o = orc.bicgstab(b, h, pc=pc, k=k, nslab=bpr, tol=1e-8, fixed_it=fixed, sync2=True)
    assert rep["status_name"] == o.status == "ok"
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(s.scalar_history(), o.scalars)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


def test_sync2_paper_problem_bitwise(bc, orc):
    f, h, faces = si.paper_problem(64)
    s = bc.Solver((64, 64, 64), h, bc=faces)
    s.set_option(bc.OPT_SYNC2, 1)
    s.set_preconditioner("gnocomm", 24)
    s.set_rhs(torch.from_numpy(f).cuda())
    rep = s.solve(tol=1e-10)
    o = orc.bicgstab(f, h, pc="gnocomm", k=24, tol=1e-10, bc=faces, sync2=True)
    assert rep["iterations"] == o.iterations and 10 <= o.iterations <= 40
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


def test_sync2_two_reductions_per_iteration(bc):
    n = 64
    s = bc.Solver(n, si.unit_cube_h(n))
    s.set_preconditioner("gnocomm", 4)
    s.set_rhs_random(si.SEED)
    calls = {}
    for flag in (0, 1):
        s.set_option(bc.OPT_SYNC2, flag)
        s.set_option(bc.OPT_PROFILE, 1)
        s.begin(fixed_iters=10)
        s.kernel_times_reset()
        s.iterate(10)
        kt = s.kernel_times()
        s.finish()
        calls[flag] = kt["finalize"]["calls"]
    assert calls == {0: 30, 1: 20}
    s.close()


def test_sync2_group_two_ranks(bc, orc):
    """Five Dot2 pairs all-gathered per ω stage, combined in rank order (R19)."""
    n3, P = (48, 48, 64), 2
    h = si.unit_cube_h(48)
    grp = bc.local_group(n3, h, P)
    reps, errs = [None] * P, []

    def work(r):
        try:
            grp[r].set_option(bc.OPT_SYNC2, 1)
            grp[r].set_preconditioner("gnocomm", 4)
            grp[r].set_rhs_random(si.SEED)
            reps[r] = grp[r].solve(tol=1e-8)
        except Exception as ex:
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    x = np.concatenate([host(s.solution()) for s in grp])
    hist = grp[1].residual_history()
    for s in grp:
        s.close()
    b = orc.rhs_random(n3[::-1], si.SEED)
    o = orc.bicgstab(b, h, pc="gnocomm", k=4, nslab=P, tol=1e-8, sync2=True)
    assert all(r["iterations"] == o.iterations for r in reps)
    assert np.array_equal(hist, o.history)
    assert np.array_equal(x, o.x)


def test_sync2_needs_fused_path(bc):
    s = bc.Solver(32, si.unit_cube_h(32))
    s.set_option(bc.OPT_SYNC2, 1)
    s.set_option(bc.OPT_KERNELS, 0)
    s.set_preconditioner("gnocomm", 4)
    s.set_rhs_random(si.SEED)
    with pytest.raises(bc.BcgsError):
        s.solve(tol=1e-8)
    s.close()
