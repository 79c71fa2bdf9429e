"""R19: every dot product of the solver is the correctly rounded value
RN(Σ a_i b_i).  The library certifies its Dot2 results with a rigorous error bound and
recomputes the rest exactly (superaccumulator, xdot.cuh); the oracle sums exactly.  These
tests drive the exact path on purpose -- inputs where no compensated sum is certifiable, and
BCGS_OPT_EXACT_DOT = 1, which sends every reduction through it -- and compare bitwise with
the oracle (and with the certified path)."""
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


def hard_vectors(n3, seed):
    """Cancellation-heavy dot over a huge dynamic range: terms of 10^100..10^150 that cancel
    exactly plus O(1) terms -- Dot2's error bound is ~u^2 * 10^150, so nothing certifies."""
    r = np.random.default_rng(seed)
    shape = n3[::-1]
    a = r.standard_normal(shape)
    b = r.standard_normal(shape)
    m = a.size // 4
    big = r.standard_normal(m) * 10.0 ** r.integers(100, 150, m)
    af, bf = a.reshape(-1), b.reshape(-1)
    af[:m] = big
    af[m:2 * m] = -big
    bf[:m] = 1.0
    bf[m:2 * m] = 1.0
    return a, b


@pytest.mark.parametrize("n3", [(9, 7, 5), (64, 48, 40), (130, 66, 24)])
def test_uncertifiable_dot_goes_exact(bc, orc, n3):
    s = bc.Solver(n3, 0.1)
    a, b = hard_vectors(n3, 5)
    v = s.dot(dev(a), dev(b))
    assert v == orc.dot(a, b)
    assert s.exact_dots() >= 1          # the certification refused Dot2 here
    s.close()


@pytest.mark.parametrize("n3", [(64, 48, 40), (130, 66, 24)])
def test_certified_and_forced_exact_agree(bc, orc, n3):
    r = np.random.default_rng(9)
    a = r.standard_normal(n3[::-1]) * 10.0 ** r.integers(-6, 6, n3[::-1])
    b = r.standard_normal(n3[::-1])
    s = bc.Solver(n3, 0.1)
    v0 = s.dot(dev(a), dev(b))
    s.set_option(bc.OPT_EXACT_DOT, 1)
    v1 = s.dot(dev(a), dev(b))
    assert v0 == v1 == orc.dot(a, b)
    s.close()


def test_nonfinite_dot_is_nan(bc):
    s = bc.Solver((16, 16, 16), 0.1)
    a = np.ones((16, 16, 16))
    a[3, 4, 5] = np.inf
    assert np.isnan(s.dot(dev(a), dev(np.ones((16, 16, 16)))))
    s.close()


@pytest.mark.parametrize("n,pc,k,bpr,kernels,sync2", [(32, "gnocomm", 4, 1, 1, 0),
                                                      (48, "bj", 3, 2, 1, 0),
                                                      (32, "none", 0, 1, 1, 0),
                                                      (40, "gnocomm", 4, 2, 0, 0),
                                                      (32, "gnocomm", 4, 1, 1, 1)])
def test_forced_exact_solve_bitwise(bc, orc, n, pc, k, bpr, kernels, sync2):
    """Every reduction parked and resolved exactly (host round trips per stage, resumed
    iterations, graph replays as no-ops while parked): the same iterates as the oracle."""
    h = si.unit_cube_h(n)
    s = bc.Solver(n, h)
    s.set_option(bc.OPT_KERNELS, kernels)
    s.set_option(bc.OPT_SYNC2, sync2)
    s.set_option(bc.OPT_EXACT_DOT, 1)
    s.set_preconditioner(pc, k, blocks_per_rank=bpr)
    s.set_rhs_random(si.SEED)
    rep = s.solve(tol=1e-8)
    b = orc.rhs_random((n, n, n), si.SEED)
    o = orc.bicgstab(b, h, pc=pc, k=k, nslab=bpr, tol=1e-8, sync2=bool(sync2))
    assert rep["iterations"] == o.iterations
    assert s.exact_dots() >= 3 * o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(s.scalar_history(), o.scalars)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


def test_forced_exact_fixed_iterations_through_begin_iterate_finish(bc, orc):
    """Fixed-iteration mode (the bench's split API): the iterations enqueued while a stage
    was parked are enqueued again after the resolution -- all of them run."""
    n, k = 32, 4
    h = si.unit_cube_h(n)
    s = bc.Solver(n, h)
    s.set_option(bc.OPT_EXACT_DOT, 1)
    s.set_preconditioner("gnocomm", k)
    s.set_rhs_random(si.SEED)
    s.begin(fixed_iters=7)
    s.iterate(3)
    s.iterate(4)
    rep = s.finish()
    assert rep["iterations"] == 7
    o = orc.bicgstab(orc.rhs_random((n, n, n), si.SEED), h, pc="gnocomm", k=k, fixed_it=7)
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


@pytest.mark.parametrize("P,pc,kernels", [(2, "gnocomm", 1), (4, "gnocomm", 1), (2, "g", 0),
                                          (2, "g", 1), (4, "bj", 0)])
def test_forced_exact_multirank_bitwise(bc, orc, P, pc, kernels):
    """In-process ranks: the superaccumulators are all-gathered and summed as integers; every
    stage parks, and the iterations enqueued meanwhile (including G(CI)'s k-deep halos and
    extended-slab copies) must leave the fields the resumed iteration needs untouched."""
    n3 = (32, 32, 64)
    h = si.unit_cube_h(32)
    grp = bc.local_group(n3, h, P)
    reps, errs = [None] * P, []

    def work(r):
        try:
            grp[r].set_option(bc.OPT_EXACT_DOT, 1)
            grp[r].set_option(bc.OPT_KERNELS, kernels)
            grp[r].set_preconditioner(pc, 4)
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
    hist = grp[0].residual_history()
    for s in grp:
        s.close()
    b = orc.rhs_random(n3[::-1], si.SEED)
    o = orc.bicgstab(b, h, pc=pc, k=4, nslab=P, tol=1e-8)
    assert all(r["iterations"] == o.iterations for r in reps)
    assert np.array_equal(hist, o.history)
    assert np.array_equal(x, o.x)


@pytest.mark.parametrize("sync2,fixed", [(0, 0), (1, 45)])
def test_certification_holds_deep_into_the_solve(bc, orc, sync2, fixed):
    """The certified path carries whole solves without the exact fallback: the r~ dots grow
    ill-conditioned as Bi-CGSTAB converges (r~ᵀs of the 2-sync rewrite reaches
    Σ|ab|/|Σab| ~ 1e20 after 20-40 iterations), which Dot3 plus a renormalised final sum
    still certifies.  Results are bitwise the oracle's either way."""
    n = 64
    h = si.unit_cube_h(n)
    s = bc.Solver(n, h)
    s.set_option(bc.OPT_SYNC2, sync2)
    s.set_preconditioner("gnocomm", 4)
    s.set_rhs_random(si.SEED)
    rep = s.solve(tol=1e-8, fixed_iters=fixed)
    assert s.exact_dots() == 0, s.certification_info()
    o = orc.bicgstab(orc.rhs_random((n, n, n), si.SEED), h, pc="gnocomm", k=4, tol=1e-8,
                     fixed_it=fixed, sync2=bool(sync2))
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()
