"""Multi-pass temporal blocking: degrees above the one-pass
kernels (the paper's k = 24) run as passes of 2-4 Chebyshev sweeps (Alg. 2 / Alg. 4,
P:216-233), each pass handing the last two iterates x_{j-1}, x_{j-2} to the next.
Same expression trees in the same sweep order as the oracle -> bitwise identical."""
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


def apply_pair(bc, orc, n3, h, pc, k, bpr, mp_min=None, faces=None):
    s = bc.Solver(n3, h, bc=faces) if faces else bc.Solver(n3, h)
    if mp_min is not None:
        s.set_option(bc.OPT_MULTIPASS, mp_min)
    s.set_option(bc.OPT_PROFILE, 1)
    s.set_preconditioner(pc, k, blocks_per_rank=bpr)
    q = np.random.default_rng(7).standard_normal(n3[::-1])
    s.kernel_times_reset()
    out = host(s.apply_preconditioner(dev(q)))
    kt = s.kernel_times()
    ivl = orc.pc_interval(n3[::-1], h, bpr, pc, bc=faces)   # the oracle's own interval
    ref = orc.apply_cheb(q, h, bpr, k, ivl[0], ivl[1], bc=faces)
    return out, ref, kt


@pytest.mark.parametrize("k,mp_min", [(5, 4), (6, 4), (7, 4), (8, 4), (9, None), (13, None),
                                      (16, None), (24, None)])
@pytest.mark.parametrize("n3,bpr", [((66, 46, 18), 1), ((40, 24, 32), 2)])
def test_multipass_preconditioner_bitwise(bc, orc, n3, bpr, k, mp_min):
    out, ref, kt = apply_pair(bc, orc, n3, 0.05, "gnocomm", k, bpr, mp_min)
    assert "fused_p_cheb" in kt and "precond_sweep" not in kt, kt   # the blocked path ran
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("pc,k,bpr", [("bj", 12, 2), ("g", 10, 1)])
def test_multipass_other_preconditioners(bc, orc, pc, k, bpr):
    out, ref, _ = apply_pair(bc, orc, (48, 40, 36), 1.0 / 37, pc, k, bpr if pc != "g" else 1)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("faces,k", [(si.PAPER_BC, 24), ((1, 1, 1, 1, 1, 0), 11)])
def test_multipass_mixed_bc_bitwise(bc, orc, faces, k):
    out, ref, kt = apply_pair(bc, orc, (70, 52, 40), 0.2, "gnocomm", k, 2, faces=faces)
    assert "precond_sweep" not in kt
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("n,k,bpr", [(64, 16, 1), (64, 24, 1), (48, 12, 4)])
def test_multipass_solve_bitwise(bc, orc, n, k, bpr):
    """Whole solves through the fused iteration (p-kernel and s-kernel passes, CUDA graph)."""
    h = si.unit_cube_h(n)
    s = bc.Solver(n, h)
    s.set_preconditioner("gnocomm", k, blocks_per_rank=bpr)
    s.set_rhs_random(si.SEED)
    rep = s.solve(tol=1e-8)
    b = orc.rhs_random((n, n, n), si.SEED)
    o = orc.bicgstab(b, h, pc="gnocomm", k=k, nslab=bpr, tol=1e-8)
    assert rep["converged"] and rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(s.scalar_history(), o.scalars)
    assert np.array_equal(host(s.solution()), o.x)


def test_multipass_equals_one_pass(bc):
    """k = 8 both ways (one-pass square-tile kernel vs 2 passes of 4): bitwise equal."""
    n3, h = (64, 64, 48), 1.0 / 65
    q = dev(np.random.default_rng(3).standard_normal(n3[::-1]))
    outs = []
    for mp in (64, 4):
        s = bc.Solver(n3, h)
        s.set_option(bc.OPT_MULTIPASS, mp)
        s.set_preconditioner("gnocomm", 8)
        outs.append(s.apply_preconditioner(q).clone())
    assert torch.equal(outs[0], outs[1])
