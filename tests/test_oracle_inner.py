"""Pins of the oracle's inner-Krylov preconditioners FBiCGS-BJ(BiCGS) / FBiCGS-G(BiCGS)
(Eq. 12-15, inner settings P:393-394; DESIGN.md §3 R29).

Sources of truth independent of oracle/: dense block matrices of Eq. 6 / Eq. 5 and their
direct solves (numpy LAPACK), a separately written numpy flexible Bi-CGSTAB (Alg. 1)
with the EXACT block-Jacobi inverse of Eq. 13 as preconditioner, and the iteration counts
the inner cap implies."""
import numpy as np
import pytest

import synth_inputs as si
from tests import dense_ref


def rng(seed=0):
    return np.random.default_rng(seed)


def block_solve(A, b, nslab):
    """Eq. 15 exactly: (R_s A R_s^T)^{-1} p_s per block by LU."""
    m = A.shape[0] // nslab
    out = np.empty_like(b)
    for s in range(nslab):
        sl = slice(s * m, (s + 1) * m)
        out[sl] = np.linalg.solve(A[sl, sl], b[sl])
    return out


def fbicgstab_numpy(A, b, Minv, tol, max_it):
    """Alg. 1 with a right preconditioner applied as p̂ = M⁻¹p, r̂ = M⁻¹s."""
    x = np.zeros_like(b)
    r = b.copy()
    rt = r.copy()
    p = r.copy()
    rho = rt @ r
    nb = np.linalg.norm(b)
    hist = [1.0]
    for i in range(1, max_it + 1):
        ph = Minv(p)
        w = A @ ph
        alpha = rho / (rt @ w)
        s = r - alpha * w
        rh = Minv(s)
        t = A @ rh
        omega = (t @ s) / (t @ t)
        x = x + alpha * ph + omega * rh
        r = s - omega * t
        hist.append(np.linalg.norm(r) / nb)
        if hist[-1] < tol:
            return x, i, np.array(hist)
        rho_new = rt @ r
        beta = (rho_new / rho) * (alpha / omega)
        rho = rho_new
        p = r + beta * (p - omega * w)
    return x, max_it, np.array(hist)


@pytest.mark.parametrize("nslab", [1, 2, 4])
@pytest.mark.parametrize("bc", [None, si.PAPER_BC])
def test_inner_apply_solves_each_block(orc, nslab, bc):
    """One application = the block solve of Eq. 15 to the inner tolerance: the block residual
    is below tol·|p_s| (the inner recurrence residual is tested, the true one agrees to
    rounding) and the result equals the LU block solve within cond·tol."""
    nx, ny, nz, h = 6, 5, 8, 0.2
    bc6 = bc or (0,) * 6
    A = dense_ref.assemble_bc(nx, ny, nz, h, bc6)
    Ab = dense_ref.block_diag_slabs(A, nx, ny, nz, nslab)
    q = rng(3).standard_normal((nz, ny, nx))
    tol = 1e-9
    out, its = orc.apply_inner(q, h, nslab, tol, 500, bc=bc)
    ref = block_solve(A, q.ravel(), nslab)
    m = nx * ny * nz // nslab
    for s in range(nslab):
        sl = slice(s * m, (s + 1) * m)
        res = np.linalg.norm(q.ravel()[sl] - Ab[sl, sl] @ out.ravel()[sl])
        assert res <= 1.01 * tol * np.linalg.norm(q.ravel()[sl])
    cond = np.linalg.cond(A[:m, :m])
    assert np.linalg.norm(out.ravel() - ref) <= cond * tol * np.linalg.norm(ref)
    assert its >= nslab


def test_inner_cap_counts(orc):
    """max_in caps every block solve: a 3-iteration cap on 4 blocks = 12 inner iterations."""
    q = rng(4).standard_normal((16, 8, 8))
    _, its = orc.apply_inner(q, 0.1, 4, 1e-14, 3)
    assert its == 12


def test_inner_zero_block(orc):
    """p_s = 0 on a block gives p̂_s = 0 without iterating (R26)."""
    q = rng(5).standard_normal((8, 6, 6))
    q[:4] = 0.0
    out, its = orc.apply_inner(q, 0.1, 2, 1e-8, 500)
    assert np.all(out[:4] == 0.0) and np.any(out[4:] != 0.0)


def test_g_bicgs_exact_inner_is_one_iteration(orc):
    """G(BiCGS) with an inner tolerance near machine precision is M⁻¹ ≈ A⁻¹: the outer
    iteration converges at i = 1 (α ≈ 1, s ≈ 0), to the dense solution."""
    n = 8
    h = si.unit_cube_h(n)
    b = orc.rhs_random((n, n, n), si.SEED)
    r = orc.bicgstab(b, h, pc="g_bicgs", tol=1e-8, inner_tol=1e-14, inner_max=2000)
    A = dense_ref.assemble(n, n, n, h)
    ref = np.linalg.solve(A, b.ravel()).reshape(b.shape)
    assert r.status == "ok" and r.iterations == 1
    assert np.max(np.abs(r.x - ref)) <= 1e-10 * np.max(np.abs(ref))


@pytest.mark.parametrize("nslab", [2, 4])
def test_bj_bicgs_tight_inner_equals_exact_block_jacobi(orc, nslab):
    """BJ(BiCGS) with a tight inner tolerance follows the flexible Bi-CGSTAB with the EXACT
    block-Jacobi inverse (Eq. 13, LU): same iteration count, histories agree to ~1e-8."""
    nx, ny, nz = 8, 6, 8
    h = 1.0 / 9
    A = dense_ref.assemble(nx, ny, nz, h)
    b = orc.rhs_random((nz, ny, nx), si.SEED)
    x_ref, it_ref, hist_ref = fbicgstab_numpy(A, b.ravel(), lambda v: block_solve(A, v, nslab),
                                              1e-8, 200)
    r = orc.bicgstab(b, h, pc="bj_bicgs", nslab=nslab, tol=1e-8, inner_tol=1e-13,
                     inner_max=2000)
    assert r.status == "ok"
    assert abs(r.iterations - it_ref) <= 1
    m = min(len(hist_ref), len(r.history))
    assert np.max(np.abs(r.history[:m] - hist_ref[:m]) / hist_ref[:m]) <= 1e-6
    assert np.linalg.norm(r.x.ravel() - x_ref) <= 1e-7 * np.linalg.norm(x_ref)


@pytest.mark.parametrize("pc,nslab", [("bj_bicgs", 2), ("g_bicgs", 1)])
def test_paper_inner_settings_converge_to_dense_solution(orc, pc, nslab):
    """P:393-394 settings (BJ: 1e-6 / 500, G: 1e-2 / 500) with mixed faces: the outer solve
    reaches tol and the dense Eq. 5/6 solution within κ·tol."""
    nx, ny, nz, h = 8, 6, 8, 0.2
    A = dense_ref.assemble_bc(nx, ny, nz, h, si.PAPER_BC)
    b = rng(8).standard_normal((nz, ny, nx))
    ref = np.linalg.solve(A, b.ravel()).reshape(b.shape)
    r = orc.bicgstab(b, h, pc=pc, nslab=nslab, tol=1e-10, max_it=500, bc=si.PAPER_BC)
    assert r.status == "ok" and r.extra["inner_iterations"] > 0
    kappa = np.linalg.cond(A)
    assert np.linalg.norm(r.x - ref) <= kappa * 1e-10 * np.linalg.norm(ref)
    assert r.true_rel < 1e-9
