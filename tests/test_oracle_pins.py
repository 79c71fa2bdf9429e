"""Pins of the CPU oracle against values that do not come from the oracle itself.

Each test names the passage it pins (P:n = PAPER.md line n) and the independent source of
truth: dense Kronecker assembly (Eq. 6), closed-form spectra (Eq. 9-11), closed-form
Chebyshev residual polynomials (Alg. 2), dense direct solves, manufactured solutions,
exact summation, and splitmix64's published test vector.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import synth_inputs as si
from tests import dense_ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rng(seed=0):
    return np.random.default_rng(seed)


# --------------------------------------------------------------------------- inputs / RNG

def test_splitmix64_published_vector(orc):
    vals = [int(l) for l in open(os.path.join(GOLDEN, "splitmix64_vigna.txt"))
            if l.strip() and not l.startswith("#")]
    assert [orc.splitmix64(1234567, g) for g in range(5)] == vals
    g = np.arange(5, dtype=np.uint64)
    assert [int(v) for v in si.splitmix64_np(1234567, g)] == vals


def test_rhs_random_oracle_equals_numpy_generator(orc):
    b_orc = orc.rhs_random((7, 5, 9), 42)
    b_np = si.rhs_random(9, 5, 7, 42)
    assert np.array_equal(b_orc, b_np)
    assert b_orc.min() >= -1.0 and b_orc.max() < 1.0
    # slab of the global field depends only on the global index
    assert np.array_equal(si.rhs_random(9, 5, 7, 42, z0=3, nzl=2), b_np[3:5])


# --------------------------------------------------------------------------- operator

SHAPES = [(1, 1, 1), (1, 1, 3), (2, 1, 1), (3, 4, 2), (5, 3, 4), (4, 6, 6), (6, 5, 4)]


@pytest.mark.parametrize("shape", SHAPES)
def test_apply_A_equals_dense_kronecker(orc, shape):
    """P:95-100 Eq. 6 assembled densely vs the matrix-free stencil, ≤1e-13."""
    nz, ny, nx = shape
    h = 0.37
    A = dense_ref.assemble(nx, ny, nz, h)
    v = rng(1).standard_normal(shape)
    ref = (A @ v.ravel()).reshape(shape)
    out = orc.apply_A(v, h)
    assert np.max(np.abs(out - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("shape,nslab", [((4, 3, 5), 2), ((6, 4, 3), 3), ((8, 2, 2), 4),
                                         ((6, 5, 4), 6)])
def test_block_operator_equals_dense_diagonal_blocks(orc, shape, nslab):
    """Eq. 12-14: the slab-local operator is R_s A R_s^T on each slab."""
    nz, ny, nx = shape
    h = 0.5
    A = dense_ref.block_diag_slabs(dense_ref.assemble(nx, ny, nz, h), nx, ny, nz, nslab)
    v = rng(2).standard_normal(shape)
    ref = (A @ v.ravel()).reshape(shape)
    assert np.max(np.abs(orc.apply_A(v, h, nslab) - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_apply_A_spec_examples(orc):
    # 1x1x1, h = 1 -> 6v: the three 1x1 factors D_1 = [2] summed.
    assert orc.apply_A(np.full((1, 1, 1), 2.5), 1.0)[0, 0, 0] == 15.0
    # 2x1x1, h = 1 -> [[6,-1],[-1,6]]
    e0 = np.array([[[1.0, 0.0]]])
    assert orc.apply_A(e0, 1.0).ravel().tolist() == [6.0, -1.0]


@pytest.mark.parametrize("n,modes", [(6, [(1, 1, 1), (2, 3, 1), (6, 6, 6)]),
                                     (9, [(1, 2, 3), (4, 9, 5)])])
def test_sine_modes_are_eigenvectors_eq9(orc, n, modes):
    """Discrete sine modes are eigenvectors with λ = Σ 4 sin²(aπ/(2(n+1)))/h² (Eq. 7-9)."""
    h = si.unit_cube_h(n)
    x = (np.arange(n) + 1.0) * h
    for a, b, c in modes:
        v = (np.sin(c * np.pi * x)[:, None, None] * np.sin(b * np.pi * x)[None, :, None]
             * np.sin(a * np.pi * x)[None, None, :])
        lam = sum(4.0 * math.sin(m * math.pi / (2 * (n + 1))) ** 2 for m in (a, b, c)) / h**2
        out = orc.apply_A(v, h)
        assert np.max(np.abs(out - lam * v)) <= 1e-12 * lam


def slab_mode(nx, ny, nz, nslab, a, b, c, h):
    """sin(aπx) sin(bπy) sin(cπ(k_loc+1)/(L+1)) in every slab: eigenvector of the block op."""
    L = nz // nslab
    xs = (np.arange(nx) + 1.0) / (nx + 1)
    ys = (np.arange(ny) + 1.0) / (ny + 1)
    zl = (np.arange(nz) % L + 1.0) / (L + 1)
    v = (np.sin(c * np.pi * zl)[:, None, None] * np.sin(b * np.pi * ys)[None, :, None]
         * np.sin(a * np.pi * xs)[None, None, :])
    lam = (4 * math.sin(a * math.pi / (2 * (nx + 1))) ** 2
           + 4 * math.sin(b * math.pi / (2 * (ny + 1))) ** 2
           + 4 * math.sin(c * math.pi / (2 * (L + 1))) ** 2) / h**2
    return v, lam


def test_slab_local_modes_are_block_eigenvectors(orc):
    v, lam = slab_mode(7, 6, 16, 2, 2, 3, 2, 0.1)
    out = orc.apply_A(v, 0.1, 2)
    assert np.max(np.abs(out - lam * v)) <= 1e-12 * lam
    # ... and NOT eigenvectors of the global operator (the cut matters)
    assert np.max(np.abs(orc.apply_A(v, 0.1, 1) - lam * v)) > 1e-3 * lam


def test_operator_symmetry(orc):
    """All-Dirichlet operator is symmetric."""
    shape = (5, 6, 7)
    v, w = rng(3).standard_normal(shape), rng(4).standard_normal(shape)
    h = 0.2
    a = np.vdot(orc.apply_A(v, h), w)
    b = np.vdot(v, orc.apply_A(w, h))
    assert abs(a - b) <= 1e-12 * abs(a)


# --------------------------------------------------------------------------- spectrum

def test_mu_closed_form_values(orc):
    # Eq. 9: n=1 -> {2}; n=2 -> {1, 3}
    assert orc.mu(1, 1) == pytest.approx(2.0, abs=1e-15)
    assert orc.mu(2, 1) == pytest.approx(1.0, abs=1e-15)
    assert orc.mu(2, 2) == pytest.approx(3.0, abs=1e-15)


@pytest.mark.parametrize("nx,ny,nz", [(2, 2, 2), (3, 4, 5), (8, 8, 4), (6, 2, 7)])
def test_bounds_equal_dense_eigensolve(orc, nx, ny, nz):
    """Eq. 10-11 vs numpy eigvalsh of the assembled Eq. 6 matrix."""
    h = 0.3
    ev = np.linalg.eigvalsh(dense_ref.assemble(nx, ny, nz, h))
    lo, hi = orc.bounds(nx, ny, nz, h)
    assert lo == pytest.approx(ev[0], rel=1e-12)
    assert hi == pytest.approx(ev[-1], rel=1e-12)


def test_bounds_spec_and_continuum_limit(orc):
    assert orc.bounds(2, 2, 2, 1.0) == pytest.approx((3.0, 9.0), abs=1e-14)
    for n in (256, 1024):
        lo, hi = orc.bounds(n, n, n, 1.0 / (n + 1))
        assert lo == pytest.approx(3 * math.pi**2, rel=2e-5 * (256 / n) ** 2 + 1e-6)
        assert hi < 12.0 * (n + 1) ** 2          # Gerschgorin: each factor ≤ 4


def test_local_block_bounds_equal_block_eigensolve(orc):
    """BJ(CI) local bounds (R10) = extreme eigenvalues of R_s A R_s^T."""
    nx, ny, nz, nslab, h = 8, 8, 8, 2, 1.0 / 9
    A = dense_ref.assemble(nx, ny, nz, h)
    m = nx * ny * (nz // nslab)
    ev = np.linalg.eigvalsh(A[:m, :m])
    lo, hi = orc.bounds(nx, ny, nz // nslab, h)
    assert lo == pytest.approx(ev[0], rel=1e-12) and hi == pytest.approx(ev[-1], rel=1e-12)
    assert lo == pytest.approx(50.4788, abs=1e-4) and hi == pytest.approx(921.5212, abs=1e-4)


# --------------------------------------------------------------------------- dot products

def _exact_dot(a, b):
    return float(sum((Fraction(x) * Fraction(y) for x, y in zip(a.tolist(), b.tolist())),
                     Fraction(0)))


@pytest.mark.parametrize("case", range(8))
def test_dot_is_correctly_rounded(orc, case):
    """R19: the dot product is RN(Σ a_i b_i) -- checked against exact rational arithmetic
    (Python's Fraction; float(Fraction) rounds to nearest, ties to even), including heavy
    cancellation and a 10^±150 dynamic range where a compensated (Dot2) sum is not exact."""
    r = rng(10 + case)
    n = [1, 7, 100, 1000, 4096, 999, 300, 2000][case]
    a = r.standard_normal(n) * 10.0 ** r.integers(-8, 8, n)
    b = r.standard_normal(n)
    if case >= 3:          # heavy cancellation
        a = np.concatenate([a, -a[: n // 2]])
        b = np.concatenate([b, b[: n // 2] * (1 + 1e-13)])
    if case >= 6:          # huge dynamic range + exact cancellation of the large terms
        big = r.standard_normal(n) * 10.0 ** r.integers(100, 150, n)
        a = np.concatenate([big, a, -big])
        b = np.concatenate([np.ones(n), b, np.ones(n)])
    assert orc.dot(a, b) == _exact_dot(a, b)


def test_dot_is_order_independent(orc):
    r = rng(21)
    a = r.standard_normal(5000) * 10.0 ** r.integers(-20, 20, 5000)
    b = r.standard_normal(5000)
    p = r.permutation(5000)
    assert orc.dot(a, b) == orc.dot(a[p], b[p]) == _exact_dot(a, b)


def test_dot_ties_round_to_even(orc):
    # 1 + 2^-53 is the midpoint of 1 and 1 + 2^-52: ties-to-even gives 1
    assert orc.dot(np.array([1.0, 2.0 ** -53]), np.ones(2)) == 1.0
    # (1 + 2^-52) + 2^-53 is the midpoint of 1 + 2^-52 and 1 + 2^-51: even is 1 + 2^-51
    assert orc.dot(np.array([1.0 + 2.0 ** -52, 2.0 ** -53]), np.ones(2)) == 1.0 + 2.0 ** -51
    # just above the midpoint rounds up
    assert orc.dot(np.array([1.0, 2.0 ** -53, 2.0 ** -200]), np.ones(3)) == 1.0 + 2.0 ** -52


def test_dot_subnormal_overflow_and_nonfinite(orc):
    # each product 2^-1080 underflows to 0 in floating point; their exact sum is 2^-1074
    a = np.full(64, 2.0 ** -540)
    assert _exact_dot(a, a) == 2.0 ** -1074
    assert orc.dot(a, a) == 2.0 ** -1074
    # 3 * 2^-1076 = 0.75 * 2^-1074 rounds to the nearest subnormal 2^-1074
    a = np.full(3, 2.0 ** -538)
    assert orc.dot(a, a) == _exact_dot(a, a) == 2.0 ** -1074
    a = np.array([2.0 ** -537, 2.0 ** -537, 3.0 * 2.0 ** -540])
    assert orc.dot(a, np.ones(3) * 2.0 ** -537) == _exact_dot(a, np.ones(3) * 2.0 ** -537)
    assert orc.dot(np.array([1e300, 1e300]), np.array([1e300, 1e300])) == np.inf
    assert np.isnan(orc.dot(np.array([1.0, np.inf]), np.array([1.0, 1.0])))
    assert np.isnan(orc.dot(np.array([1.0, 2.0]), np.array([np.nan, 1.0])))
    assert orc.dot(np.zeros(10), np.ones(10)) == 0.0


def test_dot2_cancellation_example(orc):
    a = np.array([1e16, 1.0, -1e16, 3.0])
    b = np.ones(4)
    assert orc.dot(a, b) == 4.0       # naive left-to-right sum gives 3.0


def test_dot_plane_split_matches_exact(orc):
    v = rng(5).standard_normal((6, 5, 4))
    w = rng(6).standard_normal((6, 5, 4))
    assert orc.dot(v, w) == _exact_dot(v.ravel(), w.ravel())


# --------------------------------------------------------------------------- Chebyshev

def test_cheb_setup_spec_example(orc):
    c = orc.cheb_setup(1.0, 3.0, 2)                      # θ=2, δ=1, σ=2
    assert (c["theta"], c["delta"], c["sigma"]) == (2.0, 1.0, 2.0)
    assert c["rho"][0] == 0.5                            # ρ_0 = 1/σ
    assert c["rho"][1] == pytest.approx(1.0 / 3.5)       # 1/(2σ - ρ_0)


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4, 7])
def test_cheb_residual_polynomial_closed_form(orc, k):
    """Alg. 2: for an eigenvector v with eigenvalue λ of the operator,
    M^-1 v = ((1 - T_{k+1}((θ-λ)/δ) / T_{k+1}(σ)) / λ) v  (iterMax = k)."""
    n = 8
    h = si.unit_cube_h(n)
    lo, hi = orc.bounds(n, n, n, h)
    a, b = 10 * lo, (1 - 1e-4) * hi
    theta, delta = (b + a) / 2, (b - a) / 2
    x = (np.arange(n) + 1.0) * h
    for (ma, mb, mc) in [(1, 1, 1), (3, 2, 5), (8, 8, 8)]:
        v = (np.sin(mc * np.pi * x)[:, None, None] * np.sin(mb * np.pi * x)[None, :, None]
             * np.sin(ma * np.pi * x)[None, None, :])
        lam = sum(4 * math.sin(m * math.pi / (2 * (n + 1))) ** 2 for m in (ma, mb, mc)) / h**2
        gain = (1.0 - dense_ref.cheb_T(k + 1, (theta - lam) / delta)
                / dense_ref.cheb_T(k + 1, theta / delta)) / lam
        out = orc.apply_cheb(v, h, 1, k, a, b)
        assert np.max(np.abs(out - gain * v)) <= 1e-11 * abs(gain)


def test_cheb_slab_local_closed_form(orc):
    """Same identity on slab-local modes pins the zero-ghost cuts of GNoComm/BJ."""
    nx, ny, nz, nslab, h = 6, 5, 12, 3, 0.1
    v, lam = slab_mode(nx, ny, nz, nslab, 2, 1, 3, h)
    lo, hi = orc.bounds(nx, ny, nz // nslab, h)
    k = 5
    theta, delta = (hi + lo) / 2, (hi - lo) / 2
    gain = (1.0 - dense_ref.cheb_T(k + 1, (theta - lam) / delta)
            / dense_ref.cheb_T(k + 1, theta / delta)) / lam
    out = orc.apply_cheb(v, h, nslab, k, lo, hi)
    assert np.max(np.abs(out - gain * v)) <= 1e-11 * abs(gain)


def test_cheb_k0_and_linearity(orc):
    q = rng(7).standard_normal((6, 4, 5))
    out = orc.apply_cheb(q, 0.2, 2, 0, 3.0, 50.0)
    assert np.array_equal(out, q * (1.0 / 26.5))            # z = b/θ, iterMax = 0
    u, w = rng(8).standard_normal(q.shape), rng(9).standard_normal(q.shape)
    lhs = orc.apply_cheb(2.0 * u - 3.0 * w, 0.2, 2, 4, 30.0, 500.0)
    rhs = 2.0 * orc.apply_cheb(u, 0.2, 2, 4, 30.0, 500.0) - 3.0 * orc.apply_cheb(w, 0.2, 2, 4, 30.0, 500.0)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(lhs))   # fixed, linear


def test_cheb_contraction_bound(orc):
    """||b - A M^-1 b|| ≤ ||b|| / T_{k+1}(σ) when [a, b] contains the spectrum."""
    n, k = 10, 4
    h = si.unit_cube_h(n)
    lo, hi = orc.bounds(n, n, n, h)
    q = rng(11).standard_normal((n, n, n))
    y = orc.apply_cheb(q, h, 1, k, lo, hi)
    res = np.linalg.norm(q - orc.apply_A(y, h))
    sigma = (hi + lo) / (hi - lo)
    assert res <= np.linalg.norm(q) / dense_ref.cheb_T(k + 1, sigma) * (1 + 1e-10)


def test_cheb_spec_scalar_example(orc):
    """1x1x1 grid, h=1 (A = [6]), interval [1, 11] (θ=6): the polynomial is exact at λ=θ
    for every k ≥ 0 since T_{k+1}(0)/T_{k+1}(σ) has (θ-λ)=0: residual factor T(0)/T(σ)."""
    for k in range(5):
        out = orc.apply_cheb(np.ones((1, 1, 1)), 1.0, 1, k, 1.0, 11.0)[0, 0, 0]
        gain = (1 - dense_ref.cheb_T(k + 1, 0.0) / dense_ref.cheb_T(k + 1, 6.0 / 5.0)) / 6.0
        assert out == pytest.approx(float(gain), rel=1e-14)


# --------------------------------------------------------------------------- Bi-CGSTAB

def test_bicgstab_1x1x1(orc):
    """1x1x1, h=1, b=1 -> x = 1/6 in one iteration."""
    res = orc.bicgstab(np.ones((1, 1, 1)), 1.0, tol=1e-12)
    assert res.status == "ok" and res.iterations == 1
    assert res.x[0, 0, 0] == pytest.approx(1 / 6, rel=1e-15)


@pytest.mark.parametrize("pc,nslab", [("none", 1), ("gnocomm", 1), ("gnocomm", 2),
                                      ("bj", 2), ("bj", 1)])
def test_bicgstab_matches_dense_solve(orc, pc, nslab):
    """The converged iterate solves Eq. 6's system: compare with a dense LU solve."""
    nz, ny, nx = 8, 6, 7
    h = 0.125
    b = orc.rhs_random((nz, ny, nx), 3)
    A = dense_ref.assemble(nx, ny, nz, h)
    x_ref = np.linalg.solve(A, b.ravel()).reshape(b.shape)
    res = orc.bicgstab(b, h, pc=pc, nslab=nslab, k=3, tol=1e-12)
    assert res.status == "ok"
    cond = np.linalg.cond(A)
    err = np.linalg.norm(res.x - x_ref) / np.linalg.norm(x_ref)
    assert err <= cond * 1e-12 * 10
    assert res.true_rel < 1e-11


def test_recurrence_residual_equals_true_residual(orc):
    """Alg. 3 invariant: r_i = b - A x_i in exact arithmetic; checks every x/r update sign."""
    n = 10
    h = si.unit_cube_h(n)
    b = orc.rhs_random((n, n, n), 5)
    A = dense_ref.assemble(n, n, n, h)
    for pc in ("none", "gnocomm"):
        for it in (1, 2, 5):
            res = orc.bicgstab(b, h, pc=pc, k=4, fixed_it=it)
            true = np.linalg.norm(b.ravel() - A @ res.x.ravel()) / np.linalg.norm(b)
            assert res.history[it] == pytest.approx(true, rel=1e-9)


def test_first_iteration_scalars_unpreconditioned(orc):
    """Iteration 1 with M = I: α = bᵀb / bᵀAb, ω = (As)ᵀs/(As)ᵀ(As), s = b - αAb (Alg. 1
    P:153-166), evaluated with the dense Eq. 6 matrix."""
    n, h = 6, 1.0 / 7
    b = orc.rhs_random((n, n, n), 9).ravel()
    A = dense_ref.assemble(n, n, n, h)
    res = orc.bicgstab(b.reshape(n, n, n), h, fixed_it=1)
    alpha = (b @ b) / (b @ (A @ b))
    s = b - alpha * (A @ b)
    t = A @ s
    omega = (t @ s) / (t @ t)
    rw, a1, ts, tt, om1 = res.scalars[0, :5]
    assert a1 == pytest.approx(alpha, rel=1e-12)
    assert om1 == pytest.approx(omega, rel=1e-10)
    x1 = alpha * b + omega * s
    assert np.max(np.abs(res.x.ravel() - x1)) <= 1e-10 * np.max(np.abs(x1))


def test_mms_poly_exact_discrete_solution(orc):
    """u = Π(x_d - x_d²) is reproduced exactly by the 7-point stencil: x ≈ u at the nodes."""
    f, u, h = si.mms_poly(16)
    res = orc.bicgstab(f, h, tol=1e-13, max_it=500)
    assert res.status == "ok"
    assert np.linalg.norm(res.x - u) / np.linalg.norm(u) < 1e-10


def test_mms_sine_closed_form_error(orc):
    """Sine MMS is an exact discrete eigenvector: x = u·3π²/λ_min after one iteration, so
    the error equals |3π²/λ_min - 1| (7.5559e-4 at 32³)."""
    n = 32
    f, u, h = si.mms_sine(n)
    res = orc.bicgstab(f, h, tol=1e-8)
    lam_min = 3 * 4 * math.sin(math.pi / (2 * (n + 1))) ** 2 / h**2
    err = np.linalg.norm(res.x - u) / np.linalg.norm(u)
    assert res.iterations == 1
    assert err == pytest.approx(abs(3 * math.pi**2 / lam_min - 1), rel=1e-10)
    assert err == pytest.approx(7.5559e-4, rel=1e-4)


def test_mms_polyexp_second_order(orc):
    """O(h²) discretisation error (Eq. 3 is second order): error ratio ≈ 4 per halving."""
    errs = []
    for n in (15, 31):
        f, u, h = si.mms_polyexp(n)
        res = orc.bicgstab(f, h, tol=1e-12, max_it=2000, pc="gnocomm", k=4)
        assert res.status == "ok"
        errs.append(np.linalg.norm(res.x - u) / np.linalg.norm(u))
    assert 3.7 < errs[0] / errs[1] < 4.3


def test_boundary_values_constant_solution(orc):
    """Constant Dirichlet data g on all faces and f = 0: the discrete solution is u ≡ g."""
    n, g = 9, 2.5
    h = si.unit_cube_h(n)
    b = orc.fold_boundary(np.zeros((n, n, n)), h, [g] * 6)
    res = orc.bicgstab(b, h, tol=1e-13)
    assert np.max(np.abs(res.x - g)) < 1e-10


def test_boundary_fold_matches_dense_elimination(orc):
    """Different values per face: fold == moving the ghost column of Eq. 3 to the RHS."""
    nx, ny, nz, h = 4, 3, 5, 0.25
    g6 = [1.0, -2.0, 0.5, 3.0, -1.5, 0.25]
    b = orc.fold_boundary(np.zeros((nz, ny, nx)), h, g6)
    # extended grid with ghost layer holding the boundary values; apply full-grid stencil
    ext = np.zeros((nz + 2, ny + 2, nx + 2))
    ext[:, :, 0], ext[:, :, -1] = g6[0], g6[1]
    ext[:, 0, :], ext[:, -1, :] = g6[2], g6[3]
    ext[0, :, :], ext[-1, :, :] = g6[4], g6[5]
    # The ghosts' contribution to (A u)_c is -(sum of ghost neighbours)/h²; folding moves
    # it to the right-hand side: b_c = +(sum of ghost neighbours)/h².
    ghost_sum = (ext[1:-1, 1:-1, :-2] + ext[1:-1, 1:-1, 2:] + ext[1:-1, :-2, 1:-1]
                 + ext[1:-1, 2:, 1:-1] + ext[:-2, 1:-1, 1:-1] + ext[2:, 1:-1, 1:-1])
    assert np.allclose(b, ghost_sum / h**2, rtol=1e-14, atol=0)


def test_preconditioning_reduces_iterations(orc):
    """Table II ordering at desk scale: CI variants beat none."""
    n = 24
    h = si.unit_cube_h(n)
    b = orc.rhs_random((n, n, n), si.SEED)
    none = orc.bicgstab(b, h, pc="none").iterations
    gn = orc.bicgstab(b, h, pc="gnocomm", k=4).iterations
    bj = orc.bicgstab(b, h, pc="bj", k=4, nslab=2).iterations
    assert gn < none and bj < none


def test_bj_with_global_bounds_equals_gnocomm(orc):
    """GNoComm(CI) ≡ BJ(CI) with the global (rescaled) eigenvalues."""
    n = 12
    h = si.unit_cube_h(n)
    b = orc.rhs_random((n, n, n), 1)
    lo, hi = orc.bounds(n, n, n, h)
    g = orc.bicgstab(b, h, pc="gnocomm", k=4, nslab=3, fixed_it=6)
    j = orc.bicgstab(b, h, pc="bj", k=4, nslab=3, fixed_it=6,
                     bounds_override=(10.0 * lo, (1 - 1e-4) * hi))
    assert np.array_equal(g.x, j.x) and np.array_equal(g.history, j.history)


def test_fixed_iteration_mode_and_history_shape(orc):
    n = 8
    b = orc.rhs_random((n, n, n), 2)
    res = orc.bicgstab(b, si.unit_cube_h(n), pc="gnocomm", fixed_it=5)
    assert res.iterations == 5 and len(res.history) == 6 and res.history[0] == 1.0
    assert np.all(np.isfinite(res.history))


def test_zero_rhs(orc):
    res = orc.bicgstab(np.zeros((3, 3, 3)), 0.25)
    assert res.status == "ok" and res.iterations == 0 and not res.x.any()


def test_initial_guess_reading_r26(orc):
    """R26: exact initial guess -> converged, 0 iterations; rel_0 = ||b - A x0|| / ||b||."""
    n, h = 6, 1.0 / 7
    b = orc.rhs_random((n, n, n), 4)
    A = dense_ref.assemble(n, n, n, h)
    xs = np.linalg.solve(A, b.ravel()).reshape(b.shape)
    res = orc.bicgstab(b, h, x0=xs, tol=1e-8)
    assert res.status == "ok" and res.iterations == 0
    x0 = xs + 0.01 * np.random.default_rng(0).standard_normal(xs.shape)
    res = orc.bicgstab(b, h, x0=x0, tol=1e-12)
    rel0 = np.linalg.norm(b.ravel() - A @ x0.ravel()) / np.linalg.norm(b)
    assert res.history[0] == pytest.approx(rel0, rel=1e-12)
    assert np.linalg.norm(res.x - xs) / np.linalg.norm(xs) < 1e-9


def test_gci_is_decomposition_independent_and_beats_gnocomm(orc):
    """G(CI) applies the global Chebyshev polynomial: its iterates do not depend
    on the slab count (bitwise), equal GNoComm on one slab, and on P slabs it needs
    no more iterations than GNoComm (Table II: 50 vs 140 at 64 ranks)."""
    n = 24
    h = si.unit_cube_h(n)
    b = orc.rhs_random((n, n, n), si.SEED)
    g1 = orc.bicgstab(b, h, pc="g", k=4, nslab=1)
    g4 = orc.bicgstab(b, h, pc="g", k=4, nslab=4)
    gn1 = orc.bicgstab(b, h, pc="gnocomm", k=4, nslab=1)
    gn4 = orc.bicgstab(b, h, pc="gnocomm", k=4, nslab=4)
    assert np.array_equal(g1.history, g4.history) and np.array_equal(g1.x, g4.x)
    assert np.array_equal(g1.x, gn1.x)
    assert g4.iterations <= gn4.iterations


@pytest.mark.parametrize("pc,k", [("none", 0), ("gnocomm", 4)])
def test_r7_breakdown_on_nonfinite_rw(orc, pc, k):
    """R7 (paper silent): a non-finite r~ᵀw stops the solve before any update of that
    iteration with BREAKDOWN and iterations = i - 1.  Constructed exactly: b = 1e300 at one
    point makes bᵀb overflow (exact sum beyond the double range -> +inf, R19), so
    ||b|| = inf, rel_0 = inf/inf = NaN, and r~ᵀw = Σ b_i (A p̂)_i overflows at iteration 1."""
    n = 16
    b = np.zeros((n, n, n))
    b[5, 6, 7] = 1e300
    r = orc.bicgstab(b, si.unit_cube_h(n), pc=pc, k=k, tol=1e-8)
    assert r.status == "breakdown" and r.iterations == 0
    assert len(r.history) == 1 and np.isnan(r.history[0])
    assert not r.x.any()                      # no update was applied
