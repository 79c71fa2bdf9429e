"""Pins of the oracle's 2-sync rewrite (DESIGN.md §3 R31): r~ᵀr and rᵀr of
Alg. 3 l.21-22 from the a9 reduction via the identities r = s - ω t,
r~ᵀr = r~ᵀs - ω r~ᵀt, ||r||² = sᵀs - 2ω tᵀs + ω² tᵀt, which removes MPI5.

Sources of truth independent of the rewrite: the standard (explicit-dot) oracle, itself pinned
in test_oracle_pins.py (same iterate sequence up to rounding: histories within 1e-8 over the
first 10 iterations, iteration counts +-2), dense solves (the converged solution), and the
MMS_SINE one-iteration exact solve (the clamp of a cancelled ||r||² at 0)."""
import numpy as np
import pytest

import synth_inputs as si
from tests import dense_ref


@pytest.mark.parametrize("pc,k,nslab", [("none", 0, 1), ("gnocomm", 4, 1), ("gnocomm", 4, 2),
                                        ("bj", 3, 2), ("g", 4, 1)])
def test_sync2_follows_the_standard_iteration(orc, pc, k, nslab):
    n = 24
    h = si.unit_cube_h(n)
    b = orc.rhs_random((n, n, n), si.SEED)
    o1 = orc.bicgstab(b, h, pc=pc, k=k, nslab=nslab, tol=1e-8)
    o2 = orc.bicgstab(b, h, pc=pc, k=k, nslab=nslab, tol=1e-8, sync2=True)
    assert o1.status == o2.status == "ok"
    assert abs(o1.iterations - o2.iterations) <= 2
    m = min(10, o1.iterations, o2.iterations) + 1
    assert np.max(np.abs(o1.history[:m] - o2.history[:m]) / o1.history[:m]) <= 1e-8
    # every scalar of the first iterations (rw, α, tᵀs, tᵀt, ω, ρ_new, rᵀr, β)
    rel = np.abs(o1.scalars[:3] - o2.scalars[:3]) / np.maximum(np.abs(o1.scalars[:3]), 1e-300)
    assert np.max(rel) <= 1e-9
    assert o2.true_rel < 1e-8


def test_sync2_solution_equals_dense_solve(orc):
    nx, ny, nz, h = 8, 6, 5, 0.2
    A = dense_ref.assemble_bc(nx, ny, nz, h, si.PAPER_BC)
    b = np.random.default_rng(9).standard_normal((nz, ny, nx))
    ref = np.linalg.solve(A, b.ravel()).reshape(b.shape)
    r = orc.bicgstab(b, h, pc="gnocomm", k=3, nslab=1, tol=1e-12, max_it=2000, bc=si.PAPER_BC,
                     sync2=True)
    assert r.status == "ok"
    assert np.max(np.abs(r.x - ref)) <= 1e-9 * np.max(np.abs(ref))


def test_sync2_exact_one_iteration_clamps(orc):
    """MMS_SINE is an exact eigenvector: s = r - αw cancels to rounding noise in iteration 1,
    sᵀs - 2ω tᵀs + ω² tᵀt is then noise of either sign; the clamp at 0 gives rel ~ 0 and the
    closed-form discretisation error (7.5559e-4 at 32³)."""
    f, u, h = si.mms_sine(32)
    r = orc.bicgstab(f, h, pc="none", tol=1e-8, sync2=True)
    assert r.status == "ok" and r.iterations == 1
    assert np.isfinite(r.history).all() and r.history[1] < 1e-8
    err = np.max(np.abs(r.x - u)) / np.max(np.abs(u))
    assert err == pytest.approx(7.5559e-4, rel=1e-3)
