"""Pins of the oracle's pipelined Bi-CGSTAB (bcgs_oracle.c pbicgstab, the
paper's "communication-avoiding/reducing algorithms"): the recurrences of the
communication-hiding p-BiCGStab for B = A M^-1 produce Alg. 3's iterates in exact
arithmetic, with two reductions per iteration.

Sources of truth independent of the recurrences: the standard oracle (Alg. 3 as written,
pinned in test_oracle_pins.py): same residual histories to rounding over the first
iterations and the same first-iteration scalars; dense direct solves (the converged
solution, within the tolerance band); the true residual ||b - A x|| (the recurrences for
r, r̂, w, ŵ must stay consistent with x); the MMS_SINE eigenvector RHS (one iteration)."""
import numpy as np
import pytest

import synth_inputs as si
from tests import dense_ref


@pytest.mark.parametrize("n,pc,k,nslab", [(16, "none", 0, 1), (24, "gnocomm", 4, 1),
                                          (24, "gnocomm", 4, 2), (24, "bj", 3, 2),
                                          (24, "g", 4, 2), (20, "gnocomm", 8, 1)])
def test_pipelined_follows_the_standard_iteration(orc, n, pc, k, nslab):
    h = si.unit_cube_h(n)
    b = orc.rhs_random((n, n, n), si.SEED)
    o1 = orc.bicgstab(b, h, pc=pc, k=k, nslab=nslab, tol=1e-8)
    o2 = orc.bicgstab(b, h, pc=pc, k=k, nslab=nslab, tol=1e-8, pipelined=True)
    assert o1.status == o2.status == "ok"
    assert abs(o1.iterations - o2.iterations) <= 2
    m = min(10, o1.iterations, o2.iterations) + 1
    # relative to the residual, floored at 1e-5 of ||b||: once the residual is far below
    # ||b|| the two recurrences differ by rounding of O(u ||b||) (attainable accuracy)
    d = np.abs(o1.history[:m] - o2.history[:m]) / np.maximum(o1.history[:m], 1e-5)
    assert np.max(d) <= 1e-9
    # first iteration: α, tᵀs <-> (q, y), tᵀt <-> (y, y), ω, ρ_new, rᵀr are the same numbers
    for j in (1, 2, 3, 4, 5, 6):
        assert o2.scalars[0, j] == pytest.approx(o1.scalars[0, j], rel=1e-12)
    assert o2.true_rel < 1e-7                          # recurrences consistent with x
    assert np.linalg.norm(o2.x - o1.x) <= 1e-6 * np.linalg.norm(o1.x)


def test_pipelined_solution_equals_dense_solve(orc):
    nx, ny, nz, h = 8, 6, 6, 0.2
    A = dense_ref.assemble(nx, ny, nz, h)
    b = np.random.default_rng(11).standard_normal((nz, ny, nx))
    ref = np.linalg.solve(A, b.ravel()).reshape(b.shape)
    r = orc.bicgstab(b, h, pc="gnocomm", k=3, nslab=1, tol=1e-12, max_it=2000, pipelined=True)
    assert r.status == "ok"
    assert np.linalg.norm(r.x - ref) <= 1e-9 * np.linalg.norm(ref)


def test_pipelined_mms_sine_one_iteration(orc):
    f, u, h = si.mms_sine(24)
    r = orc.bicgstab(f, h, pc="none", k=0, tol=1e-8, pipelined=True)
    assert r.iterations == 1 and r.status == "ok"


def test_pipelined_rejects_flexible_preconditioners(orc):
    n = 8
    b = orc.rhs_random((n, n, n), 1)
    r = orc.bicgstab(b, si.unit_cube_h(n), pc="bj_bicgs", tol=1e-6, pipelined=True)
    assert r.status == "config"
