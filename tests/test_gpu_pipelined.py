"""Pipelined (communication-hiding) Bi-CGSTAB (BCGS_OPT_PIPELINED; NEXT-4; DESIGN.md
R32): the GPU iteration (pipe.cuh kernels, the library's preconditioner and stencil kernels,
two reductions per iteration) against the oracle twin (bcgs_oracle.c pbicgstab, itself pinned
against the standard iteration and dense solves in test_oracle_pipelined.py): histories,
scalars and x bitwise."""
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


@pytest.mark.parametrize("n,pc,k,bpr,kernels,exact", [(32, "none", 0, 1, 1, 0),
                                                      (32, "gnocomm", 4, 1, 1, 0),
                                                      ((40, 36, 48), "gnocomm", 4, 2, 1, 0),
                                                      (48, "bj", 3, 2, 1, 0),
                                                      (32, "gnocomm", 6, 1, 1, 0),
                                                      (32, "gnocomm", 4, 1, 0, 0),
                                                      (32, "gnocomm", 4, 1, 1, 1)])
def test_pipelined_bitwise(bc, orc, n, pc, k, bpr, kernels, exact):
    n3 = (n,) * 3 if np.isscalar(n) else n
    h = si.unit_cube_h(n3[0])
    s = bc.Solver(n3, h)
    s.set_option(bc.OPT_KERNELS, kernels)
    s.set_option(bc.OPT_EXACT_DOT, exact)
    s.set_option(bc.OPT_PIPELINED, 1)
    s.set_preconditioner(pc, k, blocks_per_rank=bpr)
    s.set_rhs_random(si.SEED)
    rep = s.solve(tol=1e-8)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc=pc, k=k, nslab=bpr, tol=1e-8,
                     pipelined=True)
    assert rep["status_name"] == o.status == "ok"
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(s.scalar_history(), o.scalars)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


def test_pipelined_fixed_iterations_256(bc, orc):
    """C2 size, fixed 10 iterations through the split API (graph replay), bitwise."""
    n = 256
    h = si.unit_cube_h(n)
    s = bc.Solver(n, h)
    s.set_option(bc.OPT_PIPELINED, 1)
    s.set_preconditioner("gnocomm", 4)
    s.set_rhs_random(si.SEED)
    s.begin(fixed_iters=10)
    s.iterate(10)
    rep = s.finish()
    o = orc.bicgstab(orc.rhs_random((n, n, n), si.SEED), h, pc="gnocomm", k=4, fixed_it=10,
                     pipelined=True)
    assert rep["iterations"] == 10
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("transport", ["copy"])   # p2p: tests/test_gpu_p2p.py (processes)
def test_pipelined_two_ranks(bc, orc, transport):
    n3, P = (32, 32, 64), 2
    h = si.unit_cube_h(32)
    grp = bc.local_group(n3, h, P, transport=transport)
    reps, errs = [None] * P, []
    setup = threading.Barrier(P)   # set every rank up before any rank enters an exchange

    def work(r):
        try:
            grp[r].set_option(bc.OPT_PIPELINED, 1)
            grp[r].set_preconditioner("gnocomm", 4)
            grp[r].set_rhs_random(si.SEED)
            setup.wait()
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
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=4, nslab=P,
                     tol=1e-8, pipelined=True)
    assert all(r["iterations"] == o.iterations for r in reps)
    assert np.array_equal(hist, o.history)
    assert np.array_equal(x, o.x)


def test_pipelined_rejects_inner_krylov(bc):
    s = bc.Solver(16, 1.0 / 17)
    s.set_option(bc.OPT_PIPELINED, 1)
    s.set_preconditioner("bj_bicgs", 0)
    s.set_rhs_random(1)
    with pytest.raises(bc.BcgsError):
        s.solve(tol=1e-6)
    s.close()
