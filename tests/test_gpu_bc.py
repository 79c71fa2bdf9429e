"""GPU-vs-oracle parity of the mixed Dirichlet/Neumann path (DESIGN.md §3
R27-R28): mirror ghosts in every kernel family (reference sweeps, streaming stencil+dot,
square-tile and TMA temporally blocked Chebyshev kernels), the mixed Chebyshev interval, the
Neumann-flux fold, whole solves and the paper's own §IV workload.  Bitwise."""
import threading

import numpy as np
import pytest

import synth_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BCS = [si.PAPER_BC, (1, 1, 0, 0, 0, 0), (0, 0, 1, 1, 0, 0), (0, 0, 0, 0, 1, 1),
       (1, 0, 0, 1, 0, 1), (1, 1, 1, 1, 1, 0)]


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


@pytest.mark.parametrize("faces", BCS)
@pytest.mark.parametrize("block_local,bpr", [(0, 1), (1, 2)])
def test_operator_bc_bitwise(bc, orc, faces, block_local, bpr):
    n3 = (34, 18, 20)
    h = 0.11
    s = bc.Solver(n3, h, bc=faces)
    s.set_preconditioner("gnocomm", 1, blocks_per_rank=bpr)
    v = np.random.default_rng(1).standard_normal(n3[::-1])
    out = host(s.apply_operator(dev(v), block_local=bool(block_local)))
    assert np.array_equal(out, orc.apply_A(v, h, bpr if block_local else 1, bc=faces))


@pytest.mark.parametrize("kernels", [0, 1])
@pytest.mark.parametrize("variant", [2, 7])
@pytest.mark.parametrize("pc,k,bpr", [("gnocomm", 1, 1), ("gnocomm", 4, 2), ("bj", 3, 2),
                                      ("g", 4, 1), ("gnocomm", 5, 1), ("bj", 8, 2)])
@pytest.mark.parametrize("faces", [si.PAPER_BC, (1, 1, 1, 1, 1, 0)])
def test_preconditioner_bc_bitwise(bc, orc, faces, pc, k, bpr, variant, kernels):
    """Every kernel family with mirror ghosts; (70, 52, 40) has ragged tiles in x and y."""
    n3 = (70, 52, 40)
    h = 0.2
    s = bc.Solver(n3, h, bc=faces)
    s.set_option(bc.OPT_KERNELS, kernels)
    s.set_option(bc.OPT_TB_VARIANT, variant)
    s.set_preconditioner(pc, k, blocks_per_rank=bpr)
    q = np.random.default_rng(2).standard_normal(n3[::-1])
    out = host(s.apply_preconditioner(dev(q)))
    nslab = 1 if pc == "g" else bpr
    ivl = orc.pc_interval(n3[::-1], h, nslab, pc, bc=faces)   # the oracle's own interval
    ref = orc.apply_cheb(q, h, 1 if pc == "g" else bpr, k, ivl[0], ivl[1], bc=faces)
    assert np.array_equal(out, ref)


def test_preconditioner_bc_odd_nx(bc, orc):
    """odd nx: no TMA (16-byte rows) -> square-tile mirror kernel."""
    n3, h, k = (45, 33, 24), 0.3, 4
    s = bc.Solver(n3, h, bc=si.PAPER_BC)
    s.set_preconditioner("gnocomm", k)
    q = np.random.default_rng(5).standard_normal(n3[::-1])
    ivl = orc.pc_interval(n3[::-1], h, 1, "gnocomm", bc=si.PAPER_BC)
    assert np.array_equal(host(s.apply_preconditioner(dev(q))),
                          orc.apply_cheb(q, h, 1, k, ivl[0], ivl[1], bc=si.PAPER_BC))


def solve_pair(bc, orc, n3, h, faces, pc, k, bpr=1, kernels=1, tol=1e-10, fixed=0, b=None,
               g6=None):
    s = bc.Solver(n3, h, bc=faces)
    s.set_option(bc.OPT_KERNELS, kernels)
    s.set_preconditioner(pc, k, blocks_per_rank=bpr)
    if b is None:
        b = orc.rhs_random(n3[::-1], si.SEED)
    if g6 is not None:
        for f in range(6):
            s.set_boundary_value(f, g6[f])
    s.set_rhs(dev(b))
    rep = s.solve(tol=tol, max_iter=3000, fixed_iters=fixed)
    bf = b if g6 is None else orc.fold_boundary(b, h, g6, bc=faces)
    o = orc.bicgstab(bf, h, pc=pc, k=k, nslab=bpr, tol=tol, max_it=3000, fixed_it=fixed,
                     bc=faces)
    return s, rep, o


@pytest.mark.parametrize("kernels", [0, 1])
@pytest.mark.parametrize("pc,k,bpr", [("none", 0, 1), ("gnocomm", 4, 1), ("gnocomm", 4, 4),
                                      ("bj", 3, 2), ("g", 2, 1)])
def test_solve_bc_bitwise(bc, orc, pc, k, bpr, kernels):
    n3, h = (48, 40, 32), 0.05
    s, rep, o = solve_pair(bc, orc, n3, h, si.PAPER_BC, pc, k, bpr, kernels)
    assert rep["status_name"] == o.status == "ok"
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)


def test_neumann_flux_fold_bitwise(bc, orc):
    """R28: non-zero Neumann derivatives and Dirichlet values folded on the device."""
    n3, h = (32, 24, 16), 0.07
    faces = si.PAPER_BC
    g6 = [0.5, -1.25, 2.0, 0.75, -0.3, 1.1]
    b = orc.rhs_random(n3[::-1], si.SEED)
    s, rep, o = solve_pair(bc, orc, n3, h, faces, "gnocomm", 4, fixed=6, b=b, g6=g6)
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)


@pytest.mark.parametrize("kernels", [0, 1])
def test_paper_problem_64(bc, orc, kernels):
    """§IV workload at 64³, GNoComm(CI) k = 24, (10, 1-1e-4), tol 1e-10:
    identical iterations / history / solution to the oracle; 14 iterations in the paper
    (P:444), band 10-40."""
    f, h, faces = si.paper_problem(64)
    s, rep, o = solve_pair(bc, orc, (64, 64, 64), h, faces, "gnocomm", 24, kernels=kernels,
                           b=f)
    assert rep["status_name"] == "ok" and 10 <= rep["iterations"] <= 40
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    assert rep["true_rel_residual"] < 1e-9


@pytest.mark.parametrize("k", [4, 8])
def test_paper_problem_128_fused(bc, orc, k):
    """§IV workload at 128³ through the temporally blocked kernels (k <= 8), bitwise."""
    f, h, faces = si.paper_problem(128)
    s, rep, o = solve_pair(bc, orc, (128, 128, 128), h, faces, "gnocomm", k, b=f)
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)


@pytest.mark.parametrize("P,pc,k", [(2, "gnocomm", 4), (4, "gnocomm", 3), (2, "g", 4),
                                    (4, "g", 4), (4, "bj", 2)])
@pytest.mark.parametrize("kernels", [0, 1])
def test_local_group_bc(bc, orc, P, pc, k, kernels):
    """Neumann z faces on the first / last rank only; halos + mirrors across P slabs."""
    n3 = (40, 32, 32)
    f, h, faces = si.paper_problem(32)
    f = np.ascontiguousarray(np.broadcast_to(f[:, :, :1], (32, 32, 40)) +
                             np.random.default_rng(3).standard_normal((32, 32, 40)))
    grp = bc.local_group(n3, h, P, bc=faces)
    L = n3[2] // P
    reps, errs = [None] * P, []

    def work(r):
        try:
            s = grp[r]
            s.set_option(bc.OPT_KERNELS, kernels)
            s.set_preconditioner(pc, k)
            s.set_rhs(dev(f[r * L:(r + 1) * L]))
            reps[r] = s.solve(tol=1e-10)
        except Exception as ex:
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    x = np.concatenate([s.solution().cpu().numpy() for s in grp])
    hist = grp[0].residual_history()
    for s in grp:
        s.close()
    o = orc.bicgstab(f, h, pc=pc, k=k, nslab=P, tol=1e-10, bc=faces)
    assert reps[0]["iterations"] == o.iterations
    assert np.array_equal(hist, o.history)
    assert np.array_equal(x, o.x)


def test_bc_config_errors(bc):
    with pytest.raises(bc.BcgsError):
        bc.Solver((1, 8, 8), 0.1, bc=(1, 0, 0, 0, 0, 0))          # Neumann axis of 1 point
    s = bc.Solver((8, 8, 8), 0.1, bc=(0, 0, 0, 0, 1, 0))
    with pytest.raises(bc.BcgsError):
        s.set_preconditioner("gnocomm", 2, blocks_per_rank=8)   # 1-plane block at a z face


def _random_bc_configs(count, seed=20251019):
    """Seeded mixed-face configurations: each face Dirichlet or Neumann (never all six
    Neumann: singular), extents >= 2 along a Neumann axis and >= 2 planes per block with a
    Neumann z face (R27), odd and even nx, every preconditioner kind."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        faces = tuple(int(v) for v in rng.integers(0, 2, size=6))
        if sum(faces) == 6:
            continue
        n3 = [int(rng.integers(2, 48)) for _ in range(3)]
        pc = ["gnocomm", "bj", "g", "none"][int(rng.integers(0, 4))]
        k = 0 if pc == "none" else int(rng.integers(1, 9))
        divs = [d for d in range(1, 5) if n3[2] % d == 0 and n3[2] // d >= 2]
        bpr = 1 if pc == "g" else int(rng.choice(divs))
        out.append((tuple(n3), faces, pc, k, bpr))
    return out


@pytest.mark.parametrize("n3,faces,pc,k,bpr", _random_bc_configs(16))
def test_random_bc_configs_bitwise(bc, orc, n3, faces, pc, k, bpr):
    """Seeded random mixed Dirichlet / Neumann problems: 6 fixed iterations bitwise vs the
    oracle (mirror ghosts in every kernel family, mixed Chebyshev intervals, c_min = 1)."""
    h = 0.09
    s = bc.Solver(n3, h, bc=faces)
    s.set_preconditioner(pc, k, c_min=1.0, blocks_per_rank=bpr)
    b = orc.rhs_random(n3[::-1], si.SEED)
    s.set_rhs(dev(b))
    rep = s.solve(fixed_iters=6)
    o = orc.bicgstab(b, h, pc=pc, k=k, nslab=bpr, fixed_it=6, bc=faces, c_min=1.0)
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()
