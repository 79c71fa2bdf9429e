"""GPU-vs-oracle parity through the C ABI (libbcgs.so), on seeded synthetic inputs.

Bars (BASELINE.json north_star): per-iteration relative residuals within 1e-9 over the first
20 iterations, converged solution within 1e-8 relative L2, iteration count to 1e-8 within
±1.  With the arithmetic contract the expected outcome is bitwise identity;
single-operator tests demand it.
"""
import numpy as np
import pytest

import synth_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KERNELS = [0, 1]          # 0 = reference kernels, 1 = fused / temporally blocked


@pytest.fixture(scope="module")
def bc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_08935_b200 import bcgs
    bcgs.load()
    return bcgs


def make(bc, n, h=None, kernels=1, **pc):
    n3 = (n,) * 3 if np.isscalar(n) else tuple(n)
    h = si.unit_cube_h(n3[0]) if h is None else h
    s = bc.Solver(n3, h)
    s.set_option(bc.OPT_KERNELS, kernels)
    if pc:
        s.set_preconditioner(**pc)
    return s, n3, h


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


# --------------------------------------------------------------------------- single steps

@pytest.mark.parametrize("n", [8, (37, 29, 23), 64])
def test_rhs_random_bitwise(bc, orc, n):
    """R16 device generator == oracle generator: with M = I, iteration 1 gives
    x1 = α b + ω s, which exposes every bit of b (history, scalars and x compared)."""
    out = compare_solve(bc, orc, n, pc="none", k=0, fixed=1)
    assert_parity(*out)


@pytest.mark.parametrize("n", [(33, 17, 20), 48, (64, 64, 40)])
@pytest.mark.parametrize("block_local,bpr", [(0, 1), (1, 2), (1, 4)])
def test_operator_bitwise(bc, orc, n, block_local, bpr):
    s, n3, h = make(bc, n, pc="none", degree=0, blocks_per_rank=1)
    s.set_preconditioner("gnocomm", 1, blocks_per_rank=bpr)
    v = np.random.default_rng(1).standard_normal(n3[::-1])
    out = host(s.apply_operator(dev(v), block_local=bool(block_local)))
    ref = orc.apply_A(v, h, bpr if block_local else 1)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("kernels", KERNELS)
@pytest.mark.parametrize("pc,k,bpr", [("gnocomm", 0, 1), ("gnocomm", 1, 1), ("gnocomm", 2, 2),
                                      ("gnocomm", 4, 1), ("gnocomm", 4, 4), ("bj", 3, 2),
                                      ("bj", 7, 1), ("gnocomm", 8, 2)])
@pytest.mark.parametrize("n", [(40, 24, 32), (67, 45, 16)])
def test_preconditioner_bitwise(bc, orc, n, pc, k, bpr, kernels):
    s, n3, h = make(bc, n, kernels=kernels, pc=pc, degree=k, blocks_per_rank=bpr)
    q = np.random.default_rng(2).standard_normal(n3[::-1])
    out = host(s.apply_preconditioner(dev(q)))
    ivl = orc.pc_interval(n3[::-1], h, bpr, pc)   # the oracle's own interval (R9, R10)
    ref = orc.apply_cheb(q, h, bpr, k, ivl[0], ivl[1])
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("n", [(9, 7, 5), 64, (130, 66, 24)])
def test_dot_equals_oracle(bc, orc, n):
    s, n3, h = make(bc, n)
    r = np.random.default_rng(3)
    a = r.standard_normal(n3[::-1]) * 10.0 ** r.integers(-6, 6, n3[::-1])
    b = r.standard_normal(n3[::-1])
    assert s.dot(dev(a), dev(b)) == orc.dot(a, b)


# --------------------------------------------------------------------------- whole solves

def compare_solve(bc, orc, n, pc="gnocomm", k=4, bpr=1, kernels=1, tol=1e-8, fixed=0,
                  rhs=None, max_it=5000, c_min=10.0):
    s, n3, h = make(bc, n, kernels=kernels)
    s.set_preconditioner(pc, k, c_min=c_min, blocks_per_rank=bpr)
    if rhs is None:
        s.set_rhs_random(si.SEED)
        b = orc.rhs_random(n3[::-1], si.SEED)
    else:
        b, h = rhs
        s.set_rhs(dev(b))
    rep = s.solve(tol=tol, max_iter=max_it, fixed_iters=fixed)
    g_hist = s.residual_history()
    g_scal = s.scalar_history()
    g_x = host(s.solution())
    o = orc.bicgstab(b, h, pc=pc, k=k, nslab=bpr, tol=tol, max_it=max_it, fixed_it=fixed,
                     c_min=c_min)
    return rep, g_hist, g_scal, g_x, o


def assert_parity(rep, g_hist, g_scal, g_x, o, bitwise=True):
    assert rep["status_name"] == o.status
    assert abs(rep["iterations"] - o.iterations) <= 1
    m = min(21, len(g_hist), len(o.history))
    rel = np.abs(g_hist[:m] - o.history[:m]) / np.abs(o.history[:m])
    assert np.max(rel) <= 1e-9, rel
    err = np.linalg.norm(g_x - o.x) / np.linalg.norm(o.x)
    assert err <= 1e-8
    if bitwise:
        assert rep["iterations"] == o.iterations
        assert np.array_equal(g_hist, o.history)
        assert np.array_equal(g_scal, o.scalars)
        assert np.array_equal(g_x, o.x)


def test_c1_mms_polyexp_unpreconditioned(bc, orc):
    """BASELINE config C1: 32³, manufactured solution, unpreconditioned, to 1e-8."""
    f, u, h = si.mms_polyexp(32)
    out = compare_solve(bc, orc, 32, pc="none", k=0, rhs=(f, h))
    assert_parity(*out)
    rep, x = out[0], out[3]
    assert rep["converged"] and rep["true_rel_residual"] < 1e-7
    err = np.linalg.norm(x - u) / np.linalg.norm(u)
    assert err == pytest.approx(4.56e-4, rel=0.05)       # O(h²) discretisation error


@pytest.mark.parametrize("kernels", KERNELS)
@pytest.mark.parametrize("n,pc,k,bpr", [(32, "gnocomm", 4, 1), (48, "gnocomm", 4, 2),
                                        (64, "gnocomm", 4, 4), (64, "bj", 4, 2),
                                        ((40, 36, 48), "gnocomm", 3, 3), (32, "none", 0, 1),
                                        (64, "gnocomm", 8, 1)])
def test_solve_parity(bc, orc, n, pc, k, bpr, kernels):
    assert_parity(*compare_solve(bc, orc, n, pc, k, bpr, kernels))


@pytest.mark.parametrize("n,pc,k,bpr", [((1, 1, 1), "none", 0, 1), ((2, 1, 3), "gnocomm", 2, 1),
                                        ((3, 5, 1), "none", 0, 1), ((1, 7, 2), "bj", 3, 2),
                                        ((5, 4, 3), "gnocomm", 4, 3), ((2, 2, 9), "gnocomm", 4, 3),
                                        ((66, 1, 1), "gnocomm", 4, 1), ((2, 130, 2), "gnocomm", 3, 1)])
def test_solve_parity_degenerate_grids(bc, orc, n, pc, k, bpr):
    """Degenerate extents: a single unknown, one-plane slabs and blocks, 1-point lines along
    each axis, slab blocks thinner than the degree (R24 warning case), odd / even nx --
    every kernel family's edge handling (TMA boxes larger than the grid, one-tile grids,
    the stencil chunk model at 1-3 planes), bitwise vs the oracle.  GNoComm with c_min = 1:
    these spectra are narrower than R9's default rescaling c_min / c_max ~ 10 (next test)."""
    assert_parity(*compare_solve(bc, orc, n, pc, k, bpr, 1, c_min=1.0))


def _random_configs(count, seed=20251018):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        n3 = tuple(int(rng.integers(1, 5)) if rng.random() < 0.25 else int(rng.integers(5, 72))
                   for _ in range(3))
        pc = ["gnocomm", "bj", "g", "none"][int(rng.integers(0, 4))]
        k = 0 if pc == "none" else int(rng.integers(1, 9))
        bpr = int(rng.choice([d for d in range(1, 5) if n3[2] % d == 0]))
        if pc == "g":
            bpr = 1
        out.append((n3, pc, k, bpr))
    return out


@pytest.mark.parametrize("n3,pc,k,bpr", _random_configs(24))
def test_random_configs_fixed_iterations_bitwise(bc, orc, n3, pc, k, bpr):
    """Seeded random extents (1..71 per axis, a quarter of them 1..4; odd and even nx),
    preconditioners, degrees 1-8 and block counts: 6 fixed iterations bitwise vs the oracle
    (c_min = 1 keeps every rescaled interval non-empty)."""
    s, _, h = make(bc, n3)
    try:
        s.set_preconditioner(pc, k, c_min=1.0, blocks_per_rank=bpr)
    except bc.BcgsError as ex:   # a spectrum with a single eigenvalue (all axes of length 1)
        a, b = orc.pc_interval(n3[::-1], h, bpr, pc, c_min=1.0)
        assert "spectrum" in str(ex) and not a < b
        return
    s.set_rhs_random(si.SEED)
    rep = s.solve(fixed_iters=6)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc=pc, k=k, nslab=bpr, fixed_it=6,
                     c_min=1.0)
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


@pytest.mark.parametrize("n", [(1, 1, 1), (66, 1, 1)])
def test_narrow_spectrum_rejects_default_rescaling(bc, orc, n):
    """R9: a' = c_min λmin, b' = c_max λmax is empty when λmax / λmin < c_min / c_max -- the
    library refuses with BCGS_E_SPECTRUM, as the oracle's interval is empty too."""
    s, n3, h = make(bc, n)
    a, b = orc.pc_interval(n3[::-1], h, 1, "gnocomm")
    assert not a < b
    with pytest.raises(bc.BcgsError, match="spectrum"):
        s.set_preconditioner("gnocomm", 4)
    s.close()


@pytest.mark.parametrize("kernels", KERNELS)
def test_solve_parity_128(bc, orc, kernels):
    assert_parity(*compare_solve(bc, orc, 128, "gnocomm", 4, 1, kernels))


@pytest.mark.parametrize("n,pc,k,bpr", [(64, "gnocomm", 1, 1), (64, "gnocomm", 4, 8),
                                        (128, "gnocomm", 4, 8), (128, "bj", 4, 8),
                                        (128, "gnocomm", 8, 2), (64, "bj", 16, 4)])
def test_solve_parity_matrix(bc, orc, n, pc, k, bpr):
    """SURVEY §8(c) parity matrix rows not covered above: GNoComm k = 1, P = 8 slab blocks
    (8 / 16 planes), BJ at P = 8, and multi-pass degrees, full solves to 1e-8, bitwise."""
    assert_parity(*compare_solve(bc, orc, n, pc, k, bpr, 1))


def test_c2_256_eight_slabs_first_20(bc, orc):
    """256³ with 8 slab blocks (the P = 8 preconditioner of SURVEY §8(c)), 20 iterations."""
    assert_parity(*compare_solve(bc, orc, 256, "gnocomm", 4, 8, 1, fixed=20))


@pytest.mark.parametrize("kernels", KERNELS)
def test_c2_256_first_20_iterations(bc, orc, kernels):
    """Config C2 (256³, Chebyshev degree 4): first 20 iterations, bitwise."""
    assert_parity(*compare_solve(bc, orc, 256, "gnocomm", 4, 1, kernels, fixed=20))


def _big(bc, orc, n, pc, k, bpr, fixed):
    out = compare_solve(bc, orc, n, pc, k, bpr, 1, fixed=fixed)
    assert out[0]["iterations"] == fixed == out[4].iterations
    assert_parity(*out)
    torch.cuda.empty_cache()


def test_c3_512_first_20_iterations(bc, orc):
    """Config C3 at full size (512³, GNoComm(CI) k = 4, P = 1: the bench launch
    configuration): the north_star window of 20 iterations -- every residual, every scalar
    (r~ᵀw, α, tᵀs, tᵀt, ω, ρ, rᵀr, β) and every element of x bitwise equal to the oracle."""
    _big(bc, orc, 512, "gnocomm", 4, 1, 20)


def test_c3_512_eight_slabs_first_20_iterations(bc, orc):
    """512³ GNoComm(CI) k = 4 on 8 slab blocks (the 8-GPU preconditioner emulated with
    blocks_per_rank = 8, SURVEY §8(c) row "512³ | 1, 8"): 20 iterations bitwise."""
    _big(bc, orc, 512, "gnocomm", 4, 8, 20)


def test_c4_512_block_jacobi_first_20_iterations(bc, orc):
    """Config C4 at full size: BJ(CI) k = 4 with local exact bounds (R10) on 8 slab blocks:
    20 iterations bitwise."""
    _big(bc, orc, 512, "bj", 4, 8, 20)


def test_c4_512_block_jacobi_one_block_first_20_iterations(bc, orc):
    """Config C4 at P = 1: BJ(CI) k = 4 (= G(CI) with unscaled bounds): 20 iterations."""
    _big(bc, orc, 512, "bj", 4, 1, 20)


def test_graph_replay_matches_direct(bc):
    outs = []
    for graph in (0, 1):
        s, n3, h = make(bc, 64, pc="gnocomm", degree=4)
        s.set_option(bc.OPT_GRAPH, graph)
        s.set_rhs_random(7)
        rep = s.solve(tol=1e-8)
        outs.append((rep["iterations"], s.residual_history(), host(s.solution())))
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1], outs[1][1]) and np.array_equal(outs[0][2], outs[1][2])


def test_boundary_values_and_initial_guess(bc, orc):
    n, g = 24, 1.5
    h = si.unit_cube_h(n)
    s, n3, _ = make(bc, n, pc="gnocomm", degree=4)
    for f in range(6):
        s.set_boundary_value(f, g)
    s.set_rhs(dev(np.zeros((n, n, n))))
    rep = s.solve(tol=1e-12)
    x = host(s.solution())
    assert rep["converged"] and np.max(np.abs(x - g)) < 1e-9
    b = orc.fold_boundary(np.zeros((n, n, n)), h, [g] * 6)
    o = orc.bicgstab(b, h, pc="gnocomm", k=4, tol=1e-12)
    assert np.array_equal(x, o.x)
    # warm start from the exact solution: converged before the first iteration (R26)
    x0 = np.full((n, n, n), g)
    s.set_initial_guess(dev(x0))
    rep2 = s.solve(tol=1e-8)
    assert rep2["converged"] and rep2["iterations"] == 0
    # perturbed warm start: bitwise parity with the oracle's r0 = b - A x0 path
    x0 = x0 + 1e-3 * np.random.default_rng(4).standard_normal(x0.shape)
    s.set_initial_guess(dev(x0))
    rep3 = s.solve(tol=1e-10)
    o3 = orc.bicgstab(b, h, pc="gnocomm", k=4, tol=1e-10, x0=x0)
    assert rep3["iterations"] == o3.iterations
    assert np.array_equal(s.residual_history(), o3.history)
    assert np.array_equal(host(s.solution()), o3.x)


def test_zero_rhs_and_breakdown_reporting(bc):
    s, n3, h = make(bc, 16, pc="gnocomm", degree=2)
    s.set_rhs(dev(np.zeros((16, 16, 16))))
    rep = s.solve(tol=1e-8)
    assert rep["converged"] and rep["iterations"] == 0
    assert not host(s.solution()).any()


def test_mms_sine_one_iteration(bc):
    f, u, h = si.mms_sine(32)
    s, n3, _ = make(bc, 32, pc="none", degree=0)
    s.set_rhs(dev(f))
    rep = s.solve(tol=1e-8)
    assert rep["iterations"] == 1


def test_recurrence_equals_true_residual_any_size(bc):
    """Property that holds at any size: after a few iterations the recurrence residual
    equals ||b - A x||/||b|| to rounding (checked at the bench size 512³ too)."""
    for n in (96, 512):
        s, n3, h = make(bc, n, pc="gnocomm", degree=4)
        s.set_rhs_random(si.SEED)
        rep = s.solve(fixed_iters=5)
        assert rep["true_rel_residual"] == pytest.approx(rep["rel_residual"], rel=1e-6)
        del s
        torch.cuda.empty_cache()


@pytest.mark.slow
def test_c2_256_full_solve(bc, orc):
    """Config C2 (256³, Chebyshev degree 4) solved to 1e-8: iterations, every residual and
    the converged x bitwise equal to the oracle (bars: 1e-9 / 1e-8 / ±1)."""
    assert_parity(*compare_solve(bc, orc, 256, "gnocomm", 4, 1, 1))


def test_c3_512_k24_multipass_first_iteration(bc, orc):
    """The paper's degree k = 24 at 512³ through the multi-pass kernels (6 passes per
    application, full-size launch configuration): iteration 1 bitwise."""
    assert_parity(*compare_solve(bc, orc, 512, "gnocomm", 24, 1, 1, fixed=1))


def _host_ram_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 2**30
    except ImportError:
        return 0.0


def test_c5_1024_eight_slabs_first_5_iterations(bc, orc):
    """Config C5 size (1024³, GNoComm(CI) k = 4 on 8 slab blocks = the 8-GPU decomposition):
    SURVEY §8(c) row "1024³ | 8 | first 5 iterations", bitwise against the oracle (the GPU
    holds 15 fields of 8 GiB; the oracle ~12 fields + b, x in host RAM)."""
    free_hbm = torch.cuda.mem_get_info()[0] / 2**30
    if _host_ram_gb() < 150 or free_hbm < 135:
        pytest.skip(f"needs ~150 GiB host RAM and ~135 GiB HBM (have {_host_ram_gb():.0f}, "
                    f"{free_hbm:.0f})")
    _big(bc, orc, 1024, "gnocomm", 4, 8, 5)


def test_c5_1024_properties(bc):
    """Config C5 size (1024³; 8 slabs as on 8 GPUs): properties that hold at any size --
    the recurrence residual equals ||b - A x||/||b||, and residuals decrease."""
    s, n3, h = make(bc, 1024, pc="gnocomm", degree=4, blocks_per_rank=8)
    s.set_rhs_random(si.SEED)
    rep = s.solve(fixed_iters=4)
    hist = s.residual_history()
    assert rep["true_rel_residual"] == pytest.approx(rep["rel_residual"], rel=1e-6)
    assert np.all(np.diff(hist) < 0)
    s.close()
    del s
    torch.cuda.empty_cache()


@pytest.mark.parametrize("variant", [2, 7])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_tb_variants_bitwise(bc, orc, variant, k):
    """Every temporally blocked layout (square tile / TMA warp-row 24 warps) gives the
    oracle's Chebyshev application bitwise, including ragged tiles and a block cut."""
    n3 = (70, 52, 40)
    h = si.unit_cube_h(70)
    s = bc.Solver(n3, h)
    s.set_option(bc.OPT_TB_VARIANT, variant)
    s.set_preconditioner("gnocomm", k, blocks_per_rank=2)
    q = np.random.default_rng(7).standard_normal(n3[::-1])
    out = host(s.apply_preconditioner(dev(q)))
    ivl = orc.pc_interval(n3[::-1], h, 2, "gnocomm")
    assert np.array_equal(out, orc.apply_cheb(q, h, 2, k, ivl[0], ivl[1]))


@pytest.mark.parametrize("n3,bpr,k", [((70, 52, 40), 2, 4), ((132, 90, 33), 1, 3),
                                      ((64, 200, 48), 3, 2)])
def test_tb_segment_schedule_bitwise(bc, orc, n3, bpr, k):
    """Segment scheduling of the temporally blocked kernel (BCGS_OPT_TB_SCHEDULE = 2: one CTA
    per SM, parts spanning tile and block boundaries) gives the oracle's Chebyshev
    application and iterates bitwise (p-update + M^-1 p, s-update + M^-1 s)."""
    h = si.unit_cube_h(n3[0])
    s = bc.Solver(n3, h)
    s.set_option(bc.OPT_TB_SCHEDULE, 2)
    s.set_preconditioner("gnocomm", k, blocks_per_rank=bpr)
    q = np.random.default_rng(11).standard_normal(n3[::-1])
    ivl = orc.pc_interval(n3[::-1], h, bpr, "gnocomm")
    assert np.array_equal(host(s.apply_preconditioner(dev(q))),
                          orc.apply_cheb(q, h, bpr, k, ivl[0], ivl[1]))
    s.set_rhs_random(si.SEED)
    rep = s.solve(fixed_iters=12)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=k, nslab=bpr,
                     fixed_it=12)
    assert rep["iterations"] == o.iterations == 12
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


@pytest.mark.parametrize("n3,bpr", [((70, 52, 40), 2), ((64, 64, 64), 1)])
def test_pdl_launch_chain_bitwise(bc, orc, n3, bpr):
    """BCGS_OPT_PDL = 1 (programmatic dependent launches inside the captured iteration):
    iterates bitwise equal to the oracle's."""
    h = si.unit_cube_h(n3[0])
    s = bc.Solver(n3, h)
    s.set_option(bc.OPT_PDL, 1)
    s.set_preconditioner("gnocomm", 4, blocks_per_rank=bpr)
    s.set_rhs_random(si.SEED)
    rep = s.solve(tol=1e-8)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=4, nslab=bpr,
                     tol=1e-8)
    assert rep["converged"] and rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


@pytest.mark.parametrize("zc", [4, 5, 13, 64])
def test_stencil_chunk_lengths_bitwise(bc, orc, zc):
    """The TMA stencil+dot with forced chunk lengths (BCGS_OPT_STENCIL = planes per CTA;
    ragged last chunks, chunks longer than the block) -- iterates bitwise the oracle's."""
    n3 = (96, 80, 70)
    h = si.unit_cube_h(n3[0])
    s = bc.Solver(n3, h)
    s.set_option(bc.OPT_STENCIL, zc)
    s.set_preconditioner("gnocomm", 4, blocks_per_rank=2)
    s.set_rhs_random(si.SEED)
    rep = s.solve(fixed_iters=10)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=4, nslab=2,
                     fixed_it=10)
    assert rep["iterations"] == o.iterations == 10
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


def test_c2_256_segment_schedule_bitwise(bc, orc):
    """Config C2 (256³, k = 4, one GPU) runs the segment schedule by default (77 tiles on 148
    SMs); first 5 iterations bitwise equal to the oracle's."""
    n = 256
    h = si.unit_cube_h(n)
    s = bc.Solver(n, h)
    s.set_preconditioner("gnocomm", 4)
    s.set_rhs_random(si.SEED)
    rep = s.solve(fixed_iters=5)
    o = orc.bicgstab(orc.rhs_random((n, n, n), si.SEED), h, pc="gnocomm", k=4, fixed_it=5)
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


def test_unpreconditioned_streaming_path(bc, orc):
    """M = I on the fused path: no p̂ / r̂ copies (no precond_sweep launches), bitwise oracle."""
    n = 48
    h = si.unit_cube_h(n)
    s = bc.Solver(n, h)
    s.set_preconditioner("none", 0)
    s.set_option(bc.OPT_PROFILE, 1)
    s.set_rhs_random(si.SEED)
    rep = s.solve(tol=1e-8)
    kt = s.kernel_times()
    assert "precond_sweep" not in kt and kt["update_p"]["calls"] >= rep["iterations"] - 1
    o = orc.bicgstab(orc.rhs_random((n, n, n), si.SEED), h, pc="none", tol=1e-8)
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


def test_phase_times_spec_keys(bc):
    """bcgs_get_phase_times: the SPEC's six phase keys from the profiled kernels --
    every phase of a one-rank fused iteration but the halo is timed, total = their sum."""
    s, n3, h = make(bc, 64, pc="gnocomm", degree=4)
    s.set_rhs_random(si.SEED)
    s.set_option(bc.OPT_PROFILE, 1)
    s.kernel_times_reset()
    s.solve(fixed_iters=5)
    ph = s.phase_times()
    assert tuple(ph) == bc.PHASE_KEYS
    for key in ("preconditioner", "allreduce", "stencil_kernels", "vector_kernels"):
        assert ph[key] > 0, (key, ph)
    assert ph["halo_exchange"] == 0.0
    parts = sum(v for k, v in ph.items() if k != "total")
    assert ph["total"] == pytest.approx(parts, rel=1e-12)
    kt = s.kernel_times()
    assert ph["preconditioner"] == pytest.approx(kt["fused_p_cheb"]["ms"] + kt["fused_s_cheb"]["ms"],
                                                 rel=1e-12)
    s.close()


def test_schedule_and_stencil_options_validated(bc):
    """BCGS_OPT_TB_SCHEDULE takes 0..2, BCGS_OPT_STENCIL 0..64 (>= 2: planes per CTA; 64 keeps
    the stencil dots' per-thread chains inside the certification depth, R19)."""
    s, n3, h = make(bc, 16, pc="gnocomm", degree=2)
    for opt, bad in ((bc.OPT_TB_SCHEDULE, 3), (bc.OPT_TB_SCHEDULE, -1), (bc.OPT_STENCIL, -1),
                     (bc.OPT_STENCIL, 65), (bc.OPT_STENCIL, 5000)):
        with pytest.raises(bc.BcgsError):
            s.set_option(opt, bad)
    for opt, good in ((bc.OPT_TB_SCHEDULE, 1), (bc.OPT_STENCIL, 2), (bc.OPT_STENCIL, 0)):
        s.set_option(opt, good)
    s.close()


def test_tb_variant_option_rejects_removed_layouts(bc):
    s, n3, h = make(bc, 16, pc="gnocomm", degree=2)
    for v in (5, 8, 9, 10):
        with pytest.raises(bc.BcgsError):
            s.set_option(bc.OPT_TB_VARIANT, v)


@pytest.mark.parametrize("n3,pc,k,bpr", [((64, 48, 40), "gnocomm", 4, 1),
                                         ((130, 66, 24), "none", 0, 1),
                                         ((96, 80, 70), "bj", 3, 2),
                                         ((192, 34, 65), "gnocomm", 2, 5)])
def test_stencil_tma_equals_l1_kernel_and_oracle(bc, orc, n3, pc, k, bpr):
    """The TMA-staged stencil+dot kernels (st_tma.cu: 64 x 16 tiles, 32-plane chunks; ragged
    in x, y and z here) give the L1 kernels' and the oracle's iterates bitwise."""
    h = si.unit_cube_h(n3[0])
    outs = []
    for tma in (0, 1):
        s = bc.Solver(n3, h)
        s.set_option(bc.OPT_STENCIL, tma)
        s.set_preconditioner(pc, k, blocks_per_rank=bpr)
        s.set_rhs_random(si.SEED)
        s.solve(fixed_iters=6)
        outs.append((s.residual_history(), s.scalar_history(), host(s.solution())))
        s.close()
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc=pc, k=k, nslab=bpr, fixed_it=6)
    for hist, scal, x in outs:
        assert np.array_equal(hist, o.history)
        assert np.array_equal(scal, o.scalars)
        assert np.array_equal(x, o.x)


@pytest.mark.parametrize("graph,exact", [(0, 0), (2, 0), (2, 1)])
def test_nccl_one_rank_communicator(bc, orc, graph, exact):
    """The NCCL code path on one GPU: a 1-rank communicator (ncclCommInitRank) whose
    ncclAllGather carries every reduction (and the exact path's superaccumulators), captured
    into the CUDA graph with BCGS_OPT_GRAPH = 2; host waits poll ncclCommGetAsyncError."""
    n = 48
    h = si.unit_cube_h(n)
    s = bc.Solver(n, h, nranks=1, nccl_id=bc.nccl_unique_id())
    s.set_option(bc.OPT_GRAPH, graph)
    s.set_option(bc.OPT_EXACT_DOT, exact)
    s.set_preconditioner("gnocomm", 4)
    s.set_rhs_random(si.SEED)
    rep = s.solve(tol=1e-8)
    o = orc.bicgstab(orc.rhs_random((n, n, n), si.SEED), h, pc="gnocomm", k=4, tol=1e-8)
    assert rep["iterations"] == o.iterations
    assert np.array_equal(s.residual_history(), o.history)
    assert np.array_equal(host(s.solution()), o.x)
    s.close()


@pytest.mark.parametrize("exact", [0, 1])
def test_r7_breakdown_on_nonfinite_rw_matches_oracle(bc, orc, exact):
    """R7: r~ᵀw overflows at iteration 1 (b = 1e300 at one point): BREAKDOWN with 0
    iterations, x untouched, history [NaN] -- the same on the GPU (certified and exact dot
    paths: a non-finite Σ|ab| or sum is never certified; the exact path rounds the overflow
    to +inf) as in the oracle."""
    n = 16
    h = si.unit_cube_h(n)
    b = np.zeros((n, n, n))
    b[5, 6, 7] = 1e300
    s, n3, _ = make(bc, n, pc="gnocomm", degree=4)
    s.set_option(bc.OPT_EXACT_DOT, exact)
    s.set_rhs(dev(b))
    rep = s.solve(tol=1e-8)
    o = orc.bicgstab(b, h, pc="gnocomm", k=4, tol=1e-8)
    assert o.status == "breakdown" and rep["status_name"] == "breakdown"
    assert rep["iterations"] == o.iterations == 0
    assert np.array_equal(s.residual_history(), o.history, equal_nan=True)
    assert not host(s.solution()).any()
    s.close()
