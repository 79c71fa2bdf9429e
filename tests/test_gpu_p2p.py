"""Peer-memory transport (p2p.cuh; SURVEY §8(e), NEXT-4 one-shot reductions): halos and
reductions as device kernels storing into the peers' memory with sequence-numbered flags.

Ranks are OS processes on the SAME GPU (tests/mp_p2p.py): one CUDA context per rank, the
mailboxes mapped through CUDA IPC (bcgs_p2p_handle / bcgs_p2p_connect) -- the code path of
one process per GPU, multi-rank iterations replayed as CUDA graphs.  (In-process groups,
bcgs_create_local_p2p, share one context: a driver call that waits for the device can stall
behind another rank's spin-waiting kernel, so they are exercised here only for the timeout.)

Every case is compared bitwise with the oracle's P-slab emulation (R19: correctly rounded
dots make the rank count invisible in the reductions)."""
import numpy as np
import pytest

import synth_inputs as si
from tests import mp_p2p

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_08935_b200 import bcgs
    bcgs.load()
    return bcgs


def check(out, P, o, scalars=True):
    for r in range(P):
        assert isinstance(out[r][0], dict), out[r][0]
    x = np.concatenate([out[r][3] for r in range(P)])
    for r in range(P):
        rep, hist, scal = out[r][0], out[r][1], out[r][2]
        assert rep["iterations"] == o.iterations
        assert np.array_equal(hist, o.history)          # identical scalars on every rank
        if scalars:
            assert np.array_equal(scal, o.scalars)
    assert np.array_equal(x, o.x)


@pytest.mark.parametrize("P,n3,pc,k,kernels", [(2, (48, 40, 64), "gnocomm", 4, 1),
                                               (4, (32, 32, 64), "gnocomm", 4, 1),
                                               (2, (40, 36, 48), "bj", 3, 1),
                                               (2, (32, 32, 64), "none", 0, 1),
                                               (2, (48, 40, 64), "g", 4, 1),
                                               (4, (40, 32, 32), "g", 8, 0),
                                               (8, (32, 32, 64), "gnocomm", 4, 1)])
def test_p2p_ranks_match_oracle(bc, orc, P, n3, pc, k, kernels):
    out = mp_p2p.run(P, {"n3": n3, "pc": pc, "k": k, "options": {"OPT_KERNELS": kernels}})
    h = si.unit_cube_h(n3[0])
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc=pc, k=k, nslab=P, tol=1e-8)
    check(out, P, o)


def test_p2p_forced_exact(bc, orc):
    """The exact path's superaccumulators travel through the mailboxes too (k_limbs_p2p)."""
    n3, P = (32, 32, 64), 2
    out = mp_p2p.run(P, {"n3": n3, "pc": "gnocomm", "k": 4, "options": {"OPT_EXACT_DOT": 1}})
    h = si.unit_cube_h(32)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=4, nslab=P, tol=1e-8)
    check(out, P, o)
    assert out[0][5] >= 3 * o.iterations


def test_p2p_pipelined(bc, orc):
    """The pipelined iteration (R32) over the p2p transport."""
    n3, P = (32, 32, 64), 2
    out = mp_p2p.run(P, {"n3": n3, "pc": "gnocomm", "k": 4, "options": {"OPT_PIPELINED": 1}})
    h = si.unit_cube_h(32)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=4, nslab=P, tol=1e-8,
                     pipelined=True)
    check(out, P, o)


@pytest.mark.parametrize("P", [2, 4])
def test_p2p_g_bicgs_across_ranks(bc, orc, P):
    """FBiCGS-G(BiCGS) on P ranks: the inner solve is ONE Bi-CGSTAB over the
    whole domain whose halos and reductions span all ranks (it shares the outer transport),
    so the result is the single-domain G(BiCGS)'s: bitwise the oracle's."""
    n3 = (24, 20, 32)
    out = mp_p2p.run(P, {"n3": n3, "pc": "g_bicgs", "max_iter": 200})
    h = si.unit_cube_h(24)
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="g_bicgs", nslab=P, tol=1e-8,
                     max_it=200)
    check(out, P, o)
    assert out[0][4] == o.extra["inner_iterations"]


def test_p2p_timeout_instead_of_hang(bc):
    """A rank whose peer never answers gets BCGS_E_COMM after the configured timeout."""
    n3 = (16, 16, 32)
    grp = bc.local_group(n3, 1.0 / 17, 2, transport="p2p")
    s = grp[0]
    s.set_option(bc.OPT_COMM_TIMEOUT, 2)
    s.set_preconditioner("gnocomm", 2)
    s.set_rhs_random(1)
    with pytest.raises(bc.BcgsError) as ei:
        s.solve(tol=1e-8)          # rank 1 never runs: the first reduction times out
    assert ei.value.status == bc.E_COMM
    for g in grp:
        g.close()
