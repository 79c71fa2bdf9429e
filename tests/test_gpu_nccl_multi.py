"""NCCL transport across GPUs: one OS process per GPU, z-slab halos
by ncclSend / ncclRecv overlapped with the interior stencil, every reduction an ncclAllGather
of the ranks' correctly rounded quadruples combined in rank order -- compared bitwise with the
oracle's P-slab emulation (R19 makes the rank count invisible in the reductions).

Needs >= 2 GPUs (skipped on the one-GPU boxes of this project's round-end runs; run it on a
multi-GPU node: python -m pytest tests/test_gpu_nccl_multi.py)."""
import numpy as np
import pytest

import synth_inputs as si
from tests import mp_p2p

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bc():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_2503_08935_b200 import bcgs
    bcgs.load()
    return bcgs


def _check(out, P, o):
    for r in range(P):
        assert isinstance(out[r][0], dict), out[r][0]
        rep, hist, scal = out[r][0], out[r][1], out[r][2]
        assert rep["iterations"] == o.iterations
        assert np.array_equal(hist, o.history)
        assert np.array_equal(scal, o.scalars)
    assert np.array_equal(np.concatenate([out[r][3] for r in range(P)]), o.x)


@pytest.mark.parametrize("n3,pc,k,opts", [
    ((48, 40, 64), "gnocomm", 4, {}),
    ((48, 40, 64), "gnocomm", 4, {"OPT_GRAPH": 2}),      # NCCL captured in the CUDA graph
    ((40, 36, 48), "bj", 3, {}),
    ((48, 40, 64), "g", 4, {}),                          # G(CI): one k-deep halo
    ((32, 32, 64), "none", 0, {}),
    ((48, 40, 64), "gnocomm", 4, {"OPT_EXACT_DOT": 1}),  # superaccumulators all-gathered
])
def test_nccl_two_gpus_match_oracle(bc, orc, n3, pc, k, opts):
    P = 2
    out = mp_p2p.run(P, {"n3": n3, "pc": pc, "k": k, "options": opts, "transport": "nccl"})
    h = si.unit_cube_h(n3[0])
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc=pc, k=k, nslab=P, tol=1e-8)
    _check(out, P, o)


def test_nccl_sync2_two_gpus(bc, orc):
    n3, P = (48, 40, 64), 2
    out = mp_p2p.run(P, {"n3": n3, "pc": "gnocomm", "k": 4, "options": {"OPT_SYNC2": 1},
                         "transport": "nccl"})
    h = si.unit_cube_h(n3[0])
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=4, nslab=P,
                     tol=1e-8, sync2=True)
    _check(out, P, o)


def test_nccl_all_gpus(bc, orc):
    P = min(8, torch.cuda.device_count())
    n3 = (32, 32, 8 * P)
    out = mp_p2p.run(P, {"n3": n3, "pc": "gnocomm", "k": 4, "transport": "nccl"})
    h = si.unit_cube_h(n3[0])
    o = orc.bicgstab(orc.rhs_random(n3[::-1], si.SEED), h, pc="gnocomm", k=4, nslab=P, tol=1e-8)
    _check(out, P, o)
