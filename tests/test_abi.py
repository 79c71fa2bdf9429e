"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/bcgs.h
declares, and its host-only logic (workspace sizing, Chebyshev constants) matches the
oracle.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2503_08935_b200 import bcgs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "bcgs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bcgs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = bcgs.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(bcgs.EXPORTS) == syms


def test_abi_version_and_status_strings():
    lib = bcgs.load()
    assert lib.bcgs_abi_version() == 6
    assert lib.bcgs_status_string(7) == b"breakdown"


def test_workspace_bytes_and_config_errors():
    nb = bcgs.workspace_bytes(64, 1 / 65)
    # 13 fields of (L+2) planes plus state / history / partials
    assert nb >= 13 * 66 * 64 * 64 * 8
    assert bcgs.workspace_bytes(64, 1 / 65, nranks=3) == 0      # 64 % 3 != 0
    assert bcgs.workspace_bytes(64, 1 / 65, nranks=4) < nb
    assert bcgs.workspace_bytes((10, 20, 30), 0.1) > 0


@pytest.mark.parametrize("n,nslab,pc,k", [(32, 1, "gnocomm", 4), (64, 4, "gnocomm", 4),
                                          (64, 4, "bj", 4), (128, 8, "bj", 7),
                                          (512, 8, "gnocomm", 24), ((48, 40, 36), 3, "bj", 2),
                                          (64, 4, "g", 4)])
def test_chebyshev_constants_equal_oracle(orc, n, nslab, pc, k):
    """Host-side constants of the library (R9, R10, R18) are bit-identical to the oracle's."""
    n3 = (n,) * 3 if np.isscalar(n) else n
    h = 1.0 / (n3[0] + 1)
    ivl, cst, rho = bcgs.chebyshev_constants(n3, h, nslab, pc, k)
    if pc in ("gnocomm", "g"):
        lo, hi = orc.bounds(n3[0], n3[1], n3[2], h)
        a, b = 10.0 * lo, (1.0 - 1e-4) * hi
    else:
        a, b = orc.bounds(n3[0], n3[1], n3[2] // nslab, h)
    assert (ivl[0], ivl[1]) == (a, b)
    ref = orc.cheb_setup(a, b, k)
    assert list(cst) == [ref[key] for key in ("theta", "delta", "sigma", "cz", "g1", "A2", "B2")]
    assert np.array_equal(rho, ref["rho"])


@pytest.mark.parametrize("faces", [(0, 1, 1, 0, 1, 0), (1, 1, 0, 0, 0, 1), (0, 0, 1, 1, 1, 1)])
@pytest.mark.parametrize("pc,nslab", [("gnocomm", 1), ("gnocomm", 4), ("bj", 1), ("bj", 2),
                                      ("bj", 4), ("g", 1)])
def test_chebyshev_constants_mixed_bc_equal_oracle(orc, faces, pc, nslab):
    """R27: the library's mixed-BC interval (closed-form mixed spectra, BJ union over the
    blocks' z factors) and constants are bit-identical to the oracle's."""
    n3, h = (40, 24, 32), 0.1
    ivl, cst, rho = bcgs.chebyshev_constants(n3, h, nslab, pc, 6, bc=faces)
    a, b = orc.pc_interval(n3[::-1], h, nslab, pc, bc=faces)
    assert (ivl[0], ivl[1]) == (a, b)
    ref = orc.cheb_setup(a, b, 6)
    assert list(cst) == [ref[key] for key in ("theta", "delta", "sigma", "cz", "g1", "A2", "B2")]
    assert np.array_equal(rho, ref["rho"])


def test_chebyshev_constants_bc_config_errors():
    with pytest.raises(bcgs.BcgsError):     # 1-plane blocks next to a Neumann z face
        bcgs.chebyshev_constants((8, 8, 8), 0.1, 8, "bj", 2, bc=(0, 0, 0, 0, 1, 0))
    with pytest.raises(bcgs.BcgsError):     # Neumann axis with one point
        bcgs.chebyshev_constants((1, 8, 8), 0.1, 1, "gnocomm", 2, bc=(1, 0, 0, 0, 0, 0))
    with pytest.raises(bcgs.BcgsError):     # unknown face kind
        bcgs.chebyshev_constants((8, 8, 8), 0.1, 1, "gnocomm", 2, bc=(2, 0, 0, 0, 0, 0))


def test_chebyshev_constants_reject_bad_interval():
    with pytest.raises(bcgs.BcgsError):
        bcgs.chebyshev_constants(16, 1 / 17, 1, "gnocomm", 4, c_min=1e9)
    with pytest.raises(bcgs.BcgsError):
        bcgs.chebyshev_constants(16, 1 / 17, 1, "gnocomm", bcgs.MAX_DEGREE + 1)


def test_solver_requires_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        bcgs.Solver(8, 1 / 9)
