"""CPU ORACLE for the Bi-CGSTAB / Chebyshev Poisson hot path of arXiv 2503.08935.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2503_08935_b200``) never imports it and shares no code with it.

``bcgs_oracle.c`` holds the arithmetic (compiled to ``liboracle.so`` with
``-ffp-contract=off``); this module only marshals numpy arrays through ctypes.
``dense.py`` holds the dense Kronecker assembly of Eq. 6 used as a pin on tiny grids.

Parity status: every oracle function is pinned by ``tests/test_oracle_pins.py``,
``test_oracle_bc.py``, ``test_oracle_inner.py`` and ``test_oracle_sync2.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bcgs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# -ffp-contract=off: no FMA contraction (DESIGN.md §3 R17); -mfma only makes fma() native.
CFLAGS = ["-O2", "-mfma", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
          "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so next to the source (gcc).  Returns the path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i64, f64, P = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        _lib.orc_threads.restype = ctypes.c_int
        _lib.orc_splitmix64.restype = ctypes.c_uint64
        _lib.orc_splitmix64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        _lib.orc_rhs_random.argtypes = [i64, i64, i64, ctypes.c_uint64, P]
        _lib.orc_fold_boundary.argtypes = [i64, i64, i64, f64, P, P]
        _lib.orc_apply_A.argtypes = [i64, i64, i64, f64, i64, P, P]
        _lib.orc_dot.restype = f64
        _lib.orc_dot.argtypes = [i64, i64, P, P]
        _lib.orc_dot_pair.argtypes = [i64, i64, P, P, P]
        _lib.orc_mu.restype = f64
        _lib.orc_mu.argtypes = [i64, i64]
        _lib.orc_bounds.argtypes = [i64, i64, i64, f64, P, P]
        _lib.orc_cheb_setup.restype = ctypes.c_int
        _lib.orc_cheb_setup.argtypes = [f64, f64, ctypes.c_int, P, P]
        _lib.orc_apply_cheb.restype = ctypes.c_int
        _lib.orc_apply_cheb.argtypes = [i64, i64, i64, f64, i64, ctypes.c_int, f64, f64, P, P]
        _lib.orc_fold_boundary_bc.argtypes = [i64, i64, i64, f64, ctypes.c_int, P, P]
        _lib.orc_apply_A_bc.argtypes = [i64, i64, i64, f64, i64, ctypes.c_int, P, P]
        _lib.orc_mu_bc.restype = f64
        _lib.orc_mu_bc.argtypes = [i64, i64, ctypes.c_int]
        _lib.orc_bounds_bc.argtypes = [i64, i64, i64, f64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, P, P]
        _lib.orc_apply_cheb_bc.restype = ctypes.c_int
        _lib.orc_apply_cheb_bc.argtypes = [i64, i64, i64, f64, i64, ctypes.c_int, ctypes.c_int,
                                           f64, f64, P, P]
        _lib.orc_pc_interval.argtypes = [i64, i64, i64, f64, i64, ctypes.c_int, ctypes.c_int,
                                         f64, f64, P]
        _lib.orc_bicgstab_bc.restype = ctypes.c_int
        _lib.orc_bicgstab_bc.argtypes = [i64, i64, i64, f64, i64, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, f64, f64, f64, f64, P, P, f64,
                                         ctypes.c_int, ctypes.c_int, P, P, P, P, P]
        _lib.orc_bicgstab_ex.restype = ctypes.c_int
        _lib.orc_bicgstab_ex.argtypes = [i64, i64, i64, f64, i64, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, f64, f64, f64, f64, f64, ctypes.c_int,
                                         ctypes.c_int, P, P, f64, ctypes.c_int, ctypes.c_int, P, P, P, P, P,
                                         P]
        _lib.orc_apply_inner.restype = ctypes.c_longlong
        _lib.orc_apply_inner.argtypes = [i64, i64, i64, f64, i64, ctypes.c_int, f64,
                                         ctypes.c_int, P, P]
        _lib.orc_bicgstab.restype = ctypes.c_int
        _lib.orc_bicgstab.argtypes = [i64, i64, i64, f64, i64, ctypes.c_int, ctypes.c_int,
                                      f64, f64, f64, f64, P, P, f64, ctypes.c_int,
                                      ctypes.c_int, P, P, P, P, P]
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _shape(shape):
    nz, ny, nx = shape
    return int(nx), int(ny), int(nz)


# Problem arrays are numpy arrays of shape (nz, ny, nx) (x fastest), fp64.

def threads() -> int:
    return int(lib().orc_threads())


def splitmix64(seed: int, g: int) -> int:
    return int(lib().orc_splitmix64(seed, g))


def rhs_random(shape, seed: int) -> np.ndarray:
    nx, ny, nz = _shape(shape)
    b = np.empty((nz, ny, nx), np.float64)
    lib().orc_rhs_random(nx, ny, nz, seed, _ptr(b))
    return b


def bc_mask(bc6) -> int:
    """Face kinds (0 Dirichlet / 1 Neumann, faces x-,x+,y-,y+,z-,z+) -> bit mask."""
    if bc6 is None:
        return 0
    if isinstance(bc6, int):
        return bc6
    return sum((1 << f) for f, kind in enumerate(bc6) if kind)


def fold_boundary(b: np.ndarray, h: float, g6, bc=None) -> np.ndarray:
    nx, ny, nz = _shape(b.shape)
    out = np.ascontiguousarray(b, dtype=np.float64).copy()
    g = np.ascontiguousarray(np.asarray(g6, np.float64))
    lib().orc_fold_boundary_bc(nx, ny, nz, h, bc_mask(bc), _ptr(g), _ptr(out))
    return out


def apply_A(v: np.ndarray, h: float, nslab: int = 1, bc=None) -> np.ndarray:
    """Global operator (nslab=1) or block-diagonal slab operator (Eq. 6 / Eq. 12-14);
    bc: Neumann faces (Eq. 5 mirror ghosts)."""
    v = np.ascontiguousarray(v, np.float64)
    nx, ny, nz = _shape(v.shape)
    out = np.empty_like(v)
    lib().orc_apply_A_bc(nx, ny, nz, h, nslab, bc_mask(bc), _ptr(v), _ptr(out))
    return out


def dot(a: np.ndarray, b: np.ndarray) -> float:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    if a.ndim == 3:
        plen, npl = a.shape[1] * a.shape[2], a.shape[0]
    else:
        plen, npl = a.size, 1
    return float(lib().orc_dot(plen, npl, _ptr(a), _ptr(b)))


def dot_pair(a: np.ndarray, b: np.ndarray):
    """Dot2 (hi, lo) pair of a (nz, ny, nx) field (R19 partial)."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    out = np.zeros(2)
    lib().orc_dot_pair(a.shape[1] * a.shape[2], a.shape[0], _ptr(a), _ptr(b), _ptr(out))
    return float(out[0]), float(out[1])


def mu(n: int, i: int) -> float:
    return float(lib().orc_mu(n, i))


def bounds(nx: int, ny: int, nzb: int, h: float):
    lo, hi = np.zeros(1), np.zeros(1)
    lib().orc_bounds(nx, ny, nzb, h, _ptr(lo), _ptr(hi))
    return float(lo[0]), float(hi[0])


def mu_bc(n: int, i: int, kind: int) -> float:
    """Eigenvalue i of the 1-D factor with `kind` Neumann ends (0: Eq. 9; 1, 2: R27)."""
    return float(lib().orc_mu_bc(n, i, kind))


def bounds_bc(nx: int, ny: int, nzb: int, h: float, kinds):
    lo, hi = np.zeros(1), np.zeros(1)
    lib().orc_bounds_bc(nx, ny, nzb, h, int(kinds[0]), int(kinds[1]), int(kinds[2]),
                        _ptr(lo), _ptr(hi))
    return float(lo[0]), float(hi[0])


def pc_interval(shape, h: float, nslab: int, pc: str, c_min: float = 10.0,
                c_max: float = 1.0 - 1e-4, bc=None):
    """Chebyshev interval [a', b'] the oracle's Alg. 3 uses for preconditioner `pc`."""
    nx, ny, nz = _shape(shape)
    out = np.zeros(2)
    lib().orc_pc_interval(nx, ny, nz, h, nslab, bc_mask(bc), PC[pc], c_min, c_max, _ptr(out))
    return float(out[0]), float(out[1])


def cheb_setup(a: float, b: float, k: int):
    cst = np.zeros(7)
    rho = np.zeros(max(k, 1) + 1)
    rc = lib().orc_cheb_setup(a, b, k, _ptr(cst), _ptr(rho))
    if rc:
        raise ValueError(f"cheb_setup rc={rc}")
    keys = ["theta", "delta", "sigma", "cz", "g1", "A2", "B2"]
    d = dict(zip(keys, map(float, cst)))
    d["rho"] = rho
    return d


def apply_cheb(q: np.ndarray, h: float, nslab: int, k: int, a: float, b: float,
               bc=None) -> np.ndarray:
    q = np.ascontiguousarray(q, np.float64)
    nx, ny, nz = _shape(q.shape)
    out = np.empty_like(q)
    rc = lib().orc_apply_cheb_bc(nx, ny, nz, h, nslab, bc_mask(bc), k, a, b, _ptr(q),
                                 _ptr(out))
    if rc:
        raise ValueError(f"apply_cheb rc={rc}")
    return out


PC = {"none": 0, "gnocomm": 1, "bj": 2, "g": 3, "bj_bicgs": 4, "g_bicgs": 5}
# inner-Krylov preconditioners: default inner settings of the paper
INNER_DEFAULT = {"bj_bicgs": (1e-6, 500), "g_bicgs": (1e-2, 500)}
STATUS = {0: "ok", 1: "config", 6: "not_converged", 7: "breakdown"}


@dataclass
class Result:
    status: str
    iterations: int
    x: np.ndarray
    history: np.ndarray
    scalars: np.ndarray          # (iterations, 8): rw, alpha, ts, tt, omega, rho_new, rr, beta
    true_rel: float
    extra: dict = field(default_factory=dict)


def apply_inner(q: np.ndarray, h: float, nslab: int, tol: float, max_it: int,
                bc=None) -> tuple[np.ndarray, int]:
    """One BJ(BiCGS) application: inner unpreconditioned Bi-CGSTAB on each of the
    nslab z-blocks.  Returns (M^{-1} q, total inner iterations)."""
    q = np.ascontiguousarray(q, np.float64)
    nx, ny, nz = _shape(q.shape)
    out = np.empty_like(q)
    tot = lib().orc_apply_inner(nx, ny, nz, h, nslab, bc_mask(bc), tol, max_it, _ptr(q),
                                _ptr(out))
    return out, int(tot)


def bicgstab(b: np.ndarray, h: float, *, pc: str = "none", k: int = 4, nslab: int = 1,
             c_min: float = 10.0, c_max: float = 1.0 - 1e-4, bounds_override=None,
             x0: np.ndarray | None = None, tol: float = 1e-8, max_it: int = 5000,
             fixed_it: int = 0, bc=None, inner_tol: float | None = None,
             inner_max: int | None = None, sync2: bool = False,
             pipelined: bool = False) -> Result:
    """Alg. 3 with M = I, GNoComm(CI), BJ(CI), G(CI) on `nslab` z-slabs, or the
    inner-Krylov BJ(BiCGS) / G(BiCGS) (inner_tol / inner_max default to P:393-394's values;
    Result.extra["inner_iterations"] = total inner iterations).  sync2: the 2-sync rewrite
    (R31): ρ_new and ||r||² from the a9 reduction, no MPI5.  pipelined: the pipelined
    (communication-hiding) Bi-CGSTAB of bcgs_oracle.c's pbicgstab, two reductions per
    iteration (linear preconditioners only)."""
    dt, dm = INNER_DEFAULT.get(pc, (0.0, 0))
    inner_tol = dt if inner_tol is None else inner_tol
    inner_max = dm if inner_max is None else inner_max
    tot = ctypes.c_longlong(0)
    b = np.ascontiguousarray(b, np.float64)
    nx, ny, nz = _shape(b.shape)
    cap = (fixed_it if fixed_it > 0 else max_it)
    x = np.zeros_like(b)
    hist = np.full(cap + 1, np.nan)
    scal = np.zeros((cap, 8))
    it = ctypes.c_int(0)
    tr = ctypes.c_double(0.0)
    lmin, lmax = bounds_override if bounds_override is not None else (0.0, 0.0)
    x0p = None
    if x0 is not None:
        x0 = np.ascontiguousarray(x0, np.float64)
        x0p = _ptr(x0)
    st = lib().orc_bicgstab_ex(nx, ny, nz, h, nslab, bc_mask(bc), PC[pc], k, c_min, c_max,
                               lmin, lmax, inner_tol, inner_max,
                               (1 if sync2 else 0) | (2 if pipelined else 0),
                               _ptr(b), x0p, tol, max_it, fixed_it, _ptr(x), _ptr(hist),
                               _ptr(scal), ctypes.byref(it), ctypes.byref(tr),
                               ctypes.byref(tot))
    n = it.value
    return Result(STATUS.get(st, str(st)), n, x, hist[: n + 1].copy(), scal[:n].copy(),
                  float(tr.value), {"inner_iterations": int(tot.value)})
