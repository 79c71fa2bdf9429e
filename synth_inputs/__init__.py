"""Seeded synthetic inputs shared by the oracle-side tests and the GPU-side tests / bench.

This module holds NONE of the method's arithmetic (no stencil, no Chebyshev, no Krylov
step): only problem inputs -- right-hand sides and, for manufactured solutions, the exact
continuous solution sampled at the grid nodes.  Both `oracle/` and
`paper_2503_08935_b200/` implement the RANDOM generator independently as well (counter-based
splitmix64, DESIGN.md §3 R16); `rhs_random` here is a third, numpy, implementation used
to cross-check both.

Grid convention (DESIGN.md §3 R14): unit cube, homogeneous Dirichlet, nx*ny*nz unknowns,
spacing h, unknown (i, j, k) (0-based) at ((i+1)h, (j+1)h, (k+1)h).  Arrays have shape
(nz, ny, nx) (x fastest).
"""
from __future__ import annotations

import math

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

#: Default seed for the bench / parity workloads.
SEED = 20250311


def splitmix64_np(seed: int, g: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 output for counters g (uint64), wrap-around arithmetic."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (g.astype(np.uint64) + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def rhs_random(nx: int, ny: int, nz: int, seed: int = SEED, z0: int = 0,
               nzl: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """i.i.d. uniform [-1, 1) per point; value depends only on (seed, global index).

    Returns planes z0 .. z0+nzl-1 of the global nx*ny*nz field (a z-slab).
    """
    nzl = nz - z0 if nzl is None else nzl
    if out is None:
        out = np.empty((nzl, ny, nx), np.float64)
    plane = nx * ny
    chunk = max(1, (1 << 24) // max(plane, 1))
    for k0 in range(0, nzl, chunk):
        k1 = min(nzl, k0 + chunk)
        g = np.arange((z0 + k0) * plane, (z0 + k1) * plane, dtype=np.uint64)
        v = splitmix64_np(seed, g)
        u = (v >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        out[k0:k1] = (2.0 * u - 1.0).reshape(k1 - k0, ny, nx)
    return out


def unit_cube_h(n: int) -> float:
    """h = 1/(N+1): N unknowns strictly inside [0, 1] (DESIGN.md §3 R14)."""
    return 1.0 / (n + 1)


def _coords(n: int, h: float) -> np.ndarray:
    return (np.arange(n, dtype=np.float64) + 1.0) * h


def _grid(nx, ny, nz, h):
    x = _coords(nx, h)[None, None, :]
    y = _coords(ny, h)[None, :, None]
    z = _coords(nz, h)[:, None, None]
    return x, y, z


# --- manufactured solutions (DESIGN.md §3 R15 readings) ----------------------------------

def mms_sine(n: int):
    """u = sin(pi x) sin(pi y) sin(pi z); f = 3 pi^2 u.  Exact discrete eigenvector."""
    h = unit_cube_h(n)
    x, y, z = _grid(n, n, n, h)
    u = np.sin(math.pi * z) * np.sin(math.pi * y) * np.sin(math.pi * x)
    return 3.0 * math.pi ** 2 * u, u, h


def mms_poly(n: int):
    """u = prod_d (x_d - x_d^2); f = sum_d 2 prod_{e != d} (x_e - x_e^2).

    The 7-point stencil differentiates quadratics exactly, so A u = f at the nodes.
    """
    h = unit_cube_h(n)
    x, y, z = _grid(n, n, n, h)
    gx, gy, gz = x - x * x, y - y * y, z - z * z
    u = gz * gy * gx
    f = 2.0 * (gy * gz) + 2.0 * (gx * gz) + 2.0 * (gx * gy)
    return np.broadcast_to(f, u.shape).copy(), u, h


def mms_polyexp(n: int):
    """u = prod_d (x_d - x_d^2) e^{x_d};  -g'' = s (s + 3) e^s for g = (s - s^2) e^s."""
    h = unit_cube_h(n)
    x, y, z = _grid(n, n, n, h)

    def g(s):
        return (s - s * s) * np.exp(s)

    def mg2(s):
        return s * (s + 3.0) * np.exp(s)

    u = g(z) * g(y) * g(x)
    f = mg2(x) * g(y) * g(z) + g(x) * mg2(y) * g(z) + g(x) * g(y) * mg2(z)
    return f, u, h


# --- the paper's own workload (§IV, R27) --------------------------

#: Face kinds of the §IV problem, faces x-,x+,y-,y+,z-,z+ (0 Dirichlet, 1 Neumann):
#: "Dirichlet ... on x-, y+, z+, while Neumann ... on x+, y-, z-".
PAPER_BC = (0, 1, 1, 0, 1, 0)
PAPER_LO = (3.0, 2.5, 10.0)          # x in [3, 28.5], y in [2.5, 28], z in [10, 35.5]
PAPER_LEN = 25.5


def paper_problem(n: int, z0: int = 0, nzl: int | None = None):
    """f = sin x + cos y + 3 sin z - 2yz + 2 at the nodes of an n^3 grid over the paper's box.

    Node i of an axis sits at lo + i*h with h = 25.5/(n-1) (n = 256 gives the paper's
    Δ = 0.1 and 256 nodes per axis).  Boundary data are homogeneous (the paper does not
    state them).  Returns (f planes z0..z0+nzl-1, h, PAPER_BC).
    """
    nzl = n - z0 if nzl is None else nzl
    h = PAPER_LEN / (n - 1)
    i = np.arange(n, dtype=np.float64)
    x = (PAPER_LO[0] + i * h)[None, None, :]
    y = (PAPER_LO[1] + i * h)[None, :, None]
    z = (PAPER_LO[2] + (np.arange(z0, z0 + nzl, dtype=np.float64)) * h)[:, None, None]
    f = np.sin(x) + np.cos(y) + 3.0 * np.sin(z) - 2.0 * y * z + 2.0
    return np.ascontiguousarray(f), h, PAPER_BC
