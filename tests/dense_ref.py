"""Dense Kronecker assembly of the Poisson operator, Eq. 6, for pins on tiny grids.

Independent of the matrix-free stencil in oracle/: it builds the 1-D Dirichlet matrix D of
Eq. 4 and combines the factors with np.kron exactly as Eq. 6 writes them, with
x the fastest index (I_z ⊗ I_y ⊗ O_x).
"""
import numpy as np


def D(n: int) -> np.ndarray:
    """tridiag(-1, 2, -1), Eq. 4."""
    return 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)


def assemble(nx: int, ny: int, nz: int, h: float) -> np.ndarray:
    Ix, Iy, Iz = np.eye(nx), np.eye(ny), np.eye(nz)
    h2 = h * h
    return (np.kron(Iz, np.kron(Iy, D(nx) / h2))
            + np.kron(Iz, np.kron(D(ny) / h2, Ix))
            + np.kron(D(nz) / h2, np.kron(Iy, Ix)))


def block_diag_slabs(A: np.ndarray, nx: int, ny: int, nz: int, nslab: int) -> np.ndarray:
    """Σ_s R_s^T (R_s A R_s^T) R_s (Eq. 12-14): keep only the diagonal slab blocks."""
    L = nz // nslab
    m = nx * ny * L
    out = np.zeros_like(A)
    for s in range(nslab):
        sl = slice(s * m, (s + 1) * m)
        out[sl, sl] = A[sl, sl]
    return out


def cheb_T(n: int, x):
    """Chebyshev polynomial of the first kind via the three-term recurrence."""
    x = np.asarray(x, dtype=np.float64)
    t0, t1 = np.ones_like(x), x.copy()
    if n == 0:
        return t0
    for _ in range(n - 1):
        t0, t1 = t1, 2.0 * x * t1 - t0
    return t1


def N(n: int, left: bool, right: bool) -> np.ndarray:
    """Eq. 5: D with first row (2, -α) and last row (-β, 2); α = 2 for a Neumann
    left end, β = 2 for a Neumann right end (else 1, i.e. matrix D).  Both ends Neumann is
    the natural extension (α = β = 2)."""
    m = D(n)
    if left:
        m[0, 1] = -2.0
    if right:
        m[n - 1, n - 2] = -2.0
    return m


def assemble_bc(nx: int, ny: int, nz: int, h: float, bc6) -> np.ndarray:
    """Eq. 6 with O_d = D or N per axis; bc6 = face kinds x-,x+,y-,y+,z-,z+ (1 = Neumann)."""
    Ox, Oy, Oz = N(nx, bc6[0], bc6[1]), N(ny, bc6[2], bc6[3]), N(nz, bc6[4], bc6[5])
    Ix, Iy, Iz = np.eye(nx), np.eye(ny), np.eye(nz)
    h2 = h * h
    return (np.kron(Iz, np.kron(Iy, Ox / h2))
            + np.kron(Iz, np.kron(Oy / h2, Ix))
            + np.kron(Oz / h2, np.kron(Iy, Ix)))
