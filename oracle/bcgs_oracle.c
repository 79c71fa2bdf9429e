/*
 * bcgs_oracle.c -- CPU ORACLE for the preconditioned Bi-CGSTAB Poisson hot path of
 * arXiv 2503.08935 ("A Parallel and Highly-Portable HPC Poisson Solver: Preconditioned
 * Bi-CGSTAB with alpaka").
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code, header,
 * constant table or helper with the CUDA library under paper_2503_08935_b200/; the two are
 * written independently from the paper and from the arithmetic contract in DESIGN.md §3.
 *
 * Style: plain loops, one stencil sweep per pass, one vector operation per pass, fp64,
 * compiled with -ffp-contract=off: the compiler contracts nothing; the contract's fused
 * multiply-adds (DESIGN.md §3 R17/R18/R20) are written as explicit fma().  OpenMP is used
 * only over z-planes of element-wise passes (order-independent) and for exact dot-product
 * accumulators (integer sums: order-independent).
 *
 * Citations: "P:n" = line n of the paper's LaTeX source.  Section / equation /
 * algorithm numbers are given next to every citation.
 *
 * Layout (DESIGN.md §3 R14): unknown (i,j,k), 0-based, i fastest:  idx = i + nx*(j + ny*k).
 * The grid has nx*ny*nz unknowns; physical boundary ghosts are homogeneous Dirichlet zeros
 * (Eq. 4) or, on faces flagged Neumann in the bit mask bcm (bit f = face f,
 * 0..5 = x-,x+,y-,y+,z-,z+), mirrors of the first interior neighbour (Eq. 5;
 * "_bc" entry points); non-zero boundary data are folded into the right-hand side once
 * (orc_fold_boundary_bc).
 *
 * Parity status: every function below is pinned by tests/test_oracle_pins.py (and, for the
 * mixed faces, the inner-Krylov preconditioners and the 2-sync flag, by test_oracle_bc.py,
 * test_oracle_inner.py and test_oracle_sync2.py) against values
 * that do not come from this file (dense Kronecker assembly, closed-form spectra, closed-form
 * Chebyshev polynomials, dense direct solves, manufactured solutions, exact summation,
 * splitmix64's published test vector).  No function is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define IDX(i, j, k) ((i) + nx * ((j) + ny * (k)))

/* ------------------------------------------------------------------------------------------
 * Right-hand side: splitmix64 counter generator (DESIGN.md §3 R16).  Input generation, not
 * part of the method; each side implements it independently.
 * state = seed + (g+1)*0x9E3779B97F4A7C15, then the splitmix64 finaliser; u = (v>>11)*2^-53;
 * b = 2u - 1 (exact).  g = global linear index.
 * ---------------------------------------------------------------------------------------- */
uint64_t orc_splitmix64(uint64_t seed, uint64_t g)
{
    uint64_t z = seed + (g + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void orc_rhs_random(int64_t nx, int64_t ny, int64_t nz, uint64_t seed, double* b)
{
    int64_t n = nx * ny * nz;
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < n; ++g) {
        uint64_t v = orc_splitmix64(seed, (uint64_t)g);
        double u = (double)(v >> 11) * 0x1.0p-53;
        b[g] = 2.0 * u - 1.0;
    }
}

/* Fold constant Dirichlet boundary values into the RHS (DESIGN.md §3 R15).  For the unknown
 * next to face f the stencil row (Eq. 3) references one ghost whose value is g_f;
 * moving it to the right-hand side adds g_f/h^2.  Faces: 0=x-,1=x+,2=y-,3=y+,4=z-,5=z+.
 * Faces are folded in face order 0..5, each as b += g*h2inv. */
void orc_fold_boundary_bc(int64_t nx, int64_t ny, int64_t nz, double h, int bcm,
                          const double* g6, double* b)
{
    double h2inv = 1.0 / (h * h);
    for (int f = 0; f < 6; ++f) {
        /* Dirichlet value g: the ghost g moves to the RHS as g/h^2.  Neumann (bit f of bcm)
         * outward normal derivative g: the centred ghost rule ghost = mirror + 2 h g
         * ("Set Neumann BCs") leaves 2 h g / h^2 = 2 g / h on the RHS (R28). */
        double add = ((bcm >> f) & 1) ? (2.0 * g6[f]) / h : g6[f] * h2inv;
        if (g6[f] == 0.0) continue;
        for (int64_t k = 0; k < nz; ++k)
            for (int64_t j = 0; j < ny; ++j)
                for (int64_t i = 0; i < nx; ++i) {
                    int on = (f == 0 && i == 0) || (f == 1 && i == nx - 1) ||
                             (f == 2 && j == 0) || (f == 3 && j == ny - 1) ||
                             (f == 4 && k == 0) || (f == 5 && k == nz - 1);
                    if (on) b[IDX(i, j, k)] = b[IDX(i, j, k)] + add;
                }
    }
}

void orc_fold_boundary(int64_t nx, int64_t ny, int64_t nz, double h, const double* g6, double* b)
{
    orc_fold_boundary_bc(nx, ny, nz, h, 0, g6, b);
}

/* ------------------------------------------------------------------------------------------
 * The operator.  P:95-100 (Eq. 6): P = I⊗I⊗D_x/Δx² + I⊗D_y/Δy²⊗I + D_z/Δz²⊗I⊗I with D from
 * Eq. 4.  With uniform spacing h the row for unknown c reads
 *     (A v)_c = fma(6, v_c, -(((((v_xm + v_xp) + v_ym) + v_yp) + v_zm) + v_zp)) * h2inv,
 * h2inv = 1/(h*h), out-of-domain neighbours = +0.0 (homogeneous Dirichlet).
 * nslab > 1 gives the block-diagonal operator Σ_s R_s^T (R_s A R_s^T) R_s of Eq. 12-14
 * (P:185-205): z is cut into nslab equal slabs and neighbours across a cut are also +0.0.
 * nslab == 1 is the global operator (used by KernelBiCGS1/3).
 * ---------------------------------------------------------------------------------------- */
void orc_apply_A_bc(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab, int bcm,
                    const double* v, double* out)
{
    double h2inv = 1.0 / (h * h);
    int64_t L = nz / nslab;
    int64_t pl = nx * ny;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nz; ++k) {
        int cut_lo = (k % L) == 0;          /* plane below is outside this block */
        int cut_hi = (k % L) == L - 1;      /* plane above is outside this block */
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                int64_t c = IDX(i, j, k);
                /* Neumann face (bit of bcm): the ghost is the mirror of the first interior
                 * neighbour (ghost_{-1} = v_1), which gives Eq. 5's rows (2, -2) (R27). */
                double xm = (i > 0) ? v[c - 1] : ((bcm & 1) ? v[c + 1] : 0.0);
                double xp = (i < nx - 1) ? v[c + 1] : ((bcm & 2) ? v[c - 1] : 0.0);
                double ym = (j > 0) ? v[c - nx] : ((bcm & 4) ? v[c + nx] : 0.0);
                double yp = (j < ny - 1) ? v[c + nx] : ((bcm & 8) ? v[c - nx] : 0.0);
                double zm = (k == 0 && (bcm & 16)) ? v[c + pl] : (cut_lo ? 0.0 : v[c - pl]);
                double zp = (k == nz - 1 && (bcm & 32)) ? v[c - pl] : (cut_hi ? 0.0 : v[c + pl]);
                double nb = ((((xm + xp) + ym) + yp) + zm) + zp;
                out[c] = fma(6.0, v[c], -nb) * h2inv;      /* (6 v_c - nb) / h^2, R17 */
            }
    }
}

void orc_apply_A(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab,
                 const double* v, double* out)
{
    orc_apply_A_bc(nx, ny, nz, h, nslab, 0, v, out);
}

/* ------------------------------------------------------------------------------------------
 * Dot products (DESIGN.md §3 R19): the CORRECTLY ROUNDED value of the exact sum,
 * RN(Σ a_i b_i), round to nearest, ties to even.  The paper computes r~ᵀw, tᵀr, tᵀt, r0ᵀr,
 * rᵀr (Alg. 3) and notes that floating-point reductions give
 * order-dependent results ("numerical issues due to floating-point arithmetic", P:207;
 * iteration counts vary with the reduction order); the exact sum rounded once has a
 * plain definition that no summation order can change.
 *
 * Method (plain, no cleverness): every double is m * 2^e with an integer m < 2^53 and
 * e >= -1074, so a product is the 106-bit integer ma*mb times 2^(ea+eb) with
 * ea + eb >= -2148.  The exact sum is kept as a big two's-complement integer X with
 * Σ = X * 2^XBASE, XBASE = -2176, in XLIMB 64-bit limbs; each product is added (or
 * subtracted) at its bit offset with full carry propagation.  At the end X is rounded to
 * 53 significant bits (or to the subnormal grid 2^-1074), ties to even.  A non-finite
 * operand gives NaN; a sum beyond the double range gives +-inf.
 * ---------------------------------------------------------------------------------------- */
static inline void two_sum(double a, double b, double* s, double* e)
{
    double x = a + b;
    double z = x - a;
    *e = (a - (x - z)) + (b - z);
    *s = x;
}

static inline void two_prod(double a, double b, double* p, double* e)
{
    double x = a * b;
    *e = fma(a, b, -x);
    *p = x;
}

/* Dot2 (Ogita, Rump & Oishi) of n contiguous elements -> (hi, lo): used only by
 * orc_dot_pair below (the per-rank compensated partial of a slab decomposition). */
static void dot2_run(int64_t n, const double* a, const double* b, double* hi, double* lo)
{
    double p = 0.0, s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double h, r, q;
        two_prod(a[i], b[i], &h, &r);
        two_sum(p, h, &p, &q);
        s = s + (q + r);
    }
    *hi = p;
    *lo = s;
}

#define XBASE (-2176)
#define XLIMB 72 /* 4608 bits: products < 2^2048, sums of < 2^64 of them < 2^2112 */

typedef struct {
    uint64_t w[XLIMB]; /* two's complement, limb 0 least significant */
    int bad;           /* a non-finite operand was seen */
} exact_acc;

/* x = m * 2^e, m < 2^53 an integer (x finite) */
static void split_double(double x, uint64_t* m, int* e, int* neg)
{
    uint64_t bits;
    memcpy(&bits, &x, sizeof bits);
    *neg = (int)(bits >> 63);
    int ex = (int)((bits >> 52) & 0x7FF);
    uint64_t frac = bits & ((1ull << 52) - 1);
    if (ex == 0) {
        *m = frac;
        *e = -1074;
    } else {
        *m = frac | (1ull << 52);
        *e = ex - 1075;
    }
}

/* X += sign * v * 2^off, v < 2^128, 0 <= off */
static void acc_add(exact_acc* X, unsigned __int128 v, int off, int negative)
{
    int q = off / 64, r = off % 64;
    uint64_t part[3];
    part[0] = (uint64_t)(v << r);
    part[1] = (uint64_t)((r == 0) ? (v >> 64) : (v >> (64 - r)));
    part[2] = (uint64_t)((r == 0) ? 0 : ((v >> 64) >> (64 - r)));
    if (!negative) {
        unsigned __int128 carry = 0;
        for (int k = q; k < XLIMB; ++k) {
            unsigned __int128 t = (unsigned __int128)X->w[k] + carry +
                                  (k - q < 3 ? part[k - q] : 0);
            X->w[k] = (uint64_t)t;
            carry = t >> 64;
            if (k - q >= 2 && carry == 0) break;
        }
    } else {
        uint64_t borrow = 0;
        for (int k = q; k < XLIMB; ++k) {
            uint64_t sub = (k - q < 3 ? part[k - q] : 0);
            uint64_t old = X->w[k];
            uint64_t t = old - sub - borrow;
            borrow = (old < sub || (old - sub) < borrow) ? 1 : 0;
            X->w[k] = t;
            if (k - q >= 2 && borrow == 0) break;
        }
    }
}

static void acc_add_product(exact_acc* X, double a, double b)
{
    if (!isfinite(a) || !isfinite(b)) {
        X->bad = 1;
        return;
    }
    uint64_t ma, mb;
    int ea, eb, na, nb;
    split_double(a, &ma, &ea, &na);
    split_double(b, &mb, &eb, &nb);
    if (ma == 0 || mb == 0) return;
    unsigned __int128 M = (unsigned __int128)ma * mb;
    acc_add(X, M, ea + eb - XBASE, na != nb);
}

/* X += Y (exact) */
static void acc_merge(exact_acc* X, const exact_acc* Y)
{
    unsigned __int128 carry = 0;
    for (int k = 0; k < XLIMB; ++k) {
        unsigned __int128 t = (unsigned __int128)X->w[k] + Y->w[k] + carry;
        X->w[k] = (uint64_t)t;
        carry = t >> 64;
    }
    X->bad |= Y->bad;
}

/* round X * 2^XBASE to the nearest double, ties to even */
static double acc_round(const exact_acc* X)
{
    if (X->bad) return NAN;
    uint64_t mag[XLIMB];
    int negative = (int)(X->w[XLIMB - 1] >> 63);
    if (negative) { /* magnitude = ~X + 1 */
        unsigned __int128 carry = 1;
        for (int k = 0; k < XLIMB; ++k) {
            unsigned __int128 t = (unsigned __int128)(~X->w[k]) + carry;
            mag[k] = (uint64_t)t;
            carry = t >> 64;
        }
    } else {
        memcpy(mag, X->w, sizeof mag);
    }
    int top = XLIMB - 1;
    while (top >= 0 && mag[top] == 0) --top;
    if (top < 0) return 0.0;
    int msb = top * 64 + 63 - __builtin_clzll(mag[top]);
    int lsb = msb - 52; /* 53 significant bits ... */
    if (lsb < -1074 - XBASE) lsb = -1074 - XBASE; /* ... or the subnormal grid 2^-1074 */
#define XBIT(pos) ((pos) < 0 ? 0u : (unsigned)((mag[(pos) / 64] >> ((pos) % 64)) & 1u))
    uint64_t sig = 0;
    for (int pos = msb; pos >= lsb; --pos) sig = (sig << 1) | XBIT(pos);
    unsigned round_bit = XBIT(lsb - 1);
    int sticky = 0;
    for (int pos = lsb - 2; pos >= 0; --pos)
        if (XBIT(pos)) {
            sticky = 1;
            break;
        }
#undef XBIT
    if (round_bit && (sticky || (sig & 1u))) {
        sig += 1;
        if (sig == (1ull << 53)) {
            sig >>= 1;
            lsb += 1;
        }
    }
    double v = ldexp((double)sig, lsb + XBASE); /* exact, or inf beyond the range */
    return negative ? -v : v;
}

/* Dot over a field of nplanes planes of plen elements each: RN(exact sum).  OpenMP threads
 * accumulate disjoint planes into private exact accumulators, merged exactly. */
double orc_dot(int64_t plen, int64_t nplanes, const double* a, const double* b)
{
    exact_acc total;
    memset(&total, 0, sizeof total);
#pragma omp parallel
    {
        exact_acc mine;
        memset(&mine, 0, sizeof mine);
#pragma omp for schedule(static)
        for (int64_t k = 0; k < nplanes; ++k)
            for (int64_t i = 0; i < plen; ++i)
                acc_add_product(&mine, a[k * plen + i], b[k * plen + i]);
#pragma omp critical
        acc_merge(&total, &mine);
    }
    return acc_round(&total);
}

/* Dot2 pair (hi, lo) of a field -- the per-rank partial a z-slab decomposition would
 * contribute before the rank-ordered combination (R19). */
void orc_dot_pair(int64_t plen, int64_t nplanes, const double* a, const double* b, double* out2)
{
    double P = 0.0, S = 0.0;
    for (int64_t k = 0; k < nplanes; ++k) {
        double hi, lo, q;
        dot2_run(plen, a + k * plen, b + k * plen, &hi, &lo);
        two_sum(P, hi, &P, &q);
        S = S + (q + lo);
    }
    out2[0] = P;
    out2[1] = S;
}

/* ------------------------------------------------------------------------------------------
 * Eigenvalue bounds.  Eq. 9: eigenvalues of D_n are 4 sin²(iπ/(2(n+1))).
 * Eqs. 10-11: λmin/λmax of P = Σ_axes min/max μ / Δ².
 *   mu(n, i)  = 4.0 * (s*s),  s = sin(((double)i * M_PI) / (2.0 * (double)(n + 1)))
 *   lam       = ((mu_x * h2inv) + (mu_y * h2inv)) + (mu_z * h2inv)
 * The local block R_s A R_s^T of a z-slab of L planes is the Dirichlet box nx*ny*L
 * (Eq. 14, P:202 with zero ghosts at the cuts), so its bounds use L in place of nz.
 * ---------------------------------------------------------------------------------------- */
double orc_mu(int64_t n, int64_t i)
{
    double s = sin(((double)i * M_PI) / (2.0 * (double)(n + 1)));
    return 4.0 * (s * s);
}

void orc_bounds(int64_t nx, int64_t ny, int64_t nzb, double h, double* lmin, double* lmax)
{
    double h2inv = 1.0 / (h * h);
    *lmin = ((orc_mu(nx, 1) * h2inv) + (orc_mu(ny, 1) * h2inv)) + (orc_mu(nzb, 1) * h2inv);
    *lmax = ((orc_mu(nx, nx) * h2inv) + (orc_mu(ny, ny) * h2inv)) + (orc_mu(nzb, nzb) * h2inv);
}

/* Mixed boundary conditions (Eq. 5; DESIGN.md §3 R27).  The paper gives no closed
 * form for the eigenvalues of N and falls back on Gerschgorin's [0, 4], whose lower
 * end 0 cannot be rescaled by c_min (R9).  The 1-D factor with the mirror rule on one end
 * has the closed form 4 sin²((2i-1)π/(4n)), i = 1..n (eigenvectors cos((2i-1)π j/(2n)));
 * with Neumann on both ends 4 sin²(iπ/(2(n-1))), i = 0..n-1 (cos(iπ j/(n-1))).  Both are
 * pinned against dense eigen-solves of Eq. 5's matrices.  kind = number of Neumann ends. */
double orc_mu_bc(int64_t n, int64_t i, int kind)
{
    double s;
    if (kind == 0) return orc_mu(n, i);
    if (kind == 1) s = sin(((double)(2 * i - 1) * M_PI) / (4.0 * (double)n));
    else s = sin(((double)i * M_PI) / (2.0 * (double)(n - 1)));
    return 4.0 * (s * s);
}

static void axis_range(int64_t n, int kind, double* mn, double* mx)
{
    if (kind == 2) {
        *mn = orc_mu_bc(n, 0, 2);
        *mx = orc_mu_bc(n, n - 1, 2);
    } else {
        *mn = orc_mu_bc(n, 1, kind);
        *mx = orc_mu_bc(n, n, kind);
    }
}

/* Eqs. 10-11 with per-axis kinds (kx, ky, kz = Neumann ends of that axis' factor). */
void orc_bounds_bc(int64_t nx, int64_t ny, int64_t nzb, double h, int kx, int ky, int kz,
                   double* lmin, double* lmax)
{
    double h2inv = 1.0 / (h * h), ax, bx, ay, by, az, bz;
    axis_range(nx, kx, &ax, &bx);
    axis_range(ny, ky, &ay, &by);
    axis_range(nzb, kz, &az, &bz);
    *lmin = ((ax * h2inv) + (ay * h2inv)) + (az * h2inv);
    *lmax = ((bx * h2inv) + (by * h2inv)) + (bz * h2inv);
}

/* ------------------------------------------------------------------------------------------
 * Chebyshev iteration, Alg. 2 as implemented in Alg. 4.
 * Interval [a, b] (Eq. 15): θ = (b+a)/2, δ = (b-a)/2, σ = θ/δ.
 * ρ_0 = 1/σ; ρ_j = 1/(2σ - ρ_{j-1}) (the garbled "1/2σ - ρ_old" of
 * Alg. 4 line 2, is read as Alg. 2's 1/(2σ - ρ_old): DESIGN.md §3 R2).
 * Host constants: cz = 1/θ, g1 = 2*(ρ_1/δ), A2 = 2*σ, B2 = 2/δ (DESIGN.md §3 R18).
 * iterMax = k (DESIGN.md §3 R1): k = 0 returns z = b/θ; k = 1 returns y;
 * k >= 2 runs the loop of P:224-230 and returns w.
 * The stencil inside is the block operator (nslab cuts): GNoComm / BJ.
 * ---------------------------------------------------------------------------------------- */
#define ORC_KMAX 256

typedef struct {
    double theta, delta, sigma, cz, g1, A2, B2;
    double rho[ORC_KMAX + 2];
} orc_cheb;

int orc_cheb_setup(double a, double b, int k, double* out7, double* rho_out)
{
    orc_cheb c;
    if (k < 0 || k > ORC_KMAX) return 1;
    c.theta = (b + a) / 2.0;
    c.delta = (b - a) / 2.0;
    if (!(c.delta > 0.0) || !(a > 0.0)) return 2;
    c.sigma = c.theta / c.delta;
    c.rho[0] = 1.0 / c.sigma;
    for (int j = 1; j <= (k > 1 ? k : 1); ++j) c.rho[j] = 1.0 / (2.0 * c.sigma - c.rho[j - 1]);
    c.cz = 1.0 / c.theta;
    c.g1 = 2.0 * (c.rho[1] / c.delta);
    c.A2 = 2.0 * c.sigma;
    c.B2 = 2.0 / c.delta;
    if (out7) {
        out7[0] = c.theta; out7[1] = c.delta; out7[2] = c.sigma; out7[3] = c.cz;
        out7[4] = c.g1; out7[5] = c.A2; out7[6] = c.B2;
    }
    if (rho_out)
        for (int j = 0; j <= (k > 1 ? k : 1); ++j) rho_out[j] = c.rho[j];
    return 0;
}

int orc_apply_cheb_bc(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab, int bcm,
                      int k, double a, double b, const double* q, double* out)
{
    double cst[7], rho[ORC_KMAX + 2];
    int rc = orc_cheb_setup(a, b, k, cst, rho);
    if (rc) return rc;
    double cz = cst[3], g1 = cst[4], A2 = cst[5], B2 = cst[6];
    int64_t n = nx * ny * nz;

    if (k == 0) {                                   /* z = b/θ; iterMax = 0 exits here */
        for (int64_t c = 0; c < n; ++c) out[c] = q[c] * cz;
        return 0;
    }
    double* S = (double*)malloc(sizeof(double) * (size_t)n);
    double* y = (double*)malloc(sizeof(double) * (size_t)n);
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    double* w = (double*)malloc(sizeof(double) * (size_t)n);

    /* KernelCI1: z = b/θ ; y = 2(ρ_cur/δ)(2b - A b/θ) */
    orc_apply_A_bc(nx, ny, nz, h, nslab, bcm, q, S);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) {
        z[c] = q[c] * cz;
        y[c] = g1 * fma(-S[c], cz, 2.0 * q[c]);     /* g1 (2b - (A b) cz), R18 */
    }
    /* KernelCI2 for i = 2..iterMax, with the pointer swaps of P:361-362 */
    for (int j = 2; j <= k; ++j) {
        orc_apply_A_bc(nx, ny, nz, h, nslab, bcm, y, S);
        double rc_ = rho[j], ro_ = rho[j - 1];
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c)
            w[c] = rc_ * fma(-ro_, z[c], fma(A2, y[c], B2 * (q[c] - S[c])));   /* R18 */
        double* tmp = z; z = y; y = w; w = tmp;   /* z <- y, y <- w */
    }
    /* KernelCI3: x = w (after the swap, the last w is in y) */
    memcpy(out, y, sizeof(double) * (size_t)n);
    free(S); free(y); free(z); free(w);
    return 0;
}

int orc_apply_cheb(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab, int k,
                   double a, double b, const double* q, double* out)
{
    return orc_apply_cheb_bc(nx, ny, nz, h, nslab, 0, k, a, b, q, out);
}

/* Chebyshev interval [a', b'] of a preconditioner (pc 1 GNoComm, 3 G(CI): global bounds
 * rescaled by (c_min, c_max), R9; pc 2 BJ: exact bounds of the local blocks, R10).  The BJ
 * blocks differ only in their z factor (first block: kind of face z-, last: kind of face
 * z+, middle: Dirichlet at both cuts); one interval covers every block's spectrum (R27). */
void orc_pc_interval(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab, int bcm,
                     int pc, double c_min, double c_max, double* out2)
{
    const int kx = (bcm & 1) + ((bcm >> 1) & 1), ky = ((bcm >> 2) & 1) + ((bcm >> 3) & 1),
              kz = ((bcm >> 4) & 1) + ((bcm >> 5) & 1);
    double a_iv = 0.0, b_iv = 0.0;
    if (pc == 1 || pc == 3) {
        double lmn, lmx;
        orc_bounds_bc(nx, ny, nz, h, kx, ky, kz, &lmn, &lmx);
        a_iv = c_min * lmn;
        b_iv = c_max * lmx;
    } else if (nslab == 1) {
        orc_bounds_bc(nx, ny, nz, h, kx, ky, kz, &a_iv, &b_iv);
    } else {
        int kinds[3] = {(bcm >> 4) & 1, (bcm >> 5) & 1, 0};
        int nk = nslab > 2 ? 3 : 2;
        for (int q = 0; q < nk; ++q) {
            double lmn, lmx;
            orc_bounds_bc(nx, ny, nz / nslab, h, kx, ky, kinds[q], &lmn, &lmx);
            if (q == 0 || lmn < a_iv) a_iv = lmn;
            if (q == 0 || lmx > b_iv) b_iv = lmx;
        }
    }
    out2[0] = a_iv;
    out2[1] = b_iv;
}

/* ------------------------------------------------------------------------------------------
 * Inner-Krylov preconditioners: FBiCGS-BJ(BiCGS) and FBiCGS-G(BiCGS),
 * P:176-207.  M_i^{-1} p is computed "as a solution of the linear system
 * (R_s A R_s^T) p̂_s = p_s" on every subdomain s (Eq. 15) by "the already available
 * BiCGS method": the unpreconditioned Alg. 3 below (M = I) on the block, x0 = 0,
 * relative tolerance tol_in, at most max_in iterations (1e-6 / 500 for BJ(BiCGS),
 * 1e-2 / 500 for G(BiCGS) = one block spanning the whole domain).  The block operator has
 * zero ghosts at the cuts (Eq. 12-14) and keeps the physical faces (a Neumann z face only in
 * the first / last block).  Reading (paper silent): the inner result is used whatever the
 * inner status (converged, breakdown or iteration cap).  The outer solver is flexible
 * because Alg. 3 stores p̂ and r̂.
 * ---------------------------------------------------------------------------------------- */
int orc_bicgstab_ex(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab, int bcm,
                    int pc, int k, double c_min, double c_max, double lmin_ov, double lmax_ov,
                    double tol_in, int max_in, int flags, const double* b, const double* x0,
                    double tol,
                    int max_it, int fixed_it, double* x, double* hist, double* scal,
                    int* iters_out, double* true_rel, long long* inner_total);

static void apply_inner_bicgs(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab,
                              int bcm, double tol_in, int max_in, const double* q, double* out,
                              long long* inner_total)
{
    int64_t Lb = nz / nslab, pl = nx * ny;
    double* hist = (double*)malloc(sizeof(double) * (size_t)(max_in + 1));
    for (int64_t s = 0; s < nslab; ++s) {
        int bcm_s = (bcm & 15) | (s == 0 ? (bcm & 16) : 0) | (s == nslab - 1 ? (bcm & 32) : 0);
        int its = 0;
        orc_bicgstab_ex(nx, ny, Lb, h, 1, bcm_s, 0, 0, 0.0, 0.0, 0.0, 0.0, 0.0, 0, 0,
                        q + s * Lb * pl, NULL, tol_in, max_in, 0, out + s * Lb * pl, hist,
                        NULL, &its, NULL, NULL);
        if (inner_total) *inner_total += its;
    }
    free(hist);
}

/* ------------------------------------------------------------------------------------------
 * Preconditioned Bi-CGSTAB, Alg. 3, Alg. 1 for the scalar forms.
 *
 * pc: 0 = none (M = I), 1 = GNoComm(CI), 2 = BJ(CI), 3 = G(CI).
 * nslab = number of z-slabs of the decomposition (ranks x blocks per rank): the
 * preconditioner acts on each slab separately (Eq. 13); the global stencils of
 * KernelBiCGS1/3 ignore the cuts (halo exchange MPI1/MPI3).
 * Bounds: GNoComm uses the global Eq. 9-11 bounds rescaled by (c_min, c_max);
 * BJ uses the exact bounds of the local Dirichlet block, unscaled (DESIGN.md §3 R10).
 * lmin_ov/lmax_ov > 0 override the interval [a', b'] directly.
 *
 * Stopping rule (DESIGN.md §3 R4): rel_i = sqrt(rᵀr)/||b|| < tol.  fixed_it > 0 runs exactly
 * fixed_it iterations (tol ignored).  Breakdown (R7): r~ᵀw == 0 or non-finite -> stop before
 * any update in that iteration; after the residual update, ω == 0, ρ_new == 0 or any
 * non-finite scalar -> stop.  tᵀt == 0 -> ω = 0 (R6).
 *
 * Outputs: x (solution), hist[0..iters] (hist[0] = 1), scal[8*(i-1) + ...] per iteration =
 * {rw, alpha, ts, tt, omega, rho_new, rr, beta}.  Returns status:
 *   0 converged / fixed iterations done, 6 not converged (max_it), 7 breakdown, 1 bad config.
 * *iters_out = number of completed iterations (each appended one entry to hist); a
 * breakdown at r~ᵀw ends the run before iteration i appends anything (iters = i-1).
 * ---------------------------------------------------------------------------------------- */
/* ------------------------------------------------------------------------------------------
 * Pipelined Bi-CGSTAB (flags bit 1, the paper's "communication-
 * avoiding/reducing algorithms" future work): the communication-hiding p-BiCGStab of
 * Cools & Vanroose (2017) for the right-preconditioned operator B = A M^-1, written out from
 * Alg. 3 by the recurrences below; in exact arithmetic it produces the iterates
 * of Alg. 3.  With S = B p, z = B S, w = B r, t = B w, v = B z, q = r - α S (Alg. 3's s),
 * y = B q (Alg. 3's t), and hats = M^-1 (p̂ = M^-1 p, ...):
 *   p = r + β(p - ω S)        p̂ = r̂ + β(p̂ - ω Ŝ)
 *   S = w + β(S - ω z)        Ŝ = ŵ + β(Ŝ - ω ẑ)
 *   z = t + β(z - ω v)        ẑ = M^-1 z        v = A ẑ          (2nd stencil overlaps R1)
 *   q = r - α S      q̂ = r̂ - α Ŝ      y = w - α z
 *   R1: (q, y), (y, y) -> ω = (q, y)/(y, y)
 *   x += α p̂ + ω q̂     r = q - ω y     r̂ = q̂ - ω(ŵ - α ẑ)     w = y - ω(t - α v)
 *   ŵ = M^-1 w        t = A ŵ                                  (1st stencil overlaps R2)
 *   R2: (r~, r), (r~, w), (r~, S), (r~, z), (r, r)
 *   β = (ρ_new/ρ)(α/ω);   α = ρ_new / (β((r~, S) - ω (r~, z)) + (r~, w))
 * Two reductions per iteration (three in Alg. 3), each independent of the stencil +
 * preconditioner application that follows it.  Start: w = A r̂0, ŵ = M^-1 w, t = A ŵ,
 * α0 = ρ0/(r~, w0), β = ω = 0 (so p0 = r0, S0 = w0, z0 = t0).  Linear preconditioners only
 * (the recurrences for the hatted vectors need M^-1 fixed).  Expression trees (contract
 * R20 style): every update is the nested fma written above, a + β(b - ω c) =
 * fma(β, fma(-ω, c, b), a).  Scalars per iteration: (r~,w)-combination, α, (q,y), (y,y), ω,
 * ρ_new, (r,r), β.  Stopping and breakdown as R4 / R6 / R7.
 * ---------------------------------------------------------------------------------------- */
static int pbicgstab(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab_pc, int bcm,
                     int pc, int k, double a_iv, double b_iv, const double* b, const double* x0,
                     double tol, int max_run, int fixed_it, double* x, double* hist,
                     double* scal, int* iters_out, double* true_rel)
{
    int64_t n = nx * ny * nz, pl = nx * ny;
    double* V[18];
    for (int i = 0; i < 18; ++i) V[i] = (double*)calloc((size_t)n, sizeof(double));
    double *r = V[0], *rh = V[1], *w = V[2], *wh = V[3], *t = V[4], *p = V[5], *ph = V[6],
           *S = V[7], *Sh = V[8], *z = V[9], *zh = V[10], *q = V[11], *qh = V[12], *y = V[13],
           *v = V[14], *rt = V[15], *tmp = V[16];
#define APPLY_M(in, out)                                                                    \
    do {                                                                                    \
        if (pc == 0) memcpy((out), (in), sizeof(double) * (size_t)n);                       \
        else orc_apply_cheb_bc(nx, ny, nz, h, nslab_pc, bcm, k, a_iv, b_iv, (in), (out));   \
    } while (0)
    if (x0) {
        memcpy(x, x0, sizeof(double) * (size_t)n);
        orc_apply_A_bc(nx, ny, nz, h, 1, bcm, x, tmp);
        for (int64_t c = 0; c < n; ++c) r[c] = b[c] - tmp[c];
    } else {
        memset(x, 0, sizeof(double) * (size_t)n);
        memcpy(r, b, sizeof(double) * (size_t)n);
    }
    memcpy(rt, r, sizeof(double) * (size_t)n);
    double rho = orc_dot(pl, nz, rt, r);
    double nb = sqrt(orc_dot(pl, nz, b, b));
    int status = 6, it = 0;
    if (nb == 0.0) {
        hist[0] = 0.0;
        status = 0;
        goto done;
    }
    hist[0] = sqrt(rho) / nb;
    if (fixed_it <= 0 && hist[0] < tol) {
        status = 0;
        goto done;
    }
    /* start: r̂ = M^-1 r, w = A r̂, ŵ = M^-1 w, t = A ŵ, α0 = ρ0 / (r~, w0) */
    APPLY_M(r, rh);
    orc_apply_A_bc(nx, ny, nz, h, 1, bcm, rh, w);
    APPLY_M(w, wh);
    orc_apply_A_bc(nx, ny, nz, h, 1, bcm, wh, t);
    double den = orc_dot(pl, nz, rt, w);
    if (den == 0.0 || !isfinite(den)) { status = 7; goto done; }
    double alpha = rho / den, beta = 0.0, omega = 0.0;
    for (int i = 1; i <= max_run; ++i) {
        it = i;
        double* sc = scal ? scal + 8 * (i - 1) : NULL;
        if (sc) { sc[0] = den; sc[1] = alpha; }
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c) {
            p[c] = fma(beta, fma(-omega, S[c], p[c]), r[c]);
            ph[c] = fma(beta, fma(-omega, Sh[c], ph[c]), rh[c]);
            S[c] = fma(beta, fma(-omega, z[c], S[c]), w[c]);
            Sh[c] = fma(beta, fma(-omega, zh[c], Sh[c]), wh[c]);
            z[c] = fma(beta, fma(-omega, v[c], z[c]), t[c]);
        }
        APPLY_M(z, zh);
        orc_apply_A_bc(nx, ny, nz, h, 1, bcm, zh, v);
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c) {
            q[c] = fma(-alpha, S[c], r[c]);
            qh[c] = fma(-alpha, Sh[c], rh[c]);
            y[c] = fma(-alpha, z[c], w[c]);
        }
        double qy = orc_dot(pl, nz, q, y);                        /* R1 */
        double yy = orc_dot(pl, nz, y, y);
        omega = (yy == 0.0) ? 0.0 : qy / yy;                       /* R6 */
        if (sc) { sc[2] = qy; sc[3] = yy; sc[4] = omega; }
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c) {
            x[c] = fma(omega, qh[c], fma(alpha, ph[c], x[c]));
            r[c] = fma(-omega, y[c], q[c]);
            rh[c] = fma(-omega, fma(-alpha, zh[c], wh[c]), qh[c]);
            w[c] = fma(-omega, fma(-alpha, v[c], t[c]), y[c]);
        }
        APPLY_M(w, wh);
        orc_apply_A_bc(nx, ny, nz, h, 1, bcm, wh, t);
        double rho_new = orc_dot(pl, nz, rt, r);                  /* R2 */
        double rw = orc_dot(pl, nz, rt, w);
        double rS = orc_dot(pl, nz, rt, S);
        double rz = orc_dot(pl, nz, rt, z);
        double rr = orc_dot(pl, nz, r, r);
        double rel = sqrt(rr) / nb;
        hist[i] = rel;
        if (sc) { sc[5] = rho_new; sc[6] = rr; sc[7] = 0.0; }
        if (fixed_it > 0) {
            if (i == fixed_it) { status = 0; break; }
        } else if (rel < tol) {
            status = 0;
            break;
        }
        if (omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new) || !isfinite(rr) ||
            !isfinite(omega)) {
            status = 7;
            break;
        }
        beta = (rho_new / rho) * (alpha / omega);                  /* R20 form */
        rho = rho_new;
        if (sc) sc[7] = beta;
        den = fma(beta, fma(-omega, rz, rS), rw);
        if (den == 0.0 || !isfinite(den)) { status = 7; break; }
        alpha = rho_new / den;
        if (fixed_it <= 0 && i == max_run) status = 6;
    }
#undef APPLY_M
done:
    if (iters_out) *iters_out = it;
    if (true_rel) {
        orc_apply_A_bc(nx, ny, nz, h, 1, bcm, x, tmp);
        for (int64_t c = 0; c < n; ++c) tmp[c] = b[c] - tmp[c];
        *true_rel = nb == 0.0 ? 0.0 : sqrt(orc_dot(pl, nz, tmp, tmp)) / nb;
    }
    for (int i = 0; i < 18; ++i) free(V[i]);
    return status;
}

int orc_bicgstab_ex(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab, int bcm,
                    int pc, int k, double c_min, double c_max, double lmin_ov, double lmax_ov,
                    double tol_in, int max_in, int flags, const double* b, const double* x0,
                    double tol,
                    int max_it, int fixed_it, double* x, double* hist, double* scal,
                    int* iters_out, double* true_rel, long long* inner_total)
{
    int64_t n = nx * ny * nz, pl = nx * ny;
    if (nslab < 1 || nz % nslab != 0) return 1;
    /* mirror ghosts need a second point on a Neumann axis, and (z) inside every block */
    if (((bcm & 3) && nx < 2) || ((bcm & 12) && ny < 2) || ((bcm & 48) && nz / nslab < 2))
        return 1;
    double a_iv = 0.0, b_iv = 0.0;
    /* pc 3 = G(CI): Chebyshev on the global operator (no slab cuts) with the
     * global rescaled bounds -- the preconditioner is independent of the decomposition. */
    const int64_t nslab_pc = (pc == 3) ? 1 : nslab;
    if (pc == 1 || pc == 2 || pc == 3) {
        if (lmin_ov > 0.0 && lmax_ov > 0.0) {
            a_iv = lmin_ov; b_iv = lmax_ov;
        } else {
            double iv[2];
            orc_pc_interval(nx, ny, nz, h, nslab, bcm, pc, c_min, c_max, iv);
            a_iv = iv[0]; b_iv = iv[1];
        }
        if (!(a_iv < b_iv) || !(a_iv > 0.0)) return 1;
    } else if (pc == 4 || pc == 5) {           /* BJ(BiCGS) / G(BiCGS) */
        if (!(tol_in > 0.0) || max_in < 1) return 1;
    } else if (pc != 0) {
        return 1;
    }
    /* pc 5 = G(BiCGS): one inner solve over the whole domain (no block cuts) */
    const int64_t nslab_in = (pc == 5) ? 1 : nslab;
    int max_run = fixed_it > 0 ? fixed_it : max_it;
    if (flags & 2) {   /* pipelined Bi-CGSTAB: linear preconditioners only */
        if (pc >= 4 || (flags & 1)) return 1;
        return pbicgstab(nx, ny, nz, h, nslab_pc, bcm, pc, k, a_iv, b_iv, b, x0, tol, max_run,
                         fixed_it, x, hist, scal, iters_out, true_rel);
    }

    double* r = (double*)calloc((size_t)n, sizeof(double));
    double* rt = (double*)calloc((size_t)n, sizeof(double));
    double* p = (double*)calloc((size_t)n, sizeof(double));
    double* ph = (double*)calloc((size_t)n, sizeof(double));
    double* rh = (double*)calloc((size_t)n, sizeof(double));
    double* w = (double*)calloc((size_t)n, sizeof(double));
    double* t = (double*)calloc((size_t)n, sizeof(double));
    double* tmp = (double*)calloc((size_t)n, sizeof(double));

    /* Alg. 3 line 1: r0 = b - A x0 */
    if (x0) {
        memcpy(x, x0, sizeof(double) * (size_t)n);
        orc_apply_A_bc(nx, ny, nz, h, 1, bcm, x, tmp);
        for (int64_t c = 0; c < n; ++c) r[c] = b[c] - tmp[c];
    } else {
        memset(x, 0, sizeof(double) * (size_t)n);
        memcpy(r, b, sizeof(double) * (size_t)n);
    }
    /* line 2-4: r~ = r0, p0 = r0, ρ0 = r~ᵀ r0 */
    memcpy(rt, r, sizeof(double) * (size_t)n);
    memcpy(p, r, sizeof(double) * (size_t)n);
    double rho = orc_dot(pl, nz, rt, r);
    double nb = sqrt(orc_dot(pl, nz, b, b));     /* ||b||: relative tolerance */
    int status = 6, it = 0;
    if (nb == 0.0) {          /* b = 0: report converged with x = x0 (R26) */
        hist[0] = 0.0;
        status = 0;
        goto done;
    }
    /* R26: rel_0 = sqrt(r~ᵀr0)/||b|| (= 1 for x0 = 0); a converged initial guess stops
     * before the first iteration (tol mode). */
    hist[0] = sqrt(rho) / nb;
    if (fixed_it <= 0 && hist[0] < tol) {
        status = 0;
        goto done;
    }
    for (int i = 1; i <= max_run; ++i) {
        it = i;
        double* sc = scal ? scal + 8 * (i - 1) : NULL;
        /* line 6: solve M p̂ = p */
        if (pc == 0) memcpy(ph, p, sizeof(double) * (size_t)n);
        else if (pc >= 4) apply_inner_bicgs(nx, ny, nz, h, nslab_in, bcm, tol_in, max_in, p, ph,
                                            inner_total);
        else orc_apply_cheb_bc(nx, ny, nz, h, nslab_pc, bcm, k, a_iv, b_iv, p, ph);
        /* MPI1 + KernelBiCGS1: w = A p̂ (global), local r~ᵀw; MPI2 */
        orc_apply_A_bc(nx, ny, nz, h, 1, bcm, ph, w);
        double rw = orc_dot(pl, nz, rt, w);
        if (sc) sc[0] = rw;
        if (rw == 0.0 || !isfinite(rw)) { status = 7; it = i - 1; break; }
        double alpha = rho / rw;
        if (sc) sc[1] = alpha;
        /* KernelBiCGS2: r = r - α w   (the half-step residual, "s") */
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c) r[c] = fma(-alpha, w[c], r[c]);
        /* solve M r̂ = r */
        if (pc == 0) memcpy(rh, r, sizeof(double) * (size_t)n);
        else if (pc >= 4) apply_inner_bicgs(nx, ny, nz, h, nslab_in, bcm, tol_in, max_in, r, rh,
                                            inner_total);
        else orc_apply_cheb_bc(nx, ny, nz, h, nslab_pc, bcm, k, a_iv, b_iv, r, rh);
        /* MPI3 + KernelBiCGS3: t = A r̂, tᵀr, tᵀt; MPI4 */
        orc_apply_A_bc(nx, ny, nz, h, 1, bcm, rh, t);
        double ts = orc_dot(pl, nz, t, r);
        double tt = orc_dot(pl, nz, t, t);
        /* flags bit 0 (R31, SURVEY §8(e) 2-sync rewrite): also r~ᵀs, r~ᵀt, sᵀs here, so that
         * MPI5 disappears: ρ_new = r~ᵀs - ω r~ᵀt and ||r||² = sᵀs - 2ω tᵀs + ω² tᵀt (algebraic
         * identities for r = s - ω t) */
        double rts = 0.0, rtt = 0.0, ss = 0.0;
        if (flags & 1) {
            rts = orc_dot(pl, nz, rt, r);
            rtt = orc_dot(pl, nz, rt, t);
            ss = orc_dot(pl, nz, r, r);
        }
        double omega = (tt == 0.0) ? 0.0 : ts / tt;  /* P:293, guard R6 */
        if (sc) { sc[2] = ts; sc[3] = tt; sc[4] = omega; }
        /* KernelBiCGS4: x = x + α p̂ + ω r̂ */
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c) x[c] = fma(omega, rh[c], fma(alpha, ph[c], x[c]));
        /* KernelBiCGS5: r = r - ω t, r0ᵀr, rᵀr; MPI5 */
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c) r[c] = fma(-omega, t[c], r[c]);
        double rho_new, rr;
        if (flags & 1) {     /* R31: fma forms, ||r||² clamped at 0 (cancellation) */
            rho_new = fma(-omega, rtt, rts);
            rr = fma(-omega, fma(-omega, tt, 2.0 * ts), ss);
            if (rr < 0.0) rr = 0.0;
        } else {
            rho_new = orc_dot(pl, nz, rt, r);
            rr = orc_dot(pl, nz, r, r);
        }
        double rel = sqrt(rr) / nb;
        hist[i] = rel;
        if (sc) { sc[5] = rho_new; sc[6] = rr; sc[7] = 0.0; }
        /* P:300-302 stopping test */
        if (fixed_it > 0) {
            if (i == fixed_it) { status = 0; break; }
        } else if (rel < tol) {
            status = 0;
            break;
        }
        if (omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new) || !isfinite(rr) ||
            !isfinite(omega)) {
            status = 7;
            break;
        }
        /* ρ_i, β_i  (Alg. 1 form: β = (ρ_i/ρ_{i-1})(α/ω); R20) */
        double beta = (rho_new / rho) * (alpha / omega);
        rho = rho_new;
        if (sc) sc[7] = beta;
        /* KernelBiCGS6: p = r + β (p - ω w) */
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c) p[c] = fma(beta, fma(-omega, w[c], p[c]), r[c]);
    }
done:
    *iters_out = it;
    if (true_rel) {
        orc_apply_A_bc(nx, ny, nz, h, 1, bcm, x, tmp);
        for (int64_t c = 0; c < n; ++c) tmp[c] = b[c] - tmp[c];
        *true_rel = nb == 0.0 ? 0.0 : sqrt(orc_dot(pl, nz, tmp, tmp)) / nb;
    }
    free(r); free(rt); free(p); free(ph); free(rh); free(w); free(t); free(tmp);
    return status;
}

/* One application of the inner-Krylov preconditioner: out = M^{-1} q on nslab blocks.
 * Returns the total number of inner iterations. */
long long orc_apply_inner(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab, int bcm,
                          double tol_in, int max_in, const double* q, double* out)
{
    long long tot = 0;
    apply_inner_bicgs(nx, ny, nz, h, nslab, bcm, tol_in, max_in, q, out, &tot);
    return tot;
}

int orc_bicgstab_bc(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab, int bcm,
                    int pc, int k, double c_min, double c_max, double lmin_ov, double lmax_ov,
                    const double* b, const double* x0, double tol, int max_it, int fixed_it,
                    double* x, double* hist, double* scal, int* iters_out, double* true_rel)
{
    return orc_bicgstab_ex(nx, ny, nz, h, nslab, bcm, pc, k, c_min, c_max, lmin_ov, lmax_ov,
                           0.0, 0, 0, b, x0, tol, max_it, fixed_it, x, hist, scal, iters_out,
                           true_rel, NULL);
}

int orc_bicgstab(int64_t nx, int64_t ny, int64_t nz, double h, int64_t nslab, int pc, int k,
                 double c_min, double c_max, double lmin_ov, double lmax_ov,
                 const double* b, const double* x0, double tol, int max_it, int fixed_it,
                 double* x, double* hist, double* scal, int* iters_out, double* true_rel)
{
    return orc_bicgstab_bc(nx, ny, nz, h, nslab, 0, pc, k, c_min, c_max, lmin_ov, lmax_ov, b,
                           x0, tol, max_it, fixed_it, x, hist, scal, iters_out, true_rel);
}

/* Number of OpenMP threads the oracle's parallel loops use (reported as cpu_baseline.cores). */
int orc_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
