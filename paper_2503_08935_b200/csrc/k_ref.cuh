// k_ref.cuh -- reference kernels: one stencil sweep per launch, one Alg. 3 operation per
// launch.  They are the B200 counterparts of the paper's KernelBiCGS1..6 / KernelCI1..3
// and serve as the bitwise twin of the fused kernels (k_fused.cuh).
//
// Field layout: every vector is (L+2) planes of nx*ny doubles; `base` points at interior
// plane 0, ghost planes at base - plane and base + L*plane (zero, or halo data from the
// z-neighbours).  Stencil (R17): (6 c - (((((xm+xp)+ym)+yp)+zm)+zp)) * h2inv.
#pragma once
#include "dd.cuh"
#include "expr.cuh"
#include "ref_shapes.cuh"
#include "state.cuh"

namespace ref {

// ------------------------------------------------------------------- random RHS (R16)
__global__ void k_rhs_random(double* __restrict__ b, int64_t n, int64_t g0, uint64_t seed)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (uint64_t)(g0 + c + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
        double u = (double)(z >> 11) * 0x1.0p-53;
        b[c] = 2.0 * u - 1.0;
    }
}

// ------------------------------------------------------------------- boundary fold (R15)
__global__ void k_fold_boundary(double* __restrict__ b, Grid g, int64_t z0, int64_t nzg,
                                double a0, double a1, double a2, double a3, double a4,
                                double a5, int mask)
{
    const int64_t plane = (int64_t)g.nx * g.ny, n = plane * g.L;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(c % g.nx), j = (int)((c / g.nx) % g.ny);
        const int64_t kg = z0 + c / plane;
        double v = b[c];
        if ((mask & 1) && i == 0) v = v + a0;
        if ((mask & 2) && i == g.nx - 1) v = v + a1;
        if ((mask & 4) && j == 0) v = v + a2;
        if ((mask & 8) && j == g.ny - 1) v = v + a3;
        if ((mask & 16) && kg == 0) v = v + a4;
        if ((mask & 32) && kg == nzg - 1) v = v + a5;
        b[c] = v;
    }
}

// ------------------------------------------------------------------- stencil helpers
// Neighbour sum of the 7-point stencil at (i, j, k); z-neighbours passed in (they may be
// block-cut zeros or ghost-plane values).
// Out-of-domain x / y neighbours: 0 (Dirichlet) or, on a Neumann face (bit of m), the
// interior neighbour on the other side (R27 mirror ghost, Eq. 5).
__device__ __forceinline__ double stencil_at(const double* __restrict__ v, int64_t c, int i,
                                             int j, int nx, int ny, double vzm, double vzp,
                                             double h2inv, int m)
{
    const double xm = (i > 0) ? v[c - 1] : ((m & 1) ? v[c + 1] : 0.0);
    const double xp = (i < nx - 1) ? v[c + 1] : ((m & 2) ? v[c - 1] : 0.0);
    const double ym = (j > 0) ? v[c - nx] : ((m & 4) ? v[c + nx] : 0.0);
    const double yp = (j < ny - 1) ? v[c + nx] : ((m & 8) ? v[c - nx] : 0.0);
    return stencil_row(v[c], xm, xp, ym, yp, vzm, vzp, h2inv);
}

// ------------------------------------------------------------------- a4 / a9 (+ apply_A)
// out = A in (global operator: ghost planes hold neighbour-rank data or zeros);
// ND = 0: no dot; ND = 1: partial a·out (KernelBiCGS1);
// ND = 2: partials a·out and out·out (KernelBiCGS3).
// block_local != 0: block-diagonal operator (cuts every Lb planes), used by apply_operator.
template <int ND>
__global__ void __launch_bounds__(BX * BY) k_stencil_dot(const double* __restrict__ in,
                                                         const double* __restrict__ a,
                                                         double* __restrict__ out, Grid g,
                                                         int block_local, dd* __restrict__ part,
                                                         const DevState* __restrict__ st)
{
    if (st && st->done) return;
    const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y;
    const int k0 = blockIdx.z * ZC, k1 = min(g.L, k0 + ZC);
    constexpr int NDA = (ND > 0) ? ND : 1;
    double p[NDA] = {}, m[NDA] = {}, s[NDA] = {}, ab[NDA] = {};
    if (i < g.nx && j < g.ny) {
        const int64_t plane = (int64_t)g.nx * g.ny;
        int64_t c = i + (int64_t)g.nx * j + plane * k0;
        double vzm = in[c - plane], vc = in[c];
        for (int k = k0; k < k1; ++k, c += plane) {
            const double vzp = in[c + plane];
            const double zm = (k == g.bc.zlo) ? vzp
                              : (block_local && (k % g.Lb) == 0) ? 0.0 : vzm;
            const double zp = (k == g.bc.zhi) ? vzm
                              : (block_local && (k % g.Lb) == g.Lb - 1) ? 0.0 : vzp;
            const double o = stencil_at(in, c, i, j, g.nx, g.ny, zm, zp, g.h2inv, g.bc.m);
            out[c] = o;
            if (ND == 1) dot3_acc(p[0], m[0], s[0], ab[0], a[c], o);   // r~ᵀw: Dot3
            if (ND == 2) dot2_acc(p[0], s[0], ab[0], a[c], o);         // tᵀs: Dot2
            if (ND >= 2) dot2_acc_self(p[ND - 1], s[ND - 1], o);
            vzm = vc;
            vc = vzp;
        }
    }
    if (ND > 0) {
        const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        block_reduce_dd<NDA>(p, m, s, ab, part + (int64_t)bid * ND);
    }
}

// ------------------------------------------------------------------- Chebyshev sweeps
// Alg. 4 with the slab-block operator (zero ghosts at every block cut and Dirichlet face,
// mirror ghosts at Neumann faces):
//   sweep 1 (KernelCI1): out = g1*((2q) - (S(q)*cz))
//   sweep j (KernelCI2):     out = ρ_j*(((A2*x1) + (B2*(q - S(x1)))) - (ρ_{j-1}*x2))
//   with x2 = q*cz for j = 2 (z = b/θ is recomputed, not stored: same bits).
// `out` may alias `x2` (each point reads x2 only at its own index).
struct ChebConst {
    double cz, g1, A2, B2;
};

__global__ void __launch_bounds__(BX * BY) k_cheb_sweep(const double* __restrict__ q,
                                                        const double* __restrict__ x1,
                                                        const double* x2, double* out, Grid g,
                                                        ChebConst cc, double rho_j,
                                                        double rho_jm1, int first,
                                                        const DevState* __restrict__ st)
{
    if (st && st->done) return;
    const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y;
    const int k0 = blockIdx.z * ZC, k1 = min(g.L, k0 + ZC);
    if (i >= g.nx || j >= g.ny) return;
    const int64_t plane = (int64_t)g.nx * g.ny;
    const double* v = first ? q : x1;
    int64_t c = i + (int64_t)g.nx * j + plane * k0;
    for (int k = k0; k < k1; ++k, c += plane) {
        const double zm = (k == g.bc.zlo) ? v[c + plane]
                          : ((k % g.Lb) == 0) ? 0.0 : v[c - plane];
        const double zp = (k == g.bc.zhi) ? v[c - plane]
                          : ((k % g.Lb) == g.Lb - 1) ? 0.0 : v[c + plane];
        const double S = stencil_at(v, c, i, j, g.nx, g.ny, zm, zp, g.h2inv, g.bc.m);
        const double qc = q[c];
        double o;
        if (first) {
            o = cheb_first(qc, S, cc.g1, cc.cz);
        } else {
            const double zc = x2 ? x2[c] : qc * cc.cz;
            o = cheb_step(qc, S, v[c], zc, rho_j, rho_jm1, cc.A2, cc.B2);
        }
        out[c] = o;
    }
}

// G(CI) on an extended slab (k-deep halo planes present): one Chebyshev sweep over planes
// [kb, ke) of the GLOBAL operator; planes outside [v0, v1) are the physical boundary
// ghosts (zero).  Same per-point expressions as k_cheb_sweep.
__global__ void __launch_bounds__(BX * BY) k_cheb_sweep_rng(const double* __restrict__ q,
                                                            const double* __restrict__ x1,
                                                            const double* x2, double* out, int nx,
                                                            int ny, int kb, int ke, int v0, int v1,
                                                            double h2inv, MirrorBc bc, ChebConst cc,
                                                            double rho_j, double rho_jm1,
                                                            int first,
                                                            const DevState* __restrict__ st)
{
    if (st && st->done) return;
    const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y;
    const int k0 = kb + blockIdx.z * ZC, k1 = min(ke, k0 + ZC);
    if (i >= nx || j >= ny) return;
    const int64_t plane = (int64_t)nx * ny;
    const double* v = first ? q : x1;
    int64_t c = i + (int64_t)nx * j + plane * k0;
    for (int k = k0; k < k1; ++k, c += plane) {
        const double zm = (k == bc.zlo) ? v[c + plane] : (k - 1 < v0) ? 0.0 : v[c - plane];
        const double zp = (k == bc.zhi) ? v[c - plane] : (k + 1 >= v1) ? 0.0 : v[c + plane];
        const double S = stencil_at(v, c, i, j, nx, ny, zm, zp, h2inv, bc.m);
        const double qc = q[c];
        double o;
        if (first) {
            o = cheb_first(qc, S, cc.g1, cc.cz);
        } else {
            const double zc = x2 ? x2[c] : qc * cc.cz;
            o = cheb_step(qc, S, v[c], zc, rho_j, rho_jm1, cc.A2, cc.B2);
        }
        out[c] = o;
    }
}

// ------------------------------------------------------------------- element-wise ops
#define EW_LOOP(n) \
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < (n); \
         c += (int64_t)gridDim.x * blockDim.x)

__global__ void k_scale(const double* __restrict__ q, double* __restrict__ out, int64_t n,
                        double a, const DevState* __restrict__ st)
{
    if (st && st->done) return;
    EW_LOOP(n) out[c] = q[c] * a;
}

__global__ void k_copy(const double* __restrict__ q, double* __restrict__ out, int64_t n,
                       const DevState* __restrict__ st)
{
    if (st && st->done) return;
    EW_LOOP(n) out[c] = q[c];
}

// r0 = b - A x0 part 2: r = b - Ax (Ax precomputed in r)
__global__ void k_residual0(const double* __restrict__ b, double* __restrict__ r, int64_t n)
{
    EW_LOOP(n) r[c] = b[c] - r[c];
}

// stand-alone dots: ND = 1: {a0·b0}; ND = 2: {a0·b0, a1·b1} (setup: {b·b, r~·r0})
template <int ND>
__global__ void k_dot2(const double* __restrict__ a0, const double* __restrict__ b0,
                       const double* __restrict__ a1, const double* __restrict__ b1, int64_t n,
                       dd* __restrict__ part)
{
    double p[ND] = {}, m[ND] = {}, s[ND] = {}, ab[ND] = {};
    EW_LOOP(n)
    {
        dot3_acc(p[0], m[0], s[0], ab[0], a0[c], b0[c]);
        if (ND > 1) dot3_acc(p[ND - 1], m[ND - 1], s[ND - 1], ab[ND - 1], a1[c], b1[c]);
    }
    block_reduce_dd<ND>(p, m, s, ab, part + (int64_t)blockIdx.x * ND);
}

// a6, KernelBiCGS2: s = r - α w  (in place on r)
__global__ void k_axpy_s(double* __restrict__ r, const double* __restrict__ w, int64_t n,
                         const DevState* __restrict__ st)
{
    if (st->done) return;
    const double alpha = st->alpha;
    EW_LOOP(n) r[c] = upd_s(r[c], w[c], alpha);
}

// a11 + a12, KernelBiCGS4/5: x = (x + α p̂) + ω r̂; r = s - ω t;
// partials r~·r and r·r.
__global__ void k_update_xr(double* __restrict__ x, const double* __restrict__ ph,
                            const double* __restrict__ rh, double* __restrict__ r,
                            const double* __restrict__ t, const double* __restrict__ rt,
                            int64_t n, dd* __restrict__ part, const DevState* __restrict__ st)
{
    if (st->done) return;
    const double alpha = st->alpha, omega = st->omega;
    double p[2] = {0.0, 0.0}, m[2] = {0.0, 0.0}, s[2] = {0.0, 0.0}, ab[2] = {0.0, 0.0};
    EW_LOOP(n)
    {
        x[c] = upd_x(x[c], ph[c], rh[c], alpha, omega);
        const double rn = upd_r(r[c], t[c], omega);
        r[c] = rn;
        dot3_acc(p[0], m[0], s[0], ab[0], rt[c], rn);
        dot2_acc_self(p[1], s[1], rn);
    }
    block_reduce_dd<2>(p, m, s, ab, part + (int64_t)blockIdx.x * 2);
}

// a14, KernelBiCGS6: p = r + β (p - ω w)
__global__ void k_update_p(double* __restrict__ p, const double* __restrict__ r,
                           const double* __restrict__ w, int64_t n,
                           const DevState* __restrict__ st)
{
    if (st->done) return;
    const double beta = st->beta, omega = st->omega;
    EW_LOOP(n) p[c] = upd_p(r[c], p[c], w[c], beta, omega);
}

}  // namespace ref

// ------------------------------------------------------------------- reduction finalize
// One CTA combines `nparts` block partials (fixed order: contiguous chunks per thread,
// then the deterministic block tree) into this rank's (hi, lo, ab) triples.  nranks == 1:
// the stage is completed (certified, or parked for the exact path: finish_stage).
// nranks > 1 (or a 1-rank communicator: the caller passes 2): the quadruples go to
// `rank_out` for the all-gather; k_scalars finishes.
// depth = 2 x the longest per-thread product chain of the producer kernel; the bound D
// adds the block, finalize and rank trees (dd.cuh, DESIGN.md §4 "Reductions").
__host__ __device__ inline int reduce_depth(int depth, int nparts, int nranks)
{
    return depth + 2 * ((nparts + 1023) / 1024) + 48 + 2 * nranks;
}

template <int ND>
__global__ void __launch_bounds__(1024) k_finalize(const dd* __restrict__ part, int nparts,
                                                   int stage, DevState* st, double* hist,
                                                   double* scal, dd* rank_out, int nranks,
                                                   int depth, double nprod, int self_mask,
                                                   int k3_mask)
{
    pdl_enter();
    if (stage != STAGE_SETUP && stage != STAGE_DOT && st->done) return;
    __shared__ dd res[ND];
    // the stage's scalar step reads and writes a dozen DevState fields one after another
    // (one thread): stage a copy in shared memory now -- its loads overlap the partials'
    // -- and write it back once, instead of a chain of dependent global loads at the end
    __shared__ DevState sst;
    constexpr int NW8 = (int)(sizeof(DevState) / 8);
    static_assert(sizeof(DevState) % 8 == 0, "DevState copied as 8-byte words");
    if (threadIdx.x < 32)
        for (int i = threadIdx.x; i < NW8; i += 32)
            reinterpret_cast<uint64_t*>(&sst)[i] = reinterpret_cast<const uint64_t*>(st)[i];
    combine_partials<ND>(part, nparts, res);   // ends with __syncthreads
    if (threadIdx.x == 0) {
        if (nranks > 1) {
#pragma unroll
            for (int d = 0; d < ND; ++d) rank_out[d] = res[d];
        } else {
            dd comb[ND];
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                comb[d] = dd{0.0, 0.0, 0.0, 0.0};
                dd_add(comb[d].hi, comb[d].mid, comb[d].lo, comb[d].ab, res[d].hi, res[d].mid,
                       res[d].lo, res[d].ab);
            }
            finish_stage(&sst, stage, ND, comb, reduce_depth(depth, nparts, 1), nprod,
                         self_mask, k3_mask, hist, scal);
        }
    }
    if (nranks <= 1) {   // write the updated state back (the only writer while it runs)
        __syncthreads();
        if (threadIdx.x < 32)
            for (int i = threadIdx.x; i < NW8; i += 32)
                reinterpret_cast<uint64_t*>(st)[i] = reinterpret_cast<const uint64_t*>(&sst)[i];
    }
}

// nranks > 1: combine the gathered per-rank triples in ascending rank order (R19).
template <int ND>
__global__ void k_scalars(const dd* __restrict__ gathered, int nranks, int stage,
                          DevState* st, double* hist, double* scal, int depth, int nparts,
                          double nprod, int self_mask, int k3_mask)
{
    if (stage != STAGE_SETUP && stage != STAGE_DOT && st->done) return;
    dd comb[ND];
    for (int d = 0; d < ND; ++d) {
        comb[d] = dd{0.0, 0.0, 0.0, 0.0};
        for (int r = 0; r < nranks; ++r) {
            const dd g = gathered[r * ND + d];
            dd_add(comb[d].hi, comb[d].mid, comb[d].lo, comb[d].ab, g.hi, g.mid, g.lo, g.ab);
        }
    }
    finish_stage(st, stage, ND, comb, reduce_depth(depth, nparts, nranks), nprod, self_mask,
                 k3_mask, hist, scal);
}

