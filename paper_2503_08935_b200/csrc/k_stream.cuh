// k_stream.cuh -- HBM-streaming kernels of the fused path, written for memory-level
// parallelism: 16-byte (double2) loads, several independent loads in flight per thread
// (all operands of an unrolled group are loaded before any arithmetic), grid sized to a
// fixed multiple of the 148 SMs (deterministic partial-sum count).
//   k_stencil2_dot<ND>: a4 / a9 (KernelBiCGS1 / KernelBiCGS3)
//   k_update_xr2:       a11 + a12 (KernelBiCGS4 / KernelBiCGS5)
// Same per-point expression trees as every other variant (expr.cuh); Dot2 reductions.
#pragma once
#include "dd.cuh"
#include "expr.cuh"
#include "ref_shapes.cuh"
#include "state.cuh"

namespace stream {

// threads (x pairs) x rows, planes per thread: 32 planes keep the partial count per launch
// (one per CTA) at 8 K for 512^3 -- the finalize reads them all (measured 5.35 vs 5.41 ms)
#ifndef BCGS_SZC
#define BCGS_SZC 32
#endif
constexpr int SBX = 32, SBY = 8, SZC = BCGS_SZC;
#ifndef BCGS_ST_UNROLL
#define BCGS_ST_UNROLL 2
#endif
constexpr int kStUnroll = BCGS_ST_UNROLL;   // z-planes unrolled (loads in flight)

// w = A v (global operator; ghost planes hold halo data or zeros) and Dot2 partials of
// a·w (ND >= 1) and w·w (ND == 2).  Each thread owns 2 adjacent x points of one row and
// marches SZC planes; requires nx even (16-byte aligned rows).
// ND == 5 (2-sync, R31): a = s, rt = r~: partials tᵀs, tᵀt, r~ᵀs, r~ᵀt, sᵀs.
template <int ND, int SBX, int SBY, int SZC>
// occupancy targets (registers): ND = 0: 6 x 256 threads (<= 40), ND = 1, 2: 4 (<= 64),
// ND = 5: 2 (<= 128) -- no spills; the kernel is latency-bound (long scoreboard)
#ifndef BCGS_ST1_THREADS
#define BCGS_ST1_THREADS 1024   // ND = 1 (r~ᵀw, Dot3) resident threads per SM target
#endif
#ifndef BCGS_ST1_CHAINS
#define BCGS_ST1_CHAINS 2       // ND = 1: independent Dot3 chains (x / y point)
#endif
__global__ void __launch_bounds__(SBX * SBY, (ND == 5 ? 512 : ND == 2 ? 1024 : ND == 1 ? BCGS_ST1_THREADS : 1536) / (SBX * SBY))
k_stencil2_dot(const double* __restrict__ v,
                                                            const double* __restrict__ a,
                                                            const double* __restrict__ rt,
                                                            double* __restrict__ out, int nx,
                                                            int ny, int kb, int ke, double h2inv,
                                                            ref::MirrorBc bc,
                                                            dd* __restrict__ part,
                                                            const DevState* __restrict__ st)
{
    if (st && st->done) return;
    const int i = (blockIdx.x * SBX + threadIdx.x) * 2, j = blockIdx.y * SBY + threadIdx.y;
    const int k0 = kb + blockIdx.z * SZC, k1 = min(ke, k0 + SZC);
    constexpr int NDA = (ND > 0) ? ND : 1;
    double p[NDA] = {}, m[NDA] = {}, s[NDA] = {}, ab[NDA] = {};
    // second accumulators per dot for the odd x point -- two independent chains (ILP);
    // merged before the block reduction (the certified result is order-free, R19)
    double p2[2] = {}, m2[2] = {}, s2[2] = {};
    if (i < nx && j < ny) {
        const int64_t plane = (int64_t)nx * ny;
        int64_t c = i + (int64_t)nx * j + plane * k0;
        double2 zm = *reinterpret_cast<const double2*>(v + c - plane);
        double2 zc = *reinterpret_cast<const double2*>(v + c);
        const bool hxm = i > 0, hxp = i + 2 < nx, hym = j > 0, hyp = j < ny - 1;
#pragma unroll kStUnroll
        for (int k = k0; k < k1; ++k, c += plane) {
            const double2 zp = *reinterpret_cast<const double2*>(v + c + plane);
            // out-of-domain neighbours: 0, or the mirror on a Neumann face (R27)
            const double xm = hxm ? __ldg(v + c - 1) : ((bc.m & 1) ? zc.y : 0.0);
            const double xp = hxp ? __ldg(v + c + 2) : ((bc.m & 2) ? zc.x : 0.0);
            double2 ym = hym ? *reinterpret_cast<const double2*>(v + c - nx) : make_double2(0, 0);
            double2 yp = hyp ? *reinterpret_cast<const double2*>(v + c + nx) : make_double2(0, 0);
            if (!hym && (bc.m & 4)) ym = yp;
            if (!hyp && (bc.m & 8)) yp = ym;
            const double2 zmk = (k == bc.zlo) ? zp : zm, zpk = (k == bc.zhi) ? zm : zp;
            double2 av = make_double2(0, 0);
            if (ND >= 1) av = __ldg(reinterpret_cast<const double2*>(a + c));
            double2 o;
            o.x = stencil_row(zc.x, xm, zc.y, ym.x, yp.x, zmk.x, zpk.x, h2inv);
            o.y = stencil_row(zc.y, zc.x, xp, ym.y, yp.y, zmk.y, zpk.y, h2inv);
            *reinterpret_cast<double2*>(out + c) = o;
            if (ND >= 2) {          // tᵀs: Dot2, two chains
                dot2_acc(p[0], s[0], ab[0], av.x, o.x);
                dot2_acc(p2[0], s2[0], ab[0], av.y, o.y);
            } else if (ND == 1) {   // r~ᵀw: Dot3, one or two chains
                dot3_acc(p[0], m[0], s[0], ab[0], av.x, o.x);
                if (BCGS_ST1_CHAINS == 2) dot3_acc(p2[0], m2[0], s2[0], ab[0], av.y, o.y);
                else dot3_acc(p[0], m[0], s[0], ab[0], av.y, o.y);
            }
            if (ND == 2 || ND == 5) {
                dot2_acc_self(p[1], s[1], o.x);
                dot2_acc_self(p2[1], s2[1], o.y);
            }
            if (ND == 5) {   // one chain per extra dot: registers for occupancy (latency)
                const double2 rv = __ldg(reinterpret_cast<const double2*>(rt + c));
                dot3_acc(p[2], m[2], s[2], ab[2], rv.x, av.x);   // r~ᵀs, r~ᵀt: Dot3
                dot3_acc(p[2], m[2], s[2], ab[2], rv.y, av.y);
                dot3_acc(p[3], m[3], s[3], ab[3], rv.x, o.x);
                dot3_acc(p[3], m[3], s[3], ab[3], rv.y, o.y);
                dot2_acc_self(p[4], s[4], av.x);
                dot2_acc_self(p[4], s[4], av.y);
            }
            zm = zc;
            zc = zp;
        }
    }
    if (ND > 0) {
#pragma unroll
        for (int d = 0; d < (ND >= 2 ? 2 : ND); ++d)   // ab: one shared sum per dot
            dd_add(p[d], m[d], s[d], ab[d], p2[d], m2[d], s2[d], 0.0);
        const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        block_reduce_dd<NDA>(p, m, s, ab, part + (int64_t)bid * ND);
    }
}

inline dim3 stencil2_grid(int64_t nx, int64_t ny, int64_t nplanes)
{
    return dim3((unsigned)((nx / 2 + SBX - 1) / SBX), (unsigned)((ny + SBY - 1) / SBY),
                (unsigned)((nplanes + SZC - 1) / SZC));
}

// a11 + a12: x = fma(ω, r̂, fma(α, p̂, x)); r = fma(-ω, t, s); partials r~·r, r·r.
// n2 = number of double2 elements; UNR double2 groups per thread per iteration.
constexpr int XR_UNR = 2;
// ND = 2: partials r~ᵀr, rᵀr (a12); ND = 0 (2-sync, R31): no dots, r~ not read
template <int ND = 2>
__global__ void __launch_bounds__(256) k_update_xr2(double2* __restrict__ x,
                                                    const double2* __restrict__ ph,
                                                    const double2* __restrict__ rh,
                                                    const double2* __restrict__ s,
                                                    double2* __restrict__ r,
                                                    const double2* __restrict__ t,
                                                    const double2* __restrict__ rt, int64_t n2,
                                                    dd* __restrict__ part,
                                                    const DevState* __restrict__ st)
{
    pdl_enter();
    if (st->done) return;
    const double alpha = st->alpha, omega = st->omega;
    double p[2] = {0.0, 0.0}, m[2] = {0.0, 0.0}, q[2] = {0.0, 0.0}, ab[2] = {0.0, 0.0};
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; c + (XR_UNR - 1) * stride < n2; c += XR_UNR * stride) {
        double2 vx[XR_UNR], vph[XR_UNR], vrh[XR_UNR], vs[XR_UNR], vt[XR_UNR], vrt[XR_UNR];
#pragma unroll
        for (int u = 0; u < XR_UNR; ++u) {
            const int64_t e = c + u * stride;
            vx[u] = x[e];
            vph[u] = __ldg(ph + e);
            vrh[u] = __ldg(rh + e);
            vs[u] = __ldg(s + e);
            vt[u] = __ldg(t + e);
            if (ND) vrt[u] = __ldg(rt + e);
        }
#pragma unroll
        for (int u = 0; u < XR_UNR; ++u) {
            const int64_t e = c + u * stride;
            double2 xn, rn;
            xn.x = upd_x(vx[u].x, vph[u].x, vrh[u].x, alpha, omega);
            xn.y = upd_x(vx[u].y, vph[u].y, vrh[u].y, alpha, omega);
            rn.x = upd_r(vs[u].x, vt[u].x, omega);
            rn.y = upd_r(vs[u].y, vt[u].y, omega);
            x[e] = xn;
            r[e] = rn;
            if (ND) {
                dot3_acc(p[0], m[0], q[0], ab[0], vrt[u].x, rn.x);
                dot3_acc(p[0], m[0], q[0], ab[0], vrt[u].y, rn.y);
                dot2_acc_self(p[1], q[1], rn.x);
                dot2_acc_self(p[1], q[1], rn.y);
            }
        }
    }
    for (; c < n2; c += stride) {
        const double2 vx = x[c], vph = ph[c], vrh = rh[c], vs = s[c], vt = t[c];
        const double2 vrt = ND ? rt[c] : make_double2(0.0, 0.0);
        double2 xn, rn;
        xn.x = upd_x(vx.x, vph.x, vrh.x, alpha, omega);
        xn.y = upd_x(vx.y, vph.y, vrh.y, alpha, omega);
        rn.x = upd_r(vs.x, vt.x, omega);
        rn.y = upd_r(vs.y, vt.y, omega);
        x[c] = xn;
        r[c] = rn;
        if (ND) {
            dot3_acc(p[0], m[0], q[0], ab[0], vrt.x, rn.x);
            dot3_acc(p[0], m[0], q[0], ab[0], vrt.y, rn.y);
            dot2_acc_self(p[1], q[1], rn.x);
            dot2_acc_self(p[1], q[1], rn.y);
        }
    }
    if (ND) block_reduce_dd<2>(p, m, q, ab, part + (int64_t)blockIdx.x * 2);
}

// M = I (plain Bi-CGSTAB, P:145-174 / Alg. 3 with p̂ = p, r̂ = s): a6 s = fma(-α, w, r) into
// its own buffer, and a14 p = fma(β, fma(-ω, w, p), r) in place (element-wise), 16-byte I/O.
__global__ void __launch_bounds__(256) k_axpy_s2(double2* __restrict__ s,
                                                 const double2* __restrict__ r,
                                                 const double2* __restrict__ w, int64_t n2,
                                                 const DevState* __restrict__ st)
{
    if (st->done) return;
    const double alpha = st->alpha;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n2;
         c += (int64_t)gridDim.x * blockDim.x) {
        const double2 rv = __ldg(r + c), wv = __ldg(w + c);
        s[c] = make_double2(upd_s(rv.x, wv.x, alpha), upd_s(rv.y, wv.y, alpha));
    }
}

__global__ void __launch_bounds__(256) k_update_p2(double2* __restrict__ p,
                                                   const double2* __restrict__ r,
                                                   const double2* __restrict__ w, int64_t n2,
                                                   const DevState* __restrict__ st)
{
    if (st->done) return;
    const double beta = st->beta, omega = st->omega;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n2;
         c += (int64_t)gridDim.x * blockDim.x) {
        const double2 rv = __ldg(r + c), wv = __ldg(w + c), pv = p[c];
        p[c] = make_double2(upd_p(rv.x, pv.x, wv.x, beta, omega),
                            upd_p(rv.y, pv.y, wv.y, beta, omega));
    }
}

// a14 at the START of an iteration (the fused G(CI) multi-rank iteration): p is updated in
// place, except in iteration 1 (p0 = r0 already there) -- the element-wise twin of MODE_P
__global__ void __launch_bounds__(256) k_update_p_lead(double2* __restrict__ p,
                                                       const double2* __restrict__ r,
                                                       const double2* __restrict__ w, int64_t n2,
                                                       const DevState* __restrict__ st)
{
    if (st->done || st->iter == 0) return;
    const double beta = st->beta, omega = st->omega;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n2;
         c += (int64_t)gridDim.x * blockDim.x) {
        const double2 rv = __ldg(r + c), wv = __ldg(w + c), pv = p[c];
        p[c] = make_double2(upd_p(rv.x, pv.x, wv.x, beta, omega),
                            upd_p(rv.y, pv.y, wv.y, beta, omega));
    }
}

}  // namespace stream
