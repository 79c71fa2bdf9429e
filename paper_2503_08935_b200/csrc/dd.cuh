// dd.cuh -- the reductions of Alg. 3 (r~ᵀw P:281, tᵀs / tᵀt P:289-290, r~ᵀr / rᵀr
// P:296-297).  Contract R19: every dot product is the CORRECTLY ROUNDED value
// RN(Σ a_i b_i), which does not depend on the summation order, the block shape or the rank
// count (the paper notes that reduction order changes results, P:207 / P:417).
//
// Fast path (this file): compensated dot products in the style of Ogita, Rump & Oishi --
// TwoProd via fma, error-free TwoSum cascades -- plus a running Σ|fl(a_i b_i)| (`ab`) that
// bounds the remaining error.  Dot2 (one compensation level: hi + lo) is used for the
// well-conditioned dots (self dots aᵀa, tᵀs); Dot3 (two levels: hi + mid + lo) for the
// dots against the shadow residual r~ (r~ᵀw, r~ᵀr, r~ᵀs, r~ᵀt), whose condition number grows
// like 1/ρ as the iteration converges (10^8 at 512^3 after 30 iterations).  Partials are
// quadruples (hi, mid, lo, ab) combined with the Dot3 cascade.  A combined result is
// CERTIFIED when the rigorous error bound puts the exact value strictly inside the rounding
// interval of fl(hi + mid + lo); otherwise the stage is parked and the dot recomputed
// exactly (xdot.cuh).  The library is compiled with --fmad=false, so the plain operators
// below are single IEEE operations.
#pragma once

struct dd {
    double hi, mid, lo, ab;   // first / second compensation levels, rounded sum of the
                              // rest, and Σ|h_i| of the same products
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e)
{
    s = a + b;
    double z = s - a;
    e = (a - (s - z)) + (b - z);
}

// Dot2: a*b into (p, s, ab)
__device__ __forceinline__ void dot2_acc(double& p, double& s, double& ab, double a, double b)
{
    double h = a * b;
    double r = fma(a, b, -h);   // exact low part of the product (unless it underflows)
    double q;
    two_sum(p, h, p, q);
    s = s + (q + r);
    ab = ab + fabs(h);
}

// Dot2 of a self dot a*a into (p, s): no Σ|h| -- its terms are >= 0, so the bound uses
// |hi + mid + lo| instead (finish_stage)
__device__ __forceinline__ void dot2_acc_self(double& p, double& s, double a)
{
    double h = a * a;
    double r = fma(a, a, -h);
    double q;
    two_sum(p, h, p, q);
    s = s + (q + r);
}

// Dot3: a*b into (p, m, s, ab) -- the first-level errors (q, r) go through a second
// error-free TwoSum level m; only second-level errors are rounded into s
__device__ __forceinline__ void dot3_acc(double& p, double& m, double& s, double& ab, double a,
                                         double b)
{
    double h = a * b;
    double r = fma(a, b, -h);
    double q, e1, e2;
    two_sum(p, h, p, q);
    two_sum(m, q, m, e1);
    two_sum(m, r, m, e2);
    s = s + (e1 + e2);
    ab = ab + fabs(h);
}

// (P, M, S, AB) += (p, m, s, ab), Dot3 cascade (exact for P and M)
__device__ __forceinline__ void dd_add(double& P, double& M, double& S, double& AB, double p,
                                       double m, double s, double ab)
{
    double q, e1, e2;
    two_sum(P, p, P, q);
    two_sum(M, q, M, e1);
    two_sum(M, m, M, e2);
    S = S + ((e1 + e2) + s);
    AB = AB + ab;
}

// Deterministic block reduction of ND quadruples; result valid in thread 0.  Fixed shuffle
// pattern + fixed warp order -> bitwise run-to-run reproducible.
template <int ND>
__device__ __forceinline__ void block_reduce_dd(double (&p)[ND], double (&m)[ND],
                                                double (&s)[ND], double (&ab)[ND], dd* out)
{
    __shared__ dd sh[32][ND];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
    const int lane = tid & 31, warp = tid >> 5, nwarp = (nthr + 31) >> 5;
    // the ND trees are independent: level-outer / dot-inner loops let their dependency
    // chains interleave (same operands per dd_add as dot-outer: bitwise the same tree)
    auto warp_tree = [&]() {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            double op[ND], om[ND], os[ND], oa[ND];
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                op[d] = __shfl_down_sync(0xffffffffu, p[d], off);
                om[d] = __shfl_down_sync(0xffffffffu, m[d], off);
                os[d] = __shfl_down_sync(0xffffffffu, s[d], off);
                oa[d] = __shfl_down_sync(0xffffffffu, ab[d], off);
            }
            if (lane + off < 32) {
#pragma unroll
                for (int d = 0; d < ND; ++d) dd_add(p[d], m[d], s[d], ab[d], op[d], om[d], os[d], oa[d]);
            }
        }
    };
    warp_tree();
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < ND; ++d) sh[warp][d] = dd{p[d], m[d], s[d], ab[d]};
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            const dd v = lane < nwarp ? sh[lane][d] : dd{0.0, 0.0, 0.0, 0.0};
            p[d] = v.hi;
            m[d] = v.mid;
            s[d] = v.lo;
            ab[d] = v.ab;
        }
        warp_tree();
        if (lane == 0) {
#pragma unroll
            for (int d = 0; d < ND; ++d) out[d] = dd{p[d], m[d], s[d], ab[d]};
        }
    }
}

// This CTA's combination of `nparts` partial quadruples -> res[ND] (valid after the call in
// every thread).  Thread t combines partials t, t + T, t + 2T, ... (coalesced; 8 loads in
// flight), then the deterministic block tree.
template <int ND>
__device__ __forceinline__ void combine_partials(const dd* __restrict__ part, int nparts,
                                                 dd* res)
{
    double p[ND], m[ND], s[ND], ab[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) { p[d] = 0.0; m[d] = 0.0; s[d] = 0.0; ab[d] = 0.0; }
    const int T = blockDim.x;
    // U partials per thread in flight (a ragged last group is predicated, not a serial tail
    // of dependent loads; U x ND quadruples stay within the 64-register budget of a
    // 1024-thread CTA); the adds keep the order b, b + T, b + 2T, ...
    constexpr int U = ND >= 4 ? 1 : 4 / ND;
    for (int b = threadIdx.x; b < nparts; b += U * T) {
        dd v[U][ND];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int d = 0; d < ND; ++d)
                v[u][d] = b + u * T < nparts ? part[(int64_t)(b + u * T) * ND + d]
                                             : dd{0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (b + u * T < nparts) {
#pragma unroll
                for (int d = 0; d < ND; ++d)
                    dd_add(p[d], m[d], s[d], ab[d], v[u][d].hi, v[u][d].mid, v[u][d].lo,
                           v[u][d].ab);
            }
    }
    block_reduce_dd<ND>(p, m, s, ab, res);
    __syncthreads();
}

// Certification of a combined quadruple (DESIGN.md §3 R19).  Every product enters hi through
// error-free TwoSums; with D = the depth of the deepest summation chain (per-thread products
// + the block, finalize and rank trees, DESIGN.md §4 "Reductions"), u = 2^-53 and
// Hc = the computed Σ|fl(a_i b_i)|:
//   Dot2 chains (first-level errors rounded into lo):  |Σ a_i b_i - (hi + mid + lo)|
//                                                       <= 2 (D+1)^2 u^2 Hc + n 2^-1074
//   Dot3 chains (first-level errors exact in mid):                <= 2 (D+1)^3 u^3 Hc + n 2^-1074
// (Du < 0.01; the n 2^-1074 term covers low parts of products that underflow).  The three
// components are renormalised by three error-free VecSum passes (x2, x1, x0 <- TwoSum
// cascades from the bottom up; exact, so x0 + x1 + x2 = hi + mid + lo): when hi and
// mid + lo nearly cancel (dots with a condition number far beyond 1/u, e.g. r~ᵀs late in a
// 2-sync solve) a single pass would leave a remainder of many ulps of the leading term.
// With r = x0 and the offset o = x1 + x2: if the exact value lies strictly inside r's
// rounding interval, r is the correctly rounded dot.  The bound is doubled and widened by
// the rounding of o; the half gaps are shrunk by 2^-50.
__device__ __forceinline__ bool dd_certify(const dd& c, double AB, int D, double nprod, bool k3,
                                           double* out, double* r_out = nullptr,
                                           double* o_out = nullptr, double* E_out = nullptr)
{
    double x0 = c.hi, x1 = c.mid, x2 = c.lo;
#pragma unroll
    for (int pass = 0; pass < 3; ++pass) {
        double s1, e1, s0, e0;
        two_sum(x1, x2, s1, e1);
        two_sum(x0, s1, s0, e0);
        x0 = s0;
        x1 = e0;
        x2 = e1;
    }
    const double r = x0;
    *out = r;
    const double o = x1 + x2;
    const double d1 = (double)D + 1.0;
    const double bound = k3 ? 2.0 * (d1 * d1 * d1) * (0x1p-53 * 0x1p-53 * 0x1p-53) * AB
                            : 2.0 * (d1 * d1) * (0x1p-53 * 0x1p-53) * AB;
    const double E = 2.0 * (bound + nprod * 0x1p-1074) + 0x1p-52 * fabs(o);
    if (r_out) { *r_out = r; *o_out = o; *E_out = E; }
    if (!isfinite(r) || !isfinite(AB) || !isfinite(o) || D < 0 || d1 * 0x1p-53 > 0.01)
        return false;
    const double ar = fabs(r);
    const long long bits = __double_as_longlong(ar);
    const double up = __longlong_as_double(bits + 1) - ar;                   // gap above |r|
    const double dn = bits > 0 ? ar - __longlong_as_double(bits - 1) : 0.0;  // gap below
    const double ee = r < 0.0 ? -o : o;   // offset of hi + mid + lo from r, towards |r| up
    const double shrink = 1.0 - 0x1p-50;
    return (ee + E) < 0.5 * up * shrink && (E - ee) < 0.5 * dn * shrink;
}
