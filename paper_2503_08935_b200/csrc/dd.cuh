// dd.cuh -- compensated (Dot2) reductions for the fused dot products of Alg. 3
// (r~ᵀw P:281, tᵀs / tᵀt P:289-290, r~ᵀr / rᵀr P:296-297).  Contract R19:
// TwoProd via fma, TwoSum accumulation, (hi, lo) pairs combined with TwoSum; result
// fl(hi + lo).  The whole library is compiled with --fmad=false, so the plain operators
// below are single IEEE operations.
#pragma once

struct dd {
    double hi, lo;
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e)
{
    s = a + b;
    double z = s - a;
    e = (a - (s - z)) + (b - z);
}

// accumulate a*b into the running pair (p, s)
__device__ __forceinline__ void dot2_acc(double& p, double& s, double a, double b)
{
    double h = a * b;
    double r = fma(a, b, -h);   // exact low part of the product
    double q;
    two_sum(p, h, p, q);
    s = s + (q + r);
}

// (P, S) += (p, s)
__device__ __forceinline__ void dd_add(double& P, double& S, double p, double s)
{
    double q;
    two_sum(P, p, P, q);
    S = S + (q + s);
}

// Deterministic block reduction of ND pairs; result valid in thread 0.  Fixed shuffle
// pattern + fixed warp order -> bitwise run-to-run reproducible.
template <int ND>
__device__ __forceinline__ void block_reduce_dd(double (&p)[ND], double (&s)[ND], dd* out)
{
    __shared__ double sh_p[32][ND], sh_s[32][ND];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
    const int lane = tid & 31, warp = tid >> 5, nwarp = (nthr + 31) >> 5;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            double op = __shfl_down_sync(0xffffffffu, p[d], off);
            double os = __shfl_down_sync(0xffffffffu, s[d], off);
            if (lane + off < 32) dd_add(p[d], s[d], op, os);
        }
        if (lane == 0) { sh_p[warp][d] = p[d]; sh_s[warp][d] = s[d]; }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            p[d] = lane < nwarp ? sh_p[lane][d] : 0.0;
            s[d] = lane < nwarp ? sh_s[lane][d] : 0.0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                double op = __shfl_down_sync(0xffffffffu, p[d], off);
                double os = __shfl_down_sync(0xffffffffu, s[d], off);
                if (lane + off < 32) dd_add(p[d], s[d], op, os);
            }
            if (lane == 0) { out[d].hi = p[d]; out[d].lo = s[d]; }
        }
    }
}
