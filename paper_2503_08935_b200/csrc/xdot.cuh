// xdot.cuh -- exact dot products for the certification fallback of R19: the
// sum Σ a_i b_i is accumulated EXACTLY in a fixed-point superaccumulator and rounded once to
// nearest-even (the correctly rounded dot).  Runs only when a Dot2 result could not be
// certified (or when BCGS_OPT_EXACT_DOT forces it); integer additions are associative, so
// the result does not depend on the order, the grid or the rank count.
//
// Representation: a double x = m * 2^e with an integer m < 2^53 and e >= -1074; a product
// a*b = (ma*mb) * 2^(ea+eb) with a 106-bit integer ma*mb.  The superaccumulator X holds
// Σ a_i b_i = X * 2^XB (XB = -2176 <= the smallest product exponent -2148) as XL signed
// 64-bit limbs of 32-bit digit weight: X = Σ_k limb_k 2^(32 k).  Each product adds five
// 32-bit digits; a limb absorbs 2^31 of them before it could overflow (the driver keeps the
// per-dot product count below that).  Top bit: products < 2^2048, sums < 2^2080 -> bit 4256.
#pragma once
#include <stdint.h>

namespace xdot {

constexpr int XB = -2176;   // weight of bit 0 of limb 0
constexpr int XL = 136;     // 32-bit digits (4352 bits)

// x = m * 2^e (m < 2^53); x finite
__device__ __forceinline__ void decompose(double x, uint64_t& m, int& e, bool& neg)
{
    const uint64_t bits = (uint64_t)__double_as_longlong(x);
    neg = (bits >> 63) != 0;
    const int ex = (int)((bits >> 52) & 0x7FF);
    const uint64_t frac = bits & ((1ull << 52) - 1);
    if (ex == 0) {
        m = frac;
        e = -1074;
    } else {
        m = frac | (1ull << 52);
        e = ex - 1075;
    }
}

// acc[] += a*b (shared-memory limbs); returns false for a non-finite operand
__device__ __forceinline__ bool add_product(long long* acc, double a, double b)
{
    if (!isfinite(a) || !isfinite(b)) return false;
    uint64_t ma, mb;
    int ea, eb;
    bool na, nb;
    decompose(a, ma, ea, na);
    decompose(b, mb, eb, nb);
    if (ma == 0 || mb == 0) return true;
    const uint64_t lo = ma * mb, hi = __umul64hi(ma, mb);   // 106-bit product
    const int o = ea + eb - XB;                              // >= 28
    const int q = o >> 5, r = o & 31;
    // (hi:lo) << r as five 32-bit digits (r < 32: at most 137 bits)
    const uint64_t w0 = lo << r;
    const uint64_t w1 = (hi << r) | (r ? lo >> (64 - r) : 0);
    const uint64_t w2 = r ? hi >> (64 - r) : 0;
    const uint64_t dig[5] = {w0 & 0xFFFFFFFFull, w0 >> 32, w1 & 0xFFFFFFFFull, w1 >> 32,
                             w2 & 0xFFFFFFFFull};
    const bool neg = na != nb;
#pragma unroll
    for (int k = 0; k < 5; ++k)
        if (dig[k])
            atomicAdd(reinterpret_cast<unsigned long long*>(acc + q + k),
                      (unsigned long long)(neg ? -(long long)dig[k] : (long long)dig[k]));
    return true;
}

// Exact partial sum of a·b over this rank's n elements -> limbs[XL] (zeroed by the caller);
// *bad |= 1 for a non-finite operand (any rank's flag makes the dot NaN).  Grid-stride;
// one shared superaccumulator per block.
static __global__ void __launch_bounds__(256) k_exact_dot(const double* __restrict__ a,
                                                   const double* __restrict__ b, int64_t n,
                                                   long long* __restrict__ limbs,
                                                   long long* __restrict__ bad)
{
    __shared__ long long acc[XL];
    for (int i = threadIdx.x; i < XL; i += blockDim.x) acc[i] = 0;
    __syncthreads();
    bool ok = true;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x)
        ok &= add_product(acc, a[c], b[c]);
    if (!ok) atomicOr(reinterpret_cast<unsigned long long*>(bad), 1ull);
    __syncthreads();
    for (int i = threadIdx.x; i < XL; i += blockDim.x)
        if (acc[i]) atomicAdd(reinterpret_cast<unsigned long long*>(limbs + i),
                              (unsigned long long)acc[i]);
}

// Round Σ_r limbs[r * stride + k] 2^(32k) 2^XB (nranks superaccumulators) to the nearest
// double, ties to even.  One thread.  bad -> NaN.
__device__ inline double round_limbs(const long long* limbs, int nranks, int64_t stride, bool bad)
{
    if (bad) return __longlong_as_double(0x7FF8000000000000ll);
    long long d[XL];
    for (int k = 0; k < XL; ++k) {
        long long v = 0;
        for (int r = 0; r < nranks; ++r) v += limbs[r * stride + k];
        d[k] = v;
    }
    // carry-normalise: digits 0..XL-2 in [0, 2^32), the top limb keeps the sign
    for (int k = 0; k < XL - 1; ++k) {
        const long long cy = d[k] >> 32;   // arithmetic shift: floor division by 2^32
        d[k] -= cy * 4294967296ll;
        d[k + 1] += cy;
    }
    const bool neg = d[XL - 1] < 0;
    if (neg) {   // magnitude of a two's-complement number in base 2^32
        long long carry = 1;
        for (int k = 0; k < XL; ++k) {
            long long v = (k < XL - 1 ? (4294967295ll - d[k]) : (-d[k] - 1)) + carry;
            carry = (k < XL - 1 && v > 4294967295ll) ? 1 : 0;
            d[k] = (k < XL - 1) ? (v & 4294967295ll) : v;
        }
    }
    // most significant bit
    int top = XL - 1;
    while (top >= 0 && d[top] == 0) --top;
    if (top < 0) return 0.0;
    const int msb = top * 32 + (63 - __clzll((unsigned long long)d[top]));
    // lsb kept: 53 significant bits, but not below 2^-1074 (subnormals)
    int L = msb - 52;
    if (L < -1074 - XB) L = -1074 - XB;
    auto bit = [&](int pos) -> uint64_t {
        if (pos < 0) return 0;
        return ((uint64_t)d[pos >> 5] >> (pos & 31)) & 1u;
    };
    uint64_t sig = 0;
    for (int pos = msb; pos >= L; --pos) sig = (sig << 1) | bit(pos);
    const uint64_t rb = bit(L - 1);
    bool sticky = false;
    for (int pos = L - 2; pos >= 0 && !sticky; --pos) sticky = bit(pos) != 0;
    if (rb && (sticky || (sig & 1))) {
        ++sig;
        if (sig == (1ull << 53)) {
            sig >>= 1;
            ++L;
        }
    }
    const double v = ldexp((double)sig, L + XB);   // exact (or +inf on overflow)
    return neg ? -v : v;
}

}  // namespace xdot
