// k_fused.cuh -- fused, temporally blocked preconditioner kernel for sm_100a.
//
// k_cheb_tb applies all K Chebyshev sweeps of Alg. 2 / Alg. 4 to a
// slab block in ONE pass over HBM: a CTA owns a TX x TY column tile (plus a K-wide halo that
// it recomputes) and marches a z-wavefront through its z-chunk; level j (sweep j) trails
// level j-1 by one plane.  z-neighbours live in per-thread register windows, in-plane
// neighbours in a double-buffered shared-memory plane per level (one __syncthreads per
// z-step).  Zero ghosts at block cuts / physical faces (R8, Eq. 12-14) are exact zeros.
//
// The level-0 input is produced on the fly:
//   MODE_PLAIN: q = input field                                   (apply_preconditioner)
//   MODE_P:     q = p_i = r + β (p_{i-1} - ω w)   (KernelBiCGS6) -> also stored
//   MODE_S:     q = s   = r - α w                 (KernelBiCGS2) -> also stored
// so the vector update costs no extra pass.  Every point is evaluated with exactly the
// expression tree of the reference kernels (R17, R18, R20) -> bitwise identical results.
#pragma once
#include <stdint.h>

#include "state.cuh"

namespace fused {

constexpr int MODE_PLAIN = 0, MODE_P = 1, MODE_S = 2;
constexpr int KMAX_TB = 8;

struct TbArgs {
    const double* q;      // MODE_PLAIN input
    const double* r;      // MODE_P / MODE_S
    const double* w;
    const double* p_a;    // MODE_P: p buffers; input = parity ? p_b : p_a
    const double* p_b;
    double* side_a;       // MODE_P: output p_i = parity ? side_a : side_b (the other buffer)
    double* side_b;       // MODE_S: side_a = s
    double* out;          // level-K output: M^-1 q
    int nx, ny, Lb, zch, nchunk;
    double h2inv, cz, g1, A2, B2;
    double rho[KMAX_TB + 1];
    const DevState* st;
};

template <int K, int TX, int TY>
struct TbShape {
    static constexpr int EX = TX + 2 * K, EY = TY + 2 * K, NT = EX * EY;
    static constexpr size_t smem = sizeof(double) * 2 * K * NT;
};

template <int K, int TX, int TY, int MODE>
__global__ void __launch_bounds__(TbShape<K, TX, TY>::NT, 1) k_cheb_tb(TbArgs a)
{
    using S = TbShape<K, TX, TY>;
    constexpr int EX = S::EX, NT = S::NT;
    extern __shared__ double sm[];   // [2][K][NT]

    const DevState* st = a.st;
    if (st && st->done) return;
    double alpha = 0.0, beta = 0.0, omega = 0.0;
    bool first = false;
    const double* pin = nullptr;
    double* side = nullptr;
    if (MODE == MODE_P) {
        const int par = st->iter & 1;
        first = (st->iter == 0);
        beta = st->beta;
        omega = st->omega;
        pin = par ? a.p_b : a.p_a;
        side = par ? a.side_a : a.side_b;
    } else if (MODE == MODE_S) {
        alpha = st->alpha;
        side = a.side_a;
    }

    const int tid = threadIdx.x;
    const int ex = tid % EX, ey = tid / EX;
    const int gx = blockIdx.x * TX + ex - K, gy = blockIdx.y * TY + ey - K;
    const bool in_dom = gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny;
    // Chebyshev distance of this column outside the output tile (<= 0 inside)
    const int dist = max(max(K - ex, ex - (K + TX - 1)), max(K - ey, ey - (K + TY - 1)));
    const bool in_tile = in_dom && dist <= 0;

    const int blk = blockIdx.z / a.nchunk, ch = blockIdx.z % a.nchunk;
    const int b0 = blk * a.Lb, b1 = b0 + a.Lb;
    const int c0 = b0 + ch * a.zch, c1 = min(b1, c0 + a.zch);
    if (c0 >= b1) return;
    const int t0 = max(b0, c0 - K), t1 = c1 - 1 + K;

    const int64_t plane = (int64_t)a.nx * a.ny;
    const int64_t col = in_dom ? gx + (int64_t)a.nx * gy : 0;

    constexpr int QW = (K + 1 > 3) ? K + 1 : 3;   // q at planes t .. t-max(K,2)
    double qw[QW];
    double win[K][3];   // levels 1..K-1: planes (newest, newest-1, newest-2)
#pragma unroll
    for (int d = 0; d < QW; ++d) qw[d] = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) win[j][0] = win[j][1] = win[j][2] = 0.0;

    // prefetch of the level-0 operands of plane t (one step ahead)
    double nr = 0.0, np = 0.0, nw = 0.0;
    auto load = [&](int t) {
        if (in_dom && t < b1) {
            const int64_t c = col + plane * t;
            if (MODE == MODE_PLAIN) {
                nr = __ldg(a.q + c);
            } else if (MODE == MODE_P) {
                np = __ldg(pin + c);
                if (!first) {
                    nr = __ldg(a.r + c);
                    nw = __ldg(a.w + c);
                }
            } else {
                nr = __ldg(a.r + c);
                nw = __ldg(a.w + c);
            }
        }
    };
    load(t0);

    for (int t = t0; t <= t1; ++t) {
        // ---- level 0: q at plane t (zero outside the block / domain)
        double q0 = 0.0;
        if (in_dom && t < b1) {
            if (MODE == MODE_PLAIN) q0 = nr;
            else if (MODE == MODE_P) q0 = first ? np : nr + beta * (np - omega * nw);
            else q0 = nr - alpha * nw;
            if (MODE != MODE_PLAIN && in_tile && t >= c0 && t < c1) side[col + plane * t] = q0;
        }
        load(t + 1);
#pragma unroll
        for (int d = QW - 1; d > 0; --d) qw[d] = qw[d - 1];
        qw[0] = q0;

        const double* prev = sm + ((t - 1) & 1) * (K * NT);
        // ---- levels 1..K: level j computes plane m = t - j
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            const int m = t - j;
            double v = 0.0;
            if (in_dom && dist <= K - j && m >= b0 && m < b1) {
                const double* pl = prev + (j - 1) * NT;
                const double xm = pl[tid - 1], xp = pl[tid + 1];
                const double ym = pl[tid - EX], yp = pl[tid + EX];
                double zm, zc, zp;   // x_{j-1} at planes m-1, m, m+1
                if (j == 1) {
                    zp = qw[0]; zc = qw[1]; zm = qw[2];
                } else {
                    zp = win[j - 1][0]; zc = win[j - 1][1]; zm = win[j - 1][2];
                }
                const double Sv = (6.0 * zc - (((((xm + xp) + ym) + yp) + zm) + zp)) * a.h2inv;
                const double qc = qw[j];
                if (j == 1) {
                    v = a.g1 * ((2.0 * qc) - (Sv * a.cz));
                } else {
                    const double z2 = (j == 2) ? qc * a.cz : win[j - 2][2];
                    v = a.rho[j] * (((a.A2 * zc) + (a.B2 * (qc - Sv))) - (a.rho[j - 1] * z2));
                }
            }
            if (j < K) {
                win[j][2] = win[j][1];
                win[j][1] = win[j][0];
                win[j][0] = v;
            } else if (in_tile && m >= c0 && m < c1) {
                a.out[col + plane * m] = v;
            }
        }
        // ---- publish the newest plane of levels 0..K-1 for the next step
        double* cur = sm + (t & 1) * (K * NT);
        cur[tid] = qw[0];
#pragma unroll
        for (int j = 1; j < K; ++j) cur[j * NT + tid] = win[j][0];
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------- host side
inline int64_t max_blocks(int64_t, int64_t, int64_t) { return 0; }
inline bool supported(int64_t, int64_t, int64_t, int, int degree, bool has_pc)
{
    return has_pc && degree >= 1 && degree <= KMAX_TB;
}
bcgs_status iteration(bcgs_ctx c);
void on_begin(bcgs_ctx c);
bool precond_supported(bcgs_ctx c);
bcgs_status precond_apply(bcgs_ctx c, const double* q, double* out);

}  // namespace fused
