// k_xp.cuh -- x-pair layout of the TMA-fed temporally blocked Chebyshev kernel (sm_100a).
//
// Same wavefront, staging and arithmetic as k_cheb_tb4 (k_tb4.cuh: level j of Alg. 2 /
// Alg. 4, P:216-233 / P:345-366, computes plane t - j at z-step t), with a different
// in-plane layout: each lane owns TWO adjacent x points (x = 2 lane, 2 lane + 1) of RY rows,
// so a warp row spans 64 columns and the recomputed x-halo (HX = 4 at k = 4) costs 8 of 64
// columns instead of 8 of 32.  The level planes in shared memory are stored split by x
// parity -- row = [E: the 32 even columns][O: the 32 odd columns] -- so the only in-plane
// neighbours a lane loads, x = 2 lane - 1 (O[lane - 1]) and x = 2 lane + 2 (E[lane + 1]), are
// contiguous across the warp (conflict-free 64-bit loads); the pair's mutual x-neighbours
// and, for RY = 2, the rows' mutual y-neighbours stay in registers.  Per point and sweep:
// RY = 2: 2 loads + 1 store (k_cheb_tb4: 3 + 1); RY = 1: 3 + 1 on 7.5 % fewer recomputed
// points.  Dirichlet faces only (R27 mirrors -> k_cheb_tb4), MODE_PLAIN / MODE_P / MODE_S.
// Lanes outside the domain (x >= nx: nx is even, so both points of a pair or none) hold
// masked zeros; values outside a level's halo are finite and never reach an output.
#pragma once
#include "k_tb4.cuh"

namespace fused {

template <int K, int RY, int NW, int NS>
struct XpShape {
    static constexpr int HX = (K + 1) / 2 * 2;            // even: 16-byte TMA box starts
    static constexpr int EX = 64, EY = NW * RY, TX = EX - 2 * HX, TY = EY - 2 * K;
    static constexpr int RS = 64;                          // level-plane row [E 32][O 32]
    static constexpr int PAD = RS;                         // one zero guard row each side
    static constexpr int PLANE = RS * EY + 2 * PAD;
    static constexpr int BOX = EX * EY;                    // staged input box (doubles)
    static constexpr int QW = ((K + 1 + 2) / 3) * 3 < 6 ? 6 : ((K + 1 + 2) / 3) * 3;
    static constexpr bool CT = QW % (2 * NS) == 0;
    static constexpr size_t level_bytes = sizeof(double) * 2 * K * PLANE;
    static constexpr size_t stage_bytes = sizeof(double) * (size_t)NS * 3 * BOX;
    static constexpr size_t smem = level_bytes + stage_bytes + 128;
};

template <int K, int RY, int NW, int NS, int MODE>
struct XpThread {
    using S = XpShape<K, RY, NW, NS>;
    static constexpr int EX = S::EX, RS = S::RS, PLANE = S::PLANE, QW = S::QW, BOX = S::BOX;
    static constexpr bool CT = S::CT;

    double qw[QW][RY][2];                       // level 0 ring
    double win[K > 1 ? K : 2][3][RY][2];        // levels 1..K-1, 3 planes
    const TbArgs* a;
    const TbMaps* maps;
    double* sm;        // level planes
    double* stg;       // [NS][3][BOX] staged inputs
    uint64_t* bar;     // [NS]
    int lane, ey0, b0, b1, c0, c1, t0, t1, wdy, tx0, ty0;
    uint32_t col[RY], plane;   // 32-bit element offsets (launcher: slab < 2^32 elements)
    unsigned actmask[RY][2];
    bool in_dom[RY], in_tile[RY], first;
    double alpha, beta, omega;
    const CUtensorMap* pmap;
    double* side;

    __device__ __forceinline__ void issue(int tt)
    {   // thread 0: stage the level-0 operands of plane tt
        const int s = (tt - t0) % NS;
        double* d = stg + (size_t)s * 3 * BOX;
        if (MODE == MODE_PLAIN) {
            mbar_expect_tx(&bar[s], BOX * 8);
            tma_load_3d(d, &maps->q, tx0, ty0, tt, &bar[s]);
        } else if (MODE == MODE_P) {
            if (first) {
                mbar_expect_tx(&bar[s], BOX * 8);
                tma_load_3d(d, pmap, tx0, ty0, tt, &bar[s]);
            } else {
                mbar_expect_tx(&bar[s], 3 * BOX * 8);
                tma_load_3d(d, pmap, tx0, ty0, tt, &bar[s]);
                tma_load_3d(d + BOX, &maps->r, tx0, ty0, tt, &bar[s]);
                tma_load_3d(d + 2 * BOX, &maps->w, tx0, ty0, tt, &bar[s]);
            }
        } else {   // MODE_S
            mbar_expect_tx(&bar[s], 2 * BOX * 8);
            tma_load_3d(d + BOX, &maps->r, tx0, ty0, tt, &bar[s]);
            tma_load_3d(d + 2 * BOX, &maps->w, tx0, ty0, tt, &bar[s]);
        }
    }

    template <int PH, bool MASK>
    __device__ __forceinline__ void step(int t)
    {
        double q0[RY][2];
        if (t < b1) {
            const int s = CT ? PH % NS : (t - t0) % NS;
            mbar_wait(&bar[s], CT ? (PH / NS) & 1 : ((t - t0) / NS) & 1);
            const double* d = stg + (size_t)s * 3 * BOX + ey0 * EX + 2 * lane;
#pragma unroll
            for (int r = 0; r < RY; ++r) {
                double2 v;
                if (MODE == MODE_PLAIN) {
                    v = *reinterpret_cast<const double2*>(d + r * EX);
                } else if (MODE == MODE_P) {
                    const double2 pv = *reinterpret_cast<const double2*>(d + r * EX);
                    if (first) {
                        v = pv;
                    } else {
                        const double2 rv = *reinterpret_cast<const double2*>(d + BOX + r * EX);
                        const double2 wv = *reinterpret_cast<const double2*>(d + 2 * BOX + r * EX);
                        v.x = upd_p(rv.x, pv.x, wv.x, beta, omega);
                        v.y = upd_p(rv.y, pv.y, wv.y, beta, omega);
                    }
                } else {
                    const double2 rv = *reinterpret_cast<const double2*>(d + BOX + r * EX);
                    const double2 wv = *reinterpret_cast<const double2*>(d + 2 * BOX + r * EX);
                    v.x = upd_s(rv.x, wv.x, alpha);
                    v.y = upd_s(rv.y, wv.y, alpha);
                }
                if (MASK && !in_dom[r]) v.x = v.y = 0.0;
                q0[r][0] = v.x;
                q0[r][1] = v.y;
                if (MODE != MODE_PLAIN && in_tile[r] && t >= c0 && t < c1)
                    *reinterpret_cast<double2*>(side + (size_t)(col[r] + plane * (uint32_t)t)) = v;
            }
        } else {
#pragma unroll
            for (int r = 0; r < RY; ++r) q0[r][0] = q0[r][1] = 0.0;
        }
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            qw[PH % QW][r][0] = q0[r][0];
            qw[PH % QW][r][1] = q0[r][1];
        }
        const double* prev = sm + S::PAD + (CT ? ((PH + 1) & 1) : ((t - t0 + 1) & 1)) * (K * PLANE);
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            const int m = t - j;
            if (wdy <= K - j) {                       // warp-uniform level skip
                const double* pl = prev + (j - 1) * PLANE + ey0 * RS + lane;
                bool mok = true;
                if (MASK) mok = (unsigned)(m - b0) < (unsigned)(b1 - b0);
                // z-window of level j - 1 at plane m: zp (m + 1), zc (m), zm (m - 1)
                double zp[RY][2], zc[RY][2], zm[RY][2];
#pragma unroll
                for (int r = 0; r < RY; ++r)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if (j == 1) {
                            zp[r][c] = qw[PH % QW][r][c];
                            zc[r][c] = qw[(PH + QW - 1) % QW][r][c];
                            zm[r][c] = qw[(PH + QW - 2) % QW][r][c];
                        } else {
                            zp[r][c] = win[j - 1][PH % 3][r][c];
                            zc[r][c] = win[j - 1][(PH + 2) % 3][r][c];
                            zm[r][c] = win[j - 1][(PH + 1) % 3][r][c];
                        }
                    }
                double v[RY][2];
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    const double xm0 = pl[r * RS + 31];      // O[lane - 1]: x = 2 lane - 1
                    const double xp1 = pl[r * RS + 1];       // E[lane + 1]: x = 2 lane + 2
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const double xm = c == 0 ? xm0 : zc[r][0];
                        const double xp = c == 0 ? zc[r][1] : xp1;
                        const double ym = r > 0 ? zc[r > 0 ? r - 1 : 0][c] : pl[(r - 1) * RS + 32 * c];
                        const double yp = r < RY - 1 ? zc[r < RY - 1 ? r + 1 : 0][c]
                                                     : pl[(r + 1) * RS + 32 * c];
                        const double Sv = stencil_row(zc[r][c], xm, xp, ym, yp, zm[r][c], zp[r][c],
                                                      a->h2inv);
                        const double qc = qw[(PH + QW - j) % QW][r][c];
                        double vv;
                        if (j == 1) {
                            vv = cheb_first(qc, Sv, a->g1, a->cz);
                        } else {
                            // x_{j-2} at the centre: x_0 = q/θ
                            const double z2 = (j == 2) ? qc * a->cz : win[j - 2][(PH + 1) % 3][r][c];
                            vv = cheb_step(qc, Sv, zc[r][c], z2, a->rho[j], a->rho[j - 1], a->A2,
                                           a->B2);
                        }
                        if (MASK) vv = (((actmask[r][c] >> j) & 1u) && mok) ? vv : 0.0;
                        v[r][c] = vv;
                    }
                }
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    if (j < K) {
                        win[j][PH % 3][r][0] = v[r][0];
                        win[j][PH % 3][r][1] = v[r][1];
                    } else if (in_tile[r] && m >= c0 && m < c1) {
                        *reinterpret_cast<double2*>(a->out + (size_t)(col[r] + plane * (uint32_t)m)) =
                            make_double2(v[r][0], v[r][1]);
                    }
                }
            }
        }
        double* cur = sm + S::PAD + (CT ? (PH & 1) : ((t - t0) & 1)) * (K * PLANE) + ey0 * RS + lane;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            cur[r * RS] = q0[r][0];
            cur[r * RS + 32] = q0[r][1];
#pragma unroll
            for (int j = 1; j < K; ++j) {
                cur[j * PLANE + r * RS] = win[j][PH % 3][r][0];
                cur[j * PLANE + r * RS + 32] = win[j][PH % 3][r][1];
            }
        }
        __syncthreads();
        // the stage of plane t is free again: refill it with plane t + NS
        if (threadIdx.x == 0 && t + NS < b1 && t + NS <= t1) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(t + NS);
        }
    }

    template <bool MASK>
    __device__ __forceinline__ void run_blocks(int tb, int nblk)
    {
        constexpr int U = QW;
        for (int b = 0; b < nblk; ++b, tb += U) {
            step<0, MASK>(tb);
            step<1 % U, MASK>(tb + 1);
            step<2 % U, MASK>(tb + 2);
            if (U > 3) {
                step<3 % U, MASK>(tb + 3);
                step<4 % U, MASK>(tb + 4);
                step<5 % U, MASK>(tb + 5);
            }
            if (U > 6) {
                step<6 % U, MASK>(tb + 6);
                step<7 % U, MASK>(tb + 7);
                step<8 % U, MASK>(tb + 8);
            }
        }
    }

    __device__ __forceinline__ void run_tail(int t, int n)
    {
        constexpr int U = QW;
        if (n > 0) step<0, true>(t);
        if (n > 1) step<1 % U, true>(t + 1);
        if (U > 3) {
            if (n > 2) step<2 % U, true>(t + 2);
            if (n > 3) step<3 % U, true>(t + 3);
            if (n > 4) step<4 % U, true>(t + 4);
        }
        if (U > 6) {
            if (n > 5) step<5 % U, true>(t + 5);
            if (n > 6) step<6 % U, true>(t + 6);
            if (n > 7) step<7 % U, true>(t + 7);
        }
    }
};

template <int K, int RY, int NW, int NS, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) k_cheb_xp(const __grid_constant__ TbArgs a,
                                                   const __grid_constant__ TbMaps maps)
{
    using T = XpThread<K, RY, NW, NS, MODE>;
    using S = XpShape<K, RY, NW, NS>;
    constexpr int TX = S::TX, TY = S::TY, U = S::QW, HX = S::HX;
    extern __shared__ __align__(128) double smraw[];

    const DevState* st = a.st;
    if (st && st->done) return;
    T th;
    th.a = &a;
    th.maps = &maps;
    th.stg = smraw;                                              // 128-B aligned TMA boxes
    th.sm = smraw + (size_t)NS * 3 * S::BOX;
    th.bar = reinterpret_cast<uint64_t*>(th.sm + 2 * K * S::PLANE);
    th.alpha = th.beta = th.omega = 0.0;
    th.first = false;
    th.pmap = nullptr;
    th.side = nullptr;
    if (MODE == MODE_P) {
        const int par = st->iter & 1;
        th.first = (st->iter == 0);
        th.beta = st->beta;
        th.omega = st->omega;
        th.pmap = par ? &maps.pb : &maps.pa;
        th.side = par ? a.side_a : a.side_b;
    } else if (MODE == MODE_S) {
        th.alpha = st->alpha;
        th.side = a.side_a;
    }
    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
    th.lane = lane;
    th.ey0 = wy * RY;
    th.tx0 = (int)blockIdx.x * TX - HX;
    th.ty0 = blockIdx.y * TY - K;
    const int gx = th.tx0 + 2 * lane;                 // even; the pair is (gx, gx + 1)
    int dx[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) dx[c] = max(HX - (2 * lane + c), (2 * lane + c) - (HX + TX - 1));
    int wdy = 1 << 20;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
        const int ey = th.ey0 + r;
        const int gy = th.ty0 + ey;
        const int dy = max(K - ey, ey - (K + TY - 1));
        wdy = min(wdy, dy);
        th.in_dom[r] = gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny;   // nx even: pair
        th.in_tile[r] = th.in_dom[r] && max(dx[0], dy) <= 0 && max(dx[1], dy) <= 0;
        th.col[r] = th.in_dom[r] ? (uint32_t)(gx + a.nx * gy) : 0u;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int dist = max(dx[c], dy);
            unsigned msk = 0;
#pragma unroll
            for (int j = 1; j <= K; ++j)
                if (th.in_dom[r] && dist <= K - j) msk |= 1u << j;
            th.actmask[r][c] = msk;
        }
    }
    th.wdy = wdy;
    const int blk = blockIdx.z / a.nchunk, ch = blockIdx.z % a.nchunk;
    th.b0 = a.ext ? a.zv0 : blk * a.Lb;
    th.b1 = a.ext ? a.zv1 : th.b0 + a.Lb;
    th.c0 = (a.ext ? a.zo0 : th.b0) + ch * a.zch;
    th.c1 = min(a.ext ? a.zo1 : th.b1, th.c0 + a.zch);
    if (th.c0 >= (a.ext ? a.zo1 : th.b1)) return;
    th.t0 = max(th.b0, th.c0 - K);
    th.t1 = th.c1 - 1 + K;
    th.plane = (uint32_t)(a.nx * a.ny);
#pragma unroll
    for (int d = 0; d < S::QW; ++d)
#pragma unroll
        for (int r = 0; r < RY; ++r) th.qw[d][r][0] = th.qw[d][r][1] = 0.0;
#pragma unroll
    for (int j = 0; j < (K > 1 ? K : 2); ++j)
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int r = 0; r < RY; ++r) th.win[j][p][r][0] = th.win[j][p][r][1] = 0.0;
    for (int i = threadIdx.x; i < 2 * K * S::PLANE; i += blockDim.x) th.sm[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&th.bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int tt = th.t0; tt < th.t0 + NS && tt < th.b1 && tt <= th.t1; ++tt) th.issue(tt);

    const bool interior = th.tx0 >= 0 && th.tx0 + S::EX <= a.nx && th.ty0 >= 0 &&
                          th.ty0 + S::EY <= a.ny;
    const int nsteps = th.t1 - th.t0 + 1;
    const int NB = nsteps / U, tail = nsteps - NB * U;
    int t = th.t0;
    if (interior) {
        const int pro_end = max(th.t0, th.b0 + K);          // first unmasked step
        const int epi_beg = min(th.t1 + 1, th.b1);          // first step that must be masked
        const int npro = min(NB, (pro_end - th.t0 + U - 1) / U);
        th.template run_blocks<true>(t, npro);
        t += npro * U;
        const int nmid = max(0, min(NB - npro, (epi_beg - t) / U));
        th.template run_blocks<false>(t, nmid);
        t += nmid * U;
        th.template run_blocks<true>(t, NB - npro - nmid);
        t += (NB - npro - nmid) * U;
    } else {
        th.template run_blocks<true>(t, NB);
        t += NB * U;
    }
    th.run_tail(t, tail);
}

}  // namespace fused
