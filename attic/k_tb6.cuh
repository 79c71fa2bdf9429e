// k_tb6.cuh -- TMA-fed temporally blocked Chebyshev kernel with 2x2 register tiles.
//
// As k_cheb_tb4 (k_tb4.cuh) but every lane owns TWO adjacent columns (RX = 2) of RY rows, so
// a warp row covers a 64-column extended tile: the recomputed x-halo shrinks from 2HX/32 to
// 2HX/64 of the tile, the left/right neighbour of each point pair comes from registers for
// the inner side, and the shared-memory traffic per point and sweep drops from 32 to 24
// bytes (published rows and the segment-end rows move as 16-byte LDS/STS.128).
// Arithmetic per point is identical to every other variant (expr.cuh).
#pragma once

namespace fused {

template <int K, int RY, int NW, int NS>
struct Tb6Shape {
    static constexpr int HX = (K + 1) / 2 * 2;             // even x-halo (TMA alignment)
    static constexpr int EX = 64, EY = NW * RY, TX = EX - 2 * HX, TY = EY - 2 * K;
    static constexpr int PAD = EX;
    static constexpr int PLANE = EX * EY + 2 * PAD;
    static constexpr int BOX = EX * EY;
    static constexpr int QW = ((K + 1 + 2) / 3) * 3 < 3 ? 3 : ((K + 1 + 2) / 3) * 3;
    static constexpr size_t level_bytes = sizeof(double) * 2 * K * PLANE;
    static constexpr size_t stage_bytes = sizeof(double) * (size_t)NS * 3 * BOX;
    static constexpr size_t smem = level_bytes + stage_bytes + 128;
};

template <int K, int RY, int NW, int NS, int MODE>
struct Tb6Thread {
    using S = Tb6Shape<K, RY, NW, NS>;
    static constexpr int EX = S::EX, TX = S::TX, TY = S::TY, PLANE = S::PLANE, QW = S::QW,
                         BOX = S::BOX;
    static constexpr int NL = K > 1 ? K : 2;

    double qw[QW][RY][2];
    double win[NL][3][RY][2];
    const TbArgs* a;
    const TbMaps* maps;
    double* sm;
    double* stg;
    uint64_t* bar;
    int lane, ey0, b0, b1, c0, c1, t0, t1, wdy, tx0, ty0;
    int64_t col[RY], plane;          // offset of column 2*lane in row r
    unsigned actmask[RY][2];
    bool in_dom[RY][2], in_tile[RY][2], first;
    double alpha, beta, omega;
    const CUtensorMap* pmap;
    double* side;

    __device__ __forceinline__ void issue(int tt)
    {
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
        } else {
            mbar_expect_tx(&bar[s], 2 * BOX * 8);
            tma_load_3d(d + BOX, &maps->r, tx0, ty0, tt, &bar[s]);
            tma_load_3d(d + 2 * BOX, &maps->w, tx0, ty0, tt, &bar[s]);
        }
    }

    template <int PH, bool MASK>
    __device__ __forceinline__ void step(int t)
    {
        // ---- level 0 (both columns of each row) from the TMA stage of plane t
        double q0[RY][2];
        if (t < b1) {
            const int s = (t - t0) % NS;
            mbar_wait(&bar[s], ((t - t0) / NS) & 1);
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
                if (MASK) {
                    v.x = in_dom[r][0] ? v.x : 0.0;
                    v.y = in_dom[r][1] ? v.y : 0.0;
                }
                q0[r][0] = v.x;
                q0[r][1] = v.y;
                if (MODE != MODE_PLAIN && t >= c0 && t < c1) {
                    if (in_tile[r][0]) side[col[r] + plane * t] = v.x;
                    if (in_tile[r][1]) side[col[r] + 1 + plane * t] = v.y;
                }
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
        const double* prev = sm + S::PAD + ((t - 1) & 1) * (K * PLANE);
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            const int m = t - j;
            if (wdy <= K - j) {
                const double* pl = prev + (j - 1) * PLANE + ey0 * EX + 2 * lane;
                bool mok = true;
                if (MASK) mok = (unsigned)(m - b0) < (unsigned)(b1 - b0);
                double v[RY][2];
                // x_{j-1} at plane m for this thread's 2 x RY points (centre values)
                double zcv[RY][2];
#pragma unroll
                for (int r = 0; r < RY; ++r)
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc)
                        zcv[r][cc] = (j == 1) ? qw[(PH + QW - 1) % QW][r][cc]
                                              : win[j - 1 > 0 ? j - 1 : 1][(PH + 2) % 3][r][cc];
                // segment-end rows from shared memory (16-byte loads)
                const double2 ytop = *reinterpret_cast<const double2*>(pl - EX);
                const double2 ybot = *reinterpret_cast<const double2*>(pl + RY * EX);
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    const double xl = pl[r * EX - 1];       // left neighbour of column 0
                    const double xr = pl[r * EX + 2];       // right neighbour of column 1
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        double zm, zc, zp;
                        if (j == 1) {
                            zp = qw[PH % QW][r][cc];
                            zc = qw[(PH + QW - 1) % QW][r][cc];
                            zm = qw[(PH + QW - 2) % QW][r][cc];
                        } else {
                            zp = win[j - 1][PH % 3][r][cc];
                            zc = win[j - 1][(PH + 2) % 3][r][cc];
                            zm = win[j - 1][(PH + 1) % 3][r][cc];
                        }
                        const double xm = cc == 0 ? xl : zcv[r][0];
                        const double xp = cc == 0 ? zcv[r][1] : xr;
                        const double ym = r > 0 ? zcv[r > 0 ? r - 1 : 0][cc]
                                                : (cc == 0 ? ytop.x : ytop.y);
                        const double yp = r < RY - 1 ? zcv[r < RY - 1 ? r + 1 : 0][cc]
                                                     : (cc == 0 ? ybot.x : ybot.y);
                        const double Sv = stencil_row(zc, xm, xp, ym, yp, zm, zp, a->h2inv);
                        const double qc = qw[(PH + QW - j) % QW][r][cc];
                        double vv;
                        if (j == 1) {
                            vv = cheb_first(qc, Sv, a->g1, a->cz);
                        } else {
                            const double z2 = (j == 2) ? qc * a->cz
                                                       : win[j - 2 > 0 ? j - 2 : 1][(PH + 1) % 3][r][cc];
                            vv = cheb_step(qc, Sv, zc, z2, a->rho[j], a->rho[j - 1], a->A2, a->B2);
                        }
                        if (MASK) vv = (((actmask[r][cc] >> j) & 1u) && mok) ? vv : 0.0;
                        v[r][cc] = vv;
                    }
                }
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    if (j < K) {
                        win[j][PH % 3][r][0] = v[r][0];
                        win[j][PH % 3][r][1] = v[r][1];
                    } else if (m >= c0 && m < c1) {
                        if (in_tile[r][0]) a->out[col[r] + plane * m] = v[r][0];
                        if (in_tile[r][1]) a->out[col[r] + 1 + plane * m] = v[r][1];
                    }
                }
            }
        }
        double* cur = sm + S::PAD + (t & 1) * (K * PLANE) + ey0 * EX + 2 * lane;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            *reinterpret_cast<double2*>(cur + r * EX) = make_double2(q0[r][0], q0[r][1]);
#pragma unroll
            for (int j = 1; j < K; ++j)
                *reinterpret_cast<double2*>(cur + j * PLANE + r * EX) =
                    make_double2(win[j][PH % 3][r][0], win[j][PH % 3][r][1]);
        }
        __syncthreads();
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
    }
};

template <int K, int RY, int NW, int NS, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) k_cheb_tb6(const __grid_constant__ TbArgs a,
                                                       const __grid_constant__ TbMaps maps)
{
    static_assert(K <= 5, "tb6: K <= 5 (QW <= 6)");
    using T = Tb6Thread<K, RY, NW, NS, MODE>;
    using S = Tb6Shape<K, RY, NW, NS>;
    constexpr int TX = S::TX, TY = S::TY, U = S::QW, HX = S::HX;
    extern __shared__ __align__(128) double smraw[];

    const DevState* st = a.st;
    if (st && st->done) return;
    T th;
    th.a = &a;
    th.maps = &maps;
    th.stg = smraw;
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
    th.tx0 = blockIdx.x * TX - HX;
    th.ty0 = blockIdx.y * TY - K;
    int wdy = 1 << 20;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
        const int ey = th.ey0 + r;
        const int gy = th.ty0 + ey;
        const int dy = max(K - ey, ey - (K + TY - 1));
        wdy = min(wdy, dy);
        th.col[r] = (th.tx0 + 2 * lane) + (int64_t)a.nx * gy;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const int ex = 2 * lane + cc;
            const int gx = th.tx0 + ex;
            const int dx = max(HX - ex, ex - (HX + TX - 1));
            const int dist = max(dx, dy);
            const bool dom = gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny;
            th.in_dom[r][cc] = dom;
            th.in_tile[r][cc] = dom && dist <= 0;
            unsigned msk = 0;
#pragma unroll
            for (int j = 1; j <= K; ++j)
                if (dom && dist <= K - j) msk |= 1u << j;
            th.actmask[r][cc] = msk;
        }
    }
    th.wdy = wdy;
    const int blk = blockIdx.z / a.nchunk, ch = blockIdx.z % a.nchunk;
    th.b0 = blk * a.Lb;
    th.b1 = th.b0 + a.Lb;
    th.c0 = th.b0 + ch * a.zch;
    th.c1 = min(th.b1, th.c0 + a.zch);
    if (th.c0 >= th.b1) return;
    th.t0 = max(th.b0, th.c0 - K);
    th.t1 = th.c1 - 1 + K;
    th.plane = (int64_t)a.nx * a.ny;
#pragma unroll
    for (int d = 0; d < S::QW; ++d)
#pragma unroll
        for (int r = 0; r < RY; ++r) th.qw[d][r][0] = th.qw[d][r][1] = 0.0;
#pragma unroll
    for (int j = 0; j < T::NL; ++j)
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int r = 0; r < RY; ++r) th.win[j][d][r][0] = th.win[j][d][r][1] = 0.0;
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
        const int pro_end = max(th.t0, th.b0 + K);
        const int epi_beg = min(th.t1 + 1, th.b1);
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
