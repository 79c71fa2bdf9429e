// k_tb5.cuh -- skewed-wavefront, TMA-fed temporally blocked Chebyshev kernel (sm_100a).
//
// As k_cheb_tb4, but level j computes plane t - 2j + 1 at z-step t (a lag of 2 planes per
// level instead of 1).  Then every level of a step depends only on values of earlier
// steps, so the K sweeps of a step are K independent dependency chains (x RY rows per
// thread) instead of one K-long chain -- the FP64 pipe is fed with ILP instead of stalling
// on the DADD/DMUL latency.  Levels are evaluated in descending order inside a step, which
// lets every level keep only a 4-plane register ring:
//   level j at plane m needs x_{j-1}(m-1..m+1) (ring of j-1, newest = m+1 from step t-1),
//   x_{j-2}(m) (ring of j-2: newest m+3, so 4 slots) and q(m) (q ring, >= 2K slots);
//   in-plane neighbours of x_{j-1}(m) were published at step t-2 -> 3 rotating smem planes.
// Arithmetic per point is identical to every other kernel variant (expr.cuh).
#pragma once

namespace fused {

template <int K, int RY, int NW, int NS>
struct Tb5Shape {
    static constexpr int HX = (K + 1) / 2 * 2;            // even x-halo (TMA alignment)
    static constexpr int EX = 32, EY = NW * RY, TX = EX - 2 * HX, TY = EY - 2 * K;
    static constexpr int PAD = EX;
    static constexpr int PLANE = EX * EY + 2 * PAD;
    static constexpr int BOX = EX * EY;
    // q ring >= max(2K, 3) slots and a multiple of 4 (the level-ring length) for K >= 2
    static constexpr int QW = K == 1 ? 3 : ((2 * K + 3) / 4) * 4;
    static constexpr int U = QW;                            // unrolled steps per block
    static constexpr int NB3 = 3;                           // rotating published planes
    static constexpr size_t level_bytes = sizeof(double) * NB3 * K * PLANE;
    static constexpr size_t stage_bytes = sizeof(double) * (size_t)NS * 3 * BOX;
    static constexpr size_t smem = level_bytes + stage_bytes + 128;
};

template <int K, int RY, int NW, int NS, int MODE>
struct Tb5Thread {
    using S = Tb5Shape<K, RY, NW, NS>;
    static constexpr int EX = S::EX, TX = S::TX, TY = S::TY, PLANE = S::PLANE, QW = S::QW,
                         BOX = S::BOX;
    static constexpr int NL = K > 1 ? K : 2;

    double qw[QW][RY];
    double win[NL][4][RY];        // levels 1..K-1, 4-plane rings
    const TbArgs* a;
    const TbMaps* maps;
    double* sm;
    double* stg;
    uint64_t* bar;
    int lane, ey0, b0, b1, c0, c1, t0, t1, wdy, tx0, ty0;
    int64_t col[RY], plane;
    unsigned actmask[RY];
    bool in_dom[RY], in_tile[RY], first;
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

    __device__ __forceinline__ double* planebuf(int t) const
    {
        const int b = ((t % 3) + 3) % 3;
        return sm + S::PAD + b * (K * PLANE);
    }

    // FULL: every level is active in every row of this warp (warp-uniform), so the level
    // loop has no branches and the K independent levels can be interleaved (ILP).
    template <int PH, bool MASK, bool FULL = false>
    __device__ __forceinline__ void step(int t)
    {
        // ---- level 0 from the TMA stage of plane t
        double q0[RY];
        if (t < b1) {
            const int s = (t - t0) % NS;
            mbar_wait(&bar[s], ((t - t0) / NS) & 1);
            const double* d = stg + (size_t)s * 3 * BOX + ey0 * EX + lane;
#pragma unroll
            for (int r = 0; r < RY; ++r) {
                double v;
                if (MODE == MODE_PLAIN) {
                    v = d[r * EX];
                } else if (MODE == MODE_P) {
                    const double pv = d[r * EX];
                    v = first ? pv : upd_p(d[BOX + r * EX], pv, d[2 * BOX + r * EX], beta, omega);
                } else {
                    v = upd_s(d[BOX + r * EX], d[2 * BOX + r * EX], alpha);
                }
                if (MASK) v = in_dom[r] ? v : 0.0;
                q0[r] = v;
                if (MODE != MODE_PLAIN && in_tile[r] && t >= c0 && t < c1)
                    side[col[r] + plane * t] = v;
            }
        } else {
#pragma unroll
            for (int r = 0; r < RY; ++r) q0[r] = 0.0;
        }
#pragma unroll
        for (int r = 0; r < RY; ++r) qw[PH % QW][r] = q0[r];
        const double* pub1 = planebuf(t - 1);   // level 0 (q) of plane t-1
        const double* pub2 = planebuf(t - 2);   // levels >= 1 computed at step t-2
        // ---- levels K..1 (descending): level j computes plane m = t - 2j + 1
        double vnew[NL][RY];
#pragma unroll
        for (int j = K; j >= 1; --j) {
            const int m = t - 2 * j + 1;
            if (FULL || wdy <= K - j) {
                const double* pl = (j == 1 ? pub1 : pub2 + (j - 1) * PLANE) + ey0 * EX + lane;
                bool mok = true;
                if (MASK) mok = (unsigned)(m - b0) < (unsigned)(b1 - b0);
                double v[RY];
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    double zm, zc, zp, yc_m, yc_p;
                    if (j == 1) {   // q(t-2), q(t-1), q(t)
                        zp = qw[PH % QW][r];
                        zc = qw[(PH + QW - 1) % QW][r];
                        zm = qw[(PH + QW - 2) % QW][r];
                        yc_m = r > 0 ? qw[(PH + QW - 1) % QW][r > 0 ? r - 1 : 0] : pl[(r - 1) * EX];
                        yc_p = r < RY - 1 ? qw[(PH + QW - 1) % QW][r < RY - 1 ? r + 1 : 0]
                                          : pl[(r + 1) * EX];
                    } else {        // ring of j-1 (not yet updated this step): newest = m+1
                        zp = win[j - 1][(PH + 3) % 4][r];
                        zc = win[j - 1][(PH + 2) % 4][r];
                        zm = win[j - 1][(PH + 1) % 4][r];
                        yc_m = r > 0 ? win[j - 1][(PH + 2) % 4][r > 0 ? r - 1 : 0] : pl[(r - 1) * EX];
                        yc_p = r < RY - 1 ? win[j - 1][(PH + 2) % 4][r < RY - 1 ? r + 1 : 0]
                                          : pl[(r + 1) * EX];
                    }
                    const double xm = pl[r * EX - 1], xp = pl[r * EX + 1];
                    const double Sv = stencil_row(zc, xm, xp, yc_m, yc_p, zm, zp, a->h2inv);
                    const double qc = qw[(PH + 2 * QW - 2 * j + 1) % QW][r];   // q(m)
                    double vv;
                    if (j == 1) {
                        vv = cheb_first(qc, Sv, a->g1, a->cz);
                    } else {
                        // x_{j-2}(m): q*cz for j = 2, else ring of j-2 (newest m+3) slot PH%4
                        const double z2 = (j == 2) ? qc * a->cz : win[j - 2 > 0 ? j - 2 : 1][PH % 4][r];
                        vv = cheb_step(qc, Sv, zc, z2, a->rho[j], a->rho[j - 1], a->A2, a->B2);
                    }
                    if (MASK) vv = (((actmask[r] >> j) & 1u) && mok) ? vv : 0.0;
                    v[r] = vv;
                }
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    if (j < K) win[j][PH % 4][r] = v[r];
                    else if (in_tile[r] && m >= c0 && m < c1) a->out[col[r] + plane * m] = v[r];
                    if (j < K) vnew[j][r] = v[r];
                }
            } else if (!FULL && j < K) {
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    win[j][PH % 4][r] = 0.0;
                    vnew[j][r] = 0.0;
                }
            }
        }
        double* cur = planebuf(t) + ey0 * EX + lane;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            cur[r * EX] = q0[r];
#pragma unroll
            for (int j = 1; j < K; ++j) cur[j * PLANE + r * EX] = vnew[j][r];
        }
        __syncthreads();
        if (threadIdx.x == 0 && t + NS < b1 && t + NS <= t1) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(t + NS);
        }
    }

    template <bool MASK, bool FULL>
    __device__ __forceinline__ void run_blocks_f(int tb, int nblk)
    {
        for (int b = 0; b < nblk; ++b, tb += QW) {
            step<0, MASK, FULL>(tb);
            step<1 % QW, MASK, FULL>(tb + 1);
            step<2 % QW, MASK, FULL>(tb + 2);
            if (QW > 3) {
                step<3 % QW, MASK, FULL>(tb + 3);
            }
            if (QW > 4) {
                step<4 % QW, MASK, FULL>(tb + 4);
                step<5 % QW, MASK, FULL>(tb + 5);
                step<6 % QW, MASK, FULL>(tb + 6);
                step<7 % QW, MASK, FULL>(tb + 7);
            }
            if (QW > 8) {
                step<8 % QW, MASK, FULL>(tb + 8);
                step<9 % QW, MASK, FULL>(tb + 9);
                step<10 % QW, MASK, FULL>(tb + 10);
                step<11 % QW, MASK, FULL>(tb + 11);
            }
        }
    }

    template <bool MASK>
    __device__ __forceinline__ void run_blocks(int tb, int nblk)
    {
        // warp-uniform dispatch; both paths execute one CTA barrier per step
        if (!MASK && wdy <= 0) run_blocks_f<MASK, true>(tb, nblk);
        else run_blocks_f<MASK, false>(tb, nblk);
    }

    __device__ __forceinline__ void run_tail(int t, int n)
    {
        if (n > 0) step<0, true>(t);
        if (n > 1) step<1 % QW, true>(t + 1);
        if (n > 2) step<2 % QW, true>(t + 2);
        if (QW > 4) {
            if (n > 3) step<3 % QW, true>(t + 3);
            if (n > 4) step<4 % QW, true>(t + 4);
            if (n > 5) step<5 % QW, true>(t + 5);
            if (n > 6) step<6 % QW, true>(t + 6);
        }
        if (QW > 8) {
            if (n > 7) step<7 % QW, true>(t + 7);
            if (n > 8) step<8 % QW, true>(t + 8);
            if (n > 9) step<9 % QW, true>(t + 9);
            if (n > 10) step<10 % QW, true>(t + 10);
        }
    }
};

template <int K, int RY, int NW, int NS, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) k_cheb_tb5(const __grid_constant__ TbArgs a,
                                                       const __grid_constant__ TbMaps maps)
{
    using T = Tb5Thread<K, RY, NW, NS, MODE>;
    using S = Tb5Shape<K, RY, NW, NS>;
    constexpr int TX = S::TX, TY = S::TY, U = S::U, HX = S::HX;
    extern __shared__ __align__(128) double smraw[];

    const DevState* st = a.st;
    if (st && st->done) return;
    T th;
    th.a = &a;
    th.maps = &maps;
    th.stg = smraw;
    th.sm = smraw + (size_t)NS * 3 * S::BOX;
    th.bar = reinterpret_cast<uint64_t*>(th.sm + S::NB3 * K * S::PLANE);
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
    const int gx = th.tx0 + lane;
    const int dx = max(HX - lane, lane - (HX + TX - 1));
    int wdy = 1 << 20;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
        const int ey = th.ey0 + r;
        const int gy = th.ty0 + ey;
        const int dy = max(K - ey, ey - (K + TY - 1));
        wdy = min(wdy, dy);
        const int dist = max(dx, dy);
        th.in_dom[r] = gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny;
        th.in_tile[r] = th.in_dom[r] && dist <= 0;
        th.col[r] = th.in_dom[r] ? gx + (int64_t)a.nx * gy : 0;
        unsigned msk = 0;
#pragma unroll
        for (int j = 1; j <= K; ++j)
            if (th.in_dom[r] && dist <= K - j) msk |= 1u << j;
        th.actmask[r] = msk;
    }
    th.wdy = wdy;
    const int blk = blockIdx.z / a.nchunk, ch = blockIdx.z % a.nchunk;
    th.b0 = blk * a.Lb;
    th.b1 = th.b0 + a.Lb;
    th.c0 = th.b0 + ch * a.zch;
    th.c1 = min(th.b1, th.c0 + a.zch);
    if (th.c0 >= th.b1) return;
    th.t0 = max(th.b0, th.c0 - K);
    th.t1 = th.c1 + 2 * K - 2;                   // level K reaches plane c1-1
    th.plane = (int64_t)a.nx * a.ny;
#pragma unroll
    for (int d = 0; d < S::QW; ++d)
#pragma unroll
        for (int r = 0; r < RY; ++r) th.qw[d][r] = 0.0;
#pragma unroll
    for (int j = 0; j < T::NL; ++j)
#pragma unroll
        for (int d = 0; d < 4; ++d)
#pragma unroll
            for (int r = 0; r < RY; ++r) th.win[j][d][r] = 0.0;
    for (int i = threadIdx.x; i < S::NB3 * K * S::PLANE; i += blockDim.x) th.sm[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&th.bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int tt = th.t0; tt < th.t0 + NS && tt < th.b1 && tt <= th.t1; ++tt) th.issue(tt);

    const bool interior = th.tx0 >= 0 && th.tx0 + 32 <= a.nx && th.ty0 >= 0 &&
                          th.ty0 + S::EY <= a.ny;
    const int nsteps = th.t1 - th.t0 + 1;
    const int NB = nsteps / U, tail = nsteps - NB * U;
    int t = th.t0;
    if (interior) {
        // unmasked while every level's plane t-2j+1 lies inside [b0, b1)
        const int pro_end = max(th.t0, th.b0 + 2 * K - 1);
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
