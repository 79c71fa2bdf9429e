// k_tb4.cuh -- TMA-fed warp-row temporally blocked Chebyshev kernel (sm_100a).
//
// Same wavefront / arithmetic as k_cheb_tb3 (k_fused.cuh), plus:
//  * level-0 operands (q, or r/p/w) of plane t+1..t+NS-1 are staged in shared memory by the
//    Tensor Memory Accelerator (cp.async.bulk.tensor.3d, one elected thread, mbarrier
//    completion) -> no exposed DRAM latency on the z-march; out-of-grid columns of the box
//    are zero-filled by TMA;
//  * steps are specialised at compile time: in the steady state of an interior tile no
//    zero-ghost masking is evaluated (masks are only needed next to the physical faces, the
//    block cuts and the first/last K planes of a block).
// Values outside a level's halo are never read by an active point (the halo shrinks by one
// per level), so unmasked lanes may hold arbitrary finite values there.
#pragma once
#include <cuda.h>

namespace fused {

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

struct TbMaps {
    CUtensorMap q, r, w, pa, pb;   // 3-D maps (nx, ny, L) of the slab fields, box (32, EY, 1)
};

template <int K, int RY, int NW, int NS>
struct Tb4Shape {
    // x-halo HX = K rounded up to even: TMA needs 16-byte aligned box starts, so the first
    // staged column (tile x0 - HX) must be even.  For odd K the outermost column is unused.
    static constexpr int HX = (K + 1) / 2 * 2;
    static constexpr int EX = 32, EY = NW * RY, TX = EX - 2 * HX, TY = EY - 2 * K;
    static constexpr int PAD = EX;
    static constexpr int PLANE = EX * EY + 2 * PAD;       // level plane incl. guard rows
    static constexpr int BOX = EX * EY;                   // staged input box (doubles)
    // z-ring of the level-0 planes (>= K + 1, multiple of 3 for the phase-unrolled windows);
    // at least 6 so that, with NS dividing QW / 2, the stage slot, its mbarrier parity and the
    // level-plane double-buffer parity of a step are compile-time functions of its phase
    static constexpr int QW = ((K + 1 + 2) / 3) * 3 < 6 ? 6 : ((K + 1 + 2) / 3) * 3;
    static constexpr bool CT = QW % (2 * NS) == 0;
    static constexpr size_t level_bytes = sizeof(double) * 2 * K * PLANE;
    static constexpr size_t stage_bytes = sizeof(double) * (size_t)NS * 3 * BOX;
    static constexpr size_t smem = level_bytes + stage_bytes + 128;
};

template <int K, int RY, int NW, int NS, int MODE, bool NEU = false, bool O2 = false>
struct Tb4Thread {
    using S = Tb4Shape<K, RY, NW, NS>;
    static constexpr int EXS = S::EX;
    static constexpr int EX = S::EX, TX = S::TX, TY = S::TY, PLANE = S::PLANE, QW = S::QW,
                         BOX = S::BOX;
    static constexpr bool CT = S::CT;

    double qw[QW][RY];                   // level 0 (q; MODE_C: x_{j0-1})
    double win[K > 1 ? K : 2][3][RY];
    double qr[MODE == MODE_C ? QW : 1][RY];   // MODE_C: q ring (centre values)
    double y2c[RY];                      // MODE_C: x_{j0-2} at plane t-1
    const TbArgs* a;
    const TbMaps* maps;
    double* sm;        // level planes
    double* stg;       // [NS][3][BOX] staged inputs
    uint64_t* bar;     // [NS]
    int lane, ey0, b0, b1, c0, c1, t0, t1, wdy, tx0, ty0;
    uint32_t col[RY], plane;   // 32-bit element offsets (launcher: slab < 2^32 elements)
    unsigned actmask[RY];
    int mir;           // Neumann mirror bits: 1 x-, 2 x+, 4<<2r y-, 8<<2r y+ (row r)
    bool in_dom[RY], in_tile[RY], first;
    double alpha, beta, omega;
    const CUtensorMap* pmap;
    double* side;

    static constexpr int ninputs() { return MODE == MODE_PLAIN ? 1 : (MODE == MODE_S ? 2 : 3); }

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
        } else if (MODE == MODE_C) {   // x_{j0-1}, q, x_{j0-2}
            mbar_expect_tx(&bar[s], 3 * BOX * 8);
            tma_load_3d(d, &maps->q, tx0, ty0, tt, &bar[s]);
            tma_load_3d(d + BOX, pmap, tx0, ty0, tt, &bar[s]);
            tma_load_3d(d + 2 * BOX, &maps->w, tx0, ty0, tt, &bar[s]);
        } else {
            mbar_expect_tx(&bar[s], 2 * BOX * 8);
            tma_load_3d(d + BOX, &maps->r, tx0, ty0, tt, &bar[s]);
            tma_load_3d(d + 2 * BOX, &maps->w, tx0, ty0, tt, &bar[s]);
        }
    }

    template <int PH, bool MASK>
    __device__ __forceinline__ void step(int t)
    {
        // ---- level 0 from the TMA stage of plane t
        double q0[RY], qn[RY], y2n[RY];
        // steps run in blocks of QW from t0, so (t - t0) % QW == PH: with CT the stage slot,
        // its mbarrier phase parity and the level-plane buffer are compile-time
        if (t < b1) {
            const int s = CT ? PH % NS : (t - t0) % NS;
            mbar_wait(&bar[s], CT ? (PH / NS) & 1 : ((t - t0) / NS) & 1);
            const double* d = stg + (size_t)s * 3 * BOX + ey0 * EX + lane;
#pragma unroll
            for (int r = 0; r < RY; ++r) {
                double v;
                if (MODE == MODE_PLAIN) {
                    v = d[r * EX];
                } else if (MODE == MODE_C) {
                    v = d[r * EX];
                    qn[r] = d[BOX + r * EX];
                    y2n[r] = d[2 * BOX + r * EX];
                    if (MASK) {
                        qn[r] = in_dom[r] ? qn[r] : 0.0;
                        y2n[r] = in_dom[r] ? y2n[r] : 0.0;
                    }
                } else if (MODE == MODE_P) {
                    const double pv = d[r * EX];
                    v = first ? pv : upd_p(d[BOX + r * EX], pv, d[2 * BOX + r * EX], beta, omega);
                } else {
                    v = upd_s(d[BOX + r * EX], d[2 * BOX + r * EX], alpha);
                }
                if (MASK) v = in_dom[r] ? v : 0.0;
                q0[r] = v;
                if ((MODE == MODE_P || MODE == MODE_S) && in_tile[r] && t >= c0 && t < c1)
                    side[(size_t)(col[r] + plane * (uint32_t)t)] = v;
            }
        } else {
#pragma unroll
            for (int r = 0; r < RY; ++r) q0[r] = qn[r] = y2n[r] = 0.0;
        }
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            qw[PH % QW][r] = q0[r];
            if (MODE == MODE_C) qr[PH % QW][r] = qn[r];
        }
        const double* prev = sm + S::PAD + (CT ? ((PH + 1) & 1) : ((t - t0 + 1) & 1)) * (K * PLANE);
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            const int m = t - j;
            if (wdy <= K - j) {                       // warp-uniform level skip
                const double* pl = prev + (j - 1) * PLANE + ey0 * EXS + lane;
                bool mok = true;
                if (MASK) mok = (unsigned)(m - b0) < (unsigned)(b1 - b0);
                double v[RY];
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    double zm, zc, zp, yc_m, yc_p;
                    if (j == 1) {
                        zp = qw[PH % QW][r];
                        zc = qw[(PH + QW - 1) % QW][r];
                        zm = qw[(PH + QW - 2) % QW][r];
                        yc_m = r > 0 ? qw[(PH + QW - 1) % QW][r > 0 ? r - 1 : 0] : pl[(r - 1) * EXS];
                        yc_p = r < RY - 1 ? qw[(PH + QW - 1) % QW][r < RY - 1 ? r + 1 : 0]
                                          : pl[(r + 1) * EXS];
                    } else {
                        zp = win[j - 1][PH % 3][r];
                        zc = win[j - 1][(PH + 2) % 3][r];
                        zm = win[j - 1][(PH + 1) % 3][r];
                        yc_m = r > 0 ? win[j - 1][(PH + 2) % 3][r > 0 ? r - 1 : 0] : pl[(r - 1) * EXS];
                        yc_p = r < RY - 1 ? win[j - 1][(PH + 2) % 3][r < RY - 1 ? r + 1 : 0]
                                          : pl[(r + 1) * EXS];
                    }
                    double xm = pl[r * EXS - 1];   // x-neighbours from the level plane
                    double xp = pl[r * EXS + 1];
                    // R27 mirror ghosts: only next to a physical face, which only masked
                    // steps reach (non-interior tiles; the prologue covers plane b0)
                    if (NEU && MASK) {
                        if (mir) {
                            if (mir & 1) xm = xp;
                            if (mir & 2) xp = xm;
                            if (mir & (4 << (2 * r))) yc_m = yc_p;
                            if (mir & (8 << (2 * r))) yc_p = yc_m;
                        }
                        if (m == a->bc.zlo) zm = zp;
                        if (m == a->bc.zhi) zp = zm;
                    }
                    const double Sv = stencil_row(zc, xm, xp, yc_m, yc_p, zm, zp, a->h2inv);
                    const double qc = MODE == MODE_C ? qr[(PH + QW - j) % QW][r]
                                                     : qw[(PH + QW - j) % QW][r];
                    double vv;
                    if (j == 1 && MODE == MODE_C) {        // sweep j0: x_{j0-2} at the centre
                        vv = cheb_step(qc, Sv, zc, y2c[r], a->rho[1], a->rho[0], a->A2, a->B2);
                    } else if (j == 1) {
                        vv = cheb_first(qc, Sv, a->g1, a->cz);
                    } else {
                        // x_{j-2} at the centre: x_0 = q/θ (first pass), level 0 (MODE_C)
                        const double z2 = (j == 2) ? (MODE == MODE_C ? qw[(PH + QW - 2) % QW][r]
                                                                     : qc * a->cz)
                                                   : win[j - 2][(PH + 1) % 3][r];
                        vv = cheb_step(qc, Sv, zc, z2, a->rho[j], a->rho[j - 1], a->A2, a->B2);
                    }
                    if (MASK) vv = (((actmask[r] >> j) & 1u) && mok) ? vv : 0.0;
                    v[r] = vv;
                }
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    if (j < K) win[j][PH % 3][r] = v[r];
                    else if (in_tile[r] && m >= c0 && m < c1) a->out[(size_t)(col[r] + plane * (uint32_t)m)] = v[r];
                    if (O2 && j == K - 1 && in_tile[r] && m >= c0 && m < c1)
                        a->out2[(size_t)(col[r] + plane * (uint32_t)m)] = v[r];
                }
            }
        }
        if (MODE == MODE_C) {
#pragma unroll
            for (int r = 0; r < RY; ++r) y2c[r] = y2n[r];
        }
        double* cur = sm + S::PAD + (CT ? (PH & 1) : ((t - t0) & 1)) * (K * PLANE) + ey0 * EXS +
                      lane;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            cur[r * EXS] = q0[r];
#pragma unroll
            for (int j = 1; j < K; ++j) cur[j * PLANE + r * EXS] = win[j][PH % 3][r];
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

    // remainder of < U steps starting at phase 0
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

// One (tile, slab block, output planes [c0, c1)) part of the launch: tile geometry and
// masks, the TMA prologue and the z-march.  `again`: a later part of the same CTA (segment
// mode) -- the stage barriers are re-armed at phase 0 (every plane issued by the previous
// part was consumed, and all threads passed its last step's barrier); the register rings
// and level planes keep the previous part's finite values, which only reach the warm-up
// cone of planes below c0, never an output (same as a chunk start inside a block) -- except
// the level-0 ring at a block start, whose planes below b0 are the zero ghosts (reset).
template <int K, int RY, int NW, int NS, int MODE, bool NEU, bool O2>
__device__ __forceinline__ void tb4_part(Tb4Thread<K, RY, NW, NS, MODE, NEU, O2>& th,
                                         const TbArgs& a, int bx, int by, int blk, int c0,
                                         int c1, bool again)
{
    using S = Tb4Shape<K, RY, NW, NS>;
    constexpr int TX = S::TX, TY = S::TY, U = S::QW, HX = S::HX;
    const int lane = th.lane;
    th.tx0 = bx * TX - HX;
    th.ty0 = by * TY - K;
    const int gx = th.tx0 + lane;
    const int dx = max(HX - lane, lane - (HX + TX - 1));
    int wdy = 1 << 20;
    th.mir = ((gx == 0 && (a.bc.m & 1)) ? 1 : 0) | ((gx == a.nx - 1 && (a.bc.m & 2)) ? 2 : 0);
#pragma unroll
    for (int r = 0; r < RY; ++r) {
        const int ey = th.ey0 + r;
        const int gy = th.ty0 + ey;
        const int dy = max(K - ey, ey - (K + TY - 1));
        wdy = min(wdy, dy);
        const int dist = max(dx, dy);
        th.in_dom[r] = gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny;
        th.in_tile[r] = th.in_dom[r] && dist <= 0;
        if (gy == 0 && (a.bc.m & 4)) th.mir |= 4 << (2 * r);
        if (gy == a.ny - 1 && (a.bc.m & 8)) th.mir |= 8 << (2 * r);
        th.col[r] = th.in_dom[r] ? (uint32_t)(gx + a.nx * gy) : 0u;
        unsigned msk = 0;
#pragma unroll
        for (int j = 1; j <= K; ++j)
            if (th.in_dom[r] && dist <= K - j) msk |= 1u << j;
        th.actmask[r] = msk;
    }
    th.wdy = wdy;
    th.b0 = a.ext ? a.zv0 : blk * a.Lb;
    th.b1 = a.ext ? a.zv1 : th.b0 + a.Lb;
    th.c0 = c0;
    th.c1 = c1;
    th.t0 = max(th.b0, th.c0 - K);
    th.t1 = th.c1 - 1 + K;
    if (again && th.t0 == th.b0) {
        // a part starting at its block's first plane: the level-0 ring stands for the zero
        // ghost planes below the block (R8 block cut) -- reset it as at kernel start (the
        // previous part's values would enter level 1 at plane b0 as its z- neighbour)
#pragma unroll
        for (int d = 0; d < S::QW; ++d)
#pragma unroll
            for (int r = 0; r < RY; ++r) {
                th.qw[d][r] = 0.0;
                if (MODE == MODE_C) th.qr[d][r] = 0.0;
            }
#pragma unroll
        for (int r = 0; r < RY; ++r) th.y2c[r] = 0.0;
    }
    if (again) {
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int s = 0; s < NS; ++s) mbar_init(&th.bar[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int tt = th.t0; tt < th.t0 + NS && tt < th.b1 && tt <= th.t1; ++tt) th.issue(tt);

    // interior tile: the extended tile lies inside the grid -> masks only near block ends
    const bool interior = th.tx0 >= 0 && th.tx0 + 32 <= a.nx && th.ty0 >= 0 &&
                          th.ty0 + S::EY <= a.ny;
    const int nsteps = th.t1 - th.t0 + 1;
    const int NB = nsteps / U, tail = nsteps - NB * U;
    int t = th.t0;
    if (interior) {
        // masked prologue while a level's plane is below the block (t - K < b0), masked
        // epilogue once planes beyond the block appear (t >= b1); unmasked in between.
        const int pro_end = max(th.t0, th.b0 + K + (NEU ? 1 : 0));   // first unmasked step
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

template <int K, int RY, int NW, int NS, int MODE, bool NEU = false, bool O2 = false,
          bool SEG = false>
__global__ void __launch_bounds__(NW * 32, 1) k_cheb_tb4(const __grid_constant__ TbArgs a,
                                                    const __grid_constant__ TbMaps maps)
{
    using T = Tb4Thread<K, RY, NW, NS, MODE, NEU, O2>;
    using S = Tb4Shape<K, RY, NW, NS>;
    extern __shared__ __align__(128) double smraw[];

    pdl_enter();
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
    } else if (MODE == MODE_C) {   // q: fixed input, or this iteration's p (parity buffer)
        const bool odd = st && (st->iter & 1);
        th.pmap = !a.qsel ? &maps.r : odd ? &maps.pa : &maps.pb;
    }
    th.lane = threadIdx.x & 31;
    th.ey0 = (threadIdx.x >> 5) * RY;
    th.plane = (uint32_t)(a.nx * a.ny);
    // output planes of a tile-block: the block, or the extended slab's output window
    const int zlo = a.ext ? a.zo0 : 0, Lo = a.ext ? a.zo1 - a.zo0 : a.Lb;
    int bx = blockIdx.x, by = blockIdx.y, blk = 0, c0 = 0, c1 = 0;
    int64_t u = 0, u1 = 0;
    if (!SEG) {          // grid mode: blockIdx = (tile x, tile y, block * nchunk + chunk)
        blk = blockIdx.z / a.nchunk;
        const int ch = blockIdx.z % a.nchunk;
        const int lo = a.ext ? zlo : blk * a.Lb;
        c0 = lo + ch * a.zch;
        c1 = min(lo + Lo, c0 + a.zch);
        if (c0 >= lo + Lo) return;
    } else {             // segment mode: CTA i owns [i T / nseg, (i+1) T / nseg) of the
                         // tile-major (tile x, tile y, block, plane) order, T = tiles x Lo
        const int64_t T = (int64_t)a.ntx * a.nty * (a.ext ? 1 : a.nblk) * Lo;
        u = T * blockIdx.x / a.nseg;
        u1 = T * (blockIdx.x + 1) / a.nseg;
        if (u >= u1) return;
    }
#pragma unroll
    for (int d = 0; d < S::QW; ++d)
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            th.qw[d][r] = 0.0;
            if (MODE == MODE_C) th.qr[d][r] = 0.0;
        }
#pragma unroll
    for (int r = 0; r < RY; ++r) th.y2c[r] = 0.0;
#pragma unroll
    for (int j = 0; j < (K > 1 ? K : 2); ++j)
#pragma unroll
        for (int r = 0; r < RY; ++r) th.win[j][0][r] = th.win[j][1][r] = th.win[j][2][r] = 0.0;
    for (int i = threadIdx.x; i < 2 * K * S::PLANE; i += blockDim.x) th.sm[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&th.bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (!SEG) {
        tb4_part(th, a, bx, by, blk, c0, c1, false);
        return;
    }
    for (bool again = false; u < u1; again = true) {
        const int64_t w = u / Lo;
        const int z0 = (int)(u - w * Lo);
        const int z1 = (u1 - u) < (int64_t)(Lo - z0) ? z0 + (int)(u1 - u) : Lo;
        bx = (int)(w % a.ntx);
        by = (int)((w / a.ntx) % a.nty);
        blk = (int)(w / ((int64_t)a.ntx * a.nty));
        const int lo = a.ext ? zlo : blk * a.Lb;
        tb4_part(th, a, bx, by, blk, lo + z0, lo + z1, again);
        u += z1 - z0;
    }
}

}  // namespace fused
