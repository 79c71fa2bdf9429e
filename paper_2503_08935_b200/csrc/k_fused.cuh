// k_fused.cuh -- fused, temporally blocked preconditioner kernel for sm_100a.
//
// k_cheb_tb applies all K Chebyshev sweeps of Alg. 2 / Alg. 4 to a
// slab block in ONE pass over HBM: a CTA owns a TX x TY column tile (plus a K-wide halo that
// it recomputes) and marches a z-wavefront through its z-chunk; level j (sweep j) trails
// level j-1 by one plane.  z-neighbours live in per-thread register rings, in-plane
// neighbours in a double-buffered shared-memory plane per level (one __syncthreads per
// z-step).  Zero ghosts at block cuts / physical faces (R8, Eq. 12-14) are exact zeros.
//
// The level-0 input is produced on the fly:
//   MODE_PLAIN: q = input field                                   (apply_preconditioner)
//   MODE_P:     q = p_i = r + β (p_{i-1} - ω w)   (KernelBiCGS6) -> also stored
//   MODE_S:     q = s   = r - α w                 (KernelBiCGS2) -> also stored
// so the vector update costs no extra pass.  Degrees above KMAX_TB run as several passes of
// the TMA kernel (k_tb4.cuh): a pass applies sweeps j0..j0+KB-1 of the same recurrence,
//   MODE_C:     level 0 = x_{j0-1} (stencil operand), with q and x_{j0-2} read at the centre
// and writes the last two levels (out2 = level KB-1) for the next pass.  Every point is evaluated with exactly the
// expression tree of the reference kernels (R17, R18, R20) -> bitwise identical results.
#pragma once
#include <stdint.h>

#include "expr.cuh"
#include "ref_shapes.cuh"
#include "state.cuh"

namespace fused {

constexpr int MODE_PLAIN = 0, MODE_P = 1, MODE_S = 2, MODE_C = 3;
constexpr int KMAX_TB = 8;

struct TbArgs {
    const double* q;      // MODE_PLAIN input
    const double* r;      // MODE_P / MODE_S
    const double* w;
    const double* p_a;    // MODE_P: p buffers; input = parity ? p_b : p_a
    const double* p_b;
    double* side_a;       // MODE_P: output p_i = parity ? side_a : side_b (the other buffer)
    double* side_b;       // MODE_S: side_a = s
    double* out;          // level-K output: M^-1 q (multi-pass: x_{j0+KB-1})
    double* out2;         // multi-pass (O2): level KB-1 output x_{j0+KB-2}
    // MODE_C: q = input field (qsel = 0) or the p buffer the p-kernel of this iteration
    // wrote (qsel = 1: selected by the iteration parity like side_a/side_b)
    int qsel;
    int nx, ny, Lb, zch, nchunk;
    // segment mode (nseg > 0, k_cheb_tb4 only): a 1-D grid of nseg CTAs, each owning an
    // equal share of the tile-major (tile x, tile y, block, plane) work -- balances tile
    // counts that do not fill the SMs (256^3: 77 tiles on 148 SMs); 0 = the 3-D grid
    int nseg, ntx, nty, nblk;
    // extended-slab mode (G(CI), ext = 1): zero ghosts outside planes [zv0, zv1), outputs
    // for planes [zo0, zo1) only, one block; plane indices are extended-slab indices.
    int ext, zv0, zv1, zo0, zo1;
    // Neumann faces (R27): x/y bits and the planes whose z-/z+ neighbour is mirrored
    ref::MirrorBc bc;
    double h2inv, cz, g1, A2, B2;
    double rho[KMAX_TB + 1];   // multi-pass: rho[i] = ρ_{j0-1+i}, i = 0..KB
    const DevState* st;
};

template <int K, int TX, int TY>
struct TbShape {
    static constexpr int EX = TX + 2 * K, EY = TY + 2 * K, NT = EX * EY;
    static constexpr int PAD = EX + 1;        // guard: halo lanes may read tid±EX safely
    static constexpr int PLANE = NT + 2 * PAD;
    static constexpr size_t smem = sizeof(double) * 2 * K * PLANE;
};

// Per-thread wavefront state.  Register windows are rings indexed by the compile-time
// phase PH of the (fully unrolled) z-step, so no register moves are needed:
//   q ring (QW >= max(K+1, 3) planes, multiple of 3): q(t-d) at slot (PH-d) mod QW
//   win[j] (levels 1..K-1, 3 planes):                x_j(newest-d) at slot (PH-d) mod 3
template <int K, int TX, int TY, int MODE, bool NEU = false>
struct TbThread {
    using S = TbShape<K, TX, TY>;
    static constexpr int EX = S::EX, NT = S::NT, PLANE = S::PLANE;
    static constexpr int QW = ((K + 1 + 2) / 3) * 3 < 3 ? 3 : ((K + 1 + 2) / 3) * 3;
    static constexpr int U = QW;                 // unroll length: multiple of QW and of 3

    double qw[QW];
    double win[K > 1 ? K : 2][3];
    double nr, np, nw;                           // prefetched level-0 operands of plane t+1
    const TbArgs* a;
    double* sm;
    int tid, b0, b1, c0, c1;
    int64_t col, plane;
    unsigned actmask;                            // bit j: level j needed at this column
    int mir;                                     // Neumann mirror bits of this column
    bool in_dom, in_tile, first;
    double alpha, beta, omega;
    const double* pin;
    double* side;

    __device__ __forceinline__ void load(int t)
    {
        if (in_dom && t < b1) {
            const int64_t c = col + plane * t;
            if (MODE == MODE_PLAIN) {
                nr = __ldg(a->q + c);
            } else if (MODE == MODE_P) {
                np = __ldg(pin + c);
                if (!first) {
                    nr = __ldg(a->r + c);
                    nw = __ldg(a->w + c);
                }
            } else {
                nr = __ldg(a->r + c);
                nw = __ldg(a->w + c);
            }
        }
    }

    template <int PH>
    __device__ __forceinline__ void step(int t)
    {
        // ---- level 0: q at plane t (zero outside the block / domain)
        double q0 = 0.0;
        if (in_dom && t < b1) {
            if (MODE == MODE_PLAIN) q0 = nr;
            else if (MODE == MODE_P) q0 = first ? np : upd_p(nr, np, nw, beta, omega);
            else q0 = upd_s(nr, nw, alpha);
            if (MODE != MODE_PLAIN && in_tile && t >= c0 && t < c1) side[col + plane * t] = q0;
        }
        load(t + 1);
        qw[PH % QW] = q0;
        const double* prev = sm + S::PAD + ((t - 1) & 1) * (K * PLANE);
        // ---- levels 1..K: level j computes plane m = t - j (branch-free, masked)
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            const int m = t - j;
            const double* pl = prev + (j - 1) * PLANE;
            double xm = pl[tid - 1], xp = pl[tid + 1];
            double ym = pl[tid - EX], yp = pl[tid + EX];
            double zm, zc, zp;   // x_{j-1} at planes m-1, m, m+1
            if (j == 1) {
                zp = qw[PH % QW];
                zc = qw[(PH + QW - 1) % QW];
                zm = qw[(PH + QW - 2) % QW];
            } else {
                zp = win[j - 1][PH % 3];
                zc = win[j - 1][(PH + 2) % 3];
                zm = win[j - 1][(PH + 1) % 3];
            }
            if (NEU) {                                   // R27 mirror ghosts
                if (mir) {
                    if (mir & 1) xm = xp;
                    if (mir & 2) xp = xm;
                    if (mir & 4) ym = yp;
                    if (mir & 8) yp = ym;
                }
                if (m == a->bc.zlo) zm = zp;
                if (m == a->bc.zhi) zp = zm;
            }
            const double Sv = stencil_row(zc, xm, xp, ym, yp, zm, zp, a->h2inv);
            const double qc = qw[(PH + QW - j) % QW];
            double v;
            if (j == 1) {
                v = cheb_first(qc, Sv, a->g1, a->cz);
            } else {
                const double z2 = (j == 2) ? qc * a->cz : win[j - 2][(PH + 1) % 3];
                v = cheb_step(qc, Sv, zc, z2, a->rho[j], a->rho[j - 1], a->A2, a->B2);
            }
            const bool act = ((actmask >> j) & 1u) && (unsigned)(m - b0) < (unsigned)(b1 - b0);
            v = act ? v : 0.0;
            if (j < K) {
                win[j][PH % 3] = v;
            } else if (in_tile && m >= c0 && m < c1) {
                a->out[col + plane * m] = v;
            }
        }
        // ---- publish the newest plane of levels 0..K-1 for the next step
        double* cur = sm + S::PAD + (t & 1) * (K * PLANE);
        cur[tid] = q0;
#pragma unroll
        for (int j = 1; j < K; ++j) cur[j * PLANE + tid] = win[j][PH % 3];
        __syncthreads();
    }
};

template <int K, int TX, int TY, int MODE, bool NEU = false>
__global__ void __launch_bounds__(TbShape<K, TX, TY>::NT, 1) k_cheb_tb(TbArgs a)
{
    using T = TbThread<K, TX, TY, MODE, NEU>;
    constexpr int EX = T::EX, U = T::U;
    extern __shared__ double sm[];   // [2][K][PAD + NT + PAD]

    const DevState* st = a.st;
    if (st && st->done) return;
    T th;
    th.a = &a;
    th.sm = sm;
    th.nr = th.np = th.nw = 0.0;
    th.alpha = th.beta = th.omega = 0.0;
    th.first = false;
    th.pin = nullptr;
    th.side = nullptr;
    if (MODE == MODE_P) {
        const int par = st->iter & 1;
        th.first = (st->iter == 0);
        th.beta = st->beta;
        th.omega = st->omega;
        th.pin = par ? a.p_b : a.p_a;
        th.side = par ? a.side_a : a.side_b;
    } else if (MODE == MODE_S) {
        th.alpha = st->alpha;
        th.side = a.side_a;
    }
    const int tid = threadIdx.x;
    th.tid = tid;
    const int ex = tid % EX, ey = tid / EX;
    const int gx = blockIdx.x * TX + ex - K, gy = blockIdx.y * TY + ey - K;
    th.in_dom = gx >= 0 && gx < a.nx && gy >= 0 && gy < a.ny;
    // Chebyshev distance of this column outside the output tile (<= 0 inside)
    const int dist = max(max(K - ex, ex - (K + TX - 1)), max(K - ey, ey - (K + TY - 1)));
    th.in_tile = th.in_dom && dist <= 0;
    th.mir = ((gx == 0 && (a.bc.m & 1)) ? 1 : 0) | ((gx == a.nx - 1 && (a.bc.m & 2)) ? 2 : 0) |
             ((gy == 0 && (a.bc.m & 4)) ? 4 : 0) | ((gy == a.ny - 1 && (a.bc.m & 8)) ? 8 : 0);
    th.actmask = 0;
#pragma unroll
    for (int j = 1; j <= K; ++j)
        if (th.in_dom && dist <= K - j) th.actmask |= 1u << j;

    const int blk = blockIdx.z / a.nchunk, ch = blockIdx.z % a.nchunk;
    th.b0 = a.ext ? a.zv0 : blk * a.Lb;
    th.b1 = a.ext ? a.zv1 : th.b0 + a.Lb;
    th.c0 = (a.ext ? a.zo0 : th.b0) + ch * a.zch;
    th.c1 = min(a.ext ? a.zo1 : th.b1, th.c0 + a.zch);
    if (th.c0 >= (a.ext ? a.zo1 : th.b1)) return;
    const int t0 = max(th.b0, th.c0 - K), t1 = th.c1 - 1 + K;
    th.plane = (int64_t)a.nx * a.ny;
    th.col = th.in_dom ? gx + (int64_t)a.nx * gy : 0;
#pragma unroll
    for (int d = 0; d < T::QW; ++d) th.qw[d] = 0.0;
#pragma unroll
    for (int j = 0; j < (K > 1 ? K : 2); ++j) th.win[j][0] = th.win[j][1] = th.win[j][2] = 0.0;
    // zero both buffers (plane t0-1 and the guards) so every neighbour read is a finite 0
    for (int i = tid; i < 2 * K * T::PLANE; i += blockDim.x) sm[i] = 0.0;
    __syncthreads();

    th.load(t0);
    int t = t0;
    for (; t + U - 1 <= t1; t += U) {
        th.template step<0>(t);
        th.template step<1 % U>(t + 1);
        th.template step<2 % U>(t + 2);
        if (U > 3) {
            th.template step<3 % U>(t + 3);
            th.template step<4 % U>(t + 4);
            th.template step<5 % U>(t + 5);
        }
        if (U > 6) {
            th.template step<6 % U>(t + 6);
            th.template step<7 % U>(t + 7);
            th.template step<8 % U>(t + 8);
        }
    }
    // remainder (< U steps); phases continue from 0
    if (t <= t1) th.template step<0>(t);
    if (t + 1 <= t1) th.template step<1 % U>(t + 1);
    if (U > 3) {
        if (t + 2 <= t1) th.template step<2 % U>(t + 2);
        if (t + 3 <= t1) th.template step<3 % U>(t + 3);
        if (t + 4 <= t1) th.template step<4 % U>(t + 4);
    }
    if (U > 6) {
        if (t + 5 <= t1) th.template step<5 % U>(t + 5);
        if (t + 6 <= t1) th.template step<6 % U>(t + 6);
        if (t + 7 <= t1) th.template step<7 % U>(t + 7);
    }
}

}  // namespace fused
#include "k_tb4.cuh"
namespace fused {

// ----------------------------------------------------------------------------- host side
inline int64_t max_blocks(int64_t nx, int64_t ny, int64_t L)
{   // partial-sum slots of the stream::k_stencil2_dot grid (k_stream.cuh)
    // worst case over the stencil launch configurations (x pairs / 32, rows / 4, planes / 4)
    return ((nx / 2 + 31) / 32) * ((ny + 3) / 4) * ((L + 3) / 4 + 2);   // + 2 boundary launches
}
bool multipass_ok(bcgs_ctx c);   // tb_multi.cu
inline bool supported(bcgs_ctx c, int degree, bool has_pc)
{
    return has_pc && degree >= 1 && (degree <= KMAX_TB || multipass_ok(c));
}
bcgs_status iteration(bcgs_ctx c, int from);
bcgs_status iteration_none(bcgs_ctx c, int from);
bcgs_status iteration_g(bcgs_ctx c, int from);
bool precond_supported(bcgs_ctx c);
bcgs_status precond_apply(bcgs_ctx c, const double* q, double* out,
                          const DevState* st = nullptr);
bcgs_status precond_g_tb(bcgs_ctx c, const double* E, double* out, int v0, int v1,
                         const DevState* st);

}  // namespace fused
