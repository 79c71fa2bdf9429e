// tb_multi.cu -- multi-pass temporal blocking for Chebyshev degrees above the single-pass
// range (the paper's k = 24).
//
// Alg. 2 / Alg. 4 is a three-term recurrence: sweep j needs x_{j-1}
// (stencil operand), x_{j-2} and q (centre values only).  A pass of KB sweeps j0..j0+KB-1
// therefore needs three input fields and hands the last two iterates to the next pass:
//   pass 0 (MODE_P / MODE_S / MODE_PLAIN, O2): sweeps 1..KB, writes x_KB -> Y0, x_{KB-1} -> Y1
//   pass i (MODE_C): stencil operand x_{j0-1}, centre x_{j0-2} and q; writes x_{j0+KB-1} and
//                    x_{j0+KB-2} into the other buffer pair (neighbouring CTAs still read the
//                    old pair in their recomputed halos), the last pass writes the output.
// Every point is evaluated with the same expression trees (R17/R18) in the same sweep order
// as the one-sweep reference kernels, so the result is bitwise the same.  HBM traffic per
// application: 16 + 40 (passes - 1) + 8 B/pt instead of 16 + 32 (k - 1).
#include "tb_launch.cuh"

namespace fused {

// warps per CTA of a pass kernel (2 rows each): 20, except the 4-sweep continuation pass
// whose q / x_{j0-2} register rings need more than the 96 registers 640 threads allow
constexpr int mp_nw(int K, int mode) { return (mode == MODE_C && K >= 4) ? 16 : 20; }

template <int K, int MODE, bool O2>
static bcgs_status pass_k(bcgs_ctx c, TbArgs& a, int nz, bool neu)
{
    constexpr int NW = mp_nw(K, MODE);
    if (neu) return launch_tb4_k<K, 2, NW, 4, MODE, true, O2>(c, a, nz);
    return launch_tb4_k<K, 2, NW, 4, MODE, false, O2>(c, a, nz);
}

#ifndef TB_MULTI_CONT
// capability: TMA maps over the slab fields and >= 2 passes of >= 2 sweeps
bool multipass_ok(bcgs_ctx c)
{
    return c->degree >= 5 && c->degree <= BCGS_MAX_DEGREE && tma_ok(c);
}

// split k into ceil(k/4) passes of 2..4 sweeps, the larger ones first
static int pass_sizes(int k, int* sz)
{
    const int np = (k + 3) / 4;
    for (int i = 0; i < np; ++i) sz[i] = k / np + (i < k % np ? 1 : 0);
    return np;
}

// continuation passes: tb_multi_c.cu (a separate translation unit: parallel nvcc)
bcgs_status pass_cont(bcgs_ctx c, TbArgs& a, int K, int nz, bool o2, bool neu);

template <int K>
static bcgs_status pass_mode(bcgs_ctx c, TbArgs& a, int nz, int mode, bool o2, bool neu)
{
    switch (mode) {
    case MODE_PLAIN: return pass_k<K, MODE_PLAIN, true>(c, a, nz, neu);
    case MODE_P: return pass_k<K, MODE_P, true>(c, a, nz, neu);
    case MODE_S: return pass_k<K, MODE_S, true>(c, a, nz, neu);
    default: return pass_cont(c, a, K, nz, o2, neu);
    }
}

static bcgs_status pass(bcgs_ctx c, TbArgs& a, int K, int mode, bool o2, bool neu)
{
    // z-chunking as launch_tb: minimise waves x (planes per chunk + 2K) over the 148 SMs
    const int hx = (K + 1) / 2 * 2, tx = 32 - 2 * hx, ty = 2 * mp_nw(K, mode) - 2 * K;
    const int64_t tiles = ((a.nx + tx - 1) / tx) * (int64_t)((a.ny + ty - 1) / ty) * c->bpr;
    int64_t best_n = 1;
    double best = 1e300;
    for (int64_t nch = 1; nch <= std::max<int64_t>(1, a.Lb / 8); ++nch) {
        const int64_t zc = (a.Lb + nch - 1) / nch;
        const int64_t waves = (tiles * nch + kNumSMs - 1) / kNumSMs;
        const double cost = (double)waves * (double)(zc + 2 * K);
        if (cost < best * 0.999) {
            best = cost;
            best_n = nch;
        }
    }
    a.zch = (int)((a.Lb + best_n - 1) / best_n);
    a.nchunk = (a.Lb + a.zch - 1) / a.zch;
    const int nz = a.nchunk * c->bpr;
    if (mode != MODE_C && K >= 3) {   // first pass: 3 or 4 sweeps
        return K == 4 ? pass_mode<4>(c, a, nz, mode, true, neu)
                      : pass_mode<3>(c, a, nz, mode, true, neu);
    }
    if (mode == MODE_C && K >= 2 && K <= 4) return pass_cont(c, a, K, nz, o2, neu);
    return fail(c, BCGS_E_INVALID, "multi-pass: no kernel for a pass of %d sweeps", K);
}

// a: common fields (grid, constants, block length, mirror bits, device state) and the
// mode's inputs / outputs as for the single-pass kernel
bcgs_status launch_multipass(bcgs_ctx c, TbArgs& a, int mode)
{
    const int k = c->degree;
    int sz[BCGS_MAX_DEGREE];
    const int np = pass_sizes(k, sz);
    if (np < 2 || sz[0] < 3 || sz[np - 1] < 2)
        return fail(c, BCGS_E_INVALID, "multi-pass needs degree >= 5 (got %d)", k);
    const bool neu = a.bc.m || a.bc.zlo >= 0 || a.bc.zhi >= 0;
    double* Y[4] = {F(c, V_C1), F(c, V_C2), F(c, V_Y3), F(c, V_Y4)};
    TbArgs b = a;
    b.out = Y[0];
    b.out2 = Y[1];
    for (int i = 0; i <= sz[0]; ++i) b.rho[i] = c->rho[i];
    TRY(pass(c, b, sz[0], mode, true, neu));
    int j0 = 1 + sz[0], cur = 0;
    for (int p = 1; p < np; ++p) {
        const bool last = p == np - 1;
        const int nxt = 2 - cur;
        TbArgs d = a;
        d.q = Y[cur];            // x_{j0-1}
        d.w = Y[cur + 1];        // x_{j0-2}
        d.qsel = 0;
        if (mode == MODE_PLAIN) {
            d.r = a.q;
        } else if (mode == MODE_S) {
            d.r = a.side_a;      // s
        } else {                 // p_i: the buffer this iteration's p-kernel wrote
            d.qsel = 1;
            d.p_a = a.side_a;
            d.p_b = a.side_b;
        }
        d.out = last ? a.out : Y[nxt];
        d.out2 = last ? nullptr : Y[nxt + 1];
        for (int i = 0; i <= sz[p]; ++i) d.rho[i] = c->rho[j0 - 1 + i];
        TRY(pass(c, d, sz[p], MODE_C, !last, neu));
        j0 += sz[p];
        cur = nxt;
    }
    return BCGS_OK;
}

#else   // TB_MULTI_CONT: the continuation-pass kernels

bcgs_status pass_cont(bcgs_ctx c, TbArgs& a, int K, int nz, bool o2, bool neu)
{
    switch (K) {
    case 2: return o2 ? pass_k<2, MODE_C, true>(c, a, nz, neu) : pass_k<2, MODE_C, false>(c, a, nz, neu);
    case 3: return o2 ? pass_k<3, MODE_C, true>(c, a, nz, neu) : pass_k<3, MODE_C, false>(c, a, nz, neu);
    case 4: return o2 ? pass_k<4, MODE_C, true>(c, a, nz, neu) : pass_k<4, MODE_C, false>(c, a, nz, neu);
    }
    return fail(c, BCGS_E_INVALID, "multi-pass: no continuation kernel for %d sweeps", K);
}
#endif

}  // namespace fused
