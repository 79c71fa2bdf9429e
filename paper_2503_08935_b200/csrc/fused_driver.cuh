// fused_driver.cuh -- host driver of the fused path.  One outer iteration:
//   K1  k_cheb_tb<MODE_P>: p_i = r + β(p - ω w) (a14 of the previous iteration) and
//       p̂ = M^-1 p_i (a2), one HBM pass (reads r, p, w; writes p_i, p̂)
//   a3  halo(p̂)                        a4  w = A p̂, r~ᵀw      a5  α
//   K2  k_cheb_tb<MODE_S>: s = r - α w (a6) and r̂ = M^-1 s (a7), one pass
//   a8  halo(r̂)                        a9  t = A r̂, tᵀs, tᵀt  a10 ω
//   a11+a12 x += α p̂ + ω r̂; r = s - ω t; r~ᵀr, rᵀr         a13 test, ρ, β
// p is double-buffered (halo columns of neighbouring tiles read the old p while the new
// one is written); the buffer is selected on the device from the iteration parity, so
// one captured graph serves every iteration.
#pragma once
#include "k_stream.cuh"

namespace fused {

// a11 + a12 with s in its own buffer: x = (x + α p̂) + ω r̂; r = s - ω t; partials r~·r, r·r
__global__ void k_update_xr_s(double* __restrict__ x, const double* __restrict__ ph,
                              const double* __restrict__ rh, const double* __restrict__ s,
                              double* __restrict__ r, const double* __restrict__ t,
                              const double* __restrict__ rt, int64_t n, dd* __restrict__ part,
                              const DevState* __restrict__ st)
{
    if (st->done) return;
    const double alpha = st->alpha, omega = st->omega;
    double p[2] = {0.0, 0.0}, m[2] = {0.0, 0.0}, q[2] = {0.0, 0.0}, ab[2] = {0.0, 0.0};
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
        x[c] = upd_x(x[c], ph[c], rh[c], alpha, omega);
        const double rn = upd_r(s[c], t[c], omega);
        r[c] = rn;
        dot3_acc(p[0], m[0], q[0], ab[0], rt[c], rn);
        dot2_acc_self(p[1], q[1], rn);
    }
    block_reduce_dd<2>(p, m, q, ab, part + (int64_t)blockIdx.x * 2);
}

// 2-sync (R31): apply the stop decided at the ω stage once x and r are updated
__global__ void k_commit(DevState* st)
{
    if (!st->done && st->pend) st->done = st->pend;
}

// output tile (TX, TY) of the kernel launch_variant picks for degree k (tb_launch.cuh)
void variant_tile(bcgs_ctx c, bool neu, int k, int* tx, int* ty)
{
    const int hx = (k + 1) / 2 * 2;                        // TMA: even x-halo
    const bool tma = c->tb_variant != 2 && c->lay.nx % 2 == 0;
    if (tma && neu && k <= 5) {
        *tx = 32 - 2 * hx; *ty = 32 - 2 * k;               // 16 warps x RY = 2
    } else if (tma && !neu && k <= 4) {
        *tx = 32 - 2 * hx; *ty = 48 - 2 * k;               // 24 warps x RY = 2
    } else {                                               // square tile
        *tx = 32; *ty = 16;
        if (k >= 7) { *tx = 16; *ty = 8; } else if (k >= 5) { *tx = 32; *ty = 8; }
    }
}

template <int MODE>
bcgs_status launch_tb(bcgs_ctx c, TbArgs& a)
{
    const int k = c->degree;
    a.nx = (int)c->lay.nx;
    a.ny = (int)c->lay.ny;
    a.Lb = (int)(c->lay.L / c->bpr);
    a.h2inv = c->h2inv;
    if (!a.ext) a.bc = c->mbc;
    a.cz = c->cst[3];
    a.g1 = c->cst[4];
    a.A2 = c->cst[5];
    a.B2 = c->cst[6];
    // multi-pass: above the one-pass range, and by default from k = 5 on (measured faster
    // than the one-pass square-tile kernel); variant 2 keeps the square tile
    if (!a.ext && multipass_ok(c) &&
        (k > KMAX_TB || (k > c->mp_min && c->tb_variant != 2)))
        return launch_multipass(c, a, MODE);
    for (int j = 0; j <= k; ++j) a.rho[j] = c->rho[j];
    // z-chunking: each chunk re-computes ~2k warm-up/drain planes; more chunks fill the 148
    // SMs (one CTA per SM) more evenly.  Pick the chunk count minimising
    // waves * (planes per chunk + 2k).
    int tx, ty;
    const bool neu = a.bc.m || a.bc.zlo >= 0 || a.bc.zhi >= 0;   // see launch_variant
    variant_tile(c, neu, k, &tx, &ty);
    if (a.ext) a.Lb = a.zo1 - a.zo0;   // chunks over the output planes, one "block"
    const int nblk = a.ext ? 1 : c->bpr;
    const int64_t tiles = ((a.nx + tx - 1) / tx) * (int64_t)((a.ny + ty - 1) / ty) * nblk;
    int64_t best_n = 1;
    double best = 1e300;
    for (int64_t nch = 1; nch <= std::max<int64_t>(1, a.Lb / 8); ++nch) {
        const int64_t zc = (a.Lb + nch - 1) / nch;
            const int64_t waves = (tiles * nch + kNumSMs - 1) / kNumSMs;
        const double cost = (double)waves * (double)(zc + 2 * k);
        if (cost < best * 0.999) {
            best = cost;
            best_n = nch;
        }
    }
    a.zch = (int)((a.Lb + best_n - 1) / best_n);
    a.nchunk = (a.Lb + a.zch - 1) / a.zch;
    const int nz = a.nchunk * nblk;
    // segment mode: one CTA per SM, each an equal share of the tile-major (tile, plane)
    // work (parts pay 2k warm-up / drain planes each).  Used only where it beats the chunk
    // grid by >= 10 %: tile counts that do not fill the SMs (256^3: 77 tiles -> ~150 vs
    // 180 plane-steps per SM).  On deep grids the chunk grid keeps neighbouring tiles at
    // the same plane, so their recomputed halo boxes are still in L2 (measured).
    a.nseg = 0;
    const bool tb4 = c->tb_variant != 2 && tb_tma_ok(c) && !neu && k <= 4 && !a.ext;
    if (tb4) {
        const int64_t per = (tiles * a.Lb + kNumSMs - 1) / kNumSMs;
        const double seg = (double)per + 2.0 * k * (double)((per + a.Lb - 1) / a.Lb + 1);
        if (c->tb_schedule == 2 || (c->tb_schedule == 0 && seg < 0.9 * best)) {
            a.nseg = kNumSMs;
            a.nblk = nblk;
        }
    }
    switch (k) {
    case 1: return launch_variant<1, MODE>(c, a, nz);
    case 2: return launch_variant<2, MODE>(c, a, nz);
    case 3: return launch_variant<3, MODE>(c, a, nz);
    case 4: return launch_variant<4, MODE>(c, a, nz);
    case 5: return launch_variant<5, MODE>(c, a, nz);
    case 6: return launch_variant<6, MODE>(c, a, nz);
    case 7: return launch_variant<7, MODE>(c, a, nz);
    case 8: return launch_variant<8, MODE>(c, a, nz);
    }
    return fail(c, BCGS_E_INVALID, "temporal blocking supports degree 1..%d", KMAX_TB);
}

// G(CI) on P > 1 ranks through the temporally blocked kernel: input = the extended slab
// (k-deep halos already exchanged), zero ghosts outside [v0, v1), outputs planes [KG, KG+L).
bcgs_status precond_g_tb(bcgs_ctx c, const double* E, double* out, int v0, int v1,
                         const DevState* st)
{
    TbArgs a{};
    const int64_t KG = BCGS_MAX_DEGREE;
    a.q = E;
    a.out = out - KG * c->lay.plane;
    a.st = st;
    a.ext = 1;
    a.zv0 = v0;
    a.zv1 = v1;
    a.zo0 = (int)KG;
    a.zo1 = (int)(KG + c->lay.L);
    a.bc = ext_mirror(c, v0, v1);
    return launch_tb<MODE_PLAIN>(c, a);
}

bool precond_supported(bcgs_ctx c)
{
    return supported(c, c->degree, c->pc != BCGS_PC_NONE);
}

bcgs_status precond_apply(bcgs_ctx c, const double* q, double* out, const DevState* st)
{
    TbArgs a{};
    a.q = q;
    a.out = out;
    a.st = st;   // nullptr for the API call; the pipelined iteration passes its state
    Prof pf(c, KC_FUSED_P1, 16.0 * npts(c));
    return launch_tb<MODE_PLAIN>(c, a);
}

// a3 + a4 (a8 + a9): halo exchange of v overlapped with the stencil+dot of the interior
// planes 1..L-2 (side stream + events), then the two boundary planes once the ghost planes
// have arrived.  Writes the Dot2 partials of all launches contiguously; *nparts = count.
template <int ND>
bcgs_status halo_stencil(bcgs_ctx c, double* v, const double* a, double* out, int kc,
                         int* nparts, const double* rt = nullptr)
{
    const int nx = (int)c->lay.nx, ny = (int)c->lay.ny, L = (int)c->lay.L;
    const dim3 sb(stream::SBX, stream::SBY);
    int nb = 0;
    // TMA-staged kernel (st_tma.cu) for the bulk of the planes; the L1 kernel for Neumann
    // faces, the 2-sync five-dot variant and the single boundary planes of nranks > 1
    const bool tma = (ND == 1 || ND == 2) && c->stencil_tma && stencil_tma_ok(c);
    auto launch_bulk = [&](int kb, int ke) -> bcgs_status {
        if (!tma) return BCGS_OK;
        int np = 0;
        TRY(launch_stencil_tma<(ND == 1 ? 1 : 2)>(c, v, a, out, kb, ke,
                                                  c->part + (int64_t)nb * ND, &np));
        nb += np;
        return BCGS_OK;
    };
    auto launch = [&](int kb, int ke) {
        const dim3 g = stream::stencil2_grid(nx, ny, ke - kb);
        dd* pp = c->part + (int64_t)nb * ND;
        stream::k_stencil2_dot<ND, stream::SBX, stream::SBY, stream::SZC><<<g, sb, 0, c->s>>>(
            v, a, rt, out, nx, ny, kb, ke, c->h2inv, c->mbc, pp, c->st);
        nb += (int)(g.x * g.y * g.z);
    };
    Prof pf(c, kc, 24.0 * npts(c));
    if (c->nranks == 1) {
        if (tma) TRY(launch_bulk(0, L));
        else launch(0, L);
    } else {
        CUDA_OK(c, cudaEventRecord(c->ev_pre, c->s));
        CUDA_OK(c, cudaStreamWaitEvent(c->s_comm, c->ev_pre, 0));
        TRY(halo_on(c, v, c->s_comm));
        CUDA_OK(c, cudaEventRecord(c->ev_halo, c->s_comm));
        if (L > 2) {                                       // interior, overlapped with the halo
            if (tma) TRY(launch_bulk(1, L - 1));
            else launch(1, L - 1);
        }
        CUDA_OK(c, cudaStreamWaitEvent(c->s, c->ev_halo, 0));
        launch(0, 1);                                       // boundary planes
        if (L > 1) launch(L - 1, L);
    }
    CUDA_OK(c, cudaGetLastError());
    *nparts = nb;
    return BCGS_OK;
}

// Unpreconditioned iteration (M = I: BiCGS, Table II row 1; config C1) on the streaming
// kernels: no copies for p̂ = p and r̂ = s.  168 B/pt: w = A p + r~ᵀw (24), s (24),
// t = A s + tᵀs, tᵀt (24), x / r + r~ᵀr, rᵀr (64), p (32).
// from >= 0: resume after the resolved stage `from` (R19 fallback, bcgs_api.cu resolve).
bcgs_status iteration_none(bcgs_ctx c, int from)
{
    const int64_t n = npts(c);
    DevState* st = c->st;
    int np1 = 0, np2 = 0;
    if (from == STAGE_RHO) goto a14;
    if (from == STAGE_OMEGA) goto a11;
    if (from == STAGE_ALPHA) goto a6;
    TRY(halo_stencil<1>(c, F(c, V_P), F(c, V_RT), F(c, V_W), KC_STENCIL1, &np1));
    TRY(reduce<1>(c, np1, STAGE_ALPHA, kStencilDepth, 1, {F(c, V_RT), F(c, V_W)}));
a6:
    {
        Prof pf(c, KC_AXPY, 24.0 * n);
        stream::k_axpy_s2<<<kEwBlocks, 256, 0, c->s>>>((double2*)F(c, V_S),
                                                       (const double2*)F(c, V_R),
                                                       (const double2*)F(c, V_W), n / 2, st);
    }
    TRY(halo_stencil<2>(c, F(c, V_S), F(c, V_S), F(c, V_T), KC_STENCIL2, &np2));
    TRY(reduce<2>(c, np2, STAGE_OMEGA, kStencilDepth, 0,
                  {F(c, V_T), F(c, V_S), F(c, V_T), F(c, V_T)}));
a11:
    {
        Prof pf(c, KC_FUSED_XR, 64.0 * n);
        stream::k_update_xr2<2><<<kEwBlocks, 256, 0, c->s>>>(
            (double2*)F(c, V_X), (const double2*)F(c, V_P), (const double2*)F(c, V_S),
            (const double2*)F(c, V_S), (double2*)F(c, V_R), (const double2*)F(c, V_T),
            (const double2*)F(c, V_RT), n / 2, c->part, st);
    }
    TRY(reduce<2>(c, kEwBlocks, STAGE_RHO, ew_depth(n), 1,
                  {F(c, V_RT), F(c, V_R), F(c, V_R), F(c, V_R)}));
a14:
    {
        Prof pf(c, KC_UPDATE_P, 32.0 * n);
        stream::k_update_p2<<<kEwBlocks, 256, 0, c->s>>>((double2*)F(c, V_P),
                                                         (const double2*)F(c, V_R),
                                                         (const double2*)F(c, V_W), n / 2, st);
    }
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

bcgs_status iteration(bcgs_ctx c, int from)
{
    const int64_t n = npts(c);
    DevState* st = c->st;
    double* ph = F(c, V_PH);
    ref::Grid g = ref_grid(c, (int)c->lay.L);
    dim3 sg = stencil_grid(c), sb(ref::BX, ref::BY);
    const int nsb = (int)(sg.x * sg.y * sg.z);
    const bool vec = (c->lay.nx % 2) == 0;   // 16-byte rows: vectorised streaming kernels
    int np1 = nsb, np2 = nsb;
    if (from == STAGE_RHO) return BCGS_OK;   // a14 is folded into the next iteration's K1
    if (from == STAGE_OMEGA2) goto a11_sync2;
    if (from == STAGE_OMEGA) goto a11;
    if (from == STAGE_ALPHA) goto k2;
    {   // K1: a14 (previous iteration) + a2
        TbArgs a{};
        a.r = F(c, V_R);
        a.w = F(c, V_W);
        a.p_a = F(c, V_P);
        a.p_b = F(c, V_P2);
        a.side_a = F(c, V_P);
        a.side_b = F(c, V_P2);
        a.out = ph;
        a.st = st;
        Prof pf(c, KC_FUSED_P1, 40.0 * n);
        TRY(launch_tb<MODE_P>(c, a));
    }
    if (vec) {
        TRY(halo_stencil<1>(c, ph, F(c, V_RT), F(c, V_W), KC_STENCIL1, &np1));
    } else {
        TRY(halo(c, ph));
        Prof pf(c, KC_STENCIL1, 24.0 * n);
        ref::k_stencil_dot<1><<<sg, sb, 0, c->s>>>(ph, F(c, V_RT), F(c, V_W), g, 0,
                                                  c->part, st);
    }
    TRY(reduce<1>(c, np1, STAGE_ALPHA, kStencilDepth, 1, {F(c, V_RT), F(c, V_W)}));
k2:
    {   // K2: a6 + a7
        TbArgs a{};
        a.r = F(c, V_R);
        a.w = F(c, V_W);
        a.side_a = F(c, V_S);
        a.out = F(c, V_RH);
        a.st = st;
        Prof pf(c, KC_FUSED_P2, 32.0 * n);
        TRY(launch_tb<MODE_S>(c, a));
    }
    if (vec && c->sync2) {   // R31: MPI4 + MPI5 in one reduction of five Dot2 pairs
        TRY(halo_stencil<5>(c, F(c, V_RH), F(c, V_S), F(c, V_T), KC_STENCIL2, &np2, F(c, V_RT)));
    } else if (vec) {
        TRY(halo_stencil<2>(c, F(c, V_RH), F(c, V_S), F(c, V_T), KC_STENCIL2, &np2));
    } else {
        TRY(halo(c, F(c, V_RH)));
        Prof pf(c, KC_STENCIL2, 24.0 * n);
        ref::k_stencil_dot<2><<<sg, sb, 0, c->s>>>(F(c, V_RH), F(c, V_S), F(c, V_T), g, 0,
                                                  c->part, st);
    }
    if (c->sync2) {   // ω, ρ_new, ||r||², test, β now; the stop applies after a11 + a12
        TRY(reduce<5>(c, np2, STAGE_OMEGA2, kStencilDepth, 12,
                      {F(c, V_T), F(c, V_S), F(c, V_T), F(c, V_T), F(c, V_RT), F(c, V_S),
                       F(c, V_RT), F(c, V_T), F(c, V_S), F(c, V_S)}));
    }
a11_sync2:
    if (c->sync2) {
        Prof pf(c, KC_FUSED_XR, 56.0 * n);
        stream::k_update_xr2<0><<<kEwBlocks, 256, 0, c->s>>>(
            (double2*)F(c, V_X), (const double2*)F(c, V_PH), (const double2*)F(c, V_RH),
            (const double2*)F(c, V_S), (double2*)F(c, V_R), (const double2*)F(c, V_T),
            nullptr, n / 2, nullptr, st);
        k_commit<<<1, 1, 0, c->s>>>(st);
        CUDA_OK(c, cudaGetLastError());
        return BCGS_OK;
    }
    TRY(reduce<2>(c, np2, STAGE_OMEGA, kStencilDepth, 0,
                  {F(c, V_T), F(c, V_S), F(c, V_T), F(c, V_T)}));
a11:
    {
        Prof pf(c, KC_FUSED_XR, 64.0 * n);
        if (vec)
            CUDA_OK(c, launch_k(c, stream::k_update_xr2<2>, dim3(kEwBlocks), dim3(256), 0,
                                (double2*)F(c, V_X), (const double2*)F(c, V_PH),
                                (const double2*)F(c, V_RH), (const double2*)F(c, V_S),
                                (double2*)F(c, V_R), (const double2*)F(c, V_T),
                                (const double2*)F(c, V_RT), (int64_t)(n / 2), c->part,
                                (const DevState*)st));
        else
            k_update_xr_s<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(
                F(c, V_X), F(c, V_PH), F(c, V_RH), F(c, V_S), F(c, V_R), F(c, V_T), F(c, V_RT),
                n, c->part, st);
    }
    TRY(reduce<2>(c, kEwBlocks, STAGE_RHO, ew_depth(n), 1,
                  {F(c, V_RT), F(c, V_R), F(c, V_R), F(c, V_R)}));
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

// The fused G(CI) iteration on nranks > 1 (bcgs_api.cu g_fused / g_precond).
bcgs_status iteration_g(bcgs_ctx c, int from)
{
    const int64_t n = npts(c);
    DevState* st = c->st;
    double* p = g_interior(c, 0);
    double* s = g_interior(c, 1);
    int np1 = 0, np2 = 0;
    if (from == STAGE_RHO) return BCGS_OK;
    if (from == STAGE_OMEGA) goto a11;
    if (from == STAGE_ALPHA) goto a6;
    {
        Prof pf(c, KC_UPDATE_P, 32.0 * n);
        stream::k_update_p_lead<<<kEwBlocks, 256, 0, c->s>>>((double2*)p, (const double2*)F(c, V_R),
                                                           (const double2*)F(c, V_W), n / 2, st);
    }
    TRY(g_precond(c, 0, F(c, V_PH)));
    TRY(halo_stencil<1>(c, F(c, V_PH), F(c, V_RT), F(c, V_W), KC_STENCIL1, &np1));
    TRY(reduce<1>(c, np1, STAGE_ALPHA, kStencilDepth, 1, {F(c, V_RT), F(c, V_W)}));
a6:
    {
        Prof pf(c, KC_AXPY, 24.0 * n);
        stream::k_axpy_s2<<<kEwBlocks, 256, 0, c->s>>>((double2*)s, (const double2*)F(c, V_R),
                                                       (const double2*)F(c, V_W), n / 2, st);
    }
    TRY(g_precond(c, 1, F(c, V_RH)));
    TRY(halo_stencil<2>(c, F(c, V_RH), s, F(c, V_T), KC_STENCIL2, &np2));
    TRY(reduce<2>(c, np2, STAGE_OMEGA, kStencilDepth, 0, {F(c, V_T), s, F(c, V_T), F(c, V_T)}));
a11:
    {
        Prof pf(c, KC_FUSED_XR, 64.0 * n);
        stream::k_update_xr2<2><<<kEwBlocks, 256, 0, c->s>>>(
            (double2*)F(c, V_X), (const double2*)F(c, V_PH), (const double2*)F(c, V_RH),
            (const double2*)s, (double2*)F(c, V_R), (const double2*)F(c, V_T),
            (const double2*)F(c, V_RT), n / 2, c->part, st);
    }
    CUDA_OK(c, cudaGetLastError());
    return reduce<2>(c, kEwBlocks, STAGE_RHO, ew_depth(n), 1,
                     {F(c, V_RT), F(c, V_R), F(c, V_R), F(c, V_R)});
}

}  // namespace fused

