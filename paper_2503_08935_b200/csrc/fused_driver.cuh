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

namespace fused {

template <int K> struct Tile;
template <> struct Tile<1> { static constexpr int X = 32, Y = 16; };
template <> struct Tile<2> { static constexpr int X = 32, Y = 16; };
template <> struct Tile<3> { static constexpr int X = 32, Y = 16; };
template <> struct Tile<4> { static constexpr int X = 32, Y = 16; };
template <> struct Tile<5> { static constexpr int X = 32, Y = 8; };
template <> struct Tile<6> { static constexpr int X = 32, Y = 8; };
template <> struct Tile<7> { static constexpr int X = 16, Y = 8; };
template <> struct Tile<8> { static constexpr int X = 16, Y = 8; };

// a11 + a12 with s in its own buffer: x = (x + α p̂) + ω r̂; r = s - ω t; partials r~·r, r·r
__global__ void k_update_xr_s(double* __restrict__ x, const double* __restrict__ ph,
                              const double* __restrict__ rh, const double* __restrict__ s,
                              double* __restrict__ r, const double* __restrict__ t,
                              const double* __restrict__ rt, int64_t n, dd* __restrict__ part,
                              const DevState* __restrict__ st)
{
    if (st->done) return;
    const double alpha = st->alpha, omega = st->omega;
    double p[2] = {0.0, 0.0}, q[2] = {0.0, 0.0};
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
        x[c] = upd_x(x[c], ph[c], rh[c], alpha, omega);
        const double rn = upd_r(s[c], t[c], omega);
        r[c] = rn;
        dot2_acc(p[0], q[0], rt[c], rn);
        dot2_acc(p[1], q[1], rn, rn);
    }
    block_reduce_dd<2>(p, q, part + (int64_t)blockIdx.x * 2);
}

template <int K, int MODE>
bcgs_status launch_tb_k(bcgs_ctx c, TbArgs& a, int nchunk_total)
{
    constexpr int TX = Tile<K>::X, TY = Tile<K>::Y;
    using S = TbShape<K, TX, TY>;
    auto kern = k_cheb_tb<K, TX, TY, MODE>;
    static bool attr = false;
    if (!attr) {
        CUDA_OK(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)S::smem));
        attr = true;
    }
    dim3 grid((unsigned)((a.nx + TX - 1) / TX), (unsigned)((a.ny + TY - 1) / TY),
              (unsigned)nchunk_total);
    kern<<<grid, S::NT, S::smem, c->s>>>(a);
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

template <int K, int RY, int NW, int MODE>
bcgs_status launch_tb3_k(bcgs_ctx c, TbArgs& a, int nchunk_total)
{
    using S = Tb3Shape<K, RY, NW>;
    auto kern = k_cheb_tb3<K, RY, NW, MODE>;
    static bool attr = false;
    if (!attr) {
        CUDA_OK(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)S::smem));
        attr = true;
    }
    dim3 grid((unsigned)((a.nx + S::TX - 1) / S::TX), (unsigned)((a.ny + S::TY - 1) / S::TY),
              (unsigned)nchunk_total);
    kern<<<grid, NW * 32, S::smem, c->s>>>(a);
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

// ---- TMA tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// 3-D map over a slab field (nx, ny, L) of doubles, box (32, box_y, 1); OOB -> zeros
bool make_map(CUtensorMap* m, const double* base, int64_t nx, int64_t ny, int64_t L, int box_y)
{
    EncodeTiledFn fn = encode_fn();
    if (!fn || (nx * 8) % 16 || ((uintptr_t)base % 16)) return false;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)L};
    cuuint64_t strides[2] = {(cuuint64_t)(nx * 8), (cuuint64_t)(nx * ny * 8)};
    cuuint32_t box[3] = {32, (cuuint32_t)box_y, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

bool tma_ok(bcgs_ctx c) { return encode_fn() != nullptr && c->lay.nx % 2 == 0; }

template <int K, int RY, int NW, int NS, int MODE>
bcgs_status launch_tb4_k(bcgs_ctx c, TbArgs& a, int nchunk_total)
{
    using S = Tb4Shape<K, RY, NW, NS>;
    auto kern = k_cheb_tb4<K, RY, NW, NS, MODE>;
    static bool attr = false;
    if (!attr) {
        CUDA_OK(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)S::smem));
        attr = true;
    }
    TbMaps maps;
    memset(&maps, 0, sizeof maps);
    const int64_t nx = c->lay.nx, ny = c->lay.ny, L = c->lay.L;
    bool ok = true;
    if (MODE == MODE_PLAIN) ok = make_map(&maps.q, a.q, nx, ny, L, S::EY);
    if (MODE != MODE_PLAIN) {
        ok = make_map(&maps.r, a.r, nx, ny, L, S::EY) && make_map(&maps.w, a.w, nx, ny, L, S::EY);
        if (MODE == MODE_P)
            ok = ok && make_map(&maps.pa, a.p_a, nx, ny, L, S::EY) &&
                 make_map(&maps.pb, a.p_b, nx, ny, L, S::EY);
    }
    if (!ok) return fail(c, BCGS_E_CUDA, "cuTensorMapEncodeTiled failed");
    dim3 grid((unsigned)((a.nx + S::TX - 1) / S::TX), (unsigned)((a.ny + S::TY - 1) / S::TY),
              (unsigned)nchunk_total);
    kern<<<grid, NW * 32, S::smem, c->s>>>(a, maps);
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

// tile (TX, TY) of a kernel variant for degree k
void variant_tile(int variant, int k, int* tx, int* ty)
{
    if (variant == 2 || k > 5) {
        *tx = 32; *ty = 16;
        if (k >= 7) { *tx = 16; *ty = 8; } else if (k >= 5) { *tx = 32; *ty = 8; }
    } else if (variant == 5) {
        *tx = 32 - 2 * ((k + 1) / 2 * 2); *ty = 32 - 2 * k;   // TMA: even x-halo
    } else if (variant == 4) {
        *tx = 32 - 2 * k; *ty = 32 - 2 * k;      // RY = 4, NW = 8
    } else {
        *tx = 32 - 2 * k; *ty = 32 - 2 * k;      // RY = 2, NW = 16
    }
}

template <int K, int MODE>
bcgs_status launch_variant(bcgs_ctx c, TbArgs& a, int nz)
{
    if constexpr (K <= 5) {   // register budget: warp-row layouts up to K = 5
        if (c->tb_variant == 5 && tma_ok(c)) return launch_tb4_k<K, 2, 16, 4, MODE>(c, a, nz);
        if (c->tb_variant == 4) return launch_tb3_k<K, 4, 8, MODE>(c, a, nz);
        if (c->tb_variant == 3) return launch_tb3_k<K, 2, 16, MODE>(c, a, nz);
    }
    return launch_tb_k<K, MODE>(c, a, nz);
}

template <int MODE>
bcgs_status launch_tb(bcgs_ctx c, TbArgs& a)
{
    const int k = c->degree;
    a.nx = (int)c->lay.nx;
    a.ny = (int)c->lay.ny;
    a.Lb = (int)(c->lay.L / c->bpr);
    a.h2inv = c->h2inv;
    a.cz = c->cst[3];
    a.g1 = c->cst[4];
    a.A2 = c->cst[5];
    a.B2 = c->cst[6];
    for (int j = 0; j <= k; ++j) a.rho[j] = c->rho[j];
    // z-chunking: enough CTAs for ~8 waves of 148 SMs, chunks of >= 16 planes
    int tx, ty;
    variant_tile(c->tb_variant, k, &tx, &ty);
    const int64_t tiles = ((a.nx + tx - 1) / tx) * (int64_t)((a.ny + ty - 1) / ty) * c->bpr;
    int64_t want = (8 * kNumSMs + tiles - 1) / tiles;
    want = std::max<int64_t>(1, std::min<int64_t>(want, (a.Lb + 15) / 16));
    a.zch = (int)((a.Lb + want - 1) / want);
    a.nchunk = (a.Lb + a.zch - 1) / a.zch;
    const int nz = a.nchunk * c->bpr;
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

bool precond_supported(bcgs_ctx c)
{
    return c->pc != BCGS_PC_NONE && c->degree >= 1 && c->degree <= KMAX_TB;
}

bcgs_status precond_apply(bcgs_ctx c, const double* q, double* out)
{
    TbArgs a{};
    a.q = q;
    a.out = out;
    a.st = nullptr;
    Prof pf(c, KC_FUSED_P1, 16.0 * npts(c));
    return launch_tb<MODE_PLAIN>(c, a);
}

void on_begin(bcgs_ctx) {}

bcgs_status iteration(bcgs_ctx c)
{
    const int64_t n = npts(c);
    DevState* st = c->st;
    ref::Grid g = ref_grid(c, (int)c->lay.L);
    dim3 sg = stencil_grid(c), sb(ref::BX, ref::BY);
    const int nsb = (int)(sg.x * sg.y * sg.z);
    {   // K1: a14 (previous iteration) + a2
        TbArgs a{};
        a.r = F(c, V_R);
        a.w = F(c, V_W);
        a.p_a = F(c, V_P);
        a.p_b = F(c, V_P2);
        a.side_a = F(c, V_P);
        a.side_b = F(c, V_P2);
        a.out = F(c, V_PH);
        a.st = st;
        Prof pf(c, KC_FUSED_P1, 40.0 * n);
        TRY(launch_tb<MODE_P>(c, a));
    }
    TRY(halo(c, F(c, V_PH)));
    {
        Prof pf(c, KC_STENCIL1, 24.0 * n);
        ref::k_stencil_dot<1><<<sg, sb, 0, c->s>>>(F(c, V_PH), F(c, V_RT), F(c, V_W), g, 0,
                                                  c->part, st);
    }
    TRY(reduce<1>(c, nsb, STAGE_ALPHA));
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
    TRY(halo(c, F(c, V_RH)));
    {
        Prof pf(c, KC_STENCIL2, 24.0 * n);
        ref::k_stencil_dot<2><<<sg, sb, 0, c->s>>>(F(c, V_RH), F(c, V_S), F(c, V_T), g, 0,
                                                  c->part, st);
    }
    TRY(reduce<2>(c, nsb, STAGE_OMEGA));
    {
        Prof pf(c, KC_FUSED_XR, 64.0 * n);
        k_update_xr_s<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(
            F(c, V_X), F(c, V_PH), F(c, V_RH), F(c, V_S), F(c, V_R), F(c, V_T), F(c, V_RT), n,
            c->part, st);
    }
    TRY(reduce<2>(c, kEwBlocks, STAGE_RHO));
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

}  // namespace fused
