// tb_launch.cuh -- host launchers of the temporally blocked kernel variants.  Included
// only by the per-degree translation units tb_k<K>.cu, which instantiate launch_variant<K,.>;
// the driver (bcgs_api.cu) sees the extern declarations in fused_launch.h.
#pragma once
#include <atomic>

#include "ctx.cuh"

namespace fused {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: `done` (one per kernel
// instantiation, owned by its launcher) remembers the devices it has been set on (bit d),
// race-free across host threads.
template <typename KernelFn>
bcgs_status ensure_smem_attr(bcgs_ctx c, KernelFn kern, size_t bytes, std::atomic<uint64_t>& done)
{
    const uint64_t bit = 1ull << (c->device & 63);
    if (done.load(std::memory_order_acquire) & bit) return BCGS_OK;
    CUDA_OK(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done.fetch_or(bit, std::memory_order_acq_rel);
    return BCGS_OK;
}

template <int K> struct Tile;
template <> struct Tile<1> { static constexpr int X = 32, Y = 16; };
template <> struct Tile<2> { static constexpr int X = 32, Y = 16; };
template <> struct Tile<3> { static constexpr int X = 32, Y = 16; };
template <> struct Tile<4> { static constexpr int X = 32, Y = 16; };
template <> struct Tile<5> { static constexpr int X = 32, Y = 8; };
template <> struct Tile<6> { static constexpr int X = 32, Y = 8; };
template <> struct Tile<7> { static constexpr int X = 16, Y = 8; };
template <> struct Tile<8> { static constexpr int X = 16, Y = 8; };

template <int K, int MODE, bool NEU = false>
bcgs_status launch_tb_k(bcgs_ctx c, TbArgs& a, int nchunk_total)
{
    if (a.nseg) return fail(c, BCGS_E_STATE, "segment mode needs the TMA kernel");
    constexpr int TX = Tile<K>::X, TY = Tile<K>::Y;
    using S = TbShape<K, TX, TY>;
    auto kern = k_cheb_tb<K, TX, TY, MODE, NEU>;
    static std::atomic<uint64_t> attr_dev{0};
    TRY(ensure_smem_attr(c, kern, S::smem, attr_dev));
    dim3 grid((unsigned)((a.nx + TX - 1) / TX), (unsigned)((a.ny + TY - 1) / TY),
              (unsigned)nchunk_total);
    kern<<<grid, S::NT, S::smem, c->s>>>(a);
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

// ---- TMA tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn()
{
    static const EncodeTiledFn fn = [] {   // thread-safe one-time lookup
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return (EncodeTiledFn)p;
        return (EncodeTiledFn) nullptr;
    }();
    return fn;
}

// 3-D map over a slab field (nx, ny, L) of doubles, box (32, box_y, 1); OOB -> zeros
inline bool make_map(CUtensorMap* m, const double* base, int64_t nx, int64_t ny, int64_t L, int box_y,
                     int box_x = 32)
{
    EncodeTiledFn fn = encode_fn();
    if (!fn || (nx * 8) % 16 || ((uintptr_t)base % 16)) return false;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)L};
    cuuint64_t strides[2] = {(cuuint64_t)(nx * 8), (cuuint64_t)(nx * ny * 8)};
    cuuint32_t box[3] = {(cuuint32_t)box_x, (cuuint32_t)box_y, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

// the TMA kernels index a slab field with 32-bit element offsets
inline bool tma_ok(bcgs_ctx c)
{
    const uint64_t elems = (uint64_t)c->lay.nx * c->lay.ny * (c->lay.L + 2 * BCGS_MAX_DEGREE + 2);
    return encode_fn() != nullptr && c->lay.nx % 2 == 0 && elems < (1ull << 32);
}

inline bool make_maps(bcgs_ctx c, TbMaps* maps, const TbArgs& a, int mode, int box_y,
                      int box_x = 32)
{
    memset(maps, 0, sizeof *maps);
    const int64_t nx = c->lay.nx, ny = c->lay.ny;
    const int64_t L = a.ext ? c->lay.L + 2 * (int64_t)BCGS_MAX_DEGREE : c->lay.L;
    if (mode == MODE_PLAIN) return make_map(&maps->q, a.q, nx, ny, L, box_y, box_x);
    if (mode == MODE_C) {   // x_{j0-1} -> q, x_{j0-2} -> w, q: r (fixed) or pa/pb (qsel)
        bool ok = make_map(&maps->q, a.q, nx, ny, L, box_y, box_x) &&
                  make_map(&maps->w, a.w, nx, ny, L, box_y, box_x);
        if (a.qsel)
            return ok && make_map(&maps->pa, a.p_a, nx, ny, L, box_y, box_x) &&
                   make_map(&maps->pb, a.p_b, nx, ny, L, box_y, box_x);
        return ok && make_map(&maps->r, a.r, nx, ny, L, box_y, box_x);
    }
    bool ok = make_map(&maps->r, a.r, nx, ny, L, box_y, box_x) &&
              make_map(&maps->w, a.w, nx, ny, L, box_y, box_x);
    if (mode == MODE_P)
        ok = ok && make_map(&maps->pa, a.p_a, nx, ny, L, box_y, box_x) &&
             make_map(&maps->pb, a.p_b, nx, ny, L, box_y, box_x);
    return ok;
}

template <int K, int RY, int NW, int NS, int MODE, bool NEU = false, bool O2 = false,
          bool SEG = false>
bcgs_status launch_tb4_k(bcgs_ctx c, TbArgs& a, int nchunk_total)
{
    using S = Tb4Shape<K, RY, NW, NS>;
    static_assert(S::smem <= 227 * 1024, "tb4 shared memory budget");
    if (a.nseg > 0 && !SEG) return fail(c, BCGS_E_STATE, "segment mode: wrong kernel instance");
    auto kern = k_cheb_tb4<K, RY, NW, NS, MODE, NEU, O2, SEG>;
    static std::atomic<uint64_t> attr_dev{0};
    TRY(ensure_smem_attr(c, kern, S::smem, attr_dev));
    TbMaps maps;
    if (!make_maps(c, &maps, a, MODE, S::EY))
        return fail(c, BCGS_E_CUDA, "cuTensorMapEncodeTiled failed");
    dim3 grid((unsigned)((a.nx + S::TX - 1) / S::TX), (unsigned)((a.ny + S::TY - 1) / S::TY),
              (unsigned)nchunk_total);
    if (a.nseg > 0) {   // segment mode (launch_tb): a 1-D grid over the tile-major work
        a.ntx = (int)grid.x;
        a.nty = (int)grid.y;
        grid = dim3((unsigned)a.nseg, 1, 1);
    }
    CUDA_OK(c, launch_k(c, kern, grid, dim3(NW * 32), S::smem, a, maps));
    return BCGS_OK;
}

// Kernel layout per degree: k <= 4 the TMA warp-row kernel with 24 warps
// (BCGS_OPT_TB_VARIANT 7, default); Neumann faces the 16-warp TMA kernel with mirror ghosts
// (k <= 5); otherwise (odd nx: no TMA, variant 2, one-pass k = 5..8) the square tile.
template <int K, int MODE>
bcgs_status launch_variant(bcgs_ctx c, TbArgs& a, int nz)
{
    if (a.bc.m || a.bc.zlo >= 0 || a.bc.zhi >= 0) {   // R27 mirror-ghost instantiations
        if constexpr (K <= 5) {
            if (tma_ok(c) && c->tb_variant != 2)
                return launch_tb4_k<K, 2, 16, 4, MODE, true>(c, a, nz);
        }
        return launch_tb_k<K, MODE, true>(c, a, nz);
    }
    if constexpr (K <= 4) {   // register budget of the 24-warp layout
        if (c->tb_variant != 2 && tma_ok(c)) {
            if (a.nseg > 0) return launch_tb4_k<K, 2, 24, 3, MODE, false, false, true>(c, a, nz);
            return launch_tb4_k<K, 2, 24, 3, MODE>(c, a, nz);
        }
    }
    return launch_tb_k<K, MODE>(c, a, nz);
}

}  // namespace fused
