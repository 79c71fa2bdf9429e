// st_tma.cu -- TMA-staged stencil + dot kernels (a4 KernelBiCGS1: w = A p̂, r~ᵀw;
// a9 KernelBiCGS3: t = A r̂, tᵀs, tᵀt) -- north_star's "7-point stencil SpMV with
// shared-memory/TMA tile staging", fused with the dot products that follow it.
//
// A CTA (8 warps) owns a 64 x 16 output tile and marches z through a chunk of planes.  The
// Tensor Memory Accelerator stages, per z-step, the 68 x 18 box of v around the tile (zero
// fill outside the grid = the Dirichlet ghosts; the ghost planes -1 and L are real memory:
// zeros or halo data) and the 64 x 16 box of the dot operand a, into an NS-slot ring
// (mbarrier completion, one issuing thread), so the z-march never waits on DRAM latency.
// Each lane owns 2 adjacent x points of 2 rows; z-neighbours live in registers.  Same
// expression trees (expr.cuh) and dot accumulations (dd.cuh) as k_stencil2_dot: results are
// bitwise identical (the dots are certified / correctly rounded, R19, so the summation order
// does not matter).  Dirichlet faces only (Neumann mirrors -> k_stencil2_dot).
#include "tb_launch.cuh"

namespace fused {

namespace st {
constexpr int NW = 8, RY = 2, TXO = 64, TYO = NW * RY;      // output tile 64 x 16
constexpr int BXV = TXO + 4, BYV = TYO + 2;                   // v box 68 x 18 (x from x0 - 2)
constexpr int NS = 4;                                         // ring slots
constexpr int VSZ = (BXV * BYV * 8 + 127) / 128 * 128;        // bytes, 128-B aligned
constexpr int ASZ = TXO * TYO * 8;
constexpr int SLOT = VSZ + ASZ;
constexpr int SMEM = NS * SLOT + 128;
constexpr int ZC = 32;                      // planes per CTA (chunk) on deep slabs
constexpr int ZC_MIN = 4;                   // partial-slot capacity (ctx.cuh max_blocks)
constexpr int ZC_MAX = 64;                  // dot chains of 2 RY-row products per plane must
                                            // stay within kStencilDepth = 128 (bcgs_api.cu, R19)
}  // namespace st

struct StMaps {
    CUtensorMap v, a;
};

// Output planes [kb, ke) of the slab; the map of v spans planes -1..L (index + 1), a likewise.
template <int ND>
__global__ void __launch_bounds__(st::NW * 32, 3) k_stencil_tma(
    const __grid_constant__ StMaps maps, double* __restrict__ out, int nx, int ny, int kb, int ke,
    int zch, double h2inv, dd* __restrict__ part, const DevState* __restrict__ st)
{
    using namespace st;
    pdl_enter();
    if (st && st->done) return;
    extern __shared__ __align__(128) double smraw[];   // (same declaration as k_tb4.cuh)
    unsigned char* smb = reinterpret_cast<unsigned char*>(smraw);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smb + NS * SLOT);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = blockIdx.x * TXO, y0 = blockIdx.y * TYO;
    const int k0 = kb + blockIdx.z * zch, k1 = min(ke, k0 + zch);
    // step s (0-based) consumes v planes k0-1+s .. k0+1+s and a plane k0+s; slot s % NS
    // receives v plane k0+1+s and a plane k0+s (plane k0-1 and k0 arrive in the prologue)
    const int nsteps = k1 - k0;
    auto vslot = [&](int s) { return reinterpret_cast<double*>(smb + (s % NS) * SLOT); };
    auto aslot = [&](int s) { return reinterpret_cast<double*>(smb + (s % NS) * SLOT + VSZ); };
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // ring position p holds v plane k0 - 1 + p (p = 0, 1 prologue; p >= 2: step p - 2's zp)
    // and a plane k0 + p - 2; we index the ring by p and wait on bar[p % NS].
    auto issue = [&](int p) {
        const int z = k0 - 1 + p;            // v plane
        const int za = k0 + p - 2;           // a plane (p >= 2)
        unsigned bytes = BXV * BYV * 8;
        if (ND >= 1 && p >= 2) bytes += ASZ;
        mbar_expect_tx(&bar[p % NS], bytes);
        tma_load_3d(vslot(p), &maps.v, x0 - 2, y0 - 1, z + 1, &bar[p % NS]);
        if (ND >= 1 && p >= 2) tma_load_3d(aslot(p), &maps.a, x0, y0, za + 1, &bar[p % NS]);
    };
    const int npos = nsteps + 2;             // ring positions 0 .. nsteps + 1
    if (threadIdx.x == 0)
        for (int p = 0; p < NS && p < npos; ++p) issue(p);
    const int xl = 2 + 2 * lane;             // column of this lane's first point in the v box
    const int gx = x0 + 2 * lane;
    constexpr int NDA = ND > 0 ? ND : 1;
    double P[NDA] = {}, M[NDA] = {}, S[NDA] = {}, AB[NDA] = {};
    double P2[2] = {}, M2[2] = {}, S2[2] = {};
    // z-window per row: zm, zc (pairs), filled from positions 0 and 1
    double2 zm[RY], zc[RY];
    auto center = [&](const double* vb, int r) {
        return *reinterpret_cast<const double2*>(vb + (warp * RY + r + 1) * BXV + xl);
    };
    mbar_wait(&bar[0], 0);
    mbar_wait(&bar[1 % NS], (1 / NS) & 1);
#pragma unroll
    for (int r = 0; r < RY; ++r) {
        zm[r] = center(vslot(0), r);
        zc[r] = center(vslot(1), r);
    }
    for (int s = 0; s < nsteps; ++s) {
        const int p = s + 2;                 // position of v plane k0 + 1 + s (zp) and a plane
        mbar_wait(&bar[p % NS], (p / NS) & 1);
        const double* vc = vslot(p - 1);     // plane k: in-plane neighbours
        const double* vp = vslot(p);
        const double* ab = aslot(p);
        const int k = k0 + s;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            const int row = warp * RY + r;
            const double* crow = vc + (row + 1) * BXV + xl;
            const double2 zp = *reinterpret_cast<const double2*>(vp + (row + 1) * BXV + xl);
            const double xm = crow[-1], xp = crow[2];
            const double2 ym = *reinterpret_cast<const double2*>(crow - BXV);
            const double2 yp = *reinterpret_cast<const double2*>(crow + BXV);
            double2 o;
            o.x = stencil_row(zc[r].x, xm, zc[r].y, ym.x, yp.x, zm[r].x, zp.x, h2inv);
            o.y = stencil_row(zc[r].y, zc[r].x, xp, ym.y, yp.y, zm[r].y, zp.y, h2inv);
            const int gy = y0 + row;
            const bool in = gx < nx && gy < ny;   // nx even: both points or none
            if (in) {
                *reinterpret_cast<double2*>(out + (int64_t)k * nx * ny + (int64_t)gy * nx + gx) = o;
                if (ND >= 1) {
                    const double2 av = *reinterpret_cast<const double2*>(ab + row * TXO + 2 * lane);
                    if (ND >= 2) {   // tᵀs: Dot2, two chains; tᵀt: self
                        dot2_acc(P[0], S[0], AB[0], av.x, o.x);
                        dot2_acc(P2[0], S2[0], AB[0], av.y, o.y);
                        dot2_acc_self(P[1], S[1], o.x);
                        dot2_acc_self(P2[1], S2[1], o.y);
                    } else {         // r~ᵀw: Dot3, two chains
                        dot3_acc(P[0], M[0], S[0], AB[0], av.x, o.x);
                        dot3_acc(P2[0], M2[0], S2[0], AB[0], av.y, o.y);
                    }
                }
            }
            zm[r] = zc[r];
            zc[r] = zp;
        }
        __syncthreads();                     // everyone is done with position p - 2's slot
        if (threadIdx.x == 0 && p - 2 + NS < npos) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(p - 2 + NS);
        }
    }
    if (ND > 0) {
#pragma unroll
        for (int d = 0; d < (ND >= 2 ? 2 : 1); ++d)
            dd_add(P[d], M[d], S[d], AB[d], P2[d], M2[d], S2[d], 0.0);
        const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        block_reduce_dd<NDA>(P, M, S, AB, part + (int64_t)bid * ND);
    }
}

// the TMA-fed Chebyshev kernel (k_tb4.cuh) can run this context's slab (segment mode)
bool tb_tma_ok(bcgs_ctx c) { return tma_ok(c); }

// capability: Dirichlet faces, nx even (16-byte rows), 32-bit-safe maps
bool stencil_tma_ok(bcgs_ctx c)
{
    return encode_fn() != nullptr && c->lay.nx % 2 == 0 && !c->mbc.m && c->mbc.zlo < 0 &&
           c->mbc.zhi < 0;
}

// Planes per CTA.  Each CTA pays 2 extra v planes (the z-neighbours of its first and last
// plane) and one pipeline fill; deep slabs use ZC (many waves of 3 CTAs per SM: the tail is
// a small fraction).  On thin slabs (the per-rank shape of a multi-GPU run, 512^2 x 64 at
// P = 8) ZC leaves a fractional last wave of 3 x 148 slots, so the chunk length minimises
// waves x (planes + 2) there.  BCGS_OPT_STENCIL >= 2 fixes the length (measurement).
static int stencil_zc(bcgs_ctx c, int tiles, int planes)
{
    using namespace st;
    if (c->stencil_tma >= 2) return std::min(ZC_MAX, std::max(ZC_MIN, c->stencil_tma));
    const int64_t slots = (int64_t)kNumSMs * 3;
    const int64_t deep = (int64_t)tiles * ((planes + ZC - 1) / ZC);
    if (deep >= 4 * slots) return ZC;
    int best = ZC;
    double best_cost = 1e300;
    for (int nch = 1; nch <= (planes + ZC_MIN - 1) / ZC_MIN; ++nch) {
        const int zc = (planes + nch - 1) / nch;
        if (zc < ZC_MIN) break;
        const int64_t waves = ((int64_t)tiles * nch + slots - 1) / slots;
        const double cost = (double)waves * (zc + 2);
        if (cost < best_cost * 0.999) { best_cost = cost; best = zc; }
    }
    return best;
}

template <int ND>
bcgs_status launch_stencil_tma(bcgs_ctx c, const double* v, const double* a, double* out,
                               int kb, int ke, dd* part, int* nparts)
{
    using namespace st;
    static std::atomic<uint64_t> attr_dev{0};
    auto kern = k_stencil_tma<ND>;
    TRY(ensure_smem_attr(c, kern, SMEM, attr_dev));
    EncodeTiledFn fn = encode_fn();
    const int64_t nx = c->lay.nx, ny = c->lay.ny, L = c->lay.L, pl = nx * ny;
    StMaps maps;
    memset(&maps, 0, sizeof maps);
    auto mk = [&](CUtensorMap* m, const double* base, int bx, int by) {
        cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)(L + 2)};
        cuuint64_t strides[2] = {(cuuint64_t)(nx * 8), (cuuint64_t)(pl * 8)};
        cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
        cuuint32_t es[3] = {1, 1, 1};
        return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base - pl), dims,
                  strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
               CUDA_SUCCESS;
    };
    if (!mk(&maps.v, v, BXV, BYV) || (ND >= 1 && !mk(&maps.a, a, TXO, TYO)))
        return fail(c, BCGS_E_CUDA, "cuTensorMapEncodeTiled failed (stencil)");
    if (ND == 0) maps.a = maps.v;
    const int zc = stencil_zc(c, (int)((nx + TXO - 1) / TXO) * (int)((ny + TYO - 1) / TYO), ke - kb);
    const dim3 grid((unsigned)((nx + TXO - 1) / TXO), (unsigned)((ny + TYO - 1) / TYO),
                    (unsigned)((ke - kb + zc - 1) / zc));
    CUDA_OK(c, launch_k(c, kern, grid, dim3(NW * 32), SMEM, maps, out, (int)nx, (int)ny, kb, ke,
                        zc, c->h2inv, part, (const DevState*)c->st));
    *nparts = (int)(grid.x * grid.y * grid.z);
    return BCGS_OK;
}

template bcgs_status launch_stencil_tma<1>(bcgs_ctx, const double*, const double*, double*, int,
                                           int, dd*, int*);
template bcgs_status launch_stencil_tma<2>(bcgs_ctx, const double*, const double*, double*, int,
                                           int, dd*, int*);

}  // namespace fused
