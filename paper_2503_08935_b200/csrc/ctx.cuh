// ctx.cuh -- solver context, workspace layout and error plumbing shared by every
// translation unit of libbcgs.so (bcgs_api.cu = driver, tb_k*.cu = blocked kernels).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>

#include "../../include/bcgs.h"
#include "dd.cuh"
#include "state.cuh"
#include "ref_shapes.cuh"
#include "k_fused.cuh"
#include "p2p.cuh"

constexpr int kNumSMs = 148;
constexpr int kEwBlocks = kNumSMs * 8;   // element-wise grid: fixed -> deterministic partials
constexpr size_t kAlign = 256;

enum KClass {
    KC_PRECOND = 0, KC_STENCIL1, KC_AXPY, KC_STENCIL2, KC_UPDATE_XR, KC_UPDATE_P,
    KC_FINALIZE, KC_HALO, KC_ALLGATHER, KC_SCALARS, KC_FUSED_P1, KC_FUSED_P2, KC_FUSED_XR,
    KC_COUNT
};
inline const char* kClassName[KC_COUNT] = {
    "precond_sweep", "stencil_dot1", "axpy_s", "stencil_dot2", "update_xr", "update_p",
    "finalize", "halo", "allgather", "scalars", "fused_p_cheb", "fused_s_cheb", "fused_xr"};
// SPEC S:382 phase keys and the phase of each kernel class (bcgs_get_phase_times, NVTX)
constexpr int PH_PRECOND = 0, PH_HALO = 1, PH_ALLREDUCE = 2, PH_STENCIL = 3, PH_VECTOR = 4,
              PH_COUNT = 5;
inline const char* kPhaseName[PH_COUNT + 1] = {"preconditioner", "halo_exchange", "allreduce",
                                                "stencil_kernels", "vector_kernels", "total"};
inline int kc_phase(int kc)
{
    switch (kc) {
    case KC_PRECOND: case KC_FUSED_P1: case KC_FUSED_P2: return PH_PRECOND;
    case KC_HALO: return PH_HALO;
    case KC_FINALIZE: case KC_ALLGATHER: case KC_SCALARS: return PH_ALLREDUCE;
    case KC_STENCIL1: case KC_STENCIL2: return PH_STENCIL;
    default: return PH_VECTOR;   // KC_AXPY, KC_UPDATE_XR, KC_UPDATE_P, KC_FUSED_XR
    }
}


inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

constexpr int V_COUNT_MAX = 17;

struct Layout {
    int64_t nx, ny, nz, L, plane, vec_elems;   // vec_elems = (L + 2) * plane
    int64_t n_part;
    size_t off_vec[V_COUNT_MAX];
    int64_t ext_elems;
    size_t off_ext[3];
    size_t off_state, off_hist, off_scal, off_part, off_rank, off_gath, off_limb, off_glimb, total;
};

constexpr int V_X = 0, V_R = 1, V_RT = 2, V_P = 3, V_PH = 4, V_RH = 5, V_W = 6, V_T = 7,
              V_B = 8, V_C1 = 9, V_C2 = 10, V_IO = 11, V_W2 = 12, V_P2 = 13,
              V_S = 14, V_Y3 = 15, V_Y4 = 16, V_COUNT = 17;
// V_C1, V_C2, V_Y3, V_Y4: Chebyshev iterates (reference sweeps; multi-pass buffer pairs)

inline int64_t stencil_blocks(int64_t nx, int64_t ny, int64_t L)
{
    return ((nx + ref::BX - 1) / ref::BX) * ((ny + ref::BY - 1) / ref::BY) *
           ((L + ref::ZC - 1) / ref::ZC);
}

inline bool make_layout(const bcgs_grid_desc* g, int32_t nranks, Layout* lay)
{
    if (!g || nranks < 1) return false;
    lay->nx = g->n[0];
    lay->ny = g->n[1];
    lay->nz = g->n[2];
    if (lay->nx < 1 || lay->ny < 1 || lay->nz < 1 || lay->nz % nranks) return false;
    lay->L = lay->nz / nranks;
    lay->plane = lay->nx * lay->ny;
    lay->vec_elems = (lay->L + 2) * lay->plane;
    lay->n_part = std::max<int64_t>(
        {stencil_blocks(lay->nx, lay->ny, lay->L), (int64_t)kEwBlocks, fused::max_blocks(lay->nx, lay->ny, lay->L)});
    size_t off = 0;
    for (int v = 0; v < V_COUNT; ++v) {
        lay->off_vec[v] = off;
        off = align_up(off + sizeof(double) * (size_t)lay->vec_elems);
    }
    // G(CI) with nranks > 1: three extended fields of L + 2*KG planes (k-deep halos)
    lay->ext_elems = nranks > 1 ? (lay->L + 2 * (int64_t)BCGS_MAX_DEGREE + 2) * lay->plane : 0;
    for (int e = 0; e < 3; ++e) {
        lay->off_ext[e] = off;
        off = align_up(off + sizeof(double) * (size_t)lay->ext_elems);
    }
    lay->off_state = off; off = align_up(off + sizeof(DevState));
    lay->off_hist = off;  off = align_up(off + sizeof(double) * (BCGS_HIST_CAP + 1));
    lay->off_scal = off;  off = align_up(off + sizeof(double) * 8 * BCGS_HIST_CAP);
    // up to 5 Dot2 pairs per reduction (2-sync ω stage, R31)
    lay->off_part = off;  off = align_up(off + sizeof(dd) * 5 * (size_t)lay->n_part);
    lay->off_rank = off;  off = align_up(off + sizeof(dd) * 5);
    lay->off_gath = off;  off = align_up(off + sizeof(dd) * 5 * (size_t)nranks);
    // R19 exact path: this rank's superaccumulators [5 dots + flag][XL] and all ranks' copies
    lay->off_limb = off;  off = align_up(off + sizeof(long long) * 6 * xdot::XL);
    lay->off_glimb = off; off = align_up(off + sizeof(long long) * 6 * xdot::XL * (size_t)nranks);
    lay->total = off;
    return true;
}

struct EvRec {
    int cls;
    cudaEvent_t a, b;
    double bytes;
};

// In-process peer transport (bcgs_create_local): P contexts on one device, each driven by
// its own host thread; exchanges are device copies between the contexts' workspaces,
// ordered by events and a host barrier (the NCCL path's single-GPU twin, for testing).
struct HostBarrier {
    std::mutex m;
    std::condition_variable cv;
    int n = 0, count = 0;
    long gen = 0;
    void wait()
    {
        std::unique_lock<std::mutex> lk(m);
        const long g = gen;
        if (++count == n) {
            count = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct LocalGroup {
    int n = 0;
    std::vector<bcgs_ctx_s*> ctxs;
    HostBarrier bar;
};

struct bcgs_ctx_s {
    Layout lay;
    double h = 0.0, h2inv = 0.0;
    int32_t bc[6] = {0, 0, 0, 0, 0, 0};   // face kinds (bcgs_bc)
    ref::MirrorBc mbc{0, -1, -1};         // this rank's mirror faces, slab plane indices
    int rank = 0, nranks = 1, device = 0;
    cudaStream_t user = nullptr, s = nullptr;
    cudaEvent_t join = nullptr;
    ncclComm_t comm = nullptr;
    char* ws = nullptr;
    double* vec[V_COUNT] = {};     // interior plane 0 of each field
    double* ext[3] = {};           // G(CI) extended fields: extended plane 0 (= global z0 - KG)
    DevState* st = nullptr;
    double *hist = nullptr, *scal = nullptr;
    dd *part = nullptr, *rank_out = nullptr, *gath = nullptr;
    long long *limbs = nullptr, *glimbs = nullptr;   // R19 exact path (xdot.cuh)
    const double* src[9][10] = {};   // operand pairs of each reduction stage (exact path)
    int exact_opt = 0;               // BCGS_OPT_EXACT_DOT
    int pdl = 0;                     // BCGS_OPT_PDL: programmatic dependent launches (off:
                                     // measured no gain over graph replay)
    int tb_schedule = 0;             // BCGS_OPT_TB_SCHEDULE: 0 auto, 1 chunk grid, 2 segments
    int stencil_tma = 1;             // BCGS_OPT_STENCIL: TMA-staged stencil+dot (st_tma.cu);
                                     // >= 2: fixed planes per CTA
    int pipelined_opt = 0, pipelined = 0;   // BCGS_OPT_PIPELINED (option / active solve)
    char* pipe_mem = nullptr;        // pipelined: z, ẑ, q, q̂, y, v (library-owned fields)
    size_t pipe_bytes = 0;
    double* pipe[6] = {};
    double* h_pinned = nullptr;    // small pinned buffer for flag polls
    // options
    int kernels = 1, use_graph = 1, profile = 0, poll = 8, tb_variant = 7;
    int sync2_opt = 0, sync2 = 0;   // BCGS_OPT_SYNC2 (R31); active for the current solve
    int ablate = 0;   // BCGS_OPT_ABLATE: 1 skip halos, 2 skip cross-rank reductions (timing)
    int mp_min = 4;   // multi-pass temporal blocking for degree > mp_min (BCGS_OPT_MULTIPASS)
    // preconditioner
    bcgs_pc pc = BCGS_PC_NONE;
    int degree = 0, bpr = 1;
    double c_min = 10.0, c_max = 1.0 - 1e-4, ov_a = 0.0, ov_b = 0.0;
    double ivl[2] = {0, 0}, cst[7] = {}, rho[BCGS_MAX_DEGREE + 2] = {};
    // inner-Krylov preconditioners BJ(BiCGS) / G(BiCGS) (R29): one private unpreconditioned
    // context per block (solved concurrently, each on its own stream)
    double in_tol = 1e-6;
    int in_max = 500;
    int64_t in_iters = 0;
    std::vector<bcgs_ctx_s*> inner;
    std::vector<void*> inner_ws;
    int have_x0 = 0;
    double face[6] = {0, 0, 0, 0, 0, 0};
    // solve bookkeeping
    int begun = 0, launched = 0, fixed = 0, max_iter = 0;
    double tol = 0.0;
    std::chrono::steady_clock::time_point t0;
    // graph
    cudaGraphExec_t gexec = nullptr;
    int graph_key = -1;              // (sync2, pipelined) of the captured iteration
    // profiling
    std::vector<EvRec> pending;
    std::vector<cudaEvent_t> free_ev;
    double ktime[KC_COUNT] = {}, kbytes[KC_COUNT] = {};
    int64_t kcalls[KC_COUNT] = {};
    LocalGroup* lg = nullptr;         // in-process peers (testing transport)
    cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
    cudaStream_t s_comm = nullptr;              // halo stream (nranks > 1), overlapped
    cudaEvent_t ev_pre = nullptr, ev_halo = nullptr;
    // peer-memory transport (p2p.cuh): own mailbox (+ landing zones), the peers' mapped
    // mailboxes, and which of them were opened through CUDA IPC (closed at destroy)
    int p2p = 0, p2p_ready = 0;
    int comm_borrowed = 0;           // G(BiCGS) inner context: the outer one's NCCL comm
    int inproc = 0;                  // p2p ranks sharing this process (and GPU): no graphs
    p2p::Peers peers{};
    char* mailbox = nullptr;
    size_t mailbox_bytes = 0;
    std::vector<void*> ipc_opened;
    double comm_timeout_s = 300.0;              // NCCL: host-side wait limit before abort
    std::string err;
};

inline bcgs_status fail(bcgs_ctx c, bcgs_status s, const char* fmt, ...)
{
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return s;
}

#define CUDA_OK(c, call)                                                                    \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail((c), BCGS_E_CUDA, "%s failed: %s (%s:%d)", #call,                   \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                       \
    } while (0)

#define NCCL_OK(c, call)                                                                    \
    do {                                                                                    \
        ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess)                                                              \
            return fail((c), BCGS_E_NCCL, "%s failed: %s", #call, ncclGetErrorString(r_)); \
    } while (0)

// PDL chain (BCGS_OPT_PDL): one rank, no transport kernels or host waits in between, no
// profiling events
inline bool pdl_active(bcgs_ctx c)
{
    return c->pdl && c->nranks == 1 && !c->p2p && !c->comm && !c->profile;
}

// Launch a kernel that begins with pdl_enter(): with programmatic stream serialization
// when the PDL chain is active, as an ordinary launch otherwise.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(bcgs_ctx c, void (*kern)(KArgs...), dim3 grid, dim3 block,
                            size_t smem, Args&&... args)
{
    if (!pdl_active(c)) {
        kern<<<grid, block, smem, c->s>>>(std::forward<Args>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

inline double* F(bcgs_ctx c, int v) { return c->vec[v]; }
inline bool inner_pc(bcgs_ctx c) { return c->pc == BCGS_PC_BJ_BICGS || c->pc == BCGS_PC_G_BICGS; }
inline int64_t npts(bcgs_ctx c) { return c->lay.L * c->lay.plane; }

#define TRY(x)                        \
    do {                              \
        bcgs_status s_ = (x);         \
        if (s_ != BCGS_OK) return s_; \
    } while (0)
