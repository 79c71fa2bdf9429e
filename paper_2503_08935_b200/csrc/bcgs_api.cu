// bcgs_api.cu -- C ABI (include/bcgs.h) and solver driver of the B200-native Bi-CGSTAB
// Poisson hot path (arXiv 2503.08935).  One context per rank / GPU.  The driver enqueues
// the kernels of one outer iteration of Alg. 3 on a private stream; all
// scalars live on the device (state.cuh), the host only polls a done flag.
//
// Built with --fmad=false (R17): no FMA contraction in any kernel; fma() appears only in
// Dot2's TwoProd (dd.cuh).
#include "ctx.cuh"
#include <nvtx3/nvToolsExt.h>
#include "k_ref.cuh"
#include "k_stream.cuh"
#include "pipe.cuh"

namespace {


ref::Grid ref_grid(bcgs_ctx c, int Lb)
{
    ref::Grid g;
    g.nx = (int)c->lay.nx;
    g.ny = (int)c->lay.ny;
    g.L = (int)c->lay.L;
    g.Lb = Lb;
    g.h2inv = c->h2inv;
    g.bc = c->mbc;
    return g;
}

// Mirror faces of the extended slab of G(CI) (planes [v0, v1) valid): the physical z faces
// sit at v0 on the first rank and at v1 - 1 on the last.
ref::MirrorBc ext_mirror(bcgs_ctx c, int v0, int v1)
{
    ref::MirrorBc m = c->mbc;
    m.zlo = (c->rank == 0 && c->bc[4]) ? v0 : -1;
    m.zhi = (c->rank == c->nranks - 1 && c->bc[5]) ? v1 - 1 : -1;
    return m;
}

dim3 stencil_grid(bcgs_ctx c)
{
    return dim3((unsigned)((c->lay.nx + ref::BX - 1) / ref::BX),
                (unsigned)((c->lay.ny + ref::BY - 1) / ref::BY),
                (unsigned)((c->lay.L + ref::ZC - 1) / ref::ZC));
}

// ------------------------------------------------------------------ profiling events
cudaEvent_t get_ev(bcgs_ctx c)
{
    if (!c->free_ev.empty()) {
        cudaEvent_t e = c->free_ev.back();
        c->free_ev.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct Prof {
    bcgs_ctx c;
    int cls;
    double bytes;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    Prof(bcgs_ctx c_, int cls_, double bytes_, cudaStream_t s_ = nullptr)
        : c(c_), cls(cls_), bytes(bytes_), s(s_ ? s_ : c_->s)
    {
        if (c->profile) {
            a = get_ev(c);
            cudaEventRecord(a, s);
            // "<S:382 phase key>/<kernel class>" (host range around the launch)
            char name[64];
            snprintf(name, sizeof name, "%s/%s", kPhaseName[kc_phase(cls)], kClassName[cls]);
            nvtxRangePushA(name);
        }
    }
    ~Prof()
    {
        if (c->profile) {
            nvtxRangePop();
            cudaEvent_t b = get_ev(c);
            cudaEventRecord(b, s);
            c->pending.push_back({cls, a, b, bytes});
        }
    }
};

void harvest(bcgs_ctx c)
{
    if (c->pending.empty()) return;
    cudaStreamSynchronize(c->s);
    for (auto& r : c->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        c->ktime[r.cls] += ms;
        c->kcalls[r.cls] += 1;
        c->kbytes[r.cls] = r.bytes;
        c->free_ev.push_back(r.a);
        c->free_ev.push_back(r.b);
    }
    c->pending.clear();
}

// ------------------------------------------------------------------ host constants
// Eq. 9: μ_i = 4 sin²(iπ/(2(n+1))); Eqs. 10-11; R9, R10, R18.
double mu(int64_t n, int64_t i)
{
    double s = sin(((double)i * M_PI) / (2.0 * (double)(n + 1)));
    return 4.0 * (s * s);
}

// Extreme eigenvalues of one 1-D factor with `nn` Neumann ends (R27; Eq. 5's N):
//   nn = 0: Eq. 9, i = 1 and n;   nn = 1: 4 sin²((2i-1)π/(4n)), i = 1 and n;
//   nn = 2: 4 sin²(iπ/(2(n-1))), i = 0 and n-1.
void factor_range(int64_t n, int nn, double* lo, double* hi)
{
    auto f1 = [n](int64_t i) {
        double s = sin(((double)(2 * i - 1) * M_PI) / (4.0 * (double)n));
        return 4.0 * (s * s);
    };
    auto f2 = [n](int64_t i) {
        double s = sin(((double)i * M_PI) / (2.0 * (double)(n - 1)));
        return 4.0 * (s * s);
    };
    if (nn == 0) { *lo = mu(n, 1); *hi = mu(n, n); }
    else if (nn == 1) { *lo = f1(1); *hi = f1(n); }
    else { *lo = f2(0); *hi = f2(n - 1); }
}

// Eqs. 10-11: sums of the factor extremes; nn[3] = Neumann ends of the x, y, z factors.
void bounds_box(int64_t nx, int64_t ny, int64_t nzb, double h, const int* nn, double* lo,
                double* hi)
{
    double h2inv = 1.0 / (h * h), lx, hx, ly, hy, lz, hz;
    factor_range(nx, nn[0], &lx, &hx);
    factor_range(ny, nn[1], &ly, &hy);
    factor_range(nzb, nn[2], &lz, &hz);
    *lo = ((lx * h2inv) + (ly * h2inv)) + (lz * h2inv);
    *hi = ((hx * h2inv) + (hy * h2inv)) + (hz * h2inv);
}

// Face kinds are 0 / 1 and a Neumann axis has >= 2 points (the mirror needs a neighbour).
bool bc_ok(const bcgs_grid_desc* g)
{
    for (int f = 0; f < 6; ++f)
        if (g->bc[f] != BCGS_BC_DIRICHLET && g->bc[f] != BCGS_BC_NEUMANN) return false;
    for (int d = 0; d < 3; ++d)
        if ((g->bc[2 * d] || g->bc[2 * d + 1]) && g->n[d] < 2) return false;
    return true;
}

bcgs_status cheb_constants(const bcgs_grid_desc* g, int32_t nslab, bcgs_pc pc, int32_t k,
                           double c_min, double c_max, double ov_a, double ov_b, double* ivl,
                           double* cst, double* rho)
{
    if (k < 0 || k > BCGS_MAX_DEGREE) return BCGS_E_INVALID;
    double a, b;
    if (ov_a > 0.0 || ov_b > 0.0) {
        a = ov_a;
        b = ov_b;
    } else {
        int nn[3] = {g->bc[0] + g->bc[1], g->bc[2] + g->bc[3], g->bc[4] + g->bc[5]};
        if (pc == BCGS_PC_CHEB_GNOCOMM || pc == BCGS_PC_CHEB_G) {
            double lo, hi;
            bounds_box(g->n[0], g->n[1], g->n[2], g->h, nn, &lo, &hi);
            a = c_min * lo;
            b = c_max * hi;
        } else if (nslab == 1) {
            bounds_box(g->n[0], g->n[1], g->n[2], g->h, nn, &a, &b);   // R10
        } else {
            // R10 + R27: the blocks' z factors are (z- kind, D), (D, D), (D, z+ kind); one
            // interval spanning all of them
            const int zk[3] = {g->bc[4], g->bc[5], 0};
            for (int q = 0; q < (nslab > 2 ? 3 : 2); ++q) {
                double lo, hi;
                int nb[3] = {nn[0], nn[1], zk[q]};
                bounds_box(g->n[0], g->n[1], g->n[2] / nslab, g->h, nb, &lo, &hi);
                if (q == 0 || lo < a) a = lo;
                if (q == 0 || hi > b) b = hi;
            }
        }
    }
    if (!(a > 0.0) || !(a < b) || !std::isfinite(b)) return BCGS_E_SPECTRUM;
    double theta = (b + a) / 2.0, delta = (b - a) / 2.0;   // Eq. 15
    double sigma = theta / delta;
    rho[0] = 1.0 / sigma;
    int kk = std::max(k, 1);
    for (int j = 1; j <= kk; ++j) rho[j] = 1.0 / (2.0 * sigma - rho[j - 1]);
    ivl[0] = a;
    ivl[1] = b;
    cst[0] = theta;
    cst[1] = delta;
    cst[2] = sigma;
    cst[3] = 1.0 / theta;
    cst[4] = 2.0 * (rho[1] / delta);
    cst[5] = 2.0 * sigma;
    cst[6] = 2.0 / delta;
    return BCGS_OK;
}

// ------------------------------------------------------------------ init / state
// The parked stage with its flagged dots replaced by the exactly rounded sums of the
// superaccumulators limbs[r][d][XL] (+ a non-finite flag per rank at [r][5][0]).
__global__ void k_resolve(DevState* st, const long long* __restrict__ limbs, int nranks,
                          int64_t rank_stride, double* hist, double* scal)
{
    const int stage = st->pend_stage, mask = st->pend_mask;
    if (!mask || st->comm_err) return;   // a failed limb exchange leaves the stage parked
    bool bad = false;
    for (int r = 0; r < nranks; ++r) bad |= limbs[r * rank_stride + 5 * xdot::XL] != 0;
    double v[5];
    for (int d = 0; d < 5; ++d) {
        v[d] = st->pend_v[d];
        if (mask & (1 << d)) {
            v[d] = xdot::round_limbs(limbs + d * xdot::XL, nranks, rank_stride, bad);
            st->n_exact += 1;
        }
    }
    st->pend_mask = 0;
    if (stage != STAGE_DOT) st->done = DONE_RUNNING;
    stage_update(st, stage, v, hist, scal);
}

__global__ void k_set_exact(DevState* st, int exact) { st->exact_mode = exact; }

__global__ void k_init_state(DevState* st, double tol, int max_iter, int fixed, int exact)
{
    st->pend_stage = 0;
    st->pend_mask = 0;
    st->exact_mode = exact;
    st->n_exact = 0;
    st->tol = tol;
    st->max_iter = max_iter;
    st->fixed_iters = fixed;
    st->done = DONE_RUNNING;
    st->iter = 0;
    st->pend = DONE_RUNNING;
}

// ------------------------------------------------------------------ host waits
// Wait for the private stream.  NCCL contexts poll ncclCommGetAsyncError while waiting and
// abort the communicator on an asynchronous error or after comm_timeout_s (a dead peer
// would otherwise block the host forever); the p2p transport times out on the device.
bcgs_status sync_stream(bcgs_ctx c)
{
    if (!c->comm) {
        CUDA_OK(c, cudaStreamSynchronize(c->s));
        return BCGS_OK;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t e = cudaStreamQuery(c->s);
        if (e == cudaSuccess) return BCGS_OK;
        if (e != cudaErrorNotReady) CUDA_OK(c, e);
        ncclResult_t ae = ncclSuccess;
        ncclCommGetAsyncError(c->comm, &ae);
        const double dt =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if ((ae != ncclSuccess && ae != ncclInProgress) || dt > c->comm_timeout_s) {
            ncclCommAbort(c->comm);
            c->comm = nullptr;
            if (ae != ncclSuccess && ae != ncclInProgress)
                return fail(c, BCGS_E_NCCL, "NCCL asynchronous error: %s (communicator aborted)",
                            ncclGetErrorString(ae));
            return fail(c, BCGS_E_NCCL, "NCCL wait exceeded %.0f s (communicator aborted)",
                        c->comm_timeout_s);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

// ------------------------------------------------------------------ communication
// Face-halo exchange of a field (a3 / a8, MPI1 / MPI3 P:278): send plane 0 to rank-1
// and plane L-1 to rank+1, receive the ghost planes -1 and L.  NCCL, or the in-process
// peer transport of bcgs_create_local.
bcgs_status local_exchange_begin(bcgs_ctx c, cudaStream_t hs)
{
    CUDA_OK(c, cudaEventRecord(c->ev_ready, hs));
    c->lg->bar.wait();   // every rank has recorded its producer event
    return BCGS_OK;
}

bcgs_status local_exchange_end(bcgs_ctx c, bool all, cudaStream_t hs)
{
    CUDA_OK(c, cudaEventRecord(c->ev_done, hs));
    c->lg->bar.wait();   // every rank has issued its copies
    for (int r = 0; r < c->nranks; ++r)
        if (r != c->rank && (all || r == c->rank - 1 || r == c->rank + 1))
            CUDA_OK(c, cudaStreamWaitEvent(c->s, c->lg->ctxs[r]->ev_done, 0));
    return BCGS_OK;
}

// peer transport: send k planes of v (interior planes [0, k) down, [L - k, L) up) and land
// the neighbours' planes in [gl, gl + k planes) and [gh, gh + k planes) (p2p.cuh)
bcgs_status p2p_halo(bcgs_ctx c, const double* v, double* gl, double* gh, int k,
                     cudaStream_t hs, int guarded)
{
    if (!c->p2p_ready) return fail(c, BCGS_E_STATE, "p2p transport not connected");
    if (k > c->peers.cap)
        return fail(c, BCGS_E_CONFIG, "halo of %d planes > p2p landing capacity %lld", k,
                    (long long)c->peers.cap);
    const int nb = (int)std::min<int64_t>(kNumSMs, (k * c->lay.plane + 255) / 256);
    p2p::k_halo_ack<<<1, 32, 0, hs>>>(c->peers, c->st, guarded);
    p2p::k_halo_send<<<nb, 256, 0, hs>>>(c->peers, v, c->lay.L, k, c->st, guarded);
    p2p::k_halo_wait<<<1, 32, 0, hs>>>(c->peers, c->st, guarded);
    p2p::k_halo_land<<<nb, 256, 0, hs>>>(c->peers, gl, gh, k, c->st, guarded);
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

// The peer context's copy of my field pointer v (same layout on every rank): the workspace,
// or the library-owned pipelined fields
const double* peer_field(bcgs_ctx c, bcgs_ctx p, const void* v)
{
    const char* cv = (const char*)v;
    if (c->pipe_mem && cv >= c->pipe_mem && cv < c->pipe_mem + c->pipe_bytes && p->pipe_mem)
        return (const double*)(p->pipe_mem + (cv - c->pipe_mem));
    return (const double*)(p->ws + (cv - c->ws));
}

bcgs_status halo_on(bcgs_ctx c, double* v, cudaStream_t hs, int guarded = 1)
{
    if (c->nranks == 1 || (c->ablate & 1)) return BCGS_OK;   // ablation: timing only
    Prof pf(c, KC_HALO, 0.0, hs);
    const size_t pl = (size_t)c->lay.plane;
    if (c->p2p) return p2p_halo(c, v, v - pl, v + c->lay.L * pl, 1, hs, guarded);
    if (c->lg) {
        TRY(local_exchange_begin(c, hs));
        for (int d = -1; d <= 1; d += 2) {
            const int nb = c->rank + d;
            if (nb < 0 || nb >= c->nranks) continue;
            bcgs_ctx p = c->lg->ctxs[nb];
            const double* pv = peer_field(c, p, v);
            CUDA_OK(c, cudaStreamWaitEvent(hs, p->ev_ready, 0));
            // from rank-1: its plane L-1 -> my ghost -1; from rank+1: its plane 0 -> ghost L
            const double* src = d < 0 ? pv + (c->lay.L - 1) * pl : pv;
            double* dst = d < 0 ? v - pl : v + c->lay.L * pl;
            CUDA_OK(c, cudaMemcpyAsync(dst, src, pl * sizeof(double), cudaMemcpyDeviceToDevice,
                                       hs));
        }
        return local_exchange_end(c, false, hs);
    }
    NCCL_OK(c, ncclGroupStart());
    if (c->rank > 0) {
        NCCL_OK(c, ncclSend(v, pl, ncclDouble, c->rank - 1, c->comm, hs));
        NCCL_OK(c, ncclRecv(v - pl, pl, ncclDouble, c->rank - 1, c->comm, hs));
    }
    if (c->rank < c->nranks - 1) {
        NCCL_OK(c, ncclSend(v + (c->lay.L - 1) * pl, pl, ncclDouble, c->rank + 1, c->comm, hs));
        NCCL_OK(c, ncclRecv(v + c->lay.L * pl, pl, ncclDouble, c->rank + 1, c->comm, hs));
    }
    NCCL_OK(c, ncclGroupEnd());
    return BCGS_OK;
}

bcgs_status halo(bcgs_ctx c, double* v) { return halo_on(c, v, c->s); }
// outside an iteration (API calls, the x halo of begin / finish): not skipped when done
bcgs_status halo_api(bcgs_ctx c, double* v) { return halo_on(c, v, c->s, 0); }

// All-gather of `bytes` from every rank's `mine` (at the same workspace offset on every
// rank) into dst[rank] (NCCL, or the in-process transport).
bcgs_status allgather_bytes(bcgs_ctx c, const void* mine, void* dst, size_t bytes)
{
    if (c->lg) {
        const ptrdiff_t off = (const char*)mine - c->ws;
        TRY(local_exchange_begin(c, c->s));
        for (int r = 0; r < c->nranks; ++r) {
            bcgs_ctx p = c->lg->ctxs[r];
            if (r != c->rank) CUDA_OK(c, cudaStreamWaitEvent(c->s, p->ev_ready, 0));
            CUDA_OK(c, cudaMemcpyAsync((char*)dst + r * bytes, p->ws + off, bytes,
                                       cudaMemcpyDeviceToDevice, c->s));
        }
        return local_exchange_end(c, true, c->s);
    }
    NCCL_OK(c, ncclAllGather(mine, dst, bytes, ncclUint8, c->comm, c->s));
    return BCGS_OK;
}

// All-gather of every rank's ND Dot2 triples (MPI2/4/5).
bcgs_status allgather_pairs(bcgs_ctx c, int nd)
{
    Prof pf(c, KC_ALLGATHER, 0.0);
    if (c->ablate & 2) {   // ablation (timing only): every slot = this rank's pairs, no comm
        for (int r = 0; r < c->nranks; ++r)
            CUDA_OK(c, cudaMemcpyAsync(c->gath + (size_t)r * nd, c->rank_out, nd * sizeof(dd),
                                       cudaMemcpyDeviceToDevice, c->s));
        return BCGS_OK;
    }
    return allgather_bytes(c, c->rank_out, c->gath, nd * sizeof(dd));
}

// Chain depth of a grid-stride element-wise producer (kEwBlocks x 256 threads): 2 x the
// products per thread (R19 certification bound, dd.cuh); stencil producers pass 2 x 16.
inline int ew_depth(int64_t n)
{
    const int64_t T = (int64_t)kEwBlocks * 256;
    return (int)(2 * ((n + T - 1) / T + 2));
}
// per-thread dot chains of the stencil kernels: 2 products per plane and chain over <= 64
// planes (TMA stencil: 2 rows x st::ZC_MAX; L1 stencil: 2 x 2 x SZC), + 1 for the chain merge
constexpr int kStencilDepth = 2 * 2 * stream::SZC + 2;
static_assert(2 * 64 + 1 <= kStencilDepth, "TMA stencil chunk cap (st_tma.cu ZC_MAX)");

// Reduce `nparts` partial triples of ND dots, then complete the stage (certified) or park it
// for the exact path.  src = the ND operand pairs (a_d, b_d), recorded for that path.
// k3_mask bit d: dot d was accumulated with Dot3 chains (the r~ dots, dd.cuh)
template <int ND>
bcgs_status reduce(bcgs_ctx c, int nparts, int stage, int depth, int k3_mask,
                   std::initializer_list<const double*> src)
{
    int i = 0;
    for (const double* p : src) c->src[stage][i++] = p;
    int self_mask = 0;   // a·a dots: their producers accumulate no Σ|h| (dot2_acc_self)
    for (int d = 0; d < ND; ++d)
        if (c->src[stage][2 * d] && c->src[stage][2 * d] == c->src[stage][2 * d + 1])
            self_mask |= 1 << d;
    const double nprod = (double)c->lay.nx * (double)c->lay.ny * (double)c->lay.nz;
    if (c->p2p) {   // one kernel: finalize + one-shot peer exchange + rank-ordered combine
        if (!c->p2p_ready) return fail(c, BCGS_E_STATE, "p2p transport not connected");
        Prof pf(c, KC_FINALIZE, 0.0);
        p2p::k_reduce_p2p<ND><<<1, 256, 0, c->s>>>(c->peers, c->part, nparts, stage, c->st,
                                                    c->hist, c->scal, depth, nprod, self_mask,
                                                    k3_mask, (c->ablate & 2) ? 1 : 0);
        CUDA_OK(c, cudaGetLastError());
        return BCGS_OK;
    }
    // a communicator (also a 1-rank one: the NCCL path exercised on one GPU) -> all-gather
    const bool gather = c->nranks > 1 || c->comm;
    {
        Prof pf(c, KC_FINALIZE, 0.0);
        CUDA_OK(c, launch_k(c, k_finalize<ND>, dim3(1), dim3(1024), 0, (const dd*)c->part,
                            nparts, stage, c->st, c->hist, c->scal, c->rank_out,
                            gather ? 2 : 1, depth, nprod, self_mask, k3_mask));
    }
    if (gather) {
        TRY(allgather_pairs(c, ND));
        Prof pf(c, KC_SCALARS, 0.0);
        k_scalars<ND><<<1, 1, 0, c->s>>>(c->gath, c->nranks, stage, c->st, c->hist, c->scal,
                                         depth, nparts, nprod, self_mask, k3_mask);
    }
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

// R19 fallback: the parked stage's flagged dots recomputed exactly (superaccumulators,
// all-gathered across ranks and summed as integers) and the stage completed.  Returns the
// stage in *stage (-1: nothing was parked).
bcgs_status resolve(bcgs_ctx c, int* stage)
{
    *stage = -1;
    int32_t* h = (int32_t*)c->h_pinned;
    CUDA_OK(c, cudaMemcpyAsync(h, &c->st->pend_stage, 2 * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, c->s));
    TRY(sync_stream(c));
    const int stg = h[0], mask = h[1];
    if (!mask) return BCGS_OK;
    const int64_t XL = xdot::XL, per_rank = 6 * XL;
    CUDA_OK(c, cudaMemsetAsync(c->limbs, 0, sizeof(long long) * per_rank, c->s));
    for (int d = 0; d < 5; ++d)
        if (mask & (1 << d)) {
            const double* a = c->src[stg][2 * d];
            const double* b = c->src[stg][2 * d + 1];
            if (!a || !b) return fail(c, BCGS_E_STATE, "exact dot: no operands for stage %d", stg);
            xdot::k_exact_dot<<<kEwBlocks, 256, 0, c->s>>>(a, b, npts(c), c->limbs + d * XL,
                                                           c->limbs + 5 * XL);
        }
    CUDA_OK(c, cudaGetLastError());
    const long long* L = c->limbs;
    if (c->p2p) {
        p2p::k_limbs_p2p<<<1, 256, 0, c->s>>>(c->peers, c->limbs, c->glimbs, c->st);
        L = c->glimbs;
    } else if (c->nranks > 1 || c->comm) {
        TRY(allgather_bytes(c, c->limbs, c->glimbs, sizeof(long long) * per_rank));
        L = c->glimbs;
    }
    k_resolve<<<1, 1, 0, c->s>>>(c->st, L, c->nranks, per_rank, c->hist, c->scal);
    CUDA_OK(c, cudaGetLastError());
    *stage = stg;
    return BCGS_OK;
}


// ------------------------------------------------------------------ preconditioner (ref)
// Alg. 4 with one sweep per launch; out = M^-1 q on every block.
// G(CI) on P > 1 ranks: exact global Chebyshev polynomial.  Instead of Alg. 4's
// halo exchange before every sweep (MPI2), exchange k planes of the input once
// (communication-avoiding); sweep j is then exact on the extended slab minus
// j planes per side, so after k sweeps the rank's own L planes are exact.
bcgs_status halo_deep(bcgs_ctx c, const double* q, double* E, int k)
{
    const size_t pl = (size_t)c->lay.plane;
    const int64_t L = c->lay.L, KG = BCGS_MAX_DEGREE;
    Prof pf(c, KC_HALO, 0.0);
    if (c->p2p) return p2p_halo(c, q, E + (KG - k) * pl, E + (KG + L) * pl, k, c->s, 1);
    if (c->lg) {
        TRY(local_exchange_begin(c, c->s));
        for (int d = -1; d <= 1; d += 2) {
            const int nb = c->rank + d;
            if (nb < 0 || nb >= c->nranks) continue;
            bcgs_ctx p = c->lg->ctxs[nb];
            const double* pq = peer_field(c, p, q);
            CUDA_OK(c, cudaStreamWaitEvent(c->s, p->ev_ready, 0));
            const double* src = d < 0 ? pq + (L - k) * pl : pq;
            double* dst = d < 0 ? E + (KG - k) * pl : E + (KG + L) * pl;
            CUDA_OK(c, cudaMemcpyAsync(dst, src, k * pl * sizeof(double),
                                       cudaMemcpyDeviceToDevice, c->s));
        }
        return local_exchange_end(c, false, c->s);
    }
    NCCL_OK(c, ncclGroupStart());
    if (c->rank > 0) {
        NCCL_OK(c, ncclSend(q, k * pl, ncclDouble, c->rank - 1, c->comm, c->s));
        NCCL_OK(c, ncclRecv(E + (KG - k) * pl, k * pl, ncclDouble, c->rank - 1, c->comm, c->s));
    }
    if (c->rank < c->nranks - 1) {
        NCCL_OK(c, ncclSend(q + (L - k) * pl, k * pl, ncclDouble, c->rank + 1, c->comm, c->s));
        NCCL_OK(c, ncclRecv(E + (KG + L) * pl, k * pl, ncclDouble, c->rank + 1, c->comm, c->s));
    }
    NCCL_OK(c, ncclGroupEnd());
    return BCGS_OK;
}

bcgs_status precond_g(bcgs_ctx c, const double* q, double* out, const DevState* st)
{
    const int k = c->degree;
    const int64_t pl = c->lay.plane, L = c->lay.L, KG = BCGS_MAX_DEGREE;
    ref::ChebConst cc{c->cst[3], c->cst[4], c->cst[5], c->cst[6]};
    if (k == 0) {
        Prof pf(c, KC_PRECOND, 16.0 * npts(c));
        ref::k_scale<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(q, out, npts(c), cc.cz, st);
        CUDA_OK(c, cudaGetLastError());
        return BCGS_OK;
    }
    double* E = c->ext[0];
    double* A = c->ext[1];
    double* B = c->ext[2];
    // every write below is guarded by the device state (a parked solve, R19, leaves the
    // fields the resumed iteration still needs untouched)
    ref::k_copy<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(q, E + KG * pl, L * pl, st);
    TRY(halo_deep(c, q, E, k));
    const int v0 = (int)(c->rank == 0 ? KG : KG - k);
    const int v1 = (int)(c->rank == c->nranks - 1 ? KG + L : KG + L + k);
    if (c->kernels == 1 && k <= fused::KMAX_TB) {   // all k sweeps in one HBM pass
        Prof pf(c, KC_PRECOND, 16.0 * npts(c));
        return fused::precond_g_tb(c, E, out, v0, v1, st);
    }
    const int nx = (int)c->lay.nx, ny = (int)c->lay.ny;
    const dim3 blk(ref::BX, ref::BY);
    auto grid = [&](int kb, int ke) {
        return dim3((unsigned)((nx + ref::BX - 1) / ref::BX), (unsigned)((ny + ref::BY - 1) / ref::BY),
                    (unsigned)((ke - kb + ref::ZC - 1) / ref::ZC));
    };
    Prof pf(c, KC_PRECOND, 16.0 * npts(c));
    ref::k_cheb_sweep_rng<<<grid(v0, v1), blk, 0, c->s>>>(E, nullptr, nullptr, A, nx, ny, v0, v1,
                                                          v0, v1, c->h2inv, ext_mirror(c, v0, v1),
                                                          cc, 0.0, 0.0, 1, st);
    double* xm1 = A;
    double* xm2 = nullptr;
    for (int j = 2; j <= k; ++j) {
        double* dst = xm2 ? xm2 : B;
        ref::k_cheb_sweep_rng<<<grid(v0, v1), blk, 0, c->s>>>(E, xm1, xm2, dst, nx, ny, v0, v1, v0,
                                                              v1, c->h2inv, ext_mirror(c, v0, v1),
                                                              cc, c->rho[j],
                                                              c->rho[j - 1], 0, st);
        xm2 = xm1;
        xm1 = dst;
    }
    ref::k_copy<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(xm1 + KG * pl, out, L * pl, st);
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

bcgs_status precond_inner(bcgs_ctx c, const double* q, double* out, const DevState* st);
bcgs_status inner_all(bcgs_ctx c);

bcgs_status precond_ref(bcgs_ctx c, const double* q, double* out, const DevState* st)
{
    const int64_t n = npts(c);
    const int k = c->degree;
    if (inner_pc(c)) return precond_inner(c, q, out, st);
    if (c->pc == BCGS_PC_CHEB_G && c->nranks > 1) return precond_g(c, q, out, st);
    if (c->pc == BCGS_PC_NONE) {
        Prof pf(c, KC_PRECOND, 16.0 * n);
        ref::k_copy<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(q, out, n, st);
        CUDA_OK(c, cudaGetLastError());
        return BCGS_OK;
    }
    ref::ChebConst cc{c->cst[3], c->cst[4], c->cst[5], c->cst[6]};
    if (k == 0) {
        Prof pf(c, KC_PRECOND, 16.0 * n);
        ref::k_scale<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(q, out, n, cc.cz, st);
        CUDA_OK(c, cudaGetLastError());
        return BCGS_OK;
    }
    ref::Grid g = ref_grid(c, (int)(c->lay.L / c->bpr));
    dim3 grid = stencil_grid(c), blk(ref::BX, ref::BY);
    double* A = F(c, V_C1);
    double* B = F(c, V_C2);
    // x_1
    {
        Prof pf(c, KC_PRECOND, 16.0 * n);
        ref::k_cheb_sweep<<<grid, blk, 0, c->s>>>(q, nullptr, nullptr, k == 1 ? out : A, g, cc,
                                                 0.0, 0.0, 1, st);
    }
    // Sweeps j >= 3 write in place over x_{j-2} (each point reads x_{j-2} only at its own
    // index); x_0 = q*cz is recomputed by sweep 2 instead of stored.
    double* xm1 = A;
    double* xm2 = nullptr;
    for (int j = 2; j <= k; ++j) {
        double* dst = (j == k) ? out : (xm2 ? xm2 : B);
        {
            Prof pf(c, KC_PRECOND, (xm2 ? 32.0 : 24.0) * n);
            ref::k_cheb_sweep<<<grid, blk, 0, c->s>>>(q, xm1, xm2, dst, g, cc, c->rho[j],
                                                     c->rho[j - 1], 0, st);
        }
        xm2 = xm1;
        xm1 = dst;
    }
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

// ------------------------------------------------------------------ one outer iteration
// `from` >= 0: the remainder of an iteration whose reduction stage `from` was parked and has
// been resolved (R19 fallback): only the steps after that stage are enqueued.
bcgs_status iteration_ref(bcgs_ctx c, int from)
{
    const int64_t n = npts(c);
    DevState* st = c->st;
    ref::Grid g = ref_grid(c, (int)c->lay.L);
    dim3 sg = stencil_grid(c), sb(ref::BX, ref::BY);
    const int nsb = (int)(sg.x * sg.y * sg.z);
    if (from == STAGE_RHO) goto a14;
    if (from == STAGE_OMEGA) goto a11;
    if (from == STAGE_ALPHA) goto a6;
    // a2: p̂ = M^-1 p
    TRY(precond_ref(c, F(c, V_P), F(c, V_PH), st));
    // a3: halo p̂
    TRY(halo(c, F(c, V_PH)));
    // a4: w = A p̂, r~ᵀw
    {
        Prof pf(c, KC_STENCIL1, 24.0 * n);
        ref::k_stencil_dot<1><<<sg, sb, 0, c->s>>>(F(c, V_PH), F(c, V_RT), F(c, V_W), g, 0,
                                                  c->part, st);
    }
    // a5: α
    TRY(reduce<1>(c, nsb, STAGE_ALPHA, kStencilDepth, 1, {F(c, V_RT), F(c, V_W)}));
a6:  // a6: s = r - α w
    {
        Prof pf(c, KC_AXPY, 24.0 * n);
        ref::k_axpy_s<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(F(c, V_R), F(c, V_W), n, st);
    }
    // a7: r̂ = M^-1 s
    TRY(precond_ref(c, F(c, V_R), F(c, V_RH), st));
    // a8: halo r̂
    TRY(halo(c, F(c, V_RH)));
    // a9: t = A r̂, tᵀs, tᵀt
    {
        Prof pf(c, KC_STENCIL2, 24.0 * n);
        ref::k_stencil_dot<2><<<sg, sb, 0, c->s>>>(F(c, V_RH), F(c, V_R), F(c, V_T), g, 0,
                                                  c->part, st);
    }
    // a10: ω
    TRY(reduce<2>(c, nsb, STAGE_OMEGA, kStencilDepth, 0,
                  {F(c, V_T), F(c, V_R), F(c, V_T), F(c, V_T)}));   // s = r in place
a11:  // a11 + a12: x, r, r~ᵀr, rᵀr
    {
        Prof pf(c, KC_UPDATE_XR, 64.0 * n);
        ref::k_update_xr<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(
            F(c, V_X), F(c, V_PH), F(c, V_RH), F(c, V_R), F(c, V_T), F(c, V_RT), n, c->part, st);
    }
    // a13: test, ρ, β
    TRY(reduce<2>(c, kEwBlocks, STAGE_RHO, ew_depth(n), 1, {F(c, V_RT), F(c, V_R), F(c, V_R),
                                                         F(c, V_R)}));
a14:  // a14: p = r + β (p - ω w)
    {
        Prof pf(c, KC_UPDATE_P, 32.0 * n);
        ref::k_update_p<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(F(c, V_P), F(c, V_R), F(c, V_W),
                                                                n, st);
    }
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

// ------------------------------------------------------------------ pipelined Bi-CGSTAB
// BCGS_OPT_PIPELINED (pipe.cuh; NEXT-4): library-owned fields z, ẑ, q, q̂, y, v; the
// rest reuse the workspace: p = V_P, p̂ = V_PH, S = V_S, Ŝ = V_P2, r̂ = V_RH, w = V_W,
// ŵ = V_W2, t = V_T.
enum { PZ = 0, PZH = 1, PQ = 2, PQH = 3, PY = 4, PV = 5 };

bcgs_status pipe_alloc(bcgs_ctx c)
{
    if (c->pipe_mem) return BCGS_OK;
    const size_t one = align_up(sizeof(double) * (size_t)c->lay.vec_elems);
    c->pipe_bytes = 6 * one;
    CUDA_OK(c, cudaMalloc(&c->pipe_mem, 6 * one));
    CUDA_OK(c, cudaMemset(c->pipe_mem, 0, 6 * one));   // ghost planes: zero (Dirichlet)
    for (int i = 0; i < 6; ++i) c->pipe[i] = (double*)(c->pipe_mem + i * one) + c->lay.plane;
    return BCGS_OK;
}

bcgs_status pipe_precond(bcgs_ctx c, const double* in, double* out)
{
    if (c->kernels == 1 && fused::precond_supported(c) &&
        !(c->pc == BCGS_PC_CHEB_G && c->nranks > 1))
        return fused::precond_apply(c, in, out, c->st);
    return precond_ref(c, in, out, c->st);
}

bcgs_status pipe_stencil(bcgs_ctx c, double* in, double* out)
{
    TRY(halo(c, in));
    Prof pf(c, KC_STENCIL1, 16.0 * npts(c));
    ref::k_stencil_dot<0><<<stencil_grid(c), dim3(ref::BX, ref::BY), 0, c->s>>>(
        in, nullptr, out, ref_grid(c, (int)c->lay.L), 0, nullptr, c->st);
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

// after the setup stage: r̂ = M^-1 r, w = A r̂, ŵ = M^-1 w, t = A ŵ, α0 = ρ0 / r~ᵀw
bcgs_status pipe_start(bcgs_ctx c)
{
    TRY(pipe_precond(c, F(c, V_R), F(c, V_RH)));
    TRY(pipe_stencil(c, F(c, V_RH), F(c, V_W)));
    TRY(pipe_precond(c, F(c, V_W), F(c, V_W2)));
    TRY(pipe_stencil(c, F(c, V_W2), F(c, V_T)));
    const int64_t n = npts(c);
    ref::k_dot2<1><<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(F(c, V_RT), F(c, V_W), nullptr,
                                                           nullptr, n, c->part);
    CUDA_OK(c, cudaGetLastError());
    return reduce<1>(c, kEwBlocks, STAGE_PIPE_INIT, ew_depth(n), 1, {F(c, V_RT), F(c, V_W)});
}

bcgs_status iteration_pipe(bcgs_ctx c, int from)
{
    const int64_t n = npts(c);
    DevState* st = c->st;
    double** P = c->pipe;
    if (from == STAGE_PIPE_RHO) return BCGS_OK;
    if (from == STAGE_PIPE_OMEGA) goto after_r1;
    {
        Prof pf(c, KC_UPDATE_P, 160.0 * n);
        pbcg::k_pipe_a<<<kEwBlocks, 256, 0, c->s>>>(
            F(c, V_P), F(c, V_PH), F(c, V_S), F(c, V_P2), P[PZ], P[PZH], P[PV], F(c, V_R),
            F(c, V_RH), F(c, V_W), F(c, V_W2), F(c, V_T), P[PQ], P[PQH], P[PY], n, c->part, st);
    }
    CUDA_OK(c, cudaGetLastError());
    TRY(reduce<2>(c, kEwBlocks, STAGE_PIPE_OMEGA, ew_depth(n), 0,
                  {P[PQ], P[PY], P[PY], P[PY]}));   // R1
after_r1:
    TRY(pipe_precond(c, P[PZ], P[PZH]));
    TRY(pipe_stencil(c, P[PZH], P[PV]));
    {
        Prof pf(c, KC_UPDATE_XR, 128.0 * n);
        pbcg::k_pipe_b<<<kEwBlocks, 256, 0, c->s>>>(
            F(c, V_X), F(c, V_R), F(c, V_RH), F(c, V_W), F(c, V_PH), P[PQH], P[PQ], P[PY],
            P[PZH], F(c, V_W2), F(c, V_T), P[PV], F(c, V_RT), F(c, V_S), P[PZ], n, c->part, st);
    }
    CUDA_OK(c, cudaGetLastError());
    TRY(pipe_precond(c, F(c, V_W), F(c, V_W2)));
    TRY(pipe_stencil(c, F(c, V_W2), F(c, V_T)));
    return reduce<5>(c, kEwBlocks, STAGE_PIPE_RHO, ew_depth(n), 15,
                     {F(c, V_RT), F(c, V_R), F(c, V_RT), F(c, V_W), F(c, V_RT), F(c, V_S),
                      F(c, V_RT), P[PZ], F(c, V_R), F(c, V_R)});   // R2
}

// ------------------------------------------------------------------ G(CI) on nranks > 1, fused
// p and s live in the interiors of the extended slabs ext[0] / ext[1] (KG ghost planes per
// side), so each application's k-deep halo (NEXT-1, §7) lands directly in the ghost region
// of the preconditioner's input -- no copy of the input; a14 and a6 run as element-wise
// kernels before it (the neighbours' planes of p / s must exist before the sweeps).
bool g_fused(bcgs_ctx c)
{
    return c->pc == BCGS_PC_CHEB_G && c->nranks > 1 && c->kernels == 1 &&
           c->degree >= 1 && c->degree <= fused::KMAX_TB && c->lay.nx % 2 == 0 && !c->sync2;
}

double* g_interior(bcgs_ctx c, int e) { return c->ext[e] + BCGS_MAX_DEGREE * c->lay.plane; }

bcgs_status g_precond(bcgs_ctx c, int e, double* out)
{
    const int k = c->degree;
    const int64_t L = c->lay.L, KG = BCGS_MAX_DEGREE;
    TRY(halo_deep(c, g_interior(c, e), c->ext[e], k));
    const int v0 = (int)(c->rank == 0 ? KG : KG - k);
    const int v1 = (int)(c->rank == c->nranks - 1 ? KG + L : KG + L + k);
    Prof pf(c, KC_PRECOND, 16.0 * npts(c));
    return fused::precond_g_tb(c, c->ext[e], out, v0, v1, c->st);
}

bcgs_status iteration(bcgs_ctx c, int from)
{
    if (c->pipelined) return iteration_pipe(c, from);
    if (g_fused(c)) return fused::iteration_g(c, from);
    if (c->pc == BCGS_PC_CHEB_G && c->nranks > 1) return iteration_ref(c, from);   // k-deep halos
    if (c->kernels == 1 && fused::supported(c, c->degree, c->pc != BCGS_PC_NONE))
        return fused::iteration(c, from);
    if (c->kernels == 1 && c->pc == BCGS_PC_NONE && c->lay.nx % 2 == 0)
        return fused::iteration_none(c, from);
    return iteration_ref(c, from);
}

bcgs_status enqueue_iterations(bcgs_ctx c, int n)
{
    // graphs: single rank only (multi-rank runs launch directly; NCCL inside captured graphs
    // is supported but not exercised in round 1)
    // (inner-Krylov preconditioners synchronise the host inside an iteration: no graph)
    // graphs: one rank, or the p2p transport (kernels only); NCCL with BCGS_OPT_GRAPH = 2
    // (not for in-process p2p groups: instantiating a graph can wait for the device, i.e.
    // for another rank's kernel that spins on this rank -- a stall until the timeout)
    const bool graph_ok = c->nranks == 1 || (c->p2p && !c->inproc) || (c->comm && c->use_graph == 2);
    if (c->use_graph && graph_ok && !c->profile && !c->lg && !inner_pc(c)) {
        if (!c->gexec) {
            cudaGraph_t graph;
            CUDA_OK(c, cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
            bcgs_status st = iteration(c, -1);
            cudaError_t e = cudaStreamEndCapture(c->s, &graph);
            if (st != BCGS_OK) return st;
            CUDA_OK(c, e);
            CUDA_OK(c, cudaGraphInstantiate(&c->gexec, graph, 0));
            c->graph_key = c->sync2 | (c->pipelined << 1);
            cudaGraphDestroy(graph);
        }
        for (int i = 0; i < n; ++i) CUDA_OK(c, cudaGraphLaunch(c->gexec, c->s));
        return BCGS_OK;
    }
    for (int i = 0; i < n; ++i) TRY(iteration(c, -1));
    return BCGS_OK;
}

// destroy the private inner-solver contexts of BJ(BiCGS) / G(BiCGS) and free their memory
void drop_inner(bcgs_ctx c)
{
    for (size_t k = 0; k < c->inner.size(); ++k) {
        if (c->inner[k]) bcgs_destroy(c->inner[k]);
        if (c->inner_ws[k]) cudaFree(c->inner_ws[k]);
    }
    c->inner.clear();
    c->inner_ws.clear();
}

void drop_graph(bcgs_ctx c)
{
    if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
}

// caller stream -> private stream
bcgs_status enter(bcgs_ctx c)
{
    CUDA_OK(c, cudaSetDevice(c->device));
    CUDA_OK(c, cudaEventRecord(c->join, c->user));
    CUDA_OK(c, cudaStreamWaitEvent(c->s, c->join, 0));
    return BCGS_OK;
}

// private stream -> caller stream
bcgs_status leave(bcgs_ctx c)
{
    CUDA_OK(c, cudaEventRecord(c->join, c->s));
    CUDA_OK(c, cudaStreamWaitEvent(c->user, c->join, 0));
    return BCGS_OK;
}

bcgs_status copy_in(bcgs_ctx c, double* dst, const double* src, int32_t mem)
{
    const size_t bytes = sizeof(double) * (size_t)npts(c);
    CUDA_OK(c, cudaMemcpyAsync(dst, src, bytes,
                               mem == BCGS_MEM_HOST ? cudaMemcpyHostToDevice
                                                    : cudaMemcpyDeviceToDevice,
                               c->s));
    if (mem == BCGS_MEM_HOST) CUDA_OK(c, cudaStreamSynchronize(c->s));
    return BCGS_OK;
}

bcgs_status fold_faces(bcgs_ctx c)
{
    int mask = 0;
    double add[6];
    for (int f = 0; f < 6; ++f) {
        // R15 Dirichlet value g -> g/h²; R28 Neumann outward derivative g -> 2g/h
        add[f] = c->bc[f] ? (2.0 * c->face[f]) / c->h : c->face[f] * c->h2inv;
        if (c->face[f] != 0.0) mask |= 1 << f;
    }
    if (!mask) return BCGS_OK;
    ref::k_fold_boundary<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(
        F(c, V_B), ref_grid(c, (int)c->lay.L), c->rank * c->lay.L, c->lay.nz, add[0], add[1],
        add[2], add[3], add[4], add[5], mask);
    CUDA_OK(c, cudaGetLastError());
    return BCGS_OK;
}

bcgs_status validate_pc(bcgs_ctx c)
{
    bcgs_grid_desc g{{c->lay.nx, c->lay.ny, c->lay.nz}, c->h, {0, 0, 0, 0, 0, 0}};
    memcpy(g.bc, c->bc, sizeof g.bc);
    if (c->pc == BCGS_PC_NONE || inner_pc(c)) return BCGS_OK;
    bcgs_status s = cheb_constants(&g, c->nranks * c->bpr, c->pc, c->degree, c->c_min, c->c_max,
                                   c->ov_a, c->ov_b, c->ivl, c->cst, c->rho);
    if (s != BCGS_OK)
        return fail(c, s, "Chebyshev interval invalid (a'=%g, b'=%g, k=%d)", c->ivl[0],
                    c->ivl[1], c->degree);
    return BCGS_OK;
}

}  // namespace

#include "fused_launch.h"
#include "fused_driver.cuh"

// =================================================================== C ABI
extern "C" {

int32_t bcgs_abi_version(void) { return BCGS_ABI_VERSION; }

const char* bcgs_status_string(bcgs_status s)
{
    switch (s) {
    case BCGS_OK: return "ok";
    case BCGS_E_INVALID: return "invalid argument";
    case BCGS_E_CONFIG: return "configuration error";
    case BCGS_E_SPECTRUM: return "invalid Chebyshev interval";
    case BCGS_E_CUDA: return "CUDA error";
    case BCGS_E_NCCL: return "NCCL error";
    case BCGS_NOT_CONVERGED: return "not converged";
    case BCGS_BREAKDOWN: return "breakdown";
    case BCGS_E_STATE: return "call out of order";
    case BCGS_E_COMM: return "peer transport error (timeout)";
    }
    return "unknown";
}

size_t bcgs_workspace_bytes(const bcgs_grid_desc* grid, int32_t nranks)
{
    Layout lay;
    if (!make_layout(grid, nranks, &lay)) return 0;
    return lay.total;
}

bcgs_status bcgs_chebyshev_constants(const bcgs_grid_desc* grid, int32_t nslab, bcgs_pc pc,
                                     int32_t degree, double c_min, double c_max,
                                     double* interval2, double* out7, double* rho)
{
    if (!grid || nslab < 1 || grid->n[2] % nslab || !interval2 || !out7 || !rho)
        return BCGS_E_INVALID;
    if (!bc_ok(grid)) return BCGS_E_CONFIG;
    if ((grid->bc[4] || grid->bc[5]) && pc != BCGS_PC_CHEB_G && grid->n[2] / nslab < 2)
        return BCGS_E_CONFIG;
    if (pc != BCGS_PC_CHEB_GNOCOMM && pc != BCGS_PC_CHEB_BJ && pc != BCGS_PC_CHEB_G)
        return BCGS_E_INVALID;
    return cheb_constants(grid, nslab, pc, degree, c_min, c_max, 0.0, 0.0, interval2, out7, rho);
}

bcgs_status bcgs_nccl_unique_id(void* out128)
{
    if (!out128) return BCGS_E_INVALID;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return BCGS_E_NCCL;
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    memcpy(out128, &id, sizeof id);
    return BCGS_OK;
}

static bcgs_status create_ctx(const bcgs_grid_desc* grid, int32_t rank, int32_t nranks,
                              const void* nccl_unique_id, LocalGroup* lg, int32_t cuda_device,
                              void* d_workspace, size_t ws_bytes, void* cuda_stream,
                              bcgs_ctx* out, int p2p = 0, bcgs_ctx share = nullptr)
{
    // share: a context over the same ranks that uses `share`'s transport (the NCCL
    // communicator, or the p2p mailboxes with their sequence numbers) -- the global inner
    // solver of G(BiCGS) on nranks > 1
    if (!grid || !out || nranks < 1 || rank < 0 || rank >= nranks) return BCGS_E_INVALID;
    if (!(grid->h > 0.0)) return BCGS_E_INVALID;
    if (nranks > 1 && !nccl_unique_id && !lg && !p2p && !share) return BCGS_E_INVALID;
    if (p2p && (nranks < 2 || nranks > p2p::MAXR)) return BCGS_E_INVALID;
    if (!bc_ok(grid)) return BCGS_E_CONFIG;
    Layout lay;
    if (!make_layout(grid, nranks, &lay)) return BCGS_E_CONFIG;
    if (lay.nx > (1 << 30) || lay.ny > (1 << 30)) return BCGS_E_CONFIG;
    if (!d_workspace || ws_bytes < lay.total || ((uintptr_t)d_workspace % kAlign))
        return BCGS_E_INVALID;
    bcgs_ctx c = new bcgs_ctx_s();
    c->lay = lay;
    c->h = grid->h;
    c->h2inv = 1.0 / (grid->h * grid->h);
    memcpy(c->bc, grid->bc, sizeof c->bc);
    c->mbc.m = (grid->bc[0] ? 1 : 0) | (grid->bc[1] ? 2 : 0) | (grid->bc[2] ? 4 : 0) |
               (grid->bc[3] ? 8 : 0);
    c->mbc.zlo = (rank == 0 && grid->bc[4]) ? 0 : -1;
    c->mbc.zhi = (rank == nranks - 1 && grid->bc[5]) ? (int)lay.L - 1 : -1;
    c->rank = rank;
    c->nranks = nranks;
    c->device = cuda_device;
    c->user = (cudaStream_t)cuda_stream;
    c->ws = (char*)d_workspace;
    c->lg = lg;
    *out = c;
    CUDA_OK(c, cudaSetDevice(cuda_device));
    int prio_lo = 0, prio_hi = 0;
    CUDA_OK(c, cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CUDA_OK(c, cudaStreamCreateWithPriority(&c->s, cudaStreamNonBlocking, prio_hi));
    CUDA_OK(c, cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
    CUDA_OK(c, cudaMallocHost(&c->h_pinned, 64));
    if (nranks > 1) {
        CUDA_OK(c, cudaStreamCreateWithFlags(&c->s_comm, cudaStreamNonBlocking));
        CUDA_OK(c, cudaEventCreateWithFlags(&c->ev_pre, cudaEventDisableTiming));
        CUDA_OK(c, cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
    }
    if (lg) {
        CUDA_OK(c, cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
        CUDA_OK(c, cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
    }
    for (int v = 0; v < V_COUNT; ++v)
        c->vec[v] = (double*)(c->ws + lay.off_vec[v]) + lay.plane;
    for (int e = 0; e < 3; ++e)
        c->ext[e] = lay.ext_elems ? (double*)(c->ws + lay.off_ext[e]) + lay.plane : nullptr;
    c->st = (DevState*)(c->ws + lay.off_state);
    c->hist = (double*)(c->ws + lay.off_hist);
    c->scal = (double*)(c->ws + lay.off_scal);
    c->part = (dd*)(c->ws + lay.off_part);
    c->rank_out = (dd*)(c->ws + lay.off_rank);
    c->gath = (dd*)(c->ws + lay.off_gath);
    c->limbs = (long long*)(c->ws + lay.off_limb);
    c->glimbs = (long long*)(c->ws + lay.off_glimb);
    if (share) {
        c->comm = share->comm;
        c->comm_borrowed = 1;
        c->p2p = share->p2p;
        c->p2p_ready = share->p2p_ready;
        c->peers = share->peers;
        c->inproc = share->inproc;
    } else if (p2p) {   // mailbox + landing zones (face halos; G(CI) k-deep halos <= `cap`)
        c->p2p = 1;
        c->peers.rank = rank;
        c->peers.nranks = nranks;
        c->peers.plane = lay.plane;
        c->peers.cap = std::min<int64_t>(lay.L, 16);
        c->peers.timeout_ns = 60ull * 1000000000ull;
        c->mailbox_bytes = p2p::land_offset() +
                           sizeof(double) * 4 * (size_t)c->peers.cap * (size_t)lay.plane;
        CUDA_OK(c, cudaMalloc(&c->mailbox, c->mailbox_bytes));
        CUDA_OK(c, cudaMemset(c->mailbox, 0, c->mailbox_bytes));
        c->peers.mb[rank] = (p2p::Mailbox*)c->mailbox;
        c->peers.land[rank] = (double*)(c->mailbox + p2p::land_offset());
    }
    TRY(enter(c));
    CUDA_OK(c, cudaMemsetAsync(c->ws, 0, lay.total, c->s));   // zero ghost planes + state
    // nranks == 1 with an id: a 1-rank communicator whose all-gathers carry the reductions
    // (the NCCL code path on one GPU, for testing)
    if ((nranks > 1 || nccl_unique_id) && !lg && !p2p && !share) {
        ncclUniqueId id;
        memcpy(&id, nccl_unique_id, sizeof id);
        NCCL_OK(c, ncclCommInitRank(&c->comm, nranks, id, rank));
    }
    TRY(leave(c));
    if (lg) CUDA_OK(c, cudaStreamSynchronize(c->s));
    return BCGS_OK;
}

bcgs_status bcgs_create(const bcgs_grid_desc* grid, int32_t rank, int32_t nranks,
                        const void* nccl_unique_id, int32_t cuda_device, void* d_workspace,
                        size_t ws_bytes, void* cuda_stream, bcgs_ctx* out)
{
    return create_ctx(grid, rank, nranks, nccl_unique_id, nullptr, cuda_device, d_workspace,
                      ws_bytes, cuda_stream, out);
}

bcgs_status bcgs_create_p2p(const bcgs_grid_desc* grid, int32_t rank, int32_t nranks,
                            int32_t cuda_device, void* d_workspace, size_t ws_bytes,
                            void* cuda_stream, bcgs_ctx* out)
{
    return create_ctx(grid, rank, nranks, nullptr, nullptr, cuda_device, d_workspace, ws_bytes,
                      cuda_stream, out, 1);
}

// 128-byte record: [0, 64) cudaIpcMemHandle_t of the mailbox, then magic, rank, nranks, pid,
// mailbox bytes (int64 each)
bcgs_status bcgs_p2p_handle(bcgs_ctx c, void* out128)
{
    if (!c || !out128 || !c->p2p) return BCGS_E_INVALID;
    CUDA_OK(c, cudaSetDevice(c->device));
    cudaIpcMemHandle_t h;
    CUDA_OK(c, cudaIpcGetMemHandle(&h, c->mailbox));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
    char* o = (char*)out128;
    memset(o, 0, 128);
    memcpy(o, &h, 64);
    const int64_t rec[5] = {0x6263677332703270ll, c->rank, c->nranks, (int64_t)getpid(),
                            (int64_t)c->mailbox_bytes};
    memcpy(o + 64, rec, sizeof rec);
    return BCGS_OK;
}

bcgs_status bcgs_p2p_connect(bcgs_ctx c, const void* all_handles)
{
    if (!c || !all_handles || !c->p2p) return BCGS_E_INVALID;
    if (c->p2p_ready) return fail(c, BCGS_E_STATE, "p2p transport already connected");
    CUDA_OK(c, cudaSetDevice(c->device));
    const char* in = (const char*)all_handles;
    for (int r = 0; r < c->nranks; ++r) {
        int64_t rec[5];
        memcpy(rec, in + 128 * r + 64, sizeof rec);
        if (rec[0] != 0x6263677332703270ll || rec[1] != r || rec[2] != c->nranks ||
            rec[4] != (int64_t)c->mailbox_bytes)
            return fail(c, BCGS_E_INVALID, "p2p handle %d: wrong record (rank %lld of %lld)", r,
                        (long long)rec[1], (long long)rec[2]);
        if (r == c->rank) continue;
        if (rec[3] == (int64_t)getpid())
            return fail(c, BCGS_E_CONFIG, "p2p peer %d is in this process: use "
                        "bcgs_create_local_p2p", r);
        cudaIpcMemHandle_t h;
        memcpy(&h, in + 128 * r, 64);
        void* p = nullptr;
        CUDA_OK(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(p);
        c->peers.mb[r] = (p2p::Mailbox*)p;
        c->peers.land[r] = (double*)((char*)p + p2p::land_offset());
    }
    c->p2p_ready = 1;
    return BCGS_OK;
}

bcgs_status bcgs_create_local_p2p(const bcgs_grid_desc* grid, int32_t nranks,
                                  int32_t cuda_device, void* const* d_workspaces,
                                  size_t ws_bytes, void* cuda_stream, bcgs_ctx* outs)
{
    if (!grid || !outs || !d_workspaces || nranks < 2 || nranks > p2p::MAXR)
        return BCGS_E_INVALID;
    for (int r = 0; r < nranks; ++r) {
        bcgs_status st = create_ctx(grid, r, nranks, nullptr, nullptr, cuda_device,
                                    d_workspaces[r], ws_bytes, cuda_stream, &outs[r], 1);
        if (st != BCGS_OK) return st;
    }
    for (int r = 0; r < nranks; ++r) {   // same process: the peers' pointers directly
        for (int q = 0; q < nranks; ++q) {
            outs[r]->peers.mb[q] = outs[q]->peers.mb[q];
            outs[r]->peers.land[q] = outs[q]->peers.land[q];
        }
        outs[r]->p2p_ready = 1;
        outs[r]->inproc = 1;
    }
    return BCGS_OK;
}

bcgs_status bcgs_create_local(const bcgs_grid_desc* grid, int32_t nranks, int32_t cuda_device,
                              void* const* d_workspaces, size_t ws_bytes, void* cuda_stream,
                              bcgs_ctx* outs)
{
    if (!grid || !outs || !d_workspaces || nranks < 2) return BCGS_E_INVALID;
    LocalGroup* lg = new LocalGroup();
    lg->n = nranks;
    lg->bar.n = nranks;
    lg->ctxs.assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
        bcgs_status st = create_ctx(grid, r, nranks, nullptr, lg, cuda_device, d_workspaces[r],
                                    ws_bytes, cuda_stream, &outs[r]);
        if (st != BCGS_OK) return st;
        lg->ctxs[r] = outs[r];
    }
    return BCGS_OK;
}

void bcgs_destroy(bcgs_ctx c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->s) cudaStreamSynchronize(c->s);
    drop_inner(c);
    harvest(c);
    drop_graph(c);
    for (auto e : c->free_ev) cudaEventDestroy(e);
    if (c->comm && !c->comm_borrowed) ncclCommDestroy(c->comm);
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    if (c->mailbox) cudaFree(c->mailbox);
    if (c->pipe_mem) cudaFree(c->pipe_mem);
    if (c->ev_ready) cudaEventDestroy(c->ev_ready);
    if (c->ev_pre) cudaEventDestroy(c->ev_pre);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    if (c->s_comm) cudaStreamDestroy(c->s_comm);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    if (c->lg) {
        bool last = true;
        for (auto& p : c->lg->ctxs) {
            if (p == c) p = nullptr;
            if (p) last = false;
        }
        if (last) delete c->lg;
    }
    if (c->join) cudaEventDestroy(c->join);
    if (c->s) cudaStreamDestroy(c->s);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    delete c;
}

const char* bcgs_last_error(bcgs_ctx c) { return c ? c->err.c_str() : "null context"; }

bcgs_status bcgs_set_option(bcgs_ctx c, int32_t option, int64_t value)
{
    if (!c) return BCGS_E_INVALID;
    switch (option) {
    case BCGS_OPT_KERNELS: c->kernels = (int)value; break;
    case BCGS_OPT_GRAPH: c->use_graph = (int)value; break;
    // profiled iterations never replay the graph and polling is host-side: the captured
    // iteration stays valid (bench.py times graph replays right after switching these)
    case BCGS_OPT_PROFILE: c->profile = (int)value; return BCGS_OK;
    case BCGS_OPT_POLL: c->poll = std::max<int>(1, (int)value); return BCGS_OK;
    case BCGS_OPT_TB_VARIANT:
        if (value != 2 && value != 7)
            return fail(c, BCGS_E_INVALID, "temporally blocked layout %lld: 2 or 7",
                        (long long)value);
        c->tb_variant = (int)value;
        break;
    case BCGS_OPT_MULTIPASS: c->mp_min = std::max<int>(4, (int)value); break;
    case BCGS_OPT_ABLATE: c->ablate = (int)(value & 3); break;
    case BCGS_OPT_SYNC2: c->sync2_opt = (int)value; drop_graph(c); break;
    case BCGS_OPT_EXACT_DOT: c->exact_opt = value ? 1 : 0; break;
    case BCGS_OPT_PDL: c->pdl = value ? 1 : 0; break;
    case BCGS_OPT_TB_SCHEDULE:
        if (value < 0 || value > 2) return fail(c, BCGS_E_INVALID, "tb schedule %lld: 0..2", (long long)value);
        c->tb_schedule = (int)value;
        break;
    case BCGS_OPT_STENCIL:
        // planes per CTA <= 64: the certification bound of the stencil dots (kStencilDepth,
        // R19) covers per-thread chains of 2 products per plane over at most 64 planes
        if (value < 0 || value > 64) return fail(c, BCGS_E_INVALID, "stencil option %lld: 0..64", (long long)value);
        c->stencil_tma = (int)value;
        break;
    case BCGS_OPT_PIPELINED:   // allocate now (an allocation synchronises the device)
        c->pipelined_opt = value ? 1 : 0;
        if (c->pipelined_opt) TRY(pipe_alloc(c));
        break;
    case BCGS_OPT_COMM_TIMEOUT:   // NCCL host waits; p2p device waits (default 60 s)
        c->comm_timeout_s = value > 0 ? (double)value : 300.0;
        c->peers.timeout_ns = (value > 0 ? (unsigned long long)value : 60ull) * 1000000000ull;
        break;
    default: return fail(c, BCGS_E_INVALID, "unknown option %d", option);
    }
    drop_graph(c);
    return BCGS_OK;
}

bcgs_status bcgs_set_rhs_random(bcgs_ctx c, uint64_t seed)
{
    if (!c) return BCGS_E_INVALID;
    TRY(enter(c));
    ref::k_rhs_random<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(
        F(c, V_B), npts(c), (int64_t)c->rank * npts(c), seed);
    CUDA_OK(c, cudaGetLastError());
    TRY(fold_faces(c));
    c->begun = 0;
    return leave(c);
}

bcgs_status bcgs_set_rhs(bcgs_ctx c, const double* f, int32_t mem)
{
    if (!c || !f) return BCGS_E_INVALID;
    TRY(enter(c));
    TRY(copy_in(c, F(c, V_B), f, mem));
    TRY(fold_faces(c));
    c->begun = 0;
    return leave(c);
}

bcgs_status bcgs_set_boundary_value(bcgs_ctx c, int32_t face, double value)
{
    if (!c || face < 0 || face > 5 || !std::isfinite(value)) return BCGS_E_INVALID;
    c->face[face] = value;
    return BCGS_OK;
}

bcgs_status bcgs_set_initial_guess(bcgs_ctx c, const double* x0, int32_t mem)
{
    if (!c) return BCGS_E_INVALID;
    if (!x0) {
        c->have_x0 = 0;
        return BCGS_OK;
    }
    TRY(enter(c));
    TRY(copy_in(c, F(c, V_X), x0, mem));
    c->have_x0 = 1;
    c->begun = 0;
    return leave(c);
}

bcgs_status bcgs_set_preconditioner(bcgs_ctx c, bcgs_pc pc, int32_t degree, double c_min,
                                    double c_max, int32_t blocks_per_rank)
{
    if (!c) return BCGS_E_INVALID;
    if (pc != BCGS_PC_NONE && pc != BCGS_PC_CHEB_GNOCOMM && pc != BCGS_PC_CHEB_BJ &&
        pc != BCGS_PC_CHEB_G && pc != BCGS_PC_BJ_BICGS && pc != BCGS_PC_G_BICGS)
        return fail(c, BCGS_E_INVALID, "unknown preconditioner %d", (int)pc);
    drop_inner(c);
    if (pc == BCGS_PC_BJ_BICGS || pc == BCGS_PC_G_BICGS) {   // P:393-394 defaults
        if (pc == BCGS_PC_G_BICGS && c->lg)
            return fail(c, BCGS_E_CONFIG, "G(BiCGS) across ranks needs the NCCL or p2p "
                        "transport (not the in-process copy transport)");
        degree = 0;
        c->in_tol = pc == BCGS_PC_G_BICGS ? 1e-2 : 1e-6;
        c->in_max = 500;
    }
    if (degree < 0 || degree > BCGS_MAX_DEGREE)
        return fail(c, BCGS_E_INVALID, "degree %d outside [0, %d]", degree, BCGS_MAX_DEGREE);
    if (blocks_per_rank < 1 || c->lay.L % blocks_per_rank)
        return fail(c, BCGS_E_CONFIG, "slab of %lld planes not divisible into %d blocks (axis z)",
                    (long long)c->lay.L, blocks_per_rank);
    if ((c->bc[4] || c->bc[5]) && pc != BCGS_PC_CHEB_G && c->lay.L / blocks_per_rank < 2)
        return fail(c, BCGS_E_CONFIG, "a Neumann z face needs >= 2 planes per block");
    if (pc == BCGS_PC_CHEB_G || pc == BCGS_PC_G_BICGS) {
        blocks_per_rank = 1;   // the global operator has no block cuts
        if (c->nranks > 1 && degree > c->lay.L)
            return fail(c, BCGS_E_CONFIG, "G(CI) needs degree %d <= slab thickness %lld",
                        degree, (long long)c->lay.L);
    }
    c->pc = pc;
    c->degree = degree;
    c->c_min = c_min;
    c->c_max = c_max;
    c->bpr = blocks_per_rank;
    drop_graph(c);
    c->begun = 0;
    TRY(validate_pc(c));
    // inner-Krylov preconditioners: create the private block contexts now, not inside the
    // first solve -- their allocations synchronise the device, which must not happen while
    // ranks sharing the GPU (in-process groups) are in a peer exchange
    if (inner_pc(c)) TRY(inner_all(c));
    return BCGS_OK;
}

bcgs_status bcgs_set_inner_solver(bcgs_ctx c, double rel_tol, int32_t max_iter)
{
    if (!c) return BCGS_E_INVALID;
    if (!(rel_tol > 0.0) || max_iter < 1 || max_iter > BCGS_HIST_CAP)
        return fail(c, BCGS_E_INVALID, "inner solver: need tol > 0, 1 <= max_iter <= %d",
                    BCGS_HIST_CAP);
    c->in_tol = rel_tol;
    c->in_max = max_iter;
    return BCGS_OK;
}

int64_t bcgs_inner_iterations(bcgs_ctx c) { return c ? c->in_iters : -1; }

bcgs_status bcgs_certification_info(bcgs_ctx c, double* out9)
{
    if (!c || !out9) return BCGS_E_INVALID;
    CUDA_OK(c, cudaStreamSynchronize(c->s));
    CUDA_OK(c, cudaMemcpy(out9, c->st->cert_last, 9 * sizeof(double), cudaMemcpyDeviceToHost));
    int32_t nref = 0;
    CUDA_OK(c, cudaMemcpy(&nref, &c->st->n_refused, sizeof nref, cudaMemcpyDeviceToHost));
    out9[9] = nref;
    return BCGS_OK;
}

int32_t bcgs_exact_dots(bcgs_ctx c)
{
    if (!c) return -1;
    int32_t v = -1;
    if (cudaStreamSynchronize(c->s) != cudaSuccess ||
        cudaMemcpy(&v, &c->st->n_exact, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    return v;
}

bcgs_status bcgs_set_eigen_bounds(bcgs_ctx c, double a, double b)
{
    if (!c) return BCGS_E_INVALID;
    if (!(a == 0.0 && b == 0.0) && !(a > 0.0 && a < b))
        return fail(c, BCGS_E_SPECTRUM, "need 0 < a < b (got %g, %g)", a, b);
    c->ov_a = a;
    c->ov_b = b;
    drop_graph(c);
    return validate_pc(c);
}

bcgs_status bcgs_begin(bcgs_ctx c, double rel_tol, int32_t max_iter, int32_t fixed_iters)
{
    if (!c) return BCGS_E_INVALID;
    if (fixed_iters < 0 || fixed_iters > BCGS_HIST_CAP || max_iter < 0 ||
        (fixed_iters == 0 && (max_iter < 1 || max_iter > BCGS_HIST_CAP)))
        return fail(c, BCGS_E_INVALID, "iteration counts out of range (cap %d)", BCGS_HIST_CAP);
    c->begun = 0;   // a failed begin leaves no solve to iterate
    // configuration checks first: no device work on a configuration error
    TRY(validate_pc(c));
    if (c->sync2_opt &&   // R31 is built on the fused path (vectorised streaming kernels)
        !(c->kernels == 1 && fused::supported(c, c->degree, c->pc != BCGS_PC_NONE) &&
          c->lay.nx % 2 == 0 && !(c->pc == BCGS_PC_CHEB_G && c->nranks > 1)))
        return fail(c, BCGS_E_CONFIG, "BCGS_OPT_SYNC2 needs the fused path (kernels = 1, a "
                    "Chebyshev preconditioner, even nx)");
    if (c->pipelined_opt && (inner_pc(c) || c->sync2_opt))
        return fail(c, BCGS_E_CONFIG, "BCGS_OPT_PIPELINED needs a linear preconditioner "
                    "(none / Chebyshev) and excludes BCGS_OPT_SYNC2");
    if (c->pipelined_opt) TRY(pipe_alloc(c));
    TRY(enter(c));
    c->t0 = std::chrono::steady_clock::now();
    const int64_t n = npts(c);
    const size_t bytes = sizeof(double) * (size_t)n;
    k_init_state<<<1, 1, 0, c->s>>>(c->st, rel_tol, max_iter, fixed_iters, c->exact_opt);
    c->in_iters = 0;
    c->sync2 = c->sync2_opt ? 1 : 0;
    c->pipelined = c->pipelined_opt;
    // the captured iteration depends on the algorithm variant (not on the solve: fields,
    // scalars and the stop test live on the device), so repeated solves replay it
    if (c->graph_key != (c->sync2 | (c->pipelined << 1))) drop_graph(c);
    // Alg. 3 l.1-4: r0 = b - A x0; r~ = r0; p0 = r0; ρ0 = r~ᵀr0.  The initial
    // guess set by bcgs_set_initial_guess applies to this solve only (V_X then holds the
    // iterate); later solves start from x0 = 0 unless a new guess is set (R21).
    const bool x0 = c->have_x0;
    c->have_x0 = 0;
    if (x0) {
        TRY(halo_api(c, F(c, V_X)));
        ref::k_stencil_dot<0><<<stencil_grid(c), dim3(ref::BX, ref::BY), 0, c->s>>>(
            F(c, V_X), nullptr, F(c, V_R), ref_grid(c, (int)c->lay.L), 0, nullptr, nullptr);
        ref::k_residual0<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(F(c, V_B), F(c, V_R), n);
    } else {
        CUDA_OK(c, cudaMemsetAsync(F(c, V_X), 0, bytes, c->s));
        CUDA_OK(c, cudaMemcpyAsync(F(c, V_R), F(c, V_B), bytes, cudaMemcpyDeviceToDevice, c->s));
    }
    CUDA_OK(c, cudaMemcpyAsync(F(c, V_RT), F(c, V_R), bytes, cudaMemcpyDeviceToDevice, c->s));
    CUDA_OK(c, cudaMemcpyAsync(F(c, V_P), F(c, V_R), bytes, cudaMemcpyDeviceToDevice, c->s));
    if (g_fused(c))   // fused G(CI) on nranks > 1: p lives in the extended slab's interior
        CUDA_OK(c, cudaMemcpyAsync(g_interior(c, 0), F(c, V_R), bytes, cudaMemcpyDeviceToDevice,
                                   c->s));
    ref::k_dot2<2><<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(F(c, V_B), F(c, V_B), F(c, V_RT),
                                                           F(c, V_R), n, c->part);
    CUDA_OK(c, cudaGetLastError());
    TRY(reduce<2>(c, kEwBlocks, STAGE_SETUP, ew_depth(n), 3,
                  {F(c, V_B), F(c, V_B), F(c, V_RT), F(c, V_R)}));
    if (c->pipelined) {   // recurrence vectors start at 0 (β = ω = 0: p0 = r0, S0 = w0, ...)
        const size_t vb = sizeof(double) * (size_t)n;
        for (int v : {V_P, V_PH, V_S, V_P2}) CUDA_OK(c, cudaMemsetAsync(F(c, v), 0, vb, c->s));
        for (int i : {PZ, PZH, PV}) CUDA_OK(c, cudaMemsetAsync(c->pipe[i], 0, vb, c->s));
        TRY(pipe_start(c));
    }
    c->begun = 1;
    c->launched = 0;
    c->fixed = fixed_iters;
    c->max_iter = max_iter;
    c->tol = rel_tol;
    return BCGS_OK;
}

bcgs_status bcgs_iterate(bcgs_ctx c, int32_t n)
{
    if (!c || n < 0) return BCGS_E_INVALID;
    if (!c->begun) return fail(c, BCGS_E_STATE, "bcgs_iterate before bcgs_begin");
    TRY(enter(c));   // ordered after prior work on the caller's stream
    TRY(enqueue_iterations(c, n));
    c->launched += n;
    return BCGS_OK;
}

bcgs_status bcgs_join(bcgs_ctx c)
{
    if (!c) return BCGS_E_INVALID;
    return leave(c);
}

static bcgs_status read_state(bcgs_ctx c, int32_t* done, int32_t* iter)
{
    CUDA_OK(c, cudaMemcpyAsync(c->h_pinned, &c->st->iter, 2 * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, c->s));
    TRY(sync_stream(c));
    *iter = ((int32_t*)c->h_pinned)[0];
    *done = ((int32_t*)c->h_pinned)[1];
    if (*done == DONE_COMM_ERROR)
        return fail(c, BCGS_E_COMM, "p2p transport: a peer did not answer within the timeout");
    return BCGS_OK;
}

// Poll the device state; a parked reduction (DONE_PENDING, R19) is resolved exactly, the
// interrupted iteration completed and the iterations enqueued after it (device no-ops while
// parked) enqueued again.  Every rank sees the same parked stage (the certification runs
// on identical combined values), so the collectives of the resolution match across ranks.
static bcgs_status poll_state(bcgs_ctx c, int32_t* done, int32_t* iter)
{
    TRY(read_state(c, done, iter));
    while (*done == DONE_PENDING) {
        int stage;
        TRY(resolve(c, &stage));
        if (stage < 0) return fail(c, BCGS_E_STATE, "parked solve without a parked stage");
        if (stage == STAGE_SETUP && c->pipelined) TRY(pipe_start(c));
        else if (stage != STAGE_SETUP && stage != STAGE_PIPE_INIT) TRY(iteration(c, stage));
        TRY(read_state(c, done, iter));
        if (*done == DONE_RUNNING && c->launched > *iter) {
            TRY(enqueue_iterations(c, c->launched - *iter));
            TRY(read_state(c, done, iter));
        }
    }
    return BCGS_OK;
}

bcgs_status bcgs_finish(bcgs_ctx c, bcgs_report* out)
{
    if (!c) return BCGS_E_INVALID;
    if (!c->begun) return fail(c, BCGS_E_STATE, "bcgs_finish before bcgs_begin");
    int32_t done = 0, iter = 0;
    TRY(poll_state(c, &done, &iter));
    // true residual (R22): ||b - A x|| / ||b||, once
    double true_rel = NAN, rel = NAN;
    {
        TRY(halo_api(c, F(c, V_X)));
        ref::k_stencil_dot<0><<<stencil_grid(c), dim3(ref::BX, ref::BY), 0, c->s>>>(
            F(c, V_X), nullptr, F(c, V_IO), ref_grid(c, (int)c->lay.L), 0, nullptr, nullptr);
        ref::k_residual0<<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(F(c, V_B), F(c, V_IO), npts(c));
        ref::k_dot2<1><<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(F(c, V_IO), F(c, V_IO), nullptr,
                                                               nullptr, npts(c), c->part);
        TRY(reduce<1>(c, kEwBlocks, STAGE_DOT, ew_depth(npts(c)), 1, {F(c, V_IO), F(c, V_IO)}));
        int stg;
        TRY(resolve(c, &stg));
        double h[2];
        CUDA_OK(c, cudaMemcpyAsync(h, c->st->scratch, sizeof h, cudaMemcpyDeviceToHost, c->s));
        double nbv;
        CUDA_OK(c, cudaMemcpyAsync(&nbv, &c->st->nb, sizeof nbv, cudaMemcpyDeviceToHost, c->s));
        CUDA_OK(c, cudaMemcpyAsync(&rel, &c->st->rel, sizeof rel, cudaMemcpyDeviceToHost, c->s));
        CUDA_OK(c, cudaStreamSynchronize(c->s));
        true_rel = nbv == 0.0 ? 0.0 : sqrt(h[0]) / nbv;
    }
    harvest(c);
    TRY(leave(c));
    bcgs_status s = BCGS_OK;
    if (done == DONE_BREAKDOWN) s = BCGS_BREAKDOWN;
    else if (done == DONE_MAXIT || done == DONE_RUNNING) s = BCGS_NOT_CONVERGED;
    if (out) {
        out->status = s;
        out->converged = (done == DONE_OK);
        out->iterations = iter;
        int64_t Lb = c->lay.L / c->bpr;
        out->degree_warning = (c->pc != BCGS_PC_NONE && 2 * (int64_t)c->degree > Lb) ? 1 : 0;
        out->rel_residual = rel;
        out->true_rel_residual = true_rel;
        out->seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - c->t0).count();
    }
    return s;
}

bcgs_status bcgs_solve(bcgs_ctx c, double rel_tol, int32_t max_iter, int32_t fixed_iters,
                       bcgs_report* out)
{
    TRY(bcgs_begin(c, rel_tol, max_iter, fixed_iters));
    if (fixed_iters > 0) {
        TRY(bcgs_iterate(c, fixed_iters));
    } else {
        int32_t done = 0, iter = 0;
        TRY(poll_state(c, &done, &iter));
        while (done == DONE_RUNNING && c->launched < max_iter) {
            int batch = std::min(inner_pc(c) ? 1 : c->poll, max_iter - c->launched);
            TRY(bcgs_iterate(c, batch));
            TRY(poll_state(c, &done, &iter));
        }
    }
    return bcgs_finish(c, out);
}

int32_t bcgs_residual_history(bcgs_ctx c, double* host_out, int32_t cap)
{
    if (!c || !host_out || cap <= 0) return 0;
    int32_t iter = 0;
    if (cudaMemcpy(&iter, &c->st->iter, sizeof iter, cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    int32_t m = std::min(cap, iter + 1);
    if (cudaMemcpy(host_out, c->hist, sizeof(double) * m, cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    return m;
}

int32_t bcgs_scalar_history(bcgs_ctx c, double* host_out, int32_t cap_iters)
{
    if (!c || !host_out || cap_iters <= 0) return 0;
    int32_t iter = 0;
    if (cudaMemcpy(&iter, &c->st->iter, sizeof iter, cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    int32_t m = std::min(cap_iters, iter);
    if (m > 0 && cudaMemcpy(host_out, c->scal, sizeof(double) * 8 * m,
                            cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    return m;
}

bcgs_status bcgs_get_solution(bcgs_ctx c, double* x, int32_t mem)
{
    if (!c || !x) return BCGS_E_INVALID;
    TRY(enter(c));
    const size_t bytes = sizeof(double) * (size_t)npts(c);
    CUDA_OK(c, cudaMemcpyAsync(x, F(c, V_X), bytes,
                               mem == BCGS_MEM_HOST ? cudaMemcpyDeviceToHost
                                                    : cudaMemcpyDeviceToDevice,
                               c->s));
    if (mem == BCGS_MEM_HOST) CUDA_OK(c, cudaStreamSynchronize(c->s));
    return leave(c);
}

bcgs_status bcgs_apply_operator(bcgs_ctx c, const double* d_in, double* d_out,
                                int32_t block_local)
{
    if (!c || !d_in || !d_out) return BCGS_E_INVALID;
    TRY(enter(c));
    const size_t bytes = sizeof(double) * (size_t)npts(c);
    double* io = F(c, V_IO);
    CUDA_OK(c, cudaMemcpyAsync(io, d_in, bytes, cudaMemcpyDeviceToDevice, c->s));
    if (!block_local) TRY(halo_api(c, io));
    else {
        CUDA_OK(c, cudaMemsetAsync(io - c->lay.plane, 0, sizeof(double) * c->lay.plane, c->s));
        CUDA_OK(c, cudaMemsetAsync(io + npts(c), 0, sizeof(double) * c->lay.plane, c->s));
    }
    ref::k_stencil_dot<0><<<stencil_grid(c), dim3(ref::BX, ref::BY), 0, c->s>>>(
        io, nullptr, d_out, ref_grid(c, (int)(c->lay.L / c->bpr)), block_local, nullptr,
        nullptr);
    CUDA_OK(c, cudaGetLastError());
    return leave(c);
}

bcgs_status bcgs_apply_preconditioner(bcgs_ctx c, const double* d_in, double* d_out)
{
    if (!c || !d_in || !d_out) return BCGS_E_INVALID;
    TRY(validate_pc(c));
    TRY(enter(c));
    const size_t bytes = sizeof(double) * (size_t)npts(c);
    double* io = F(c, V_IO);
    CUDA_OK(c, cudaMemcpyAsync(io, d_in, bytes, cudaMemcpyDeviceToDevice, c->s));
    double* o = F(c, V_W2);
    if (c->kernels == 1 && fused::precond_supported(c) &&
        !(c->pc == BCGS_PC_CHEB_G && c->nranks > 1))
        TRY(fused::precond_apply(c, io, o));
    else
        TRY(precond_ref(c, io, o, nullptr));
    CUDA_OK(c, cudaMemcpyAsync(d_out, o, bytes, cudaMemcpyDeviceToDevice, c->s));
    return leave(c);
}

bcgs_status bcgs_dot(bcgs_ctx c, const double* d_a, const double* d_b, double* host_out)
{
    if (!c || !d_a || !d_b || !host_out) return BCGS_E_INVALID;
    TRY(enter(c));
    k_set_exact<<<1, 1, 0, c->s>>>(c->st, c->exact_opt);
    ref::k_dot2<1><<<kEwBlocks, ref::EW_THREADS, 0, c->s>>>(d_a, d_b, nullptr, nullptr, npts(c),
                                                           c->part);
    CUDA_OK(c, cudaGetLastError());
    TRY(reduce<1>(c, kEwBlocks, STAGE_DOT, ew_depth(npts(c)), 1, {d_a, d_b}));
    int stg;
    TRY(resolve(c, &stg));
    CUDA_OK(c, cudaMemcpyAsync(c->h_pinned, c->st->scratch, sizeof(double),
                               cudaMemcpyDeviceToHost, c->s));
    CUDA_OK(c, cudaStreamSynchronize(c->s));
    *host_out = ((double*)c->h_pinned)[0];
    return leave(c);
}

int32_t bcgs_kernel_times(bcgs_ctx c, char* names_out, int32_t names_cap, double* ms_out,
                          int64_t* calls_out, double* bytes_out, int32_t cap)
{
    if (!c) return 0;
    harvest(c);
    std::string names;
    int m = std::min<int>(cap, KC_COUNT);
    for (int i = 0; i < KC_COUNT; ++i) {
        names += kClassName[i];
        names += '\n';
        if (i < m) {
            if (ms_out) ms_out[i] = c->ktime[i];
            if (calls_out) calls_out[i] = c->kcalls[i];
            if (bytes_out) bytes_out[i] = c->kbytes[i];
        }
    }
    if (names_out && names_cap > 0) {
        strncpy(names_out, names.c_str(), names_cap - 1);
        names_out[names_cap - 1] = 0;
    }
    return m;
}

bcgs_status bcgs_get_phase_times(bcgs_ctx c, double* host_out6)
{
    if (!c || !host_out6) return BCGS_E_INVALID;
    harvest(c);
    for (int p = 0; p <= PH_COUNT; ++p) host_out6[p] = 0.0;
    for (int i = 0; i < KC_COUNT; ++i) {
        host_out6[kc_phase(i)] += c->ktime[i];
        host_out6[PH_COUNT] += c->ktime[i];
    }
    return BCGS_OK;
}

void bcgs_kernel_times_reset(bcgs_ctx c)
{
    if (!c) return;
    harvest(c);
    for (int i = 0; i < KC_COUNT; ++i) {
        c->ktime[i] = 0.0;
        c->kcalls[i] = 0;
    }
}

}  // extern "C"

// ------------------------------------------------------------------ inner-Krylov preconditioners
// BJ(BiCGS) / G(BiCGS) (R29): M^-1 q = on every block s the result of an inner,
// unpreconditioned Bi-CGSTAB (the same Alg. 3 driver, M = I) on (R_s A R_s^T) p̂_s = q_s
// (Eq. 15), x0 = 0, relative tolerance in_tol, at most in_max iterations; the inner result is
// used whatever the inner status.  Each block's inner problem is a private context (zero
// Dirichlet ghosts at the cuts, the physical faces kept; a Neumann z face only in the first /
// last block of the global decomposition) created on first use, with a workspace the library
// allocates and its own stream: the blocks' inner solves run concurrently, each polled
// separately.  Their reductions are GPU-local (no NCCL: BJ(BiCGS) is "communication-free",
// P:207).
namespace {

bcgs_status inner_ctx(bcgs_ctx c, int s, int key, bcgs_ctx* out)
{
    if ((int)c->inner.size() <= s) {
        c->inner.resize(s + 1, nullptr);
        c->inner_ws.resize(s + 1, nullptr);
    }
    if (!c->inner[s]) {
        const int nb = c->pc == BCGS_PC_G_BICGS ? 1 : c->bpr;
        // G(BiCGS) on nranks > 1: ONE inner solve over the whole domain, spread over the
        // same ranks -- a multi-rank context sharing the outer transport
        const bool global = c->pc == BCGS_PC_G_BICGS && c->nranks > 1;
        bcgs_grid_desc g{};
        g.n[0] = c->lay.nx;
        g.n[1] = c->lay.ny;
        g.n[2] = global ? c->lay.nz : c->lay.L / nb;
        g.h = c->h;
        for (int f = 0; f < 4; ++f) g.bc[f] = c->bc[f];
        g.bc[4] = (key & 1) ? BCGS_BC_NEUMANN : BCGS_BC_DIRICHLET;
        g.bc[5] = (key & 2) ? BCGS_BC_NEUMANN : BCGS_BC_DIRICHLET;
        const int inr = global ? c->nranks : 1;
        const size_t bytes = bcgs_workspace_bytes(&g, inr);
        if (!bytes) return fail(c, BCGS_E_CONFIG, "inner solver: invalid block grid");
        void* ws = nullptr;
        CUDA_OK(c, cudaMalloc(&ws, bytes));
        bcgs_ctx ic = nullptr;
        bcgs_status st = global ? create_ctx(&g, c->rank, c->nranks, nullptr, nullptr, c->device,
                                             ws, bytes, c->s, &ic, 0, c)
                                : create_ctx(&g, 0, 1, nullptr, nullptr, c->device, ws, bytes,
                                             c->s, &ic);
        if (st != BCGS_OK) {
            std::string e = ic ? ic->err : "";
            if (ic) bcgs_destroy(ic);
            cudaFree(ws);
            return fail(c, st, "inner solver context: %s", e.c_str());
        }
        c->inner[s] = ic;
        c->inner_ws[s] = ws;
    }
    *out = c->inner[s];
    return BCGS_OK;
}

// Neumann z faces (R27) of inner block s: the global problem's first / last block only
int inner_key(bcgs_ctx c, int s)
{
    const int nb = c->pc == BCGS_PC_G_BICGS ? 1 : c->bpr;
    const int total = c->nranks * nb, gb = c->rank * nb + s;
    if (c->pc == BCGS_PC_G_BICGS && c->nranks > 1)   // the global problem's own faces
        return (c->bc[4] ? 1 : 0) | (c->bc[5] ? 2 : 0);
    return ((c->bc[4] && gb == 0) ? 1 : 0) | ((c->bc[5] && gb == total - 1) ? 2 : 0);
}

bcgs_status inner_all(bcgs_ctx c)
{
    const int nb = c->pc == BCGS_PC_G_BICGS ? 1 : c->bpr;
    for (int s = 0; s < nb; ++s) {
        bcgs_ctx ic;
        TRY(inner_ctx(c, s, inner_key(c, s), &ic));
    }
    return BCGS_OK;
}

bcgs_status precond_inner(bcgs_ctx c, const double* q, double* out, const DevState* st)
{
    if (st) {   // an outer stop earlier in this iteration (breakdown at α): nothing to do
        CUDA_OK(c, cudaMemcpyAsync(c->h_pinned, &st->done, sizeof(int32_t),
                                   cudaMemcpyDeviceToHost, c->s));
        CUDA_OK(c, cudaStreamSynchronize(c->s));
        if (((int32_t*)c->h_pinned)[0] != DONE_RUNNING) return BCGS_OK;
    }
    Prof pf(c, KC_PRECOND, 0.0);
    const int nb = c->pc == BCGS_PC_G_BICGS ? 1 : c->bpr;
    const int64_t blk = (c->lay.L / nb) * c->lay.plane;
    const int total = c->nranks * nb;
    std::vector<bcgs_ctx> ics(nb, nullptr);
    // start every block's solve (bcgs_solve split into begin / iterate / poll / finish)
    for (int s = 0; s < nb; ++s) {
        TRY(inner_ctx(c, s, inner_key(c, s), &ics[s]));
        bcgs_ctx ic = ics[s];
        bcgs_status e = bcgs_set_rhs(ic, q + s * blk, BCGS_MEM_DEVICE);
        if (e == BCGS_OK) e = bcgs_begin(ic, c->in_tol, c->in_max, 0);
        if (e != BCGS_OK) return fail(c, e, "inner solve: %s", ic->err.c_str());
    }
    std::vector<char> active(nb, 1);
    int left = nb;
    while (left > 0) {
        for (int s = 0; s < nb; ++s) {
            if (!active[s]) continue;
            bcgs_ctx ic = ics[s];
            int32_t done = 0, iter = 0;
            bcgs_status e = poll_state(ic, &done, &iter);
            if (e != BCGS_OK) return fail(c, e, "inner poll: %s", ic->err.c_str());
            if (done == DONE_RUNNING && ic->launched < c->in_max) {
                e = bcgs_iterate(ic, std::min(ic->poll, c->in_max - ic->launched));
                if (e != BCGS_OK) return fail(c, e, "inner iterate: %s", ic->err.c_str());
                continue;
            }
            bcgs_report rep{};
            e = bcgs_finish(ic, &rep);
            if (e != BCGS_OK && e != BCGS_NOT_CONVERGED && e != BCGS_BREAKDOWN)
                return fail(c, e, "inner finish: %s", ic->err.c_str());
            c->in_iters += rep.iterations;
            e = bcgs_get_solution(ic, out + s * blk, BCGS_MEM_DEVICE);
            if (e != BCGS_OK) return fail(c, e, "inner get_solution: %s", ic->err.c_str());
            active[s] = 0;
            --left;
        }
    }
    return BCGS_OK;
}

}  // namespace
