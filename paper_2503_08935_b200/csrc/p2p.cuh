// p2p.cuh -- peer-memory transport of the z-slab decomposition (SURVEY §8(e), NEXT-4
// "one-shot NVLink reductions"): the face halos (MPI1 / MPI3, P:278 / P:286) and the scalar
// reductions (MPI2 / MPI4 / MPI5) of Alg. 3 as device kernels
// that store into the peers' memory (NVLink / NVSwitch P2P, or the same GPU) and signal
// sequence-numbered flags -- no host involvement, so a multi-rank iteration is one CUDA graph.
//
// Every rank owns a Mailbox (library cudaMalloc; peers map it with CUDA IPC, or use the
// pointer directly inside one process).  Sequence numbers live in the own mailbox and advance
// on the device, identically on every rank (bulk-synchronous: every rank performs the same
// exchanges in the same order; a parked or finished solve skips them on every rank alike).
//   halo seq q (sender):  wait until the receiver acknowledged q - 2 (same landing slot),
//                         copy planes into its landing slot q & 1, fence, flag = q
//   halo seq q (receiver): wait for flag >= q from each neighbour, copy landing -> ghost
//                         planes, acknowledge q to the sender
//   reduction seq q:      one CTA: combine this rank's partials, store the triples into
//                         every rank's red[q & 1][me], fence, flag = q in every mailbox,
//                         wait for all flags >= q, combine in ascending rank order (R19)
// Two slots per stream suffice: a rank can start exchange q only after every rank has
// finished q - 1 (which needed their data of q - 1, written after consuming q - 2).
// Every wait has a timeout (%globaltimer): on expiry the solve stops with DONE_COMM_ERROR
// (the host returns BCGS_E_COMM) instead of hanging.
#pragma once
#include <stdint.h>

#include "dd.cuh"
#include "state.cuh"
#include "xdot.cuh"

namespace p2p {

constexpr int MAXR = 64;                  // ranks per communicator (BCGS_P2P_MAX_RANKS)

struct Mailbox {
    unsigned long long halo_flag[2];      // halo seq delivered from below (0) / above (1)
    unsigned long long halo_ack[2];       // halo seq the lower (0) / upper (1) rank consumed
    unsigned long long red_flag[MAXR];    // per source rank: reduction seq of its data
    unsigned ctr_send, ctr_land;          // block-completion counters (own rank only)
    // this rank's exchange sequence numbers (own rank only; shared by every context that
    // uses the mailbox, e.g. the inner solver of G(BiCGS))
    unsigned long long seq_halo_sent, seq_halo_recv, seq_red;
    unsigned long long pad[6];
    dd red[2][MAXR][5];                   // reduction triples [seq & 1][source rank][dot]
    long long limbs[2][MAXR][6 * xdot::XL];   // exact-path superaccumulators
    // landing zones follow at land_offset(): [dir][slot][cap planes][plane]
};

inline size_t land_offset() { return (sizeof(Mailbox) + 255) / 256 * 256; }

struct Peers {
    Mailbox* mb[MAXR];        // every rank's mailbox (mb[rank] = own), device-visible pointers
    double* land[MAXR];       // their landing zones
    int rank, nranks;
    int64_t plane;            // doubles per z-plane
    int64_t cap;              // landing planes per (dir, slot)
    unsigned long long timeout_ns;   // every wait gives up after this (BCGS_E_COMM)
};

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long now_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// spin until *flag >= want; false on timeout
__device__ __forceinline__ bool wait_ge(const unsigned long long* flag, unsigned long long want,
                                        unsigned long long timeout_ns)
{
    const unsigned long long t0 = now_ns();
    while (ld_acquire(flag) < want) {
        if (now_ns() - t0 > timeout_ns) return false;
        __nanosleep(200);
    }
    return true;
}

__device__ __forceinline__ void comm_error(DevState* st)
{
    st->comm_err = 1;
    st->done = DONE_COMM_ERROR;
}

// landing slot of direction dir (0: data coming from the lower rank, 1: from the upper)
__device__ __forceinline__ double* land_slot(double* land, int dir, unsigned long long seq,
                                             int64_t cap, int64_t plane)
{
    return land + ((int64_t)(dir * 2 + (int)(seq & 1)) * cap) * plane;
}

// Sender: planes [z0, z0 + k) of field v to the lower neighbour (dir 1 of its landing) and
// planes [L - k, L) to the upper neighbour (dir 0 of its landing).  Grid-stride copy; the
// last block to finish publishes the flags.  seq = seq_halo_sent + 1.
// guarded != 0 (inside an iteration): skipped once the solve is done or parked, on every
// rank alike; API calls (apply_operator, the x halo of begin / finish) pass 0.
// Every spin is done by ONE small block (k_halo_ack, k_halo_wait, the reduction's thread
// 0), so ranks that share a GPU (in-process groups) keep SMs free for each other.
//
// Sender, part 1 (one warp): the receivers must have consumed seq - 2 (the same landing
// slot) before it is overwritten.
static __global__ void k_halo_ack(Peers P, DevState* st, int guarded)
{
    if ((guarded && st->done) || threadIdx.x) return;
    const unsigned long long seq = P.mb[P.rank]->seq_halo_sent + 1;
    const int r = P.rank;
    Mailbox* me = P.mb[r];
    bool ok = true;
    if (r > 0 && seq > 2) ok &= wait_ge(&me->halo_ack[0], seq - 2, P.timeout_ns);
    if (r < P.nranks - 1 && seq > 2) ok &= wait_ge(&me->halo_ack[1], seq - 2, P.timeout_ns);
    if (!ok) comm_error(st);
}

// Sender, part 2
static __global__ void k_halo_send(Peers P, const double* __restrict__ v, int64_t L, int k,
                            DevState* st, int guarded)
{
    if ((guarded && st->done) || st->comm_err) return;
    const unsigned long long seq = P.mb[P.rank]->seq_halo_sent + 1;
    const int r = P.rank;
    const bool lo = r > 0, hi = r < P.nranks - 1;
    Mailbox* me = P.mb[r];
    unsigned* done_ctr = &me->ctr_send;
    const int64_t n = (int64_t)k * P.plane;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (lo) {   // my lowest planes -> lower rank, arriving "from above" (dir 1)
        double* dst = land_slot(P.land[r - 1], 1, seq, P.cap, P.plane);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
            dst[i] = v[i];
    }
    if (hi) {   // my highest planes -> upper rank, arriving "from below" (dir 0)
        double* dst = land_slot(P.land[r + 1], 0, seq, P.cap, P.plane);
        const double* src = v + (L - k) * P.plane;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
            dst[i] = src[i];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(done_ctr, 1u);
        if (prev == gridDim.x - 1) {   // last block: every copy is globally visible
            __threadfence_system();
            if (lo) st_release(&P.mb[r - 1]->halo_flag[1], seq);
            if (hi) st_release(&P.mb[r + 1]->halo_flag[0], seq);
            *done_ctr = 0;
            me->seq_halo_sent = seq;
        }
    }
}

// Receiver, part 1 (one warp): wait for the neighbours' data of seq = seq_halo_recv + 1
static __global__ void k_halo_wait(Peers P, DevState* st, int guarded)
{
    if ((guarded && st->done) || threadIdx.x) return;
    const unsigned long long seq = P.mb[P.rank]->seq_halo_recv + 1;
    const int r = P.rank;
    Mailbox* me = P.mb[r];
    bool ok = true;
    if (r > 0) ok &= wait_ge(&me->halo_flag[0], seq, P.timeout_ns);
    if (r < P.nranks - 1) ok &= wait_ge(&me->halo_flag[1], seq, P.timeout_ns);
    if (!ok) comm_error(st);
}

// Receiver, part 2: landing -> ghost region (k planes below `gl`, k planes at `gh`),
// then acknowledge seq to the senders.
static __global__ void k_halo_land(Peers P, double* gl, double* gh, int k, DevState* st, int guarded)
{
    if ((guarded && st->done) || st->comm_err) return;
    unsigned* done_ctr = &P.mb[P.rank]->ctr_land;
    const unsigned long long seq = P.mb[P.rank]->seq_halo_recv + 1;
    const int r = P.rank;
    const int64_t n = (int64_t)k * P.plane;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (r > 0) {
        const double* src = land_slot(P.land[r], 0, seq, P.cap, P.plane);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
            gl[i] = __ldcv(src + i);
    }
    if (r < P.nranks - 1) {
        const double* src = land_slot(P.land[r], 1, seq, P.cap, P.plane);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
            gh[i] = __ldcv(src + i);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(done_ctr, 1u);
        if (prev == gridDim.x - 1) {   // last block: the landing slots are free again
            __threadfence_system();
            if (r > 0) st_release(&P.mb[r - 1]->halo_ack[1], seq);
            if (r < P.nranks - 1) st_release(&P.mb[r + 1]->halo_ack[0], seq);
            *done_ctr = 0;
            P.mb[r]->seq_halo_recv = seq;
        }
    }
}

// One-shot all-gather of a small record (thread 0): mine -> slot[seq & 1][me] of every
// rank, flags, wait for every rank's flag.  Returns false on timeout.
__device__ inline bool exchange(const Peers& P, DevState* st, unsigned long long seq)
{
    const int me = P.rank;
    __threadfence_system();
    for (int r = 0; r < P.nranks; ++r) st_release(&P.mb[r]->red_flag[me], seq);
    Mailbox* my = P.mb[me];
    for (int r = 0; r < P.nranks; ++r)
        if (!wait_ge(&my->red_flag[r], seq, P.timeout_ns)) return false;
    return true;
}

// Fused reduction (one CTA of 1024 threads): this rank's partials -> triples (as
// k_finalize), one-shot exchange, rank-ordered combination, stage completion (R19).
template <int ND>
__global__ void __launch_bounds__(256) k_reduce_p2p(Peers P, const dd* __restrict__ part,
                                                     int nparts, int stage, DevState* st,
                                                     double* hist, double* scal, int depth,
                                                     double nprod, int self_mask, int k3_mask,
                                                     int local_only)
{
    if (stage != STAGE_SETUP && stage != STAGE_DOT && st->done) return;
    __shared__ dd res[ND];
    combine_partials<ND>(part, nparts, res);
    if (threadIdx.x) return;
    const int me = P.rank;
    dd comb[ND];
    if (local_only) {   // ablation (timing only): this rank's triples, no exchange
        for (int d = 0; d < ND; ++d) {
            comb[d] = dd{0.0, 0.0, 0.0, 0.0};
            dd_add(comb[d].hi, comb[d].mid, comb[d].lo, comb[d].ab, res[d].hi, res[d].mid,
                   res[d].lo, res[d].ab);
        }
    } else {
        const unsigned long long seq = P.mb[me]->seq_red + 1;
        const int slot = (int)(seq & 1);
        for (int r = 0; r < P.nranks; ++r)
            for (int d = 0; d < ND; ++d) P.mb[r]->red[slot][me][d] = res[d];
        if (!exchange(P, st, seq)) {
            comm_error(st);
            return;
        }
        P.mb[me]->seq_red = seq;
        Mailbox* my = P.mb[me];
        for (int d = 0; d < ND; ++d) {
            comb[d] = dd{0.0, 0.0, 0.0, 0.0};
            for (int r = 0; r < P.nranks; ++r) {
                const dd* gp = &my->red[slot][r][d];
                const dd g{__ldcv(&gp->hi), __ldcv(&gp->mid), __ldcv(&gp->lo), __ldcv(&gp->ab)};
                dd_add(comb[d].hi, comb[d].mid, comb[d].lo, comb[d].ab, g.hi, g.mid, g.lo, g.ab);
            }
        }
    }
    finish_stage(st, stage, ND, comb, depth + 2 * ((nparts + 255) / 256) + 48 + 2 * P.nranks,
                 nprod, self_mask, k3_mask, hist, scal);
}

// Exact path (R19): this rank's superaccumulators -> every rank's mailbox, exchange, and the
// gathered copy [rank][6 XL] into `out` for k_resolve.  One CTA.
static __global__ void k_limbs_p2p(Peers P, const long long* __restrict__ mine, long long* out,
                            DevState* st)
{
    __shared__ unsigned long long seq_s;
    __shared__ int ok_s;
    const int me = P.rank;
    const int64_t per = 6 * xdot::XL;
    if (threadIdx.x == 0) seq_s = P.mb[me]->seq_red + 1;
    __syncthreads();
    const int slot = (int)(seq_s & 1);
    for (int r = 0; r < P.nranks; ++r)
        for (int64_t i = threadIdx.x; i < per; i += blockDim.x)
            P.mb[r]->limbs[slot][me][i] = mine[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        ok_s = exchange(P, st, seq_s) ? 1 : 0;
        if (ok_s) P.mb[me]->seq_red = seq_s;
        else comm_error(st);
    }
    __syncthreads();
    if (!ok_s) return;
    const Mailbox* my = P.mb[me];
    for (int r = 0; r < P.nranks; ++r)
        for (int64_t i = threadIdx.x; i < per; i += blockDim.x)
            out[r * per + i] = __ldcv(&my->limbs[slot][r][i]);
}

}  // namespace p2p
