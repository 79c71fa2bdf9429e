/*
 * bcgs.h -- C ABI of the B200-native preconditioned Bi-CGSTAB Poisson hot path
 * (arXiv 2503.08935, "A Parallel and Highly-Portable HPC Poisson Solver: Preconditioned
 * Bi-CGSTAB with alpaka").  Implemented by paper_2503_08935_b200/lib/libbcgs.so.
 *
 * Citations: P:n = line n of the paper's LaTeX source, with the equation /
 * algorithm it falls in.  R-numbers refer to the arithmetic contract in DESIGN.md §3.
 *
 * Problem (Eq. 1-6): -Δφ = f on a box of nx*ny*nz unknowns with uniform spacing
 * h and homogeneous Dirichlet ghosts; constant Dirichlet face values are folded into the
 * right-hand side (R15).  Matrix-free 7-point operator A (Eq. 6).
 *
 * Decomposition: the z axis is split into `nranks` equal slabs, one per process
 * (one GPU each); rank r owns global planes [r*L, (r+1)*L), L = nz/nranks.  Each slab may
 * further be split into `blocks_per_rank` preconditioner blocks (single-GPU emulation of a
 * larger slab count; the preconditioner acts on nranks*blocks_per_rank z-slabs).
 *
 * Data layout of every field argument: this rank's slab, fp64, x fastest then y then z,
 * nx*ny*L contiguous values (no ghost planes, no padding).  `mem` says whether a pointer
 * is host (BCGS_MEM_HOST, pageable or pinned) or device (BCGS_MEM_DEVICE) memory.
 *
 * Ownership: the caller owns the device workspace (bcgs_workspace_bytes) and the CUDA
 * stream passed to bcgs_create; both must outlive the context.  The library never frees
 * caller memory; inputs are copied in, results copied out.  The context owns its private
 * CUDA stream, events, graphs and (nranks > 1) NCCL communicator.
 *
 * Streams: set_* / get_* / apply_* calls are ordered after prior work on the caller's
 * stream and the caller's stream is ordered after them (event joins); host-memory
 * variants synchronise the host.  bcgs_solve returns after the solve ends.
 *
 * Errors: every call returns a bcgs_status; bcgs_last_error gives a one-line diagnostic.
 * Configuration errors are detected before any device work.  Breakdown and non-convergence
 * are reported as statuses with the report filled, never as crashes.
 *
 * Collective semantics (nranks > 1): every rank calls create, set_*, solve, dot, apply_*
 * in the same order (bulk synchronous); scalars and the residual history are identical
 * on every rank.  A context is not thread-safe.
 */
#ifndef BCGS_H
#define BCGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BCGS_ABI_VERSION 6
#define BCGS_MAX_DEGREE 64       /* Chebyshev degree k (sweeps per application) cap      */
#define BCGS_HIST_CAP 16384      /* max outer iterations recorded per solve              */

typedef struct bcgs_ctx_s* bcgs_ctx;

typedef enum {
    BCGS_OK = 0,
    BCGS_E_INVALID = 1,       /* bad argument (null pointer, out-of-range value)          */
    BCGS_E_CONFIG = 2,        /* inconsistent configuration (e.g. nz % nranks != 0)        */
    BCGS_E_SPECTRUM = 3,      /* empty / non-positive Chebyshev interval                  */
    BCGS_E_CUDA = 4,          /* CUDA runtime error (message in bcgs_last_error)          */
    BCGS_E_NCCL = 5,          /* NCCL error                                               */
    BCGS_NOT_CONVERGED = 6,   /* max_iter reached without rel residual < tol (R23)        */
    BCGS_BREAKDOWN = 7,       /* exact zero / non-finite r~ᵀw, ω or ρ (R7)                */
    BCGS_E_STATE = 8,         /* call out of order (e.g. iterate before begin)            */
    BCGS_E_COMM = 9           /* p2p transport: a peer did not answer within the timeout  */
} bcgs_status;

/* Preconditioner M of Alg. 3 l.6/12; Table I. */
typedef enum {
    BCGS_PC_NONE = 0,          /* M = I: plain Bi-CGSTAB (Alg. 1)               */
    BCGS_PC_CHEB_GNOCOMM = 1,  /* GNoComm(CI): Chebyshev on each slab block with   */
                               /* the global Eq. 9-11 bounds rescaled by (c_min, c_max)    */
    BCGS_PC_CHEB_BJ = 2,       /* BJ(CI): Chebyshev on each slab block with the    */
                               /* exact local-block bounds (R10)                           */
    BCGS_PC_CHEB_G = 3,        /* G(CI): Chebyshev on the GLOBAL operator with */
                               /* the rescaled global bounds; multi-rank: one k-deep halo  */
                               /* exchange per application instead of Alg. 4's per-sweep   */
                               /* MPI2 (requires k <= L); blocks_per_rank is ignored       */
    BCGS_PC_BJ_BICGS = 4,      /* BJ(BiCGS) (Eq. 15): inner unpreconditioned    */
                               /* Bi-CGSTAB on every slab block (zero ghosts at the cuts), */
                               /* x0 = 0, default tol 1e-6 / 500 iterations; the   */
                               /* outer Alg. 3 is flexible.  degree is ignored     */
    BCGS_PC_G_BICGS = 5        /* G(BiCGS): the inner solve on the whole       */
                               /* domain, default tol 1e-2 / 500; nranks == 1 only */
} bcgs_pc;

typedef enum { BCGS_MEM_DEVICE = 0, BCGS_MEM_HOST = 1 } bcgs_mem;

/* Implementation switches (bcgs_set_option). */
typedef enum {
    BCGS_OPT_KERNELS = 0,      /* 0 = reference kernels (one sweep per launch, one op per */
                               /*     launch); 1 = fused / temporally blocked (default)   */
    BCGS_OPT_GRAPH = 1,        /* 1 = replay iterations from a captured CUDA graph (default;*/
                               /*     one rank or the p2p transport; not while profiling   */
                               /*     or with bcgs_create_local); 2 = also capture NCCL    */
    BCGS_OPT_PROFILE = 2,      /* 1 = CUDA events around every kernel (bcgs_kernel_times) */
    BCGS_OPT_POLL = 3,         /* iterations launched between done-flag polls (tol mode)  */
    BCGS_OPT_TB_VARIANT = 4,   /* temporally blocked kernel layout: 7 = TMA warp-row      */
                               /* kernel (default; 24 warps for k <= 4, 16 warps with     */
                               /* Neumann faces), 2 = square tile (also used for odd nx). */
                               /* Other values: BCGS_E_INVALID.  (Options 5-7 of ABI 3,   */
                               /* layouts measured slower, were removed in ABI 4.)        */
    BCGS_OPT_MULTIPASS = 8,    /* multi-pass temporal blocking (passes of 2..4 sweeps) for */
                               /* degree > value (default 4; clamped to >= 4).  Degrees   */
                               /* above 8 always run multi-pass when the TMA kernels can  */
                               /* (nx even).  Bitwise the same result either way.         */
    BCGS_OPT_ABLATE = 9,       /* comm ablation for timing the exposed halo / reduction     */
                               /* share: bit 0 skips the face halos, bit 1  */
                               /* the cross-rank reductions (each rank uses its own pairs).*/
                               /* The maths is WRONG while set; 0 = off (default)          */
    BCGS_OPT_SYNC2 = 10,       /* 1 = 2-sync rewrite (R31): r~ᵀs, r~ᵀt, sᵀs  */
                               /* join the a9 reduction, ρ_new and ||r||² follow from the  */
                               /* identities for r = s - ω t -> 2 reductions per iteration */
                               /* instead of 3 (fused path only; rounding differs from the */
                               /* default, the oracle implements the same flag)            */
    BCGS_OPT_EXACT_DOT = 11,   /* 1 = every dot product through the exact superaccumulator */
                               /* path (R19 fallback) instead of certified   */
                               /* Dot2; the results are the same (correctly rounded) --   */
                               /* for testing the fallback.  0 = certified Dot2 (default) */
    BCGS_OPT_COMM_TIMEOUT = 12,/* seconds a transport wait may take: NCCL host waits abort  */
                               /* the communicator after it (default 300; async errors    */
                               /* abort at once); p2p device waits give up (default 60).  */
                               /* Both end the solve with an error status, never a hang.  */
    BCGS_OPT_PIPELINED = 13,   /* 1 = pipelined (communication-hiding) Bi-CGSTAB for      */
                               /* B = A M^-1 (NEXT-4; R32): 2 reductions  */
                               /* per iteration, each independent of the preconditioner + */
                               /* stencil that follows it; linear preconditioners only;   */
                               /* six more fields (library-owned).  Same iterates as Alg. 3 */
                               /* in exact arithmetic; the oracle implements the same flag */
    BCGS_OPT_PDL = 16,         /* 1 = consecutive kernels of an iteration use programmatic */
                               /* dependent launch (one rank, NCCL / p2p off, not while    */
                               /* profiling): the next kernel is launched as soon as every */
                               /* CTA of its predecessor has exited and waits for the      */
                               /* predecessor's completion; 0 = ordinary launches (default: */
                               /* graph replay already hides the launch gaps)*/
                               /* Bitwise the same results                                 */
    BCGS_OPT_TB_SCHEDULE = 15, /* work split of the temporally blocked kernel (24-warp TMA */
                               /* layout): 0 = auto (default: segments where a wave cost  */
                               /* model gains >= 10 %), 1 = tile x z-chunk grid, 2 = one  */
                               /* CTA per SM, each an equal share of the tile-major work  */
                               /* (DESIGN.md §4).  Bitwise the same results               */
    BCGS_OPT_STENCIL = 14      /* stencil+dot kernels of a4 / a9: 1 = TMA-staged z-march  */
                               /* (default; Dirichlet faces, even nx; planes per CTA from */
                               /* a wave cost model), v >= 2 = TMA with v planes per CTA  */
                               /* (clamped to 4..64; measurement), 0 = L1-cached z-march. */
                               /* Bitwise the same results; values outside 0..64:         */
                               /* BCGS_E_INVALID (64 bounds the certified dot chains)     */
} bcgs_option;

/* Boundary condition kind of a physical face (Eq. 4 / Eq. 5). */
typedef enum {
    BCGS_BC_DIRICHLET = 0,     /* ghost = boundary value, folded into b (R15)              */
    BCGS_BC_NEUMANN = 1        /* ghost = mirror of the first interior neighbour, i.e. the */
                               /* rows (2, -2) of Eq. 5's N ("Set Neumann BCs");    */
                               /* a face value is the outward normal derivative (R28)      */
} bcgs_bc;

typedef struct {
    int64_t n[3];   /* global unknowns along x, y, z (each >= 1; >= 2 on a Neumann axis)  */
    double h;       /* uniform grid spacing (> 0); unit cube: h = 1/(n+1)                  */
    int32_t bc[6];  /* bcgs_bc of faces x-, x+, y-, y+, z-, z+ (all 0 = all Dirichlet).   */
                    /* Chebyshev bounds follow the face kinds (R27).  A Neumann z face    */
                    /* needs >= 2 planes per preconditioner block.                        */
} bcgs_grid_desc;

typedef struct {
    int32_t status;            /* bcgs_status of the solve                                 */
    int32_t converged;         /* 1 if rel_residual < tol (or fixed iterations completed)  */
    int32_t iterations;        /* completed outer iterations                               */
    int32_t degree_warning;    /* 1 if k > L_block/2 (R24)                           */
    double rel_residual;       /* recurrence residual sqrt(rᵀr)/||b|| of the last iteration */
    double true_rel_residual;  /* ||b - A x|| / ||b|| computed once at the end (R22)       */
    double seconds;            /* wall time of the solve                                   */
} bcgs_report;

/* BCGS_ABI_VERSION of the library; one-line text of a status. */
int32_t bcgs_abi_version(void);
const char* bcgs_status_string(bcgs_status s);

/* Device workspace the caller must provide to bcgs_create for this grid and rank count:
 * the vectors of one rank's slab of Alg. 3 (x, r, r~, p, p̂, r̂, w, t, b, ... -- P:272-305)
 * each with one ghost plane below and above (the halo planes of MPI1 / MPI3, P:278, P:286;
 * DESIGN.md §4), the G(CI) extended slabs for nranks > 1, the device scalars and history,
 * and the reduction partials.  Returns 0 for an invalid grid / rank count (nz % nranks). */
size_t bcgs_workspace_bytes(const bcgs_grid_desc* grid, int32_t nranks);

/* Chebyshev interval and constants for a configuration, computed on the host exactly as
 * the solver computes them (Eq. 9-11, Eq. 15, Alg. 2, R9,
 * R10, R18).  out7 = {θ, δ, σ, 1/θ, 2ρ₁/δ, 2σ, 2/δ}; rho = ρ_0..ρ_k (k+1 values, at least
 * 2).  Host-only; no GPU needed.  nslab = nranks*blocks_per_rank. */
bcgs_status bcgs_chebyshev_constants(const bcgs_grid_desc* grid, int32_t nslab, bcgs_pc pc,
                                     int32_t degree, double c_min, double c_max,
                                     double* interval2, double* out7, double* rho);

/* 128-byte NCCL unique id for a new communicator (call on rank 0 only; broadcast it). */
bcgs_status bcgs_nccl_unique_id(void* out128);

/* Create a context.  nccl_unique_id: 128-byte ncclUniqueId from rank 0 (broadcast by the
 * caller); NULL for nranks == 1 (an id with nranks == 1 creates a 1-rank communicator whose
 * all-gathers carry the reductions: the NCCL code path on one GPU, for testing).
 * cuda_stream: caller's cudaStream_t (may be 0).
 * d_workspace: >= bcgs_workspace_bytes device bytes, 256-byte aligned. */
bcgs_status bcgs_create(const bcgs_grid_desc* grid, int32_t rank, int32_t nranks,
                        const void* nccl_unique_id, int32_t cuda_device, void* d_workspace,
                        size_t ws_bytes, void* cuda_stream, bcgs_ctx* out);
/* In-process multi-rank group on ONE device (testing transport): creates nranks contexts
 * (ranks 0..nranks-1 of the z-slab decomposition) whose halo exchanges and reductions are
 * device copies between their workspaces instead of NCCL.  Each context must then be driven
 * by its own host thread (exchanges block on a host barrier).  d_workspaces[r] as for
 * bcgs_create; outs[r] receives rank r's context. */
bcgs_status bcgs_create_local(const bcgs_grid_desc* grid, int32_t nranks, int32_t cuda_device,
                              void* const* d_workspaces, size_t ws_bytes, void* cuda_stream,
                              bcgs_ctx* outs);
/* Peer-memory transport: halos and reductions are
 * kernels that store into the peers' memory and signal sequence-numbered flags (one-shot
 * reductions, no host synchronisation, multi-rank iterations replayed as CUDA graphs).
 * One process per rank: bcgs_create_p2p, then every rank exchanges its 128-byte
 * bcgs_p2p_handle record (the caller's process group: all-gather) and calls
 * bcgs_p2p_connect with the nranks records in rank order (CUDA IPC; ranks on the same or
 * on NVLink-connected devices).  The mailbox (and the landing zones of the halos) is
 * allocated and freed by the library.  In one process: bcgs_create_local_p2p (direct
 * pointers; drive each context from its own host thread; set CUDA_MODULE_LOADING=EAGER
 * before the CUDA context exists -- a lazy module load at a kernel's first launch can stall
 * behind another rank's spin-waiting kernel on the same GPU).  Peer waits time out after
 * 60 s (BCGS_E_COMM) instead of hanging. */
bcgs_status bcgs_create_p2p(const bcgs_grid_desc* grid, int32_t rank, int32_t nranks,
                            int32_t cuda_device, void* d_workspace, size_t ws_bytes,
                            void* cuda_stream, bcgs_ctx* out);
bcgs_status bcgs_p2p_handle(bcgs_ctx ctx, void* out128);
bcgs_status bcgs_p2p_connect(bcgs_ctx ctx, const void* all_handles);
bcgs_status bcgs_create_local_p2p(const bcgs_grid_desc* grid, int32_t nranks,
                                  int32_t cuda_device, void* const* d_workspaces,
                                  size_t ws_bytes, void* cuda_stream, bcgs_ctx* outs);
/* Destroy a context (waits for its stream; frees what the library allocated, never the
 * caller's workspace or stream).  last_error: one-line diagnostic of the last failed call
 * (owned by the context).  set_option: bcgs_option switches (implementation choices; the
 * maths of Alg. 3 is unchanged unless an option says otherwise). */
void bcgs_destroy(bcgs_ctx ctx);
const char* bcgs_last_error(bcgs_ctx ctx);
bcgs_status bcgs_set_option(bcgs_ctx ctx, int32_t option, int64_t value);

/* Right-hand side b (Eq. 1; Alg. 3 l.1).  Random: R16, generated on the device from
 * the global index (identical bits for any rank count).  bcgs_set_rhs copies this rank's
 * slab.  Face values (R15): face 0..5 = x-,x+,y-,y+,z-,z+; the values set are folded
 * into b by every subsequent set_rhs* call: a Dirichlet value g adds g/h² to the first
 * plane of unknowns (R15), a Neumann outward derivative g adds 2g/h (R28). */
bcgs_status bcgs_set_rhs_random(bcgs_ctx ctx, uint64_t seed);
bcgs_status bcgs_set_rhs(bcgs_ctx ctx, const double* f, int32_t mem);
bcgs_status bcgs_set_boundary_value(bcgs_ctx ctx, int32_t face, double value);
/* Initial guess x0 (Alg. 3 l.1); NULL -> 0 (R21). */
bcgs_status bcgs_set_initial_guess(bcgs_ctx ctx, const double* x0, int32_t mem);

/* Preconditioner: kind, degree k (R1, 0..BCGS_MAX_DEGREE), rescaling (c_min, c_max) for
 * GNoComm (R9), blocks_per_rank >= 1 with L % blocks_per_rank == 0. */
bcgs_status bcgs_set_preconditioner(bcgs_ctx ctx, bcgs_pc pc, int32_t degree, double c_min,
                                    double c_max, int32_t blocks_per_rank);
/* Inner solver of BJ(BiCGS) / G(BiCGS): relative tolerance and iteration cap of every inner
 * solve (set after bcgs_set_preconditioner, which restores the paper's defaults).  The
 * inner result is used whatever the inner status (R29).  Inner solves run on the library's
 * stream through private contexts (workspaces allocated and owned by the library) and
 * synchronise the host, so these preconditioners are not graph-captured. */
bcgs_status bcgs_set_inner_solver(bcgs_ctx ctx, double rel_tol, int32_t max_iter);
/* Total inner iterations since the last bcgs_begin (Table II "it. / outer it."). */
int64_t bcgs_inner_iterations(bcgs_ctx ctx);
/* Dot products recomputed on the exact path since the last bcgs_begin (R19: a Dot2 result
 * that could not be certified as correctly rounded, or BCGS_OPT_EXACT_DOT); -1 on error. */
int32_t bcgs_exact_dots(bcgs_ctx ctx);
/* Diagnostics of the last Dot2 result the certification refused (R19): stage, dot index,
 * chain depth D, r = fl(hi + lo), e = (hi + lo) - r, the error bound E, the gaps above and
 * below |r|, Σ|a_i b_i|, then the number of refusals since bcgs_create (10 doubles). */
bcgs_status bcgs_certification_info(bcgs_ctx ctx, double* out10);
/* Override the Chebyshev interval [a', b'] of Alg. 2 (0 < a' < b'); (0, 0)
 * restores the default bounds of Eq. 9-11 (R9, R10). */
bcgs_status bcgs_set_eigen_bounds(bcgs_ctx ctx, double a, double b);

/* Solve A x = b with Alg. 3.  fixed_iters > 0: run exactly that many iterations
 * (tol ignored); else stop when rel < rel_tol (R4) or after max_iter (<= BCGS_HIST_CAP). */
bcgs_status bcgs_solve(bcgs_ctx ctx, double rel_tol, int32_t max_iter, int32_t fixed_iters,
                       bcgs_report* out);

/* Split form of bcgs_solve for timing: begin = Alg. 3 l.1-4 (setup, row a1); iterate
 * enqueues n more outer iterations (rows a2-a14) on the stream and returns without host
 * synchronisation (fixed-iteration semantics); finish waits and fills the report. */
bcgs_status bcgs_begin(bcgs_ctx ctx, double rel_tol, int32_t max_iter, int32_t fixed_iters);
bcgs_status bcgs_iterate(bcgs_ctx ctx, int32_t n);
bcgs_status bcgs_finish(bcgs_ctx ctx, bcgs_report* out);
/* Order the caller's stream after all work enqueued so far (no host synchronisation). */
bcgs_status bcgs_join(bcgs_ctx ctx);

/* Residual history rel_0..rel_iters of the last solve: rel_i = sqrt(rᵀr)/||b|| of Alg. 3
 * l.21-24 (R4; rel_0 = sqrt(r~ᵀr0)/||b|| = 1 for x0 = 0, R26); host_out holds
 * cap doubles; returns the count copied (min(cap, iterations + 1); 0 on error).  Identical
 * on every rank. */
int32_t bcgs_residual_history(bcgs_ctx ctx, double* host_out, int32_t cap);
/* Per-iteration scalars of Alg. 3, 8 per iteration: r~ᵀw, α, tᵀs, tᵀt, ω,
 * ρ_new, rᵀr, β (pipelined, R32: α's denominator, α, qᵀy, yᵀy, ω, ρ_new, rᵀr, β);
 * host_out holds 8 * cap_iters doubles; returns the iterations copied. */
int32_t bcgs_scalar_history(bcgs_ctx ctx, double* host_out, int32_t cap_iters);
/* Solution x of Alg. 3 l.20 (the converged iterate, R25): this rank's slab,
 * nx*ny*L doubles, x fastest, into device or host memory `x` (mem); the caller owns x. */
bcgs_status bcgs_get_solution(bcgs_ctx ctx, double* x, int32_t mem);

/* Single steps of the path on device slabs, for parity tests and micro-benchmarks.
 * apply_operator: out = A in (global operator with halo exchange; block_local != 0 gives
 * the block-diagonal slab operator of Eq. 12-14).  apply_preconditioner: out = M^-1 in
 * with the configured preconditioner.  dot: the global dot product, correctly rounded
 * (R19: certified Dot2, else the exact path) -> *host_out. */
bcgs_status bcgs_apply_operator(bcgs_ctx ctx, const double* d_in, double* d_out,
                                int32_t block_local);
bcgs_status bcgs_apply_preconditioner(bcgs_ctx ctx, const double* d_in, double* d_out);
bcgs_status bcgs_dot(bcgs_ctx ctx, const double* d_a, const double* d_b, double* host_out);

/* Kernel timings accumulated while BCGS_OPT_PROFILE = 1 (CUDA events on the launching
 * stream; the paper's per-kernel profiling of Alg. 3, P:493 -- KernelBiCGS1-6, CI sweeps,
 * MPI calls).  Returns the number of kernel classes; names are '\n'-separated in names_out.
 * ms_out[i] = total milliseconds, calls_out[i] = launches; bytes_out[i] = algorithmic
 * bytes per launch of class i. */
int32_t bcgs_kernel_times(bcgs_ctx ctx, char* names_out, int32_t names_cap, double* ms_out,
                          int64_t* calls_out, double* bytes_out, int32_t cap);
void bcgs_kernel_times_reset(bcgs_ctx ctx);

/* The same timings grouped into the SPEC's six phase keys (in this order):
 * [0] "preconditioner"  (a2 / a7: the Chebyshev kernels -- the fused ones also carry the
 *                        p / s vector updates a14 / a6 -- and reference sweeps)
 * [1] "halo_exchange"   (a3 / a8 on the comm stream; overlaps the interior stencil)
 * [2] "allreduce"       (a5 / a10 / a13: finalize, all-gather, scalar step)
 * [3] "stencil_kernels" (a4 / a9: stencil + dot)
 * [4] "vector_kernels"  (a6, a11, a12, a14 when not fused into the preconditioner)
 * [5] "total"           (sum of [0..4]; [1] overlaps [3], so this exceeds wall time)
 * host_out6[i] = milliseconds accumulated while BCGS_OPT_PROFILE = 1 (zeros otherwise).
 * With BCGS_OPT_PROFILE = 1 every timed launch is also wrapped in an NVTX range
 * "<phase key>/<kernel class>" (visible to nsys / ncu --nvtx; no-ops without a tool).
 * BCGS_E_INVALID for a null context or output. */
bcgs_status bcgs_get_phase_times(bcgs_ctx ctx, double* host_out6);

#ifdef __cplusplus
}
#endif
#endif /* BCGS_H */
