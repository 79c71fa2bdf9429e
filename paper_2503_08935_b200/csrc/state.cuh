// state.cuh -- device-resident solver state and the scalar steps of Alg. 3.
// The paper computes α, ω, β on the host after each MPI_Allreduce; here they are
// computed on the device by one thread right after the reduction, so an iteration needs no
// host round trip.  Formulas: R4, R6, R7, R20, R25.
#pragma once
#include <stdint.h>

#include "dd.cuh"
#include "xdot.cuh"

// DONE_PENDING: a reduction could not be certified (R19); every later kernel of the solve
// is a no-op until the host has recomputed the flagged dots exactly and resumed (resolve).
// DONE_COMM_ERROR: a peer-transport wait timed out (p2p.cuh); the host returns BCGS_E_COMM.
enum : int32_t { DONE_RUNNING = 0, DONE_OK = 1, DONE_BREAKDOWN = 2, DONE_MAXIT = 3,
                 DONE_PENDING = 4, DONE_COMM_ERROR = 5 };

// Programmatic dependent launch (PDL, DESIGN.md §4 "Launch chain"): a kernel launched with
// programmatic stream serialization is launched once every CTA of its predecessor has
// exited (no explicit trigger: dependents that became resident earlier would hold SM
// resources the predecessor's later CTAs need -- measured slower), before the predecessor's
// grid completion is processed; it waits here -- before touching any data -- until the
// predecessor has completed and its memory is visible.  Every kernel the library launches
// that way calls this first (completion stays transitive along the chain); a no-op for
// ordinary launches.
__device__ __forceinline__ void pdl_enter()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

struct DevState {
    double rho, alpha, omega, beta, nb;
    double den;           // pipelined: the α denominator r~ᵀw + β (r~ᵀS - ω r~ᵀz)
    double rw, ts, tt, rho_new, rr, rel;
    double tol;
    int32_t iter;         // completed outer iterations
    int32_t done;         // DONE_*
    int32_t fixed_iters;  // > 0: run exactly this many
    int32_t max_iter;
    double scratch[8];    // results of stand-alone dot calls
    int32_t pend;         // 2-sync (R31): stop decided at the ω stage, applied after a11/a12
    // R19 certification fallback
    int32_t pend_stage;   // stage whose reduction is parked (valid while pend_mask != 0)
    int32_t pend_mask;    // bit d: dot d of that stage needs the exact recomputation
    double pend_v[5];     // the stage's values (certified ones final, the others replaced)
    int32_t exact_mode;   // BCGS_OPT_EXACT_DOT = 1: every dot through the exact path
    int32_t n_exact;      // dots recomputed exactly since bcgs_begin
    int32_t comm_err;     // peer transport (p2p.cuh): a wait timed out
    // the last refused certification: stage, dot, D, r, e, E, |r| gap up, gap down, Hc
    double cert_last[9];
    int32_t n_refused;    // certifications refused since bcgs_create
};

// Reduction stages (one per MPI_Allreduce site of Alg. 3).
enum : int32_t {
    STAGE_SETUP = 0,   // {bᵀb, r~ᵀr0}         Alg. 3 l.4
    STAGE_ALPHA = 1,   // {r~ᵀw}               MPI2 + α
    STAGE_OMEGA = 2,   // {tᵀs, tᵀt}           MPI4 + ω
    STAGE_RHO = 3,     // {r~ᵀr, rᵀr}          MPI5 + test + ρ, β
    STAGE_DOT = 4,     // stand-alone dot -> scratch
    STAGE_OMEGA2 = 5,  // 2-sync (R31): {tᵀs, tᵀt, r~ᵀs, r~ᵀt, sᵀs} -> ω, ρ_new, ||r||², test
    // pipelined Bi-CGSTAB (pipe.cuh; NEXT-4): two reductions per iteration
    STAGE_PIPE_INIT = 6,    // {r~ᵀw0} -> α0
    STAGE_PIPE_OMEGA = 7,   // R1 {qᵀy, yᵀy} -> ω
    STAGE_PIPE_RHO = 8      // R2 {r~ᵀr, r~ᵀw, r~ᵀS, r~ᵀz, rᵀr} -> test, β, α
};

// Executed by a single thread once the global Dot2 values are known.
__device__ __forceinline__ void stage_update(DevState* st, int stage, const double* v,
                                             double* hist, double* scal)
{
    switch (stage) {
    case STAGE_SETUP: {
        st->nb = sqrt(v[0]);
        st->rho = v[1];
        st->iter = 0;
        if (st->nb == 0.0) {                     // b = 0 (R26)
            hist[0] = 0.0;
            st->rel = 0.0;
            st->done = DONE_OK;
            break;
        }
        st->rel = sqrt(v[1]) / st->nb;           // R26: rel_0 (= 1 for x0 = 0)
        hist[0] = st->rel;
        st->done = (st->fixed_iters <= 0 && st->rel < st->tol) ? DONE_OK : DONE_RUNNING;
        break;
    }
    case STAGE_ALPHA: {
        const int i = st->iter + 1;
        double* sc = scal + 8 * (i - 1);
        const double rw = v[0];
        st->rw = rw;
        sc[0] = rw;
        if (rw == 0.0 || !isfinite(rw)) {        // R7: stop before any update
            st->done = DONE_BREAKDOWN;
            break;
        }
        st->alpha = st->rho / rw;
        sc[1] = st->alpha;
        break;
    }
    case STAGE_OMEGA: {
        const int i = st->iter + 1;
        double* sc = scal + 8 * (i - 1);
        st->ts = v[0];
        st->tt = v[1];
        st->omega = (v[1] == 0.0) ? 0.0 : v[0] / v[1];   // P:293, R6
        sc[2] = v[0];
        sc[3] = v[1];
        sc[4] = st->omega;
        break;
    }
    case STAGE_RHO: {
        const int i = st->iter + 1;
        double* sc = scal + 8 * (i - 1);
        const double rho_new = v[0], rr = v[1];
        st->rho_new = rho_new;
        st->rr = rr;
        const double rel = sqrt(rr) / st->nb;    // R4
        st->rel = rel;
        st->iter = i;
        hist[i] = rel;
        sc[5] = rho_new;
        sc[6] = rr;
        sc[7] = 0.0;
        if (st->fixed_iters > 0) {
            if (i == st->fixed_iters) { st->done = DONE_OK; break; }
        } else if (rel < st->tol) {
            st->done = DONE_OK;
            break;
        }
        if (st->omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new) || !isfinite(rr) ||
            !isfinite(st->omega)) {
            st->done = DONE_BREAKDOWN;
            break;
        }
        const double beta = (rho_new / st->rho) * (st->alpha / st->omega);   // R20
        st->beta = beta;
        st->rho = rho_new;
        sc[7] = beta;
        if (st->fixed_iters <= 0 && i >= st->max_iter) st->done = DONE_MAXIT;
        break;
    }
    case STAGE_PIPE_INIT: {
        st->den = v[0];
        st->beta = 0.0;
        st->omega = 0.0;
        if (v[0] == 0.0 || !isfinite(v[0])) {    // R7
            st->done = DONE_BREAKDOWN;
            break;
        }
        st->alpha = st->rho / v[0];
        break;
    }
    case STAGE_PIPE_OMEGA: {
        const int i = st->iter + 1;
        double* sc = scal + 8 * (i - 1);
        sc[0] = st->den;
        sc[1] = st->alpha;
        st->ts = v[0];
        st->tt = v[1];
        st->omega = (v[1] == 0.0) ? 0.0 : v[0] / v[1];   // R6
        sc[2] = v[0];
        sc[3] = v[1];
        sc[4] = st->omega;
        break;
    }
    case STAGE_PIPE_RHO: {
        const int i = st->iter + 1;
        double* sc = scal + 8 * (i - 1);
        const double rho_new = v[0], rw = v[1], rS = v[2], rz = v[3], rr = v[4];
        st->rho_new = rho_new;
        st->rr = rr;
        const double rel = sqrt(rr) / st->nb;    // R4
        st->rel = rel;
        st->iter = i;
        hist[i] = rel;
        sc[5] = rho_new;
        sc[6] = rr;
        sc[7] = 0.0;
        if (st->fixed_iters > 0) {
            if (i == st->fixed_iters) { st->done = DONE_OK; break; }
        } else if (rel < st->tol) {
            st->done = DONE_OK;
            break;
        }
        const double omega = st->omega;
        if (omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new) || !isfinite(rr) ||
            !isfinite(omega)) {
            st->done = DONE_BREAKDOWN;
            break;
        }
        const double beta = (rho_new / st->rho) * (st->alpha / omega);   // R20
        st->beta = beta;
        st->rho = rho_new;
        sc[7] = beta;
        const double den = fma(beta, fma(-omega, rz, rS), rw);
        st->den = den;
        if (den == 0.0 || !isfinite(den)) {
            st->done = DONE_BREAKDOWN;
            break;
        }
        st->alpha = rho_new / den;
        if (st->fixed_iters <= 0 && i >= st->max_iter) st->done = DONE_MAXIT;
        break;
    }
    case STAGE_OMEGA2: {
        // MPI4 + MPI5 in one reduction: r = s - ω t gives
        // r~ᵀr = r~ᵀs - ω r~ᵀt and ||r||² = sᵀs - 2ω tᵀs + ω² tᵀt (clamped at 0).  The stop
        // is recorded in `pend` and applied after the x / r update kernel (k_commit).
        const int i = st->iter + 1;
        double* sc = scal + 8 * (i - 1);
        const double ts = v[0], tt = v[1];
        st->ts = ts;
        st->tt = tt;
        const double omega = (tt == 0.0) ? 0.0 : ts / tt;   // P:293, R6
        st->omega = omega;
        sc[2] = ts;
        sc[3] = tt;
        sc[4] = omega;
        const double rho_new = fma(-omega, v[3], v[2]);
        double rr = fma(-omega, fma(-omega, tt, 2.0 * ts), v[4]);
        if (rr < 0.0) rr = 0.0;
        st->rho_new = rho_new;
        st->rr = rr;
        const double rel = sqrt(rr) / st->nb;    // R4
        st->rel = rel;
        st->iter = i;
        hist[i] = rel;
        sc[5] = rho_new;
        sc[6] = rr;
        sc[7] = 0.0;
        if (st->fixed_iters > 0) {
            if (i == st->fixed_iters) { st->pend = DONE_OK; break; }
        } else if (rel < st->tol) {
            st->pend = DONE_OK;
            break;
        }
        if (omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new) || !isfinite(rr) ||
            !isfinite(omega)) {
            st->pend = DONE_BREAKDOWN;
            break;
        }
        const double beta = (rho_new / st->rho) * (st->alpha / omega);   // R20
        st->beta = beta;
        st->rho = rho_new;
        sc[7] = beta;
        if (st->fixed_iters <= 0 && i >= st->max_iter) st->pend = DONE_MAXIT;
        break;
    }
    default: {
        st->scratch[0] = v[0];
        st->scratch[1] = v[1];
        break;
    }
    }
}

// Completion of a reduction stage from the combined Dot2 triples (one thread): certified
// values go straight to the stage's scalar update; otherwise the stage is parked
// (DONE_PENDING, or pend_mask alone for the stand-alone STAGE_DOT) for the exact path.
// D = depth bound of the summation chains, nprod = number of products per dot (R19).
// self_mask bit d: dot d is a·a (no Σ|h| accumulated): its terms are >= 0, so
// Σ|a_i a_i| = Σ a_i a_i <= |hi + mid + lo| + E, and the bound holds with 1.001 |...|.
// k3_mask bit d: dot d was accumulated with Dot3 chains (dd.cuh).
__device__ __forceinline__ void finish_stage(DevState* st, int stage, int nd, const dd* comb,
                                             int D, double nprod, int self_mask, int k3_mask,
                                             double* hist, double* scal)
{
    double v[5] = {0, 0, 0, 0, 0};
    int mask = 0;
    for (int d = 0; d < nd; ++d) {
        const dd& c = comb[d];
        const double ab = (self_mask >> d) & 1 ? fabs((c.hi + c.mid) + c.lo) * 1.001 + 0x1p-1022
                                               : c.ab;
        double r, o, E;
        const bool ok = dd_certify(c, ab, D, nprod, (k3_mask >> d) & 1, &v[d], &r, &o, &E);
        if (!ok) {
            const double ar = fabs(r);
            const long long bits = __double_as_longlong(ar);
            const double cl[9] = {(double)stage, (double)d, (double)D, r, o, E,
                                  __longlong_as_double(bits + 1) - ar,
                                  bits > 0 ? ar - __longlong_as_double(bits - 1) : 0.0, ab};
            for (int i = 0; i < 9; ++i) st->cert_last[i] = cl[i];
            st->n_refused += 1;
        }
        if (!ok || st->exact_mode) mask |= 1 << d;
    }
    if (mask) {
        st->pend_stage = stage;
        st->pend_mask = mask;
        for (int d = 0; d < 5; ++d) st->pend_v[d] = v[d];
        if (stage != STAGE_DOT) st->done = DONE_PENDING;
        return;
    }
    stage_update(st, stage, v, hist, scal);
}

