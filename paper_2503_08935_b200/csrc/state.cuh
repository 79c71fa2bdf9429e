// state.cuh -- device-resident solver state and the scalar steps of Alg. 3.
// The paper computes α, ω, β on the host after each MPI_Allreduce; here they are
// computed on the device by one thread right after the reduction, so an iteration needs no
// host round trip.  Formulas: R4, R6, R7, R20, R25.
#pragma once
#include <stdint.h>

#include "dd.cuh"

enum : int32_t { DONE_RUNNING = 0, DONE_OK = 1, DONE_BREAKDOWN = 2, DONE_MAXIT = 3 };

struct DevState {
    double rho, alpha, omega, beta, nb;
    double rw, ts, tt, rho_new, rr, rel;
    double tol;
    int32_t iter;         // completed outer iterations
    int32_t done;         // DONE_*
    int32_t fixed_iters;  // > 0: run exactly this many
    int32_t max_iter;
    double scratch[8];    // results of stand-alone dot calls
    int32_t pend;         // 2-sync (R31): stop decided at the ω stage, applied after a11/a12
};

// Reduction stages (one per MPI_Allreduce site of Alg. 3).
enum : int32_t {
    STAGE_SETUP = 0,   // {bᵀb, r~ᵀr0}         Alg. 3 l.4
    STAGE_ALPHA = 1,   // {r~ᵀw}               MPI2 + α
    STAGE_OMEGA = 2,   // {tᵀs, tᵀt}           MPI4 + ω
    STAGE_RHO = 3,     // {r~ᵀr, rᵀr}          MPI5 + test + ρ, β
    STAGE_DOT = 4,     // stand-alone dot -> scratch
    STAGE_OMEGA2 = 5   // 2-sync (R31): {tᵀs, tᵀt, r~ᵀs, r~ᵀt, sᵀs} -> ω, ρ_new, ||r||², test
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
