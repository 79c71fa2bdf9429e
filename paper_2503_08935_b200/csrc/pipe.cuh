// pipe.cuh -- element-wise kernels of the pipelined Bi-CGSTAB (BCGS_OPT_PIPELINED; SURVEY
// §8(f) NEXT-4, the paper's "communication-avoiding/reducing algorithms" future work).
// The recurrences of the communication-hiding p-BiCGStab (Cools & Vanroose) for the right-
// preconditioned operator B = A M^-1, written out from Alg. 3; the oracle twin is
// bcgs_oracle.c pbicgstab, with the same expression trees (fma where written):
//   a + β (b - ω c) = fma(β, fma(-ω, c, b), a),  q = fma(-α, S, r), ...
// Two reductions per iteration: R1 = (q, y), (y, y) after k_pipe_a; R2 = (r~, r), (r~, w),
// (r~, S), (r~, z), (r, r) after k_pipe_b.  Neither depends on the preconditioner + stencil
// application that follows it (ẑ, v = A ẑ after R1; ŵ, t = A ŵ after R2).
#pragma once
#include "dd.cuh"
#include "state.cuh"

namespace pbcg {

#define PIPE_LOOP(n)                                                                        \
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < (n);               \
         c += (int64_t)gridDim.x * blockDim.x)

// p, p̂, S, Ŝ, z recurrences, then q, q̂, y; partials (q, y) [Dot2], (y, y) [self]
__global__ void __launch_bounds__(256) k_pipe_a(
    double* __restrict__ p, double* __restrict__ ph, double* __restrict__ S,
    double* __restrict__ Sh, double* __restrict__ z, const double* __restrict__ zh,
    const double* __restrict__ v, const double* __restrict__ r, const double* __restrict__ rh,
    const double* __restrict__ w, const double* __restrict__ wh, const double* __restrict__ t,
    double* __restrict__ q, double* __restrict__ qh, double* __restrict__ y, int64_t n,
    dd* __restrict__ part, const DevState* __restrict__ st)
{
    if (st->done) return;
    const double alpha = st->alpha, beta = st->beta, omega = st->omega;
    double P[2] = {0, 0}, M[2] = {0, 0}, Sx[2] = {0, 0}, AB[2] = {0, 0};
    PIPE_LOOP(n)
    {
        const double rc = r[c], rhc = rh[c], wc = w[c], whc = wh[c];
        const double pn = fma(beta, fma(-omega, S[c], p[c]), rc);
        const double phn = fma(beta, fma(-omega, Sh[c], ph[c]), rhc);
        const double Sn = fma(beta, fma(-omega, z[c], S[c]), wc);
        const double Shn = fma(beta, fma(-omega, zh[c], Sh[c]), whc);
        const double zn = fma(beta, fma(-omega, v[c], z[c]), t[c]);
        p[c] = pn;
        ph[c] = phn;
        S[c] = Sn;
        Sh[c] = Shn;
        z[c] = zn;
        const double qn = fma(-alpha, Sn, rc);
        const double yn = fma(-alpha, zn, wc);
        q[c] = qn;
        qh[c] = fma(-alpha, Shn, rhc);
        y[c] = yn;
        dot2_acc(P[0], Sx[0], AB[0], qn, yn);
        dot2_acc_self(P[1], Sx[1], yn);
    }
    block_reduce_dd<2>(P, M, Sx, AB, part + (int64_t)blockIdx.x * 2);
}

// x, r, r̂, w updates; partials (r~, r), (r~, w), (r~, S), (r~, z) [Dot3], (r, r) [self]
__global__ void __launch_bounds__(256) k_pipe_b(
    double* __restrict__ x, double* __restrict__ r, double* __restrict__ rh,
    double* __restrict__ w, const double* __restrict__ ph, const double* __restrict__ qh,
    const double* __restrict__ q, const double* __restrict__ y, const double* __restrict__ zh,
    const double* __restrict__ wh, const double* __restrict__ t, const double* __restrict__ v,
    const double* __restrict__ rt, const double* __restrict__ S, const double* __restrict__ z,
    int64_t n, dd* __restrict__ part, const DevState* __restrict__ st)
{
    if (st->done) return;
    const double alpha = st->alpha, omega = st->omega;
    double P[5] = {0, 0, 0, 0, 0}, M[5] = {0, 0, 0, 0, 0}, Sx[5] = {0, 0, 0, 0, 0},
           AB[5] = {0, 0, 0, 0, 0};
    PIPE_LOOP(n)
    {
        x[c] = fma(omega, qh[c], fma(alpha, ph[c], x[c]));
        const double rn = fma(-omega, y[c], q[c]);
        r[c] = rn;
        rh[c] = fma(-omega, fma(-alpha, zh[c], wh[c]), qh[c]);
        const double wn = fma(-omega, fma(-alpha, v[c], t[c]), y[c]);
        w[c] = wn;
        const double rtc = rt[c];
        dot3_acc(P[0], M[0], Sx[0], AB[0], rtc, rn);
        dot3_acc(P[1], M[1], Sx[1], AB[1], rtc, wn);
        dot3_acc(P[2], M[2], Sx[2], AB[2], rtc, S[c]);
        dot3_acc(P[3], M[3], Sx[3], AB[3], rtc, z[c]);
        dot2_acc_self(P[4], Sx[4], rn);
    }
    block_reduce_dd<5>(P, M, Sx, AB, part + (int64_t)blockIdx.x * 5);
}

#undef PIPE_LOOP

}  // namespace pbcg
