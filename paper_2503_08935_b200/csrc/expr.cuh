// expr.cuh -- the per-point expression trees of the arithmetic contract,
// shared by every CUDA kernel so that all kernel variants are bitwise identical by
// construction.  The paper's expressions evaluated with fused multiply-adds where written
// (fma = one rounding).  The whole library is built with --fmad=false: no other contraction.
#pragma once

// R17: 7-point operator row (Eq. 3 / Eq. 6), uniform spacing.
__device__ __forceinline__ double stencil_row(double c, double xm, double xp, double ym,
                                              double yp, double zm, double zp, double h2inv)
{
    const double nb = ((((xm + xp) + ym) + yp) + zm) + zp;
    return fma(6.0, c, -nb) * h2inv;
}

// R18: KernelCI1 (P:353-354 / Alg. 2 l.4): y = 2(ρ1/δ)(2b - Ab/θ) = g1 * (2q - S*cz)
__device__ __forceinline__ double cheb_first(double q, double S, double g1, double cz)
{
    return g1 * fma(-S, cz, 2.0 * q);
}

// R18: KernelCI2 (P:360 / Alg. 2 l.8): w = ρ_cur (2σ y + (2/δ)(b - A y) - ρ_old z)
__device__ __forceinline__ double cheb_step(double q, double S, double y, double z, double rho_j,
                                            double rho_jm1, double A2, double B2)
{
    return rho_j * fma(-rho_jm1, z, fma(A2, y, B2 * (q - S)));
}

// R20: vector updates of Alg. 3
__device__ __forceinline__ double upd_s(double r, double w, double alpha)
{
    return fma(-alpha, w, r);
}
__device__ __forceinline__ double upd_x(double x, double ph, double rh, double alpha,
                                        double omega)
{
    return fma(omega, rh, fma(alpha, ph, x));
}
__device__ __forceinline__ double upd_r(double s, double t, double omega)
{
    return fma(-omega, t, s);
}
__device__ __forceinline__ double upd_p(double r, double p, double w, double beta,
                                        double omega)
{
    return fma(beta, fma(-omega, w, p), r);
}
