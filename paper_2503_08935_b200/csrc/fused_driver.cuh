// fused_driver.cuh -- driver side of the fused path (filled in by the performance path).
#pragma once
namespace fused {
bcgs_status iteration(bcgs_ctx c) { return iteration_ref(c); }
void on_begin(bcgs_ctx) {}
bool precond_supported(bcgs_ctx) { return false; }
bcgs_status precond_apply(bcgs_ctx c, const double* q, double* out)
{
    return precond_ref(c, q, out, nullptr);
}
}  // namespace fused
