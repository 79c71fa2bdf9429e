// k_fused.cuh -- fused / temporally blocked kernels (filled in by the performance path).
#pragma once
#include <stdint.h>

namespace fused {
inline int64_t max_blocks(int64_t, int64_t, int64_t) { return 0; }
inline bool supported(int64_t, int64_t, int64_t, int, int, bool) { return false; }
bcgs_status iteration(bcgs_ctx c);
void on_begin(bcgs_ctx c);
bool precond_supported(bcgs_ctx c);
bcgs_status precond_apply(bcgs_ctx c, const double* q, double* out);
}  // namespace fused
