// tb_k5.cu -- instantiates the temporally blocked Chebyshev kernels for degree K = 5.
#include "tb_launch.cuh"

namespace fused {
template bcgs_status launch_variant<5, 0>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<5, 1>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<5, 2>(bcgs_ctx, TbArgs&, int);
}  // namespace fused
