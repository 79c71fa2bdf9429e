// tb_k4.cu -- instantiates the temporally blocked Chebyshev kernels for degree K = 4.
#include "tb_launch.cuh"

namespace fused {
template bcgs_status launch_variant<4, 0>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<4, 1>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<4, 2>(bcgs_ctx, TbArgs&, int);
}  // namespace fused
