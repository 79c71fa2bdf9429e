// tb_k6.cu -- instantiates the temporally blocked Chebyshev kernels for degree K = 6.
#include "tb_launch.cuh"

namespace fused {
template bcgs_status launch_variant<6, 0>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<6, 1>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<6, 2>(bcgs_ctx, TbArgs&, int);
}  // namespace fused
