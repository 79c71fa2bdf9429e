// tb_k8.cu -- instantiates the temporally blocked Chebyshev kernels for degree K = 8.
#include "tb_launch.cuh"

namespace fused {
template bcgs_status launch_variant<8, 0>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<8, 1>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<8, 2>(bcgs_ctx, TbArgs&, int);
}  // namespace fused
