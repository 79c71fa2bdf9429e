// tb_k3.cu -- instantiates the temporally blocked Chebyshev kernels for degree K = 3.
#include "tb_launch.cuh"

namespace fused {
template bcgs_status launch_variant<3, 0>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<3, 1>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<3, 2>(bcgs_ctx, TbArgs&, int);
}  // namespace fused
