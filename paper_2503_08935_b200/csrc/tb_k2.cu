// tb_k2.cu -- instantiates the temporally blocked Chebyshev kernels for degree K = 2.
#include "tb_launch.cuh"

namespace fused {
template bcgs_status launch_variant<2, 0>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<2, 1>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<2, 2>(bcgs_ctx, TbArgs&, int);
}  // namespace fused
