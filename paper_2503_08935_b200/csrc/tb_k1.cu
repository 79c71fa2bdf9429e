// tb_k1.cu -- instantiates the temporally blocked Chebyshev kernels for degree K = 1.
#include "tb_launch.cuh"

namespace fused {
template bcgs_status launch_variant<1, 0>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<1, 1>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<1, 2>(bcgs_ctx, TbArgs&, int);
}  // namespace fused
