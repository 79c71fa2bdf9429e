// tb_k7.cu -- instantiates the temporally blocked Chebyshev kernels for degree K = 7.
#include "tb_launch.cuh"

namespace fused {
template bcgs_status launch_variant<7, 0>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<7, 1>(bcgs_ctx, TbArgs&, int);
template bcgs_status launch_variant<7, 2>(bcgs_ctx, TbArgs&, int);
}  // namespace fused
