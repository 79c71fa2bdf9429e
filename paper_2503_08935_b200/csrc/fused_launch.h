// fused_launch.h -- launch_variant<K, MODE> is defined in tb_launch.cuh and explicitly
// instantiated once per degree K in tb_k<K>.cu (parallel compilation).
#pragma once
namespace fused {
bool stencil_tma_ok(bcgs_ctx c);   // st_tma.cu
bool tb_tma_ok(bcgs_ctx c);        // st_tma.cu: k_cheb_tb4 usable (segment mode)
template <int ND>
bcgs_status launch_stencil_tma(bcgs_ctx c, const double* v, const double* a, double* out,
                               int kb, int ke, dd* part, int* nparts);
bcgs_status launch_multipass(bcgs_ctx c, TbArgs& a, int mode);   // tb_multi.cu
template <int K, int MODE>
bcgs_status launch_variant(bcgs_ctx c, TbArgs& a, int nz);
#define BCGS_TB_EXTERN(K)                                                  \
    extern template bcgs_status launch_variant<K, 0>(bcgs_ctx, TbArgs&, int); \
    extern template bcgs_status launch_variant<K, 1>(bcgs_ctx, TbArgs&, int); \
    extern template bcgs_status launch_variant<K, 2>(bcgs_ctx, TbArgs&, int);
BCGS_TB_EXTERN(1) BCGS_TB_EXTERN(2) BCGS_TB_EXTERN(3) BCGS_TB_EXTERN(4)
BCGS_TB_EXTERN(5) BCGS_TB_EXTERN(6) BCGS_TB_EXTERN(7) BCGS_TB_EXTERN(8)
}  // namespace fused
