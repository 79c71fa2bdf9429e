// tb_multi_c.cu -- the continuation-pass kernels (MODE_C) of the multi-pass temporal
// blocking, compiled in their own translation unit (parallel nvcc); see tb_multi.cu.
#define TB_MULTI_CONT
#include "tb_multi.cu"
