// gemm_v7.cu -- instantiation unit of the K2 kernel for variant 7 (see gemm.cu).
#include "gemm_impl.cuh"

namespace bf16x {
BF16X_DEFINE_VARIANT(7)
}  // namespace bf16x
