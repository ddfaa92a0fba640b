// gemm_v9.cu -- instantiation unit of the K2 kernel for variant 9 (see gemm.cu).
#include "gemm_impl.cuh"

namespace bf16x {
BF16X_DEFINE_VARIANT(9)
}  // namespace bf16x
