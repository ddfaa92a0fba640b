// gemm_v1.cu -- instantiation unit of the K2 kernel for variant 1 (see gemm.cu).
#include "gemm_impl.cuh"

namespace bf16x {
BF16X_DEFINE_VARIANT(1)
}  // namespace bf16x
