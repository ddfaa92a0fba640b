// gemm_v5.cu -- instantiation unit of the K2 kernel for variant 5 (see gemm.cu).
#include "gemm_impl.cuh"

namespace bf16x {
BF16X_DEFINE_VARIANT(5)
}  // namespace bf16x
