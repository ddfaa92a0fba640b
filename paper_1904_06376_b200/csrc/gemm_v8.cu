// gemm_v8.cu -- instantiation unit of the K2 kernel for variant 8 (see gemm.cu).
#include "gemm_impl.cuh"

namespace bf16x {
BF16X_DEFINE_VARIANT(8)
}  // namespace bf16x
