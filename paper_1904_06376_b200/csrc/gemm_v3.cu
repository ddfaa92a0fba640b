// gemm_v3.cu -- instantiation unit of the K2 kernel for variant 3 (see gemm.cu).
#include "gemm_impl.cuh"

namespace bf16x {
BF16X_DEFINE_VARIANT(3)
}  // namespace bf16x
