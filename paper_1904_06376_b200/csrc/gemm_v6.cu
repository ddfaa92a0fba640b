// gemm_v6.cu -- instantiation unit of the K2 kernel for variant 6 (see gemm.cu).
#include "gemm_impl.cuh"

namespace bf16x {
BF16X_DEFINE_VARIANT(6)
}  // namespace bf16x
