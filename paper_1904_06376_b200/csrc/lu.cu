// lu.cu -- LU with partial pivoting + FP64 iterative refinement (section III).
#include "common.cuh"
#include "kernels.cuh"

extern "C" int bf16x_gesv_ir(int n, const float *A, int lda, const double *b, double *x, int variant, int nb,
                             int max_iter, double *residual_history, bf16x_ir_report *report) {
    if (n < 0) return -1;
    if (lda < (n > 1 ? n : 1)) return -3;
    if (variant != 3 && variant != 6 && variant != 9) return -6;
    if (!report) return -10;
    (void)A; (void)b; (void)x; (void)nb; (void)max_iter; (void)residual_history;
    return BF16X_ERR_CUDA;  // implemented in a later milestone
}
