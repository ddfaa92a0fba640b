// Same-box comparators (SURVEY section 0.8 / BASELINE.md section 3): cuBLAS FP32 SGEMM (pedantic, no
// TF32), cuBLAS's own Blackwell FP32 emulation (CUBLAS_COMPUTE_32F_EMULATED_16BFX9), and this
// repository's bf16x3/x6/x8/x9 through its C ABI, on the same device inputs.  Accuracy is the
// north-star normwise error ||C - C64||_F / (||A||_F ||B||_F) with C64 from cuBLAS DGEMM.
//
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -I include tools/cublas_compare.cu \
//        -L/usr/local/cuda/lib64 -lcublas -Lpaper_1904_06376_b200 -lbf16x -o tools/cublas_compare
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bf16x.h"

#define CK(x)                                                                       \
    do {                                                                            \
        auto _e = (x);                                                              \
        if ((int)_e != 0) { fprintf(stderr, "%s:%d %s -> %d\n", __FILE__, __LINE__, #x, (int)_e); exit(1); } \
    } while (0)

// counter-based uniform [-1, 1): FP64 draw rounded to FP32 (splitmix64 of the index)
__global__ void fill_uniform(float *x, size_t n, unsigned long long seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (i + 1);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
        x[i] = (float)(2.0 * u - 1.0);
    }
}
__global__ void to_double(const float *x, double *y, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        y[i] = (double)x[i];
}
__global__ void diff_sq(const float *c, const double *c64, size_t n, double *out) {
    __shared__ double s[256];
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double d = (double)c[i] - c64[i];
        acc += d * d;
    }
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) atomicAdd(out, s[0]);
}

static double norm_f32(const float *x, size_t n) {
    std::vector<float> h(n);
    CK(cudaMemcpy(h.data(), x, n * 4, cudaMemcpyDeviceToHost));
    double s = 0;
    for (float v : h) s += (double)v * v;
    return std::sqrt(s);
}

template <class F>
static double time_ms(F f, int iters = 10) {
    for (int i = 0; i < 3; ++i) f();
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> ts;
    for (int i = 0; i < iters; ++i) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

int main(int argc, char **argv) {
    std::vector<int> sizes = {4096, 8192};
    if (argc > 1) {
        sizes.clear();
        for (int i = 1; i < argc; ++i) sizes.push_back(atoi(argv[i]));
    }
    cublasHandle_t h;
    CK(cublasCreate(&h));
    for (int n : sizes) {
        const size_t nn = (size_t)n * n;
        float *A, *B, *C;
        double *A64, *B64, *C64, *err;
        CK(cudaMalloc(&A, nn * 4)); CK(cudaMalloc(&B, nn * 4)); CK(cudaMalloc(&C, nn * 4));
        CK(cudaMalloc(&A64, nn * 8)); CK(cudaMalloc(&B64, nn * 8)); CK(cudaMalloc(&C64, nn * 8));
        CK(cudaMalloc(&err, 8));
        fill_uniform<<<1184, 256>>>(A, nn, 1);
        fill_uniform<<<1184, 256>>>(B, nn, 2);
        to_double<<<1184, 256>>>(A, A64, nn);
        to_double<<<1184, 256>>>(B, B64, nn);
        const double one64 = 1.0, zero64 = 0.0;
        CK(cublasSetMathMode(h, CUBLAS_DEFAULT_MATH));
        CK(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one64, A64, n, B64, n, &zero64, C64, n));
        const double den = norm_f32(A, nn) * norm_f32(B, nn);
        auto error = [&]() {
            CK(cudaMemset(err, 0, 8));
            diff_sq<<<1184, 256>>>(C, C64, nn, err);
            double e;
            CK(cudaMemcpy(&e, err, 8, cudaMemcpyDeviceToHost));
            return std::sqrt(e) / den;
        };
        const float one = 1.f, zero = 0.f;
        const double flops = 2.0 * n * (double)n * n;
        auto report = [&](const char *name, double ms) {
            printf("{\"n\": %d, \"impl\": \"%s\", \"ms\": %.4f, \"tflops\": %.2f, \"normwise_error\": %.3e}\n", n, name,
                   ms, flops / ms / 1e9, error());
            fflush(stdout);
        };
        // cuBLAS FP32, pedantic (no TF32)
        CK(cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH));
        double ms = time_ms([&] {
            CK(cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, CUDA_R_32F, n, B, CUDA_R_32F, n, &zero, C,
                            CUDA_R_32F, n, CUBLAS_COMPUTE_32F_PEDANTIC, CUBLAS_GEMM_DEFAULT));
        });
        report("cublas_sgemm_fp32", ms);
        // cuBLAS BF16x9 FP32 emulation
        CK(cublasSetMathMode(h, CUBLAS_DEFAULT_MATH));
        CK(cublasSetEmulationStrategy(h, CUBLAS_EMULATION_STRATEGY_EAGER));
        ms = time_ms([&] {
            CK(cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, CUDA_R_32F, n, B, CUDA_R_32F, n, &zero, C,
                            CUDA_R_32F, n, CUBLAS_COMPUTE_32F_EMULATED_16BFX9, CUBLAS_GEMM_DEFAULT));
        });
        report("cublas_emulated_bf16x9", ms);
        // this repository, through the C ABI (split + GEMM per call)
        for (int v : {3, 6, 8, 9}) {
            ms = time_ms([&] { CK(bf16x_gemm(n, n, n, 1.f, A, n, B, n, 0.f, C, n, v)); });
            char name[32];
            snprintf(name, sizeof(name), "bf16x%d", v);
            report(name, ms);
        }
        cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(A64); cudaFree(B64); cudaFree(C64); cudaFree(err);
    }
    cublasDestroy(h);
    return 0;
}
