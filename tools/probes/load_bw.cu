// Per-SM L2 -> SM load bandwidth probe: G CTAs (one per SM at most, 1024 threads, 8 independent
// 16-byte loads in flight per thread) stream an L2-resident 48 MB buffer `reps` times; prints the
// per-CTA and aggregate rate for G = 8 .. 148.  (Companion of store_bw.cu.)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024) load_l2(const float4 *__restrict__ X, size_t n4, int reps, float *out) {
    float acc = 0.f;
    const size_t per = n4 / gridDim.x;
    const float4 *base = X + (size_t)blockIdx.x * per;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = threadIdx.x; i + 7 * 1024 < per; i += 8 * 1024) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(base + i + u * 1024);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    const size_t bytes = 48u << 20, n4 = bytes / 16;
    float4 *X;
    float *out;
    cudaMalloc(&X, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(X, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int Gs[] = {8, 16, 37, 74, 148};
    for (int gi = 0; gi < 5; ++gi) {
        const int G = Gs[gi], reps = 40;
        for (int rep = 0; rep < 3; ++rep) {
            load_l2<<<G, 1024>>>(X, n4, reps, out);
            cudaEventRecord(e0);
            load_l2<<<G, 1024>>>(X, n4, reps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const size_t per = n4 / G;
            const double done = (double)G * (per / (8 * 1024)) * (8 * 1024) * 16.0 * reps;
            if (rep == 2)
                printf("G %3d CTAs: %.1f us, %.1f GB/s per CTA, %.0f GB/s total (L2-resident 48 MB)\n", G, ms * 1e3,
                       done / G / (ms * 1e-3) / 1e9, done / (ms * 1e-3) / 1e9);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
