// Per-SM store rate while the same SM also loads from L2: G CTAs of 512 threads; warps 0-7 write
// 128 KB column blocks of a 4096-row FP32 matrix (as store_bw.cu), warps 8-15 stream an L2-resident
// 48 MB buffer (as load_bw.cu) for as long as the stores run.  Prints both rates per CTA.  Mode 0:
// stores only (warps 8-15 idle), mode 1: stores + loads.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) mixed(float *C, int ldc, int tiles_per_cta, const float4 *__restrict__ X,
                                             size_t n4, int mode, unsigned *done, unsigned long long *loaded,
                                             float *out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ unsigned s_done;
    if (threadIdx.x == 0) s_done = 0;
    __syncthreads();
    if (warp < 8) {
        for (int t = 0; t < tiles_per_cta; ++t) {
            const int tile = blockIdx.x * tiles_per_cta + t;
            const int tm = tile % 32, tn = tile / 32;
            float *base = C + (size_t)tn * 256 * ldc + tm * 128;
            for (int c = warp; c < 256; c += 8)
                reinterpret_cast<float4 *>(base + (size_t)c * ldc)[lane] = make_float4(c, lane, t, 1.f);
        }
        __syncwarp();
        if (lane == 0) atomicAdd(&s_done, 1u);
    } else if (mode == 1) {
        const size_t per = n4 / gridDim.x;
        const float4 *base = X + (size_t)blockIdx.x * per;
        float acc = 0.f;
        unsigned long long n = 0;
        size_t i = (size_t)(threadIdx.x - 256);
        while (*(volatile unsigned *)&s_done < 8u) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(base + (i + u * 256) % per);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
            i += 8 * 256;
            n += 8;
        }
        atomicAdd(loaded, n * 16ull);
        if (acc == 12345.f) out[0] = acc;
    }
}

int main() {
    const int ldc = 4096, ncols = 8192 * 4;
    float *C, *out;
    float4 *X;
    unsigned *done;
    unsigned long long *loaded, h;
    const size_t xb = 48u << 20;
    cudaMalloc(&C, (size_t)ldc * ncols * 4);
    cudaMalloc(&X, xb);
    cudaMemset(X, 0, xb);
    cudaMalloc(&out, 4);
    cudaMalloc(&done, 4);
    cudaMalloc(&loaded, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int Gs[] = {8, 74, 148};
    for (int mode = 0; mode < 2; ++mode)
        for (int gi = 0; gi < 3; ++gi) {
            const int G = Gs[gi];
            const int tpc = (32 * (ncols / 256)) / G > 32 ? 32 : (32 * (ncols / 256)) / G;
            float ms = 0.f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(loaded, 0, 8);
                cudaEventRecord(e0);
                mixed<<<G, 512>>>(C, ldc, tpc, X, xb / 16, mode, done, loaded, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            cudaMemcpy(&h, loaded, 8, cudaMemcpyDeviceToHost);
            const double sb = (double)tpc * 128 * 256 * 4;
            printf("mode %d (%s) G %3d: %.1f us, stores %.1f GB/s per CTA, loads %.1f GB/s per CTA\n", mode,
                   mode ? "stores + loads" : "stores only", G, ms * 1e3, sb / (ms * 1e-3) / 1e9,
                   (double)h / G / (ms * 1e-3) / 1e9);
        }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
