// Per-SM global store bandwidth probe: G CTAs (one per SM at most) each write a 128-row x 256-column
// FP32 block of a column-major 4096-row matrix (the K2 C tile of one CTA, 128 KB) `reps` times over
// fresh blocks, with 16-byte stores (each warp: 512 B runs = one column's 128 rows).  Prints the
// time and the per-CTA / aggregate write rate for G = 8 .. 148.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) store_tiles(float *C, int ldc, int tiles_per_cta, int ntile_cols) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = 0; t < tiles_per_cta; ++t) {
        const int tile = blockIdx.x * tiles_per_cta + t;
        const int tm = tile % 32, tn = tile / 32;          // 32 row-tiles of 128 rows
        float *base = C + (size_t)tn * 256 * ldc + tm * 128;
        // warp w stores columns w, w+8, ...: 128 rows = 32 lanes x float4
        for (int c = warp; c < 256; c += 8) {
            float4 v = make_float4(c, lane, t, 1.f);
            reinterpret_cast<float4 *>(base + (size_t)c * ldc)[lane] = v;
        }
    }
}

int main() {
    const int ldc = 4096, ncols = 8192 * 4;              // 4096 x 32768 FP32 = 512 MB
    float *C;
    cudaMalloc(&C, (size_t)ldc * ncols * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int Gs[] = {8, 16, 37, 74, 148};
    for (int gi = 0; gi < 5; ++gi) {
        const int G = Gs[gi];
        const int tpc = (32 * (ncols / 256)) / G > 32 ? 32 : (32 * (ncols / 256)) / G;
        for (int rep = 0; rep < 3; ++rep) {
            store_tiles<<<G, 256>>>(C, ldc, tpc, ncols / 256);
            cudaEventRecord(e0);
            store_tiles<<<G, 256>>>(C, ldc, tpc, ncols / 256);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = (double)G * tpc * 128 * 256 * 4;
            if (rep == 2)
                printf("G %3d CTAs x %2d tiles of 128 KB: %.1f us, %.1f GB/s per CTA, %.0f GB/s total\n", G, tpc,
                       ms * 1e3, bytes / G / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
