// Latency of a dependent chain of warp-wide max reductions: redux.sync (2 per 64-bit key, as
// in the LU sub-panel) vs a 5-step shfl.xor butterfly on the 64-bit key.  One warp, clock64.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t key_redux(uint32_t hi, uint32_t lo) {
    const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return ((uint64_t)mh << 32) | ml;
}
__device__ __forceinline__ uint64_t key_shfl(uint64_t k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t q = __shfl_xor_sync(0xffffffffu, k, o);
        k = q > k ? q : k;
    }
    return k;
}
__global__ void lat(unsigned long long *out, int iters) {
    const int lane = threadIdx.x & 31;
    uint64_t k = ((uint64_t)(lane * 7919u % 32u) << 32) | (0xFFFFFFFFu - lane);
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { k = key_redux((uint32_t)(k >> 32) ^ (uint32_t)(lane * i), (uint32_t)k); }
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) { k = key_shfl(k ^ ((uint64_t)(lane * i) << 32)); }
    long long t2 = clock64();
    // shared-memory round trip + bar.sync of 512 threads
    __shared__ volatile uint32_t sv[32];
    for (int i = 0; i < iters; ++i) { sv[lane] = (uint32_t)k + i; __syncthreads(); k += sv[(lane + 1) & 31]; }
    long long t3 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = k; }
}
int main() {
    unsigned long long *d, h[4];
    cudaMalloc(&d, 32);
    const int it = 1000;
    for (int threads : {32, 512}) {
        lat<<<1, threads>>>(d, it);
        lat<<<1, threads>>>(d, it);
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("threads %3d: redux key %.1f cyc, shfl key %.1f cyc, sts+bar.sync+lds %.1f cyc per step\n", threads,
               (double)h[0] / it, (double)h[1] / it, (double)h[2] / it);
    }
    return 0;
}
