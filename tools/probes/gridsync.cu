// Microbenchmark: cost of grid-wide barriers on a cooperative launch (148 CTAs x 256 threads).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_acq(const unsigned *p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_rlx(const unsigned *p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(unsigned *p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void st_rlx(unsigned *p, unsigned v) { asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

template <int MODE>
__global__ void k(unsigned *arrive, unsigned *release, unsigned *counter, int iters) {
    for (int it = 1; it <= iters; ++it) {
        __syncthreads();
        if (MODE == 0) {            // flags + fences (lu.cu design)
            if (threadIdx.x == 0) { __threadfence(); st_rel(arrive + blockIdx.x, it); }
            if (blockIdx.x == 0) {
                for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) while (ld_acq(arrive + i) < (unsigned)it) {}
                __syncthreads();
                if (threadIdx.x == 0) st_rel(release, it);
            }
            if (threadIdx.x == 0) { while (ld_acq(release) < (unsigned)it) {} __threadfence(); }
        } else if (MODE == 1) {     // flags, release/acquire only
            if (threadIdx.x == 0) st_rel(arrive + blockIdx.x, it);
            if (blockIdx.x == 0) {
                for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) while (ld_acq(arrive + i) < (unsigned)it) {}
                __syncthreads();
                if (threadIdx.x == 0) st_rel(release, it);
            }
            if (threadIdx.x == 0) while (ld_acq(release) < (unsigned)it) {}
        } else if (MODE == 2) {     // single atomic counter, monotonic target
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
                const unsigned target = it * gridDim.x;
                while (ld_acq(counter) < target) {}
            }
        } else {                    // relaxed polling + one fence
            if (threadIdx.x == 0) { __threadfence(); atomicAdd(counter, 1); const unsigned target = it * gridDim.x; while (ld_rlx(counter) < target) {} __threadfence(); }
        }
        __syncthreads();
    }
}

int main() {
    unsigned *a, *r, *c;
    cudaMalloc(&a, 4096); cudaMalloc(&r, 64); cudaMalloc(&c, 64);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 2000;
    void (*fns[4])(unsigned *, unsigned *, unsigned *, int) = {k<0>, k<1>, k<2>, k<3>};
    for (int grid : {nsm, nsm / 2, 16}) {
        for (int m = 0; m < 4; ++m) {
            cudaMemset(a, 0, 4096); cudaMemset(r, 0, 64); cudaMemset(c, 0, 64);
            int it = iters;
            void *args[] = {&a, &r, &c, &it};
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void *)fns[m], grid, 256, args, 0, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("grid %3d mode %d: %.3f us per barrier (%s)\n", grid, m, ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
