// Feasibility probe: two green contexts (a 16-SM partition + the rest) on one B200, a 16-CTA
// cluster kernel in the small one running concurrently with a grid-filling kernel in the big
// one.  Prints partition sizes and both kernels' %globaltimer windows.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char *s; cuGetErrorString(r_, &s); \
    printf("%s failed: %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(e_)); \
    return 1; } } while (0)

__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void __cluster_dims__(16, 1, 1) panel_like(unsigned long long *out, int iters) {
    unsigned long long t0 = gt();
    float x = threadIdx.x;
    for (int i = 0; i < iters; ++i) x = x * 1.0000001f + 0.5f;
    if (threadIdx.x == 0) { out[2 * blockIdx.x] = t0; out[2 * blockIdx.x + 1] = gt(); }
    if (x == 12345.f) out[0] = 0;
}

__global__ void big_like(unsigned long long *out, int iters) {
    unsigned long long t0 = gt();
    float x = threadIdx.x;
    for (int i = 0; i < iters; ++i) x = x * 1.0000001f + 0.5f;
    if (threadIdx.x == 0) { out[2 * blockIdx.x] = t0; out[2 * blockIdx.x + 1] = gt(); }
    if (x == 12345.f) out[0] = 0;
}

int main() {
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    RK(cudaSetDevice(0));
    RK(cudaFree(0));   // primary context
    CUdevResource all;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", all.sm.smCount);
    CUdevResource small[1], rest;
    unsigned int ng = 1;
    CK(cuDevSmResourceSplitByCount(small, &ng, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, 16));
    printf("groups %u: small %u SMs, rest %u SMs\n", ng, small[0].sm.smCount, rest.sm.smCount);
    CUdevResourceDesc dsmall, drest;
    CK(cuDevResourceGenerateDesc(&dsmall, small, 1));
    CK(cuDevResourceGenerateDesc(&drest, &rest, 1));
    CUgreenCtx gs, gr;
    CK(cuGreenCtxCreate(&gs, dsmall, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&gr, drest, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream ss, sr;
    CK(cuGreenCtxStreamCreate(&ss, gs, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&sr, gr, CU_STREAM_NON_BLOCKING, 0));
    unsigned long long *buf;
    RK(cudaMalloc(&buf, sizeof(unsigned long long) * 2 * 4096));
    RK(cudaMemset(buf, 0, sizeof(unsigned long long) * 2 * 4096));
    CUcontext cs, cr;
    CK(cuCtxFromGreenCtx(&cs, gs));
    CK(cuCtxFromGreenCtx(&cr, gr));
    int nbig = rest.sm.smCount;
    for (int rep = 0; rep < 2; ++rep) {
        CK(cuCtxSetCurrent(cr));
        big_like<<<nbig, 256, 0, (cudaStream_t)sr>>>(buf + 64, 2000000);
        cudaError_t e1 = cudaGetLastError();
        CK(cuCtxSetCurrent(cs));
        cudaFuncSetAttribute(panel_like, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        panel_like<<<16, 256, 0, (cudaStream_t)ss>>>(buf, 500000);
        cudaError_t e2 = cudaGetLastError();
        printf("launch errors: big %s, panel %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2));
        CK(cuStreamSynchronize(ss));
        CK(cuStreamSynchronize(sr));
    }
    std::vector<unsigned long long> h(2 * 4096);
    CK(cuCtxSetCurrent(cs));
    RK(cudaMemcpy(h.data(), buf, h.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long p0 = ~0ull, p1 = 0, b0 = ~0ull, b1 = 0;
    for (int i = 0; i < 16; ++i) { p0 = std::min(p0, h[2 * i]); p1 = std::max(p1, h[2 * i + 1]); }
    for (int i = 0; i < nbig; ++i) { b0 = std::min(b0, h[64 + 2 * i]); b1 = std::max(b1, h[64 + 2 * i + 1]); }
    unsigned long long t0 = std::min(p0, b0);
    printf("panel-like (16-CTA cluster, small ctx): %.1f .. %.1f us\n", (p0 - t0) / 1e3, (p1 - t0) / 1e3);
    printf("big-like (%d CTAs, rest ctx):           %.1f .. %.1f us\n", nbig, (b0 - t0) / 1e3, (b1 - t0) / 1e3);
    printf("overlap: %s\n", (p0 < b1 && b0 < p1) ? "yes" : "no");
    return 0;
}
