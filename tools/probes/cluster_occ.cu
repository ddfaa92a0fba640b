// Co-resident clusters per cluster size for a 1-CTA-per-SM kernel (as the GEMM: ~200 KB of shared
// memory per CTA): cudaOccupancyMaxActiveClusters for sizes 1..16 -> how many SMs each size can use.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_dummy(int *p) { extern __shared__ int s[]; if (p) p[blockIdx.x] = s[threadIdx.x]; }

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    printf("SMs %d\n", sms);
    for (int cl = 1; cl <= 16; ++cl) {
        cudaLaunchConfig_t c = {};
        c.gridDim = dim3(cl * (sms / cl));
        c.blockDim = dim3(384);
        c.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cl;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        c.attrs = a;
        c.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &c);
        printf("cluster %2d: %3d clusters = %3d SMs %s\n", cl, n, n * cl, e == cudaSuccess ? "" : cudaGetErrorString(e));
        cudaGetLastError();
    }
    return 0;
}
