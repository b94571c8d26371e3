// cluster_probe.cu — how many thread-block clusters of each size fit at once
// on this GPU when every CTA takes a whole SM (the cluster integrator's
// shape: ~223 KB of shared memory, 352 threads), and which SMs a full wave
// of 4-CTA clusters leaves idle.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -o scripts/cluster_probe scripts/cluster_probe.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void probe(int* smid_out) {
    extern __shared__ char s[];
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    if (threadIdx.x == 0) {
        s[0] = 1;
        smid_out[blockIdx.x] = id;
    }
    // hold the SM long enough for the whole wave to be resident together
    long long t0 = clock64();
    while (clock64() - t0 < 20000000) {}
}

int main() {
    const size_t smem = 223 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", nsm);
    for (int cl : {1, 2, 3, 4, 5, 6, 7, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl * 64);
        cfg.blockDim = dim3(352);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d SMs busy (%s)\n", cl, n, n * cl,
               e == cudaSuccess ? "ok" : cudaGetErrorString(e));
        if (e != cudaSuccess || n <= 0) { cudaGetLastError(); continue; }
        int* d;
        cudaMalloc(&d, sizeof(int) * n * cl);
        cfg.gridDim = dim3(n * cl);
        e = cudaLaunchKernelEx(&cfg, probe, d);
        cudaDeviceSynchronize();
        std::vector<int> h(n * cl);
        cudaMemcpy(h.data(), d, sizeof(int) * n * cl, cudaMemcpyDeviceToHost);
        std::vector<int> used(nsm, 0);
        for (int x : h) if (x >= 0 && x < nsm) used[x]++;
        std::printf("   idle SMs:");
        for (int i = 0; i < nsm; ++i) if (!used[i]) std::printf(" %d", i);
        std::printf("\n   clusters (smids):");
        for (int c = 0; c < std::min(n, 40); ++c) {
            std::printf(" [");
            for (int k = 0; k < cl; ++k) std::printf("%s%d", k ? "," : "", h[c * cl + k]);
            std::printf("]");
        }
        std::printf("\n");
        cudaFree(d);
    }
    return 0;
}
