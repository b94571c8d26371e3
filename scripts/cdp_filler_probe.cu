// cdp_filler_probe.cu — can a persistent grid of 4-CTA clusters (one CTA per
// SM, the cluster integrator's shape) launch, from the device, a one-SM
// "filler" grid that runs CONCURRENTLY on the SMs no 4-CTA cluster can use?
// Variants: (a) device launch (CUDA dynamic parallelism, fire-and-forget) by
// the last cluster to start; (b) host launch on a second stream after the
// cluster grid.  Prints the filler CTAs' SM ids and start times relative to
// the first cluster start, and whether any filler SM is also a cluster SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true
//        -o scripts/cdp_filler_probe scripts/cdp_filler_probe.cu -lcudadevrt
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    return id;
}

struct Rec {
    unsigned long long t_start, t_end;
    int sm;
};

__global__ void filler(Rec* out, long long spin) {
    extern __shared__ char s[];
    if (threadIdx.x == 0) {
        s[0] = 1;
        out[blockIdx.x].t_start = gtime();
        out[blockIdx.x].sm = static_cast<int>(smid());
    }
    const long long t0 = clock64();
    while (clock64() - t0 < spin) {}
    if (threadIdx.x == 0) out[blockIdx.x].t_end = gtime();
}

__global__ void clusters(Rec* out, int* started, int nclus, Rec* fout, int nfill, size_t fsmem, long long spin,
                         int device_launch) {
    extern __shared__ char s[];
    cg::cluster_group cl = cg::this_cluster();
    const int c = blockIdx.x / 4;
    if (threadIdx.x == 0) {
        s[0] = 1;
        out[blockIdx.x].t_start = gtime();
        out[blockIdx.x].sm = static_cast<int>(smid());
    }
    cl.sync();
    if (device_launch && cl.block_rank() == 0 && threadIdx.x == 0) {
        if (atomicAdd(started, 1) == nclus - 1)  // the last cluster to start
            filler<<<nfill, 1024, fsmem, cudaStreamFireAndForget>>>(fout, spin / 2);
    }
    const long long t0 = clock64();
    while (clock64() - t0 < spin) {}
    cl.sync();
    if (threadIdx.x == 0) out[blockIdx.x].t_end = gtime();
}

int main() {
    const size_t smem = 223 * 1024, fsmem = 100 * 1024;
    cudaFuncSetAttribute(clusters, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(filler, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(352);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(4);
    int nclus = 0;
    cudaOccupancyMaxActiveClusters(&nclus, clusters, &cfg);
    const int nfill = nsm - 4 * nclus;
    std::printf("SMs %d, co-resident 4-CTA clusters %d, filler CTAs %d\n", nsm, nclus, nfill);
    Rec *d, *fd;
    int* started;
    cudaMalloc(&d, sizeof(Rec) * 4 * nclus);
    cudaMalloc(&fd, sizeof(Rec) * nfill);
    cudaMalloc(&started, sizeof(int));
    cudaStream_t side;
    cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    const long long spin = 200000000;  // ~100 ms at 1.9 GHz
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(d, 0, sizeof(Rec) * 4 * nclus);
        cudaMemset(fd, 0, sizeof(Rec) * nfill);
        cudaMemset(started, 0, sizeof(int));
        cudaDeviceSynchronize();
        cfg.gridDim = dim3(4 * nclus);
        cudaError_t e = cudaLaunchKernelEx(&cfg, clusters, d, started, nclus, fd, nfill, fsmem, spin, mode == 0 ? 1 : 0);
        if (mode == 1) filler<<<nfill, 1024, fsmem, side>>>(fd, spin / 2);
        cudaError_t e2 = cudaDeviceSynchronize();
        std::printf("\n%s: launch %s, sync %s\n", mode == 0 ? "device launch (CDP fire-and-forget)" : "host launch, 2nd stream",
                    cudaGetErrorString(e), cudaGetErrorString(e2));
        std::vector<Rec> h(4 * nclus), f(nfill);
        cudaMemcpy(h.data(), d, sizeof(Rec) * h.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(f.data(), fd, sizeof(Rec) * f.size(), cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull, tend = 0;
        std::vector<int> used(nsm, 0);
        for (auto& r : h) {
            t0 = std::min(t0, r.t_start);
            tend = std::max(tend, r.t_end);
            if (r.sm >= 0 && r.sm < nsm) used[r.sm] = 1;
        }
        std::printf("cluster span %.3f ms, last cluster start %.3f ms\n", (tend - t0) * 1e-6,
                    (std::max_element(h.begin(), h.end(), [](const Rec& a, const Rec& b) { return a.t_start < b.t_start; })
                         ->t_start - t0) * 1e-6);
        int overlap = 0;
        for (auto& r : f) {
            std::printf("  filler sm %3d start %+.3f ms end %+.3f ms%s\n", r.sm, (double)(r.t_start - t0) * 1e-6,
                        (double)(r.t_end - t0) * 1e-6, used[r.sm] ? "  (cluster SM!)" : "");
            overlap += used[r.sm];
        }
        std::printf("filler CTAs on cluster SMs: %d\n", overlap);
    }
    return 0;
}
