// microbench_fp64.cu — FP64 latency / throughput on the B200 (design input
// for the integrator).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// --fmad=false scripts/microbench_fp64.cu -o /tmp/mb && /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__device__ __forceinline__ double op(double a, double b) {
    if (OP == 0) return a + b;          // DADD
    if (OP == 1) return a * b;          // DMUL
    if (OP == 2) return fma(a, b, 1e-300);  // DFMA
    double r;                           // MUFU.RCP64H (approx)
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    return r + 0.0 * b;
}

// latency: one thread, dependent chain
template <int OP>
__global__ void lat(double* out, long long* cyc, int n, double b) {
    double x = out[0];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = op<OP>(x, b);
    long long t1 = clock64();
    out[1] = x;
    cyc[0] = t1 - t0;
}

// throughput: ILP independent chains per thread, all threads of the grid
template <int OP, int ILP>
__global__ void thr(double* out, int n, double b) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = 1.0 + threadIdx.x * 1e-9 + k;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = op<OP>(x[k], b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    if (s == 1.2345) out[blockIdx.x] = s;
}

__global__ void lds_lat(long long* cyc, int n) {
    __shared__ unsigned idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    unsigned p = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) p = idx[p];
    long long t1 = clock64();
    if (p == 12345) cyc[1] = p;
    cyc[0] = t1 - t0;
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 1 << 20);
    cudaMalloc(&c, 64);
    double h[2] = {1.0, 0};
    cudaMemcpy(d, h, 16, cudaMemcpyHostToDevice);
    const char* names[4] = {"DADD", "DMUL", "DFMA", "MUFU.RCP64H"};
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int o = 0; o < 4; ++o) {
        long long cy;
        const int n = 4096;
        auto L = o == 0 ? lat<0> : o == 1 ? lat<1> : o == 2 ? lat<2> : lat<3>;
        L<<<1, 1>>>(d, c, n, 1.0000001);
        L<<<1, 1>>>(d, c, n, 1.0000001);
        cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("%-12s dependent latency: %.2f cycles\n", names[o], double(cy) / n);
    }
    {
        long long cy;
        lds_lat<<<1, 32>>>(c, 4096);
        lds_lat<<<1, 32>>>(c, 4096);
        cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("LDS.32 pointer-chase latency: %.2f cycles\n", double(cy) / 4096);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int o = 0; o < 3; ++o)
        for (int warps_per_sm : {4, 8, 16, 32}) {
            for (int ilp : {1, 2, 4, 8}) {
                const int n = 1 << 12;
                void (*k)(double*, int, double) = nullptr;
#define PICK(OP) \
    k = ilp == 1 ? thr<OP, 1> : ilp == 2 ? thr<OP, 2> : ilp == 4 ? thr<OP, 4> : thr<OP, 8>;
                if (o == 0) { PICK(0) } else if (o == 1) { PICK(1) } else { PICK(2) }
                k<<<sms, warps_per_sm * 32>>>(d, n, 1.0000001);
                cudaEventRecord(e0);
                k<<<sms, warps_per_sm * 32>>>(d, n, 1.0000001);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double ops = double(sms) * warps_per_sm * 32 * n * ilp;
                const double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
                printf("%-5s warps/SM %2d ILP %d: %.1f lane-ops/clk/SM (at %d MHz nominal)\n", names[o], warps_per_sm,
                       ilp, per_sm_clk, clk / 1000);
            }
        }
    return 0;
}
