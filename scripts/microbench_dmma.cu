// microbench_dmma.cu — FP64 tensor-core (DMMA, mma.sync .f64) throughput vs
// DFMA on the B200: the measurement behind the decode MLP's NS-1 decision
// (DESIGN.md §3).  tcgen05.mma has no f64 kind, so FP64 MMA on sm_100a is the
// warp-level mma.sync family (m8n8k4 and the sm_90+ m16n8k{4,8,16} shapes).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/microbench_dmma.cu -o /tmp/mbd && /tmp/mbd
//
// Each warp keeps ILP independent accumulator tiles in flight; flops counted
// as 2*M*N*K per mma.  Also reports DFMA (2 flop) with the same grid for a
// side-by-side, and the SASS opcode check is `cuobjdump -sass /tmp/mbd | grep DMMA`.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dmma_m8n8k4(double* out, int n) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 - threadIdx.x * 1e-9;
    double c[ILP][2];
#pragma unroll
    for (int k = 0; k < ILP; ++k) c[k][0] = c[k][1] = 0.0;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += c[k][0] + c[k][1];
    if (s == 1.2345) out[blockIdx.x] = s;
}

template <int ILP>
__global__ void dmma_m16n8k16(double* out, int n) {
    double a[8], b[4];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = 1.0 + (threadIdx.x + q) * 1e-9;
#pragma unroll
    for (int q = 0; q < 4; ++q) b[q] = 0.5 - (threadIdx.x + q) * 1e-9;
    double c[ILP][4];
#pragma unroll
    for (int k = 0; k < ILP; ++k) c[k][0] = c[k][1] = c[k][2] = c[k][3] = 0.0;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
                : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                  "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    if (s == 1.2345) out[blockIdx.x] = s;
}

template <int ILP>
__global__ void dfma(double* out, int n, double b) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = 1.0 + threadIdx.x * 1e-9 + k;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], b, 1e-300);
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    if (s == 1.2345) out[blockIdx.x] = s;
}

template <class F>
static double run(F launch, double flops) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return flops / (best * 1e-3) / 1e12;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* d;
    cudaMalloc(&d, 1 << 20);
    const int n = 4096;
    printf("SMs %d, max SM clock %.0f MHz\n", sms, clk / 1e3);
    for (int wps : {4, 8, 16, 32}) {
        int blocks = sms * 2, threads = wps * 16;  // two CTAs per SM
        double warps = double(blocks) * threads / 32;
        double t;
        t = run([&] { dmma_m8n8k4<4><<<blocks, threads>>>(d, n); }, warps * n * 4 * 2.0 * 8 * 8 * 4);
        printf("DMMA m8n8k4   warps/SM %2d ILP 4: %6.2f TFLOP/s\n", wps, t);
        t = run([&] { dmma_m8n8k4<8><<<blocks, threads>>>(d, n); }, warps * n * 8 * 2.0 * 8 * 8 * 4);
        printf("DMMA m8n8k4   warps/SM %2d ILP 8: %6.2f TFLOP/s\n", wps, t);
        t = run([&] { dmma_m16n8k16<2><<<blocks, threads>>>(d, n / 4); }, warps * (n / 4) * 2 * 2.0 * 16 * 8 * 16);
        printf("DMMA m16n8k16 warps/SM %2d ILP 2: %6.2f TFLOP/s\n", wps, t);
        t = run([&] { dmma_m16n8k16<4><<<blocks, threads>>>(d, n / 4); }, warps * (n / 4) * 4 * 2.0 * 16 * 8 * 16);
        printf("DMMA m16n8k16 warps/SM %2d ILP 4: %6.2f TFLOP/s\n", wps, t);
        t = run([&] { dfma<8><<<blocks, threads>>>(d, n, 0.999); }, double(blocks) * threads * n * 8 * 2.0);
        printf("DFMA          warps/SM %2d ILP 8: %6.2f TFLOP/s\n", wps, t);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
