// FP64 throughput microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64)
// versus plain DFMA. Used to pick the roofline denominator for the FP64
// projection GEMMs (MEASURED_PEAKS.json carries no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            asm volatile(
                "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                : "+d"(c[k][0]), "+d"(c[k][1])
                : "d"(a), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    const double m = 0.999999, ad = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], m, ad);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16}) {
        const int iters = 20000;
        dim3 grid(sms * 2), block(32 * warps);
        dmma_loop<<<grid, block>>>(d, 100);
        cudaEventRecord(e0);
        dmma_loop<<<grid, block>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid.x * warps;
        printf("DMMA warps/cta=%d: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
        dfma_loop<<<grid, block>>>(d, 100);
        cudaEventRecord(e0);
        dfma_loop<<<grid, block>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 8 * (double)iters * grid.x * block.x;
        printf("DFMA warps/cta=%d: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
