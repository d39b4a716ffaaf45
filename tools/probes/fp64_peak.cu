// FP64 throughput probe on B200: DFMA (FP64 pipe) vs DMMA (mma.sync m8n8k4
// f64 tensor-core path).  Evaluates the north star's question of whether the
// n <= 16 contractions would gain from FP64 tensor cores.
// Build/run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b)
{
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = threadIdx.x + q;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += x[q];
    if (s == 1.2345) out[0] = s;
}

__global__ void dmma_kernel(double* out, double a0, double b0)
{
    double a = a0 + threadIdx.x, b = b0;
    double c[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q][0] = c[q][1] = 0.0;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
    if (s == 1.2345) out[0] = s;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        dfma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double dfma_flops = 2.0 * blocks * threads * kIters * 8;
        dmma_kernel<<<blocks, threads>>>(out, 1.0, 1e-9);
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, 1.0, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms2;
        cudaEventElapsedTime(&ms2, e0, e1);
        const double dmma_flops = 2.0 * 8 * 8 * 4 * (blocks * threads / 32) * (double)kIters * 4;
        if (rep == 1)
            printf("{\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"sms\": %d}\n",
                   dfma_flops / ms / 1e9, dmma_flops / ms2 / 1e9, sms);
    }
    return 0;
}
