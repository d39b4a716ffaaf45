// Back-to-back eager launch rate of an (almost) empty kernel with a small vs
// an 7.7 KB parameter struct (the size of the Ax kernel's folded-D block).
#include <cstdio>
#include <cuda_runtime.h>

struct Big { double d[960]; };
struct Small { double d[4]; };

__global__ void k_big(Big p, double* out) { if (threadIdx.x == 0 && blockIdx.x == 0 && p.d[7] == 12345.0) *out = p.d[3]; }
__global__ void k_small(Small p, double* out) { if (threadIdx.x == 0 && blockIdx.x == 0 && p.d[1] == 12345.0) *out = p.d[3]; }

int main()
{
    double* out;
    cudaMalloc(&out, 8);
    Big b = {};
    Small s = {};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int N = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        for (int i = 0; i < 100; ++i) k_big<<<4096, 128>>>(b, out);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < N; ++i) k_big<<<4096, 128>>>(b, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float mb = 0;
        cudaEventElapsedTime(&mb, e0, e1);
        for (int i = 0; i < 100; ++i) k_small<<<4096, 128>>>(s, out);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < N; ++i) k_small<<<4096, 128>>>(s, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"us_per_launch_big_params\": %.3f, \"us_per_launch_small_params\": %.3f}\n",
               mb * 1e3 / N, ms * 1e3 / N);
    }
    return 0;
}
