// FP64 peak microbenchmarks on B200 (sm_100a): DFMA (SIMT pipe), DMMA m8n8k4 (warp mma.sync,
// lowered to DMMA.8x8x4), both at once, and shared-memory LDS.64 throughput. Each kernel runs
// long enough (~0.5 s) to reach the sustained clock; times by CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peaks tools/fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b)
{
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters)
{
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void mixed_kernel(double* out, int iters, double a0, double b0)
{
    // even warps DFMA, odd warps DMMA
    if ((threadIdx.x >> 5) & 1) {
        double acc[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
        double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(acc[i], a, b);
        }
        double s = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
        if (s == 12345.678) out[threadIdx.x] = s;
    } else {
        double x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
        for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a0, b0);
        }
        double s = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) s += x[i];
        if (s == 12345.678) out[threadIdx.x] = s;
    }
}

__global__ void lds_kernel(double* out, int iters)
{
    __shared__ double sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    double s = 0;
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) s += sm[(idx + i * 64) & 4095];
        idx = (idx + 1) & 4095;
    }
    if (s == 12345.678) out[threadIdx.x] = s;
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* out;
    CK(cudaMalloc(&out, 1 << 20));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 512, blocks = sms * 2;
    float ms;
    // DFMA: 16 chains x iters x threads x blocks FMAs
    {
        int iters = 40000;
        dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 16 * iters * (double)threads * blocks;
        printf("{\"kernel\": \"dfma\", \"tflops\": %.3f, \"ms\": %.2f}\n", flops / ms / 1e9, ms);
    }
    {
        int iters = 20000;
        dmma_kernel<<<blocks, threads>>>(out, 100);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 8 * iters * (double)(threads / 32) * blocks;   // 8x8x4 FMA per mma
        printf("{\"kernel\": \"dmma_m8n8k4\", \"tflops\": %.3f, \"ms\": %.2f}\n", flops / ms / 1e9, ms);
    }
    {
        int iters = 10000;
        mixed_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        mixed_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double f_mma = 2.0 * 256 * 8 * iters * (double)(threads / 64) * blocks;
        double f_fma = 2.0 * 16 * iters * 8 * (double)(threads / 2) * blocks;
        printf("{\"kernel\": \"dfma+dmma\", \"tflops\": %.3f, \"ms\": %.2f}\n", (f_mma + f_fma) / ms / 1e9, ms);
    }
    {
        int iters = 200000;
        lds_kernel<<<blocks, threads>>>(out, 100);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        lds_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double bytes = 8.0 * 8 * iters * (double)threads * blocks;
        printf("{\"kernel\": \"lds64\", \"tbytes_per_s\": %.3f, \"bytes_per_clk_per_sm_at_1965\": %.1f, \"ms\": %.2f}\n",
               bytes / ms / 1e9, bytes / (ms * 1e-3) / sms / 1.965e9, ms);
    }
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    printf("{\"sms\": %d, \"clock_khz_attr\": %d}\n", sms, clk);
    return 0;
}
