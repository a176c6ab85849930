// pipebench.cu -- B200 arithmetic pipe throughput (tooling, not product):
// DFMA, DADD, F2F.F64.F32, F2F.F32.F64, FFMA, SHFL, and DFMA with 1 active lane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipebench pipebench.cu
#include <cuda_runtime.h>
#include <cstdio>

constexpr int ITERS = 4096;

__global__ void k_dfma(double *out, double s)
{
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < ITERS; ++i) {
        a0 = fma(a0, s, 0.5); a1 = fma(a1, s, 0.5); a2 = fma(a2, s, 0.5); a3 = fma(a3, s, 0.5);
        a4 = fma(a4, s, 0.5); a5 = fma(a5, s, 0.5); a6 = fma(a6, s, 0.5); a7 = fma(a7, s, 0.5);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dfma_1lane(double *out, double s)
{
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    if ((threadIdx.x & 31) == 0) {
        for (int i = 0; i < ITERS; ++i) {
            a0 = fma(a0, s, 0.5); a1 = fma(a1, s, 0.5); a2 = fma(a2, s, 0.5); a3 = fma(a3, s, 0.5);
            a4 = fma(a4, s, 0.5); a5 = fma(a5, s, 0.5); a6 = fma(a6, s, 0.5); a7 = fma(a7, s, 0.5);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_ffma(float *out, float s)
{
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < ITERS; ++i) {
        a0 = fmaf(a0, s, 0.5f); a1 = fmaf(a1, s, 0.5f); a2 = fmaf(a2, s, 0.5f); a3 = fmaf(a3, s, 0.5f);
        a4 = fmaf(a4, s, 0.5f); a5 = fmaf(a5, s, 0.5f); a6 = fmaf(a6, s, 0.5f); a7 = fmaf(a7, s, 0.5f);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// float -> double -> float round trips: 2 conversions per step, 8 chains
__global__ void k_f2f(float *out, float s)
{
    float a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            double d = (double)a[j];
            asm volatile("" : "+d"(d));
            a[j] = (float)d;
        }
    }
    float t = 0;
    for (int j = 0; j < 8; ++j) t += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_shfl(float *out, float s)
{
    float a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = __shfl_down_sync(0xffffffffu, a[j], 1);
    }
    float t = 0;
    for (int j = 0; j < 8; ++j) t += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <typename F>
float timeit(F f)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main()
{
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *dout; float *fout;
    cudaMalloc(&dout, sizeof(double) * sms * 8 * 256 * 4);
    cudaMalloc(&fout, sizeof(float) * sms * 8 * 256 * 4);
    const int blocks = sms * 8, threads = 256;
    const double n = double(blocks) * threads * ITERS * 8;     // ops (per thread lane)
    const double ghz = clk / 1e6;
    auto rep = [&](const char *name, float ms, double ops) {
        const double per_s = ops / (ms * 1e-3);
        printf("%-28s %9.3f ms  %8.1f Gop/s  %6.1f /clk/SM (at %.2f GHz)\n", name, ms, per_s / 1e9, per_s / (sms * ghz * 1e9), ghz);
    };
    rep("DFMA", timeit([&] { k_dfma<<<blocks, threads>>>(dout, 0.999); }), n);
    rep("DFMA 1 lane/warp (lane ops)", timeit([&] { k_dfma_1lane<<<blocks, threads>>>(dout, 0.999); }), n / 32);
    rep("FFMA", timeit([&] { k_ffma<<<blocks, threads>>>(fout, 0.999f); }), n);
    rep("F2F f32->f64->f32 (2 conv)", timeit([&] { k_f2f<<<blocks, threads>>>(fout, 0.999f); }), 2 * n);
    rep("SHFL", timeit([&] { k_shfl<<<blocks, threads>>>(fout, 0.999f); }), n);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
