// membench.cu -- B200 memory-pattern microbenchmarks (tooling, not product).
// Which HBM access pattern of a 2-D row-walking stencil reaches copy speed?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int W = 16384, H = 16384;

__global__ void copy_f4(const float4 *__restrict__ in, float4 *__restrict__ out, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

// per-warp row walk: warp owns 128 columns [x0, x0+128) of rows [r0, r1); LDG.128, D rows in flight
template <int D, int MODE>
__global__ void __launch_bounds__(128) rowwalk(const float *__restrict__ in, float *__restrict__ out, int nbands)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int groups = W / 512;
    const int group = blockIdx.x % groups, band = blockIdx.x / groups;
    const int x0 = (group * 4 + warp) * 128;
    const int r0 = (int)((long long)H * band / nbands), r1 = (int)((long long)H * (band + 1) / nbands);
    float4 buf[D];
#pragma unroll
    for (int d = 0; d < D; ++d) buf[d] = (r0 + d < r1) ? __ldcs(reinterpret_cast<const float4 *>(in + (size_t)(r0 + d) * W + x0) + lane) : make_float4(0, 0, 0, 0);
    for (int r = r0; r < r1; r += D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const int rr = r + d;
            if (rr >= r1) break;
            float4 v = buf[d];
            if (rr + D < r1) buf[d] = __ldcs(reinterpret_cast<const float4 *>(in + (size_t)(rr + D) * W + x0) + lane);
            if (MODE == 0) {
                __stcs(reinterpret_cast<float4 *>(out + (size_t)rr * W + x0) + lane, v);
            } else {
                // quadrant pattern: row pair -> 4 streams of 256 B (float2 per lane)
                const int n = rr >> 1, mq = (x0 >> 1) + 2 * lane;
                float *ll = out + (size_t)n * W + mq, *hl = ll + W / 2;
                float *lh = out + (size_t)(H / 2 + n) * W + mq, *hh = lh + W / 2;
                if (rr & 1) {
                    __stcs(reinterpret_cast<float2 *>(lh), make_float2(v.x, v.z));
                    __stcs(reinterpret_cast<float2 *>(hh), make_float2(v.y, v.w));
                } else {
                    __stcs(reinterpret_cast<float2 *>(ll), make_float2(v.x, v.z));
                    __stcs(reinterpret_cast<float2 *>(hl), make_float2(v.y, v.w));
                }
            }
        }
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// per-warp TMA ring: box BW x BH at (x0 - XOFF, r), S stages; consume = copy box interior to out
template <int BW, int BH, int XOFF, int S, int MODE>
__global__ void __launch_bounds__(128) tmawalk(const __grid_constant__ CUtensorMap map, float *__restrict__ out, int nbands)
{
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int SF = (BW * BH + 31) / 32 * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *ring = reinterpret_cast<float *>(sm) + warp * S * SF;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + 4 * S * SF * 4) + warp * S;
    if (lane == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    const int groups = W / 512;
    const int group = blockIdx.x % groups, band = blockIdx.x / groups;
    const int x0 = (group * 4 + warp) * 128;
    const int r0 = (int)((long long)H * band / nbands), r1 = (int)((long long)H * (band + 1) / nbands);
    const int rows_per = BH - (XOFF ? 1 : 0);
    const int nst = (r1 - r0 + rows_per - 1) / rows_per;
    auto issue = [&](int j) {
        if (lane == 0) {
            const int slot = j % S;
            asm volatile("fence.proxy.async.shared::cta;");
            asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[slot])), "r"(BW * BH * 4));
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(smem_u32(ring + slot * SF)), "l"((uint64_t)&map), "r"(x0 - XOFF), "r"(r0 + j * rows_per), "r"(smem_u32(&bars[slot])) : "memory");
        }
    };
    for (int j = 0; j < S && j < nst; ++j) issue(j);
    for (int j = 0; j < nst; ++j) {
        const int slot = j % S;
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bars[slot])), "r"((j / S) & 1) : "memory");
        const float *sl = ring + slot * SF;
        for (int i = 0; i < rows_per; ++i) {
            const int rr = r0 + j * rows_per + i;
            if (rr >= r1) break;
            const float4 v = *reinterpret_cast<const float4 *>(sl + i * BW + XOFF + 4 * lane);
            if (MODE == 0) {
                __stcs(reinterpret_cast<float4 *>(out + (size_t)rr * W + x0) + lane, v);
            } else {
                const int n = rr >> 1, mq = (x0 >> 1) + 2 * lane;
                float *ll = out + (size_t)n * W + mq, *hl = ll + W / 2;
                float *lh = out + (size_t)(H / 2 + n) * W + mq, *hh = lh + W / 2;
                if (rr & 1) {
                    __stcs(reinterpret_cast<float2 *>(lh), make_float2(v.x, v.z));
                    __stcs(reinterpret_cast<float2 *>(hh), make_float2(v.y, v.w));
                } else {
                    __stcs(reinterpret_cast<float2 *>(ll), make_float2(v.x, v.z));
                    __stcs(reinterpret_cast<float2 *>(hl), make_float2(v.y, v.w));
                }
            }
        }
        __syncwarp();
        if (j + S < nst) issue(j + S);
    }
}

template <typename F>
float timeit(F f, int iters = 20)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < iters; ++i) f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    CK(cudaGetLastError());
    return ms / iters;
}

int main()
{
    size_t n = (size_t)W * H;
    float *in, *out;
    CK(cudaMalloc(&in, n * 4)); CK(cudaMalloc(&out, n * 4));
    CK(cudaMemset(in, 0, n * 4));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double bytes = 2.0 * n * 4;
    auto rep = [&](const char *name, float ms) { printf("%-40s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / ms / 1e6); };

    rep("copy_f4 grid 148x8x256", timeit([&] { copy_f4<<<sms * 8, 256>>>((const float4 *)in, (float4 *)out, n / 4); }));
    rep("copy_f4 grid 148x4x1024", timeit([&] { copy_f4<<<sms * 2, 1024>>>((const float4 *)in, (float4 *)out, n / 4); }));

    const int groups = W / 512;
    for (int nb : {9, 18, 36}) {
        char b[80];
        snprintf(b, 80, "rowwalk D=8 copy nbands=%d", nb);
        rep(b, timeit([&] { rowwalk<8, 0><<<groups * nb, 128>>>(in, out, nb); }));
        snprintf(b, 80, "rowwalk D=8 quad-stores nbands=%d", nb);
        rep(b, timeit([&] { rowwalk<8, 1><<<groups * nb, 128>>>(in, out, nb); }));
        snprintf(b, 80, "rowwalk D=16 quad-stores nbands=%d", nb);
        rep(b, timeit([&] { rowwalk<16, 1><<<groups * nb, 128>>>(in, out, nb); }));
    }

    void *pfn = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &pfn, cudaEnableDefault, &q));
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)pfn;
    auto mk = [&](int bw, int bh, CUtensorMapL2promotion prom) {
        CUtensorMap m;
        cuuint64_t dims[2] = {W, H}; cuuint64_t str[1] = {W * 4}; cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}; cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, in, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("encode failed %d\n", r);
        return m;
    };
#define TMA_CASE(BW, BH, XOFF, S, MODE, PROM, NB, NAME)                                                          \
    {                                                                                                               \
        auto k = tmawalk<BW, BH, XOFF, S, MODE>;                                                                    \
        size_t smem = 4 * S * ((BW * BH + 31) / 32 * 32) * 4 + 4 * S * 8;                                          \
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));                       \
        CUtensorMap m = mk(BW, BH, PROM);                                                                           \
        int nb = NB;                                                                                                \
        rep(NAME, timeit([&] { k<<<groups * nb, 128, smem>>>(m, out, nb); }));                                      \
    }
    TMA_CASE(128, 16, 0, 3, 0, CU_TENSOR_MAP_L2_PROMOTION_NONE, 9, "tma 128x16 aligned S3 copy nb9");
    TMA_CASE(128, 16, 0, 3, 1, CU_TENSOR_MAP_L2_PROMOTION_NONE, 9, "tma 128x16 aligned S3 quad nb9");
    TMA_CASE(136, 17, 4, 3, 0, CU_TENSOR_MAP_L2_PROMOTION_NONE, 9, "tma 136x17 x0-4 S3 copy nb9");
    TMA_CASE(136, 17, 4, 3, 1, CU_TENSOR_MAP_L2_PROMOTION_NONE, 9, "tma 136x17 x0-4 S3 quad nb9");
    TMA_CASE(136, 17, 4, 3, 1, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, 9, "tma 136x17 x0-4 S3 quad prom128 nb9");
    TMA_CASE(136, 17, 4, 3, 1, CU_TENSOR_MAP_L2_PROMOTION_NONE, 18, "tma 136x17 x0-4 S3 quad nb18");
    TMA_CASE(136, 9, 4, 4, 1, CU_TENSOR_MAP_L2_PROMOTION_NONE, 18, "tma 136x9 x0-4 S4 quad nb18");
    TMA_CASE(136, 33, 4, 2, 1, CU_TENSOR_MAP_L2_PROMOTION_NONE, 9, "tma 136x33 x0-4 S2 quad nb9");
    TMA_CASE(128, 32, 0, 3, 0, CU_TENSOR_MAP_L2_PROMOTION_NONE, 9, "tma 128x32 aligned S3 copy nb9");
    return 0;
}
