// Standalone check of the row-grouped TMA pattern (dwt2.cu, GRP loader):
// a 3-D tensor map {G P, rows / G, 1} over a buffer whose row pitch P is not a
// multiple of 16 bytes, boxes {136, h, 1} at (cls P + x, g, 0).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

struct alignas(64) Args { CUtensorMap a, b; int x, g, mode; };

__device__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ Args args, float *out)
{
    __shared__ __align__(128) float buf[3 * 136 + 32];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(3 * 136 * 4));
        const CUtensorMap *m = args.mode ? &args.b : &args.a;
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su32(buf)), "l"((uint64_t)m), "r"(args.x), "r"(args.g), "r"(0), "r"(su32(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(&bar)) : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * 136; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char **argv)
{
    const int P = argc > 1 ? atoi(argv[1]) : 4095, R = 31, G = argc > 2 ? atoi(argv[2]) : 4;
    std::vector<float> h(P * R);
    for (int i = 0; i < P * R; ++i) h[i] = i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 3 * 136 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void *fp; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    Args args;
    cuuint64_t dims[3] = {(cuuint64_t)G * P, (cuuint64_t)R / G, 1};
    cuuint64_t strides[2] = {(cuuint64_t)G * P * 4, (cuuint64_t)G * P * 4};
    cuuint32_t box[3] = {136, 3, 1}, estr[3] = {1, 1, 1};
    CUresult r = enc(&args.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode a: %d\n", (int)r);
    cuuint64_t strides2[2] = {(cuuint64_t)G * P * 4, (cuuint64_t)G * P * 4 * (R / G)};
    r = enc(&args.b, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides2, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode b: %d\n", (int)r);
    for (int mode = 0; mode < 2; ++mode) {
        args.x = 1 * P + (argc > 3 ? atoi(argv[3]) : 96); args.g = 2; args.mode = mode;
        k<<<1, 128>>>(args, o);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<float> ho(3 * 136);
        cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int rr = 0; rr < 3; ++rr)
            for (int c = 0; c < 136; ++c) {
                const long long fr = (2 + rr) * G + 1;
                const float want = fr < R ? float(fr * P + 96 + c) : 0.f;
                if (ho[rr * 136 + c] != want) ++bad;
            }
        printf("mode %d: %d mismatches; first row %g..%g\n", mode, bad, ho[0], ho[135]);
    }
    return 0;
}
