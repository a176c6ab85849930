/* Plain-C use of the C ABI (include/dwt2.h, libdwt2.so): no Python, no torch.
 * Transforms a W x H image with a linear ramp f(x, y) = 3x + 5y + 7 through
 * `levels` levels and checks what the 5/3 wavelet must give for it
 * (PAPER.md L57-70 with whole-sample symmetric extension): every detail
 * coefficient of an interior quad is 0 (two vanishing moments), the coarsest
 * LL holds the ramp's samples, and the inverse returns the input.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/forward_c.c -L paper_1708_07853_b200 -ldwt2 \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1708_07853_b200 -o forward_c
 *   ./forward_c [W H levels]                                  (exit 0 = pass) */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "dwt2.h"

#define CHECK(x)                                                                         \
    do {                                                                                 \
        int32_t rc_ = (x);                                                               \
        if (rc_ != DWT2_OK) {                                                            \
            fprintf(stderr, "%s failed: %s\n", #x, dwt2_error_string(rc_));              \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

int main(int argc, char **argv)
{
    const int W = argc > 1 ? atoi(argv[1]) : 1000, H = argc > 2 ? atoi(argv[2]) : 777;
    const int levels = argc > 3 ? atoi(argv[3]) : 3;
    const size_t n = (size_t)W * H;
    float *h_in = (float *)malloc(n * sizeof(float)), *h_out = (float *)malloc(n * sizeof(float));
    float *h_rec = (float *)malloc(n * sizeof(float));
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) h_in[(size_t)y * W + x] = (float)(3 * x + 5 * y + 7);

    float *d_in, *d_out, *d_rec;
    if (cudaMalloc((void **)&d_in, n * 4) || cudaMalloc((void **)&d_out, n * 4) || cudaMalloc((void **)&d_rec, n * 4)) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    cudaMemcpy(d_in, h_in, n * 4, cudaMemcpyHostToDevice);

    dwt2_plan *plan = dwt2_plan_create(W, H, levels, DWT2_BOUNDARY_SYMMETRIC);
    if (!plan) {
        fprintf(stderr, "dwt2_plan_create: %s\n", dwt2_error_string(dwt2_last_error()));
        return 1;
    }
    CHECK(dwt2_forward(plan, d_in, d_out, 0));
    CHECK(dwt2_inverse(plan, d_out, d_rec, 0));
    cudaMemcpy(h_out, d_out, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h_rec, d_rec, n * 4, cudaMemcpyDeviceToHost);
    dwt2_destroy(plan);

    /* level 1 details of interior quads (away from the right / bottom mirror) */
    const int Wq = (W + 1) / 2, Hq = (H + 1) / 2, Wh = W / 2, Hh = H / 2;
    double worst = 0.0;
    for (int q = 0; q < Hh - 2; ++q)
        for (int m = 0; m < Wh - 2; ++m) {
            worst = fmax(worst, fabs(h_out[(size_t)q * W + Wq + m]));                   /* HL */
            worst = fmax(worst, fabs(h_out[(size_t)(Hq + q) * W + m]));                 /* LH */
            worst = fmax(worst, fabs(h_out[(size_t)(Hq + q) * W + Wq + m]));            /* HH */
        }
    /* the coarsest LL: the ramp sampled every 2^levels pixels (interior quads) */
    int s = 1, wL = W, hL = H;
    for (int k = 0; k < levels; ++k) {
        s *= 2;
        wL = (wL + 1) / 2;
        hL = (hL + 1) / 2;
    }
    double ll_err = 0.0;
    for (int q = 0; q < hL - 2; ++q)
        for (int m = 0; m < wL - 2; ++m)
            ll_err = fmax(ll_err, fabs(h_out[(size_t)q * W + m] - (3.0 * s * m + 5.0 * s * q + 7.0)));
    double rec_err = 0.0;
    for (size_t i = 0; i < n; ++i) rec_err = fmax(rec_err, fabs(h_rec[i] - h_in[i]));
    printf("%s: %dx%d, %d levels: max |detail| %.3g, max |LL - ramp| %.3g, max |inverse - input| %.3g\n",
           dwt2_version(), W, H, levels, worst, ll_err, rec_err);
    free(h_in);
    free(h_out);
    free(h_rec);
    cudaFree(d_in);
    cudaFree(d_out);
    cudaFree(d_rec);
    return (worst == 0.0 && ll_err < 1e-3 && rec_err < 1e-3) ? 0 : 2;
}
