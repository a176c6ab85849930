/* Plain-C use of the peer-strip C ABI (include/dwt2.h "peer strip context"):
 * G row-strip ranks of one W x H image, `levels` levels, emulated in ONE
 * process on one GPU (DWT2_PEER_SEQUENTIAL): every rank gets a strip plan and a
 * context, the contexts exchange their descriptors (plain bytes -- here by
 * assignment, across processes through any channel) and connect to their
 * neighbours, and each level runs as every rank's PUBLISH launch, then every
 * rank's fused launch, whose boundary-role CTAs read the neighbours' rows from
 * the neighbours' memory.  The strip-local pyramids, placed into the global
 * Mallat layout, must equal the single-image dwt2_forward bit for bit.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/peer_strips_c.c -L paper_1708_07853_b200 -ldwt2 \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1708_07853_b200 -o peer_strips_c
 *   ./peer_strips_c [W H levels ranks]                         (exit 0 = pass) */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dwt2.h"

#define MAXG 16
#define CHECK(x)                                                                         \
    do {                                                                                 \
        int32_t rc_ = (x);                                                               \
        if (rc_ != DWT2_OK) {                                                            \
            fprintf(stderr, "%s failed: %s\n", #x, dwt2_error_string(rc_));              \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

/* rank g's rows [lo, hi): balanced runs of 2^levels-row units (distributed.strip_rows_levels) */
static void strip_rows(int H, int g, int G, int levels, int *lo, int *hi)
{
    const long long unit = 1LL << levels, nunits = (H + unit - 1) / unit;
    *lo = (int)(unit * ((g * nunits) / G));
    *hi = g == G - 1 ? H : (int)(unit * (((g + 1) * nunits) / G));
}

/* copy a strip-local pyramid (W x (r1 - r0), pitch W) into the global one (W x H)
 * (distributed.place_pyramid_output) */
static void place(float *full, const float *strip, int W, int H, int r0, int r1, int levels)
{
    int w = W, h = H, rb = r0, re = r1;
    for (int k = 0; k < levels; ++k) {
        const int Hq = (h + 1) / 2, Hh = h / 2, Wq = (w + 1) / 2;
        const int qs = rb / 2, qe = (re + 1) / 2, hq_loc = qe - qs;
        const int c0 = k == levels - 1 ? 0 : Wq;                 /* inner levels' LL is not output */
        for (int r = 0; r < hq_loc; ++r)
            memcpy(full + (size_t)(qs + r) * W + c0, strip + (size_t)r * W + c0, (size_t)(w - c0) * 4);
        const int h0 = qs < Hh ? qs : Hh, h1 = qe < Hh ? qe : Hh;
        for (int r = 0; r < h1 - h0; ++r)
            memcpy(full + (size_t)(Hq + h0 + r) * W, strip + (size_t)(hq_loc + r) * W, (size_t)w * 4);
        w = Wq; h = Hq; rb = qs; re = qe;
    }
}

int main(int argc, char **argv)
{
    const int W = argc > 1 ? atoi(argv[1]) : 1000, H = argc > 2 ? atoi(argv[2]) : 1024;
    const int L = argc > 3 ? atoi(argv[3]) : 3, G = argc > 4 ? atoi(argv[4]) : 4;
    if (G < 1 || G > MAXG) return 2;
    const size_t n = (size_t)W * H;
    float *h_in = (float *)malloc(n * 4), *h_ref = (float *)malloc(n * 4), *h_got = (float *)malloc(n * 4);
    unsigned s = 12345u;
    for (size_t i = 0; i < n; ++i) {                     /* integer pixels in [0, 255], LCG */
        s = s * 1664525u + 1013904223u;
        h_in[i] = (float)(s >> 24);
    }
    /* the single-image transform */
    float *d_in, *d_out;
    if (cudaMalloc((void **)&d_in, n * 4) || cudaMalloc((void **)&d_out, n * 4)) return 1;
    cudaMemcpy(d_in, h_in, n * 4, cudaMemcpyHostToDevice);
    dwt2_plan *plan = dwt2_plan_create(W, H, L, DWT2_BOUNDARY_SYMMETRIC);
    if (!plan) {
        fprintf(stderr, "dwt2_plan_create: %s\n", dwt2_error_string(dwt2_last_error()));
        return 1;
    }
    CHECK(dwt2_forward(plan, d_in, d_out, 0));
    cudaMemcpy(h_ref, d_out, n * 4, cudaMemcpyDeviceToHost);

    /* the ranks: plan, context, level-0 rows, descriptor */
    dwt2_plan *sp[MAXG];
    dwt2_peer_strip *ctx[MAXG];
    dwt2_peer_desc_t desc[MAXG];
    float *d_sout[MAXG];
    int r0[MAXG], r1[MAXG];
    for (int g = 0; g < G; ++g) {
        strip_rows(H, g, G, L, &r0[g], &r1[g]);
        sp[g] = dwt2_plan_create_strip_levels(W, H, r0[g], r1[g], L, DWT2_BOUNDARY_SYMMETRIC);
        ctx[g] = sp[g] ? dwt2_peer_strip_create(sp[g], 2000) : NULL;
        if (!ctx[g]) {
            fprintf(stderr, "rank %d: %s\n", g, dwt2_error_string(dwt2_last_error()));
            return 1;
        }
        float *own;
        int64_t pitch;
        CHECK(dwt2_peer_strip_buffer(ctx[g], 0, &own, &pitch));
        cudaMemcpy2D(own, (size_t)pitch * 4, h_in + (size_t)r0[g] * W, (size_t)W * 4, (size_t)W * 4,
                     (size_t)(r1[g] - r0[g]), cudaMemcpyHostToDevice);
        if (cudaMalloc((void **)&d_sout[g], (size_t)W * (r1[g] - r0[g]) * 4)) return 1;
        CHECK(dwt2_peer_strip_export(ctx[g], &desc[g]));
    }
    for (int g = 0; g < G; ++g)
        CHECK(dwt2_peer_strip_connect(ctx[g], g > 0 ? &desc[g - 1] : NULL, g + 1 < G ? &desc[g + 1] : NULL,
                                      DWT2_PEER_SEQUENTIAL));
    /* one step, level by level: every rank publishes, then every rank's fused launch */
    for (int k = 0; k < L; ++k) {
        for (int g = 0; g < G; ++g) CHECK(dwt2_peer_strip_level(ctx[g], k, DWT2_STRIP_PUBLISH, d_sout[g], 0));
        for (int g = 0; g < G; ++g) CHECK(dwt2_peer_strip_level(ctx[g], k, DWT2_STRIP_ALL, d_sout[g], 0));
    }
    if (cudaDeviceSynchronize() != cudaSuccess) {
        fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(cudaGetLastError()));
        return 1;
    }
    for (int g = 0; g < G; ++g) {
        CHECK(dwt2_peer_strip_status(ctx[g]));
        float *tmp = (float *)malloc((size_t)W * (r1[g] - r0[g]) * 4);
        cudaMemcpy(tmp, d_sout[g], (size_t)W * (r1[g] - r0[g]) * 4, cudaMemcpyDeviceToHost);
        place(h_got, tmp, W, H, r0[g], r1[g], L);
        free(tmp);
    }
    size_t bad = 0;
    for (size_t i = 0; i < n; ++i) bad += h_got[i] != h_ref[i];
    printf("%d x %d, %d levels, %d ranks: elements differing from the single-image transform %zu\n", W, H, L, G, bad);
    for (int g = 0; g < G; ++g) {
        dwt2_peer_strip_destroy(ctx[g]);
        dwt2_destroy(sp[g]);
        cudaFree(d_sout[g]);
    }
    dwt2_destroy(plan);
    cudaFree(d_in);
    cudaFree(d_out);
    free(h_in);
    free(h_ref);
    free(h_got);
    return bad == 0 ? 0 : 1;
}
