/*
 * oracle/dwt53_oracle.c -- CPU oracle for the forward 2-D CDF 5/3 DWT.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may load, link or
 * call this file.  The only permitted users are tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs.  It
 * shares no code, header, table or constant with paper_1708_07853_b200/csrc.
 *
 * What it computes.  PAPER.md L100 ("Usually, the 2-D transform is defined as
 * the tensor product of 1-D transforms"): the non-separable scheme of Eq. (5)
 * reaches exactly this result with fewer steps, so the
 * oracle is that plain definition written out, in double precision:
 *
 *   A. separable lifting (Eq. (2); 2-D sequence Eq. (3),
 *      L100-137): every row is split by parity (L57-59) and lifted with one
 *      predict/update pair, then every column of the result likewise.
 *   B. brute-force polyphase convolution (Eq. (1); Eq. (4),
 *      L160-171): every output coefficient is an independent 2-D weighted sum
 *      of the (extended) input with the tensor-product filter taps.
 *   C. inverse lifting (steps reversed, signs flipped).
 *   D. multi-level recursion on LL with Mallat placement (BASELINE.json
 *      north_star "a multi-level driver recursing on LL").
 *
 * Readings (DESIGN.md section 3 lists them all):
 *   - CDF 5/3 lifting pair P = -1/2 (1 + z), U = 1/4 (1 + z^-1), K = 1, no
 *     scaling (Eq. (2) has no scaling matrix).  z^+1 reads the
 *     next sample.
 *   - L = even 0-based samples, H = odd; ceil(N/2) L and floor(N/2) H
 *     ("according to a parity of its samples").
 *   - boundaries: whole-sample symmetric extension of the input signal
 *     x[-k] = x[k], x[N-1+k] = x[N-1-k] (the paper is silent).
 *   - Mallat layout: LL top-left, HL top-right (horizontal high), LH
 *     bottom-left, HH bottom-right.
 *   - precision: fp64.  With round_f32 != 0 each level's output is rounded
 *     to fp32 before the next level reads it (the storage type of the GPU
 *     path); with round_f32 == 0 everything stays fp64.
 *
 * Every function below is deliberately plain: no blocking, no fusion, no
 * reordering beyond the definitions cited.
 */
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* Boundary extension                                                      */
/* ---------------------------------------------------------------------- */

/* Whole-sample symmetric reflection of index k into [0, n): the extended
 * signal is periodic with period 2(n-1) and mirrored about 0 and n-1
 * ("mirror without repeating the edge sample").  n == 1 maps
 * every index to 0. */
static long wss(long k, long n)
{
    long p;
    if (n == 1)
        return 0;
    p = 2 * (n - 1);
    k %= p;
    if (k < 0)
        k += p;
    if (k >= n)
        k = p - k;
    return k;
}

/* ---------------------------------------------------------------------- */
/* A. 1-D lifting (Eq. (2) with K = 1)                                     */
/* ---------------------------------------------------------------------- */

/* Forward 1-D CDF 5/3 lifting of x[0..n) (elements `stride` apart).
 * Writes ceil(n/2) L samples to low[] and floor(n/2) H samples to high[].
 * Predict ("the first step is called the predict step"):
 *     d[i] = x[2i+1] + P(x)[i] = x[2i+1] - 1/2 (x[2i] + x[2i+2])
 * Update (L76 "the second one as the update step"):
 *     s[i] = x[2i]   + U(d)[i] = x[2i]   + 1/4 (d[i-1] + d[i])
 * The predict is evaluated on the symmetrically extended input for every
 * i the update reads (i = -1 .. ceil(n/2)-1), so the boundary rule is the
 * input extension itself, not a separate rule on d. */
static void lift_fwd_1d(const double *x, long n, long stride, double *low, double *high)
{
    long nl = (n + 1) / 2, nh = n / 2, i;
    double *d;
    if (n == 1) {
        low[0] = x[0];
        return;
    }
    d = (double *)malloc((size_t)(nl + 1) * sizeof(double)); /* d[i] at d[i + 1] */
    for (i = -1; i <= nl - 1; i++)
        d[i + 1] = x[wss(2 * i + 1, n) * stride]
                   - 0.5 * (x[wss(2 * i, n) * stride] + x[wss(2 * i + 2, n) * stride]);
    for (i = 0; i < nh; i++)
        high[i] = d[i + 1];
    for (i = 0; i < nl; i++)
        low[i] = x[2 * i * stride] + 0.25 * (d[i] + d[i + 1]);
    free(d);
}

/* Inverse of lift_fwd_1d (lifting steps run in reverse
 * order with their signs flipped).  low[] has ceil(n/2), high[] floor(n/2)
 * samples; the result goes to x[0..n) (elements `stride` apart).
 *   undo update:  x[2i]   = s[i] - 1/4 (d[i-1] + d[i])
 *   undo predict: x[2i+1] = d[i] + 1/2 (x[2i] + x[2i+2])
 * The forward step's extension, restated on d: d[-1] = d[0] and, for odd n,
 * d[nl-1] = d[nl-2] (both follow from the whole-sample symmetric input);
 * x[n] = x[n-2] for even n. */
static void lift_inv_1d(const double *low, const double *high, long n, double *x, long stride)
{
    long nl = (n + 1) / 2, nh = n / 2, i;
    double *e;
    if (n == 1) {
        x[0] = low[0];
        return;
    }
    e = (double *)malloc((size_t)nl * sizeof(double));
    for (i = 0; i < nl; i++) {
        double dl = high[i - 1 < 0 ? 0 : (i - 1 >= nh ? nh - 1 : i - 1)];
        double dr = high[i >= nh ? nh - 1 : i];
        e[i] = low[i] - 0.25 * (dl + dr);
    }
    for (i = 0; i < nl; i++)
        x[2 * i * stride] = e[i];
    for (i = 0; i < nh; i++) {
        double right = (2 * i + 2 < n) ? e[i + 1] : e[i]; /* x[n] = x[n-2] */
        x[(2 * i + 1) * stride] = high[i] + 0.5 * (e[i] + right);
    }
    free(e);
}

/* ---------------------------------------------------------------------- */
/* One 2-D level, separable lifting (Eq. (3); rows first, then columns --  */
/* the order of the horizontal and vertical steps is free)  */
/* ---------------------------------------------------------------------- */

/* in: W x H region with row pitch in_pitch; out: W x H Mallat region with
 * row pitch out_pitch.  in and out may be the same region. */
static void level_fwd_lifting(const double *in, long in_pitch, double *out, long out_pitch,
                              long W, long H)
{
    long nlx = (W + 1) / 2, nly = (H + 1) / 2, x, y;
    double *tmp = (double *)malloc((size_t)W * (size_t)H * sizeof(double));
    double *row = (double *)malloc((size_t)(W > H ? W : H) * sizeof(double));
    /* rows: L to columns [0, nlx), H to [nlx, W) */
    for (y = 0; y < H; y++) {
        lift_fwd_1d(in + y * in_pitch, W, 1, row, row + nlx);
        memcpy(tmp + y * W, row, (size_t)W * sizeof(double));
    }
    /* columns: L to rows [0, nly), H to rows [nly, H) */
    for (x = 0; x < W; x++) {
        double *col = (double *)malloc((size_t)H * sizeof(double));
        lift_fwd_1d(tmp + x, H, W, col, col + nly);
        for (y = 0; y < H; y++)
            out[y * out_pitch + x] = col[y];
        free(col);
    }
    free(row);
    free(tmp);
}

/* Inverse of level_fwd_lifting: columns first, then rows (reverse order). */
static void level_inv_lifting(const double *in, long in_pitch, double *out, long out_pitch,
                              long W, long H)
{
    long nlx = (W + 1) / 2, nly = (H + 1) / 2, x, y;
    double *tmp = (double *)malloc((size_t)W * (size_t)H * sizeof(double));
    double *col = (double *)malloc((size_t)H * sizeof(double));
    double *row = (double *)malloc((size_t)W * sizeof(double));
    for (x = 0; x < W; x++) {
        for (y = 0; y < H; y++)
            col[y] = in[y * in_pitch + x];
        lift_inv_1d(col, col + nly, H, tmp + x, W);
    }
    for (y = 0; y < H; y++) {
        memcpy(row, tmp + y * W, (size_t)W * sizeof(double));
        lift_inv_1d(row, row + nlx, W, out + y * out_pitch, 1);
    }
    free(row);
    free(col);
    free(tmp);
}

/* ---------------------------------------------------------------------- */
/* B. Brute-force polyphase convolution (Eq. (1) / Eq. (4))                */
/* ---------------------------------------------------------------------- */

/* Analysis taps of the CDF 5/3 pair, obtained by expanding the lifting pair
 * of Eq. (2) into the convolution form of Eq. (1):
 *   H: d[i] = x[2i+1] - 1/2 x[2i] - 1/2 x[2i+2]
 *        -> g1 = (-1/2, 1, -1/2) on offsets -1, 0, +1 around sample 2i+1
 *   L: s[i] = x[2i] + 1/4 (d[i-1] + d[i])
 *        = -1/8 x[2i-2] + 1/4 x[2i-1] + 3/4 x[2i] + 1/4 x[2i+1] - 1/8 x[2i+2]
 *        -> h0 = (-1/8, 1/4, 3/4, 1/4, -1/8) on offsets -2 .. +2 around 2i
 * ("g0 has 5 taps, g1 has 3 taps"). */
static const double H0[5] = {-0.125, 0.25, 0.75, 0.25, -0.125};
static const double G1[3] = {-0.5, 1.0, -0.5};

/* band: 0 = LL, 1 = HL, 2 = LH, 3 = HH.  (m, n) = (column, row) of the
 * coefficient inside its subband.  Reads the W x H image img (pitch) with
 * whole-sample symmetric extension on both axes.  64 MACs per quad.
 * Pointwise: any subset of outputs can be computed independently. */
static double conv_coeff(const double *img, long pitch, long W, long H, int band, long m, long n)
{
    int hx_high = (band == 1 || band == 3); /* horizontal high-pass for HL, HH */
    int vy_high = (band == 2 || band == 3); /* vertical high-pass for LH, HH */
    const double *fx = hx_high ? G1 : H0, *fy = vy_high ? G1 : H0;
    int rx = hx_high ? 1 : 2, ry = vy_high ? 1 : 2; /* tap radius */
    long cx = hx_high ? 2 * m + 1 : 2 * m, cy = vy_high ? 2 * n + 1 : 2 * n;
    double acc = 0.0;
    int i, j;
    for (j = -ry; j <= ry; j++)
        for (i = -rx; i <= rx; i++)
            acc += fy[j + ry] * fx[i + rx] * img[wss(cy + j, H) * pitch + wss(cx + i, W)];
    return acc;
}

static void level_fwd_conv(const double *in, long in_pitch, double *out, long out_pitch,
                           long W, long H)
{
    long nlx = (W + 1) / 2, nly = (H + 1) / 2, nhx = W / 2, nhy = H / 2, m, n;
    double *res = (double *)malloc((size_t)W * (size_t)H * sizeof(double));
    for (n = 0; n < nly; n++)
        for (m = 0; m < nlx; m++)
            res[n * W + m] = conv_coeff(in, in_pitch, W, H, 0, m, n);
    for (n = 0; n < nly; n++)
        for (m = 0; m < nhx; m++)
            res[n * W + nlx + m] = conv_coeff(in, in_pitch, W, H, 1, m, n);
    for (n = 0; n < nhy; n++)
        for (m = 0; m < nlx; m++)
            res[(nly + n) * W + m] = conv_coeff(in, in_pitch, W, H, 2, m, n);
    for (n = 0; n < nhy; n++)
        for (m = 0; m < nhx; m++)
            res[(nly + n) * W + nlx + m] = conv_coeff(in, in_pitch, W, H, 3, m, n);
    for (n = 0; n < H; n++)
        memcpy(out + n * out_pitch, res + n * W, (size_t)W * sizeof(double));
    free(res);
}

/* ---------------------------------------------------------------------- */
/* D. Multi-level recursion on LL                                          */
/* ---------------------------------------------------------------------- */

static void round_region_f32(double *buf, long pitch, long W, long H)
{
    long x, y;
    for (y = 0; y < H; y++)
        for (x = 0; x < W; x++)
            buf[y * pitch + x] = (double)(float)buf[y * pitch + x];
}

/* Level k transforms the top-left ceil(W/2^(k-1)) x ceil(H/2^(k-1)) region
 * of out (holding LL_{k-1}) in place; level 1 reads in.  Returns the number
 * of levels done, or -1 on invalid arguments. */
static long multilevel(const double *in, double *out, long W, long H, long levels, int round_f32,
                       int use_conv)
{
    long k, w = W, h = H;
    if (W < 1 || H < 1 || levels < 0)
        return -1;
    memcpy(out, in, (size_t)W * (size_t)H * sizeof(double));
    for (k = 0; k < levels; k++) {
        if (use_conv)
            level_fwd_conv(out, W, out, W, w, h);
        else
            level_fwd_lifting(out, W, out, W, w, h);
        if (round_f32)
            round_region_f32(out, W, w, h);
        w = (w + 1) / 2;
        h = (h + 1) / 2;
    }
    return levels;
}

/* ---------------------------------------------------------------------- */
/* Exported entry points (ctypes; tests/ and bench only)                   */
/* ---------------------------------------------------------------------- */

/* 1-D forward: out[0..ceil(n/2)) = L, out[ceil(n/2)..n) = H. */
void oracle_dwt53_fwd_1d(const double *x, long n, double *out)
{
    lift_fwd_1d(x, n, 1, out, out + (n + 1) / 2);
}

/* 1-D inverse of oracle_dwt53_fwd_1d. */
void oracle_dwt53_inv_1d(const double *in, long n, double *x)
{
    lift_inv_1d(in, in + (n + 1) / 2, n, x, 1);
}

/* Algorithm A: levels of separable lifting, W x H row-major (pitch W) in,
 * Mallat pyramid out.  round_f32: round each level's output to fp32. */
long oracle_dwt53_fwd_lifting(const double *in, double *out, long W, long H, long levels,
                              int round_f32)
{
    return multilevel(in, out, W, H, levels, round_f32, 0);
}

/* Algorithm B: the same through brute-force convolution at every level. */
long oracle_dwt53_fwd_conv(const double *in, double *out, long W, long H, long levels,
                           int round_f32)
{
    return multilevel(in, out, W, H, levels, round_f32, 1);
}

/* Algorithm C: inverse of A (levels in reverse order, each level inverted).
 * round_f32: round each level's reconstruction to fp32 before the next
 * (finer) level reads it -- the storage type of the GPU path (DESIGN.md
 * reading C-A13); 0 keeps everything fp64. */
long oracle_dwt53_inv_lifting(const double *in, double *out, long W, long H, long levels,
                              int round_f32)
{
    long k, *ws, *hs;
    if (W < 1 || H < 1 || levels < 0)
        return -1;
    ws = (long *)malloc((size_t)(levels + 1) * sizeof(long));
    hs = (long *)malloc((size_t)(levels + 1) * sizeof(long));
    ws[0] = W;
    hs[0] = H;
    for (k = 1; k <= levels; k++) {
        ws[k] = (ws[k - 1] + 1) / 2;
        hs[k] = (hs[k - 1] + 1) / 2;
    }
    memcpy(out, in, (size_t)W * (size_t)H * sizeof(double));
    for (k = levels - 1; k >= 0; k--) {
        level_inv_lifting(out, W, out, W, ws[k], hs[k]);
        if (round_f32)
            round_region_f32(out, W, ws[k], hs[k]);
    }
    free(ws);
    free(hs);
    return levels;
}

/* Algorithm B, pointwise, on an fp32 image (each pixel widened exactly to
 * fp64): for i < count, res[i] = coefficient (band[i], m[i], n[i]) of one
 * level applied to the W x H image img with row pitch `pitch`. */
void oracle_dwt53_conv_sample_f32(const float *img, long pitch, long W, long H, long count,
                                  const int *band, const long *m, const long *n, double *res)
{
    long i;
    int j, k;
    for (i = 0; i < count; i++) {
        /* copy the 5x5 neighbourhood (after reflection) into a small fp64 image */
        int hx_high = (band[i] == 1 || band[i] == 3), vy_high = (band[i] == 2 || band[i] == 3);
        const double *fx = hx_high ? G1 : H0, *fy = vy_high ? G1 : H0;
        int rx = hx_high ? 1 : 2, ry = vy_high ? 1 : 2;
        long cx = hx_high ? 2 * m[i] + 1 : 2 * m[i], cy = vy_high ? 2 * n[i] + 1 : 2 * n[i];
        double acc = 0.0;
        for (j = -ry; j <= ry; j++)
            for (k = -rx; k <= rx; k++)
                acc += fy[j + ry] * fx[k + rx]
                       * (double)img[wss(cy + j, H) * pitch + wss(cx + k, W)];
        res[i] = acc;
    }
}

/* Pointwise algorithm B on an fp64 image (used by the multi-level sampled
 * checks, where the level input is an oracle LL image). */
void oracle_dwt53_conv_sample(const double *img, long pitch, long W, long H, long count,
                              const int *band, const long *m, const long *n, double *res)
{
    long i;
    for (i = 0; i < count; i++)
        res[i] = conv_coeff(img, pitch, W, H, band[i], m[i], n[i]);
}

/* The reflection rule itself, exported so the tests can pin it. */
long oracle_wss_index(long k, long n)
{
    return wss(k, n);
}
