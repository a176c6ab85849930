/*
 * oracle/dwt97_oracle.c -- CPU oracle for the forward / inverse 2-D CDF 9/7
 * DWT ("the paper claims generality").
 *
 * TEST INFRASTRUCTURE ONLY (same rules as dwt53_oracle.c): nothing on the
 * product path may load, link or call this file; it shares no code, header,
 * table or constant with paper_1708_07853_b200/csrc.
 *
 * What it computes.  PAPER.md L39 ("the presented schemes are general and
 * they are not limited to any particular wavelet") and L365-367; the lifting
 * factorisation of Eq. (2) (L71-92) with K = 2 predict/update pairs and a
 * scaling step ("cdf97 ... K = 2 with a nontrivial scaling
 * step").  The 2-D transform is the tensor product of 1-D transforms
 * (PAPER.md L100), rows then columns, recursing on LL, Mallat layout -- the
 * same plain definition as the 5/3 oracle.
 *
 * Readings (C-B1 .. C-B3):
 *   - lifting constants of the CDF 9/7 factorisation (Daubechies & Sweldens,
 *     "Factoring wavelet transforms into lifting steps", 1998), as used by
 *     JPEG 2000's irreversible transform:
 *        predict 1  d += ALPHA (s[i] + s[i+1])
 *        update  1  s += BETA  (d[i-1] + d[i])
 *        predict 2  d += GAMMA (s[i] + s[i+1])
 *        update  2  s += DELTA (d[i-1] + d[i])
 *        scaling    low = s / KAPPA, high = d * KAPPA
 *     (low-pass DC gain 1, as the 5/3 pair; JPEG 2000 normalisation);
 *   - phase (L even), z direction and Mallat layout as the 5/3 oracle;
 *   - boundaries: the transform of the whole-sample symmetric extension of
 *     the input, computed literally: the signal is extended by PAD samples on
 *     each side, every lifting step runs over the extended signal, and the
 *     central n samples are kept (no separate boundary rule is written).
 *
 *   A97. separable lifting (the four steps above + scaling, per axis);
 *   B97. brute-force convolution with the published CDF 9/7 analysis filter
 *        bank (9-tap low-pass H97, 7-tap high-pass G97; JPEG 2000 Part 1),
 *        every coefficient an independent 2-D weighted sum -- written from
 *        the published taps, NOT derived from A97, so A97 == B97 (to the taps'
 *        16 printed digits) pins the lifting constants, their order and signs;
 *   C97. inverse lifting (steps reversed, signs flipped, scaling undone) on
 *        the symmetric extension of the interleaved coefficient signal.
 */
#include <stdlib.h>
#include <string.h>

#define PAD 8

static void lift_step(double *e, long len, int par, long lo, long hi, double coef);
static long wss97(long k, long n);

static const double ALPHA = -1.586134342059924;
static const double BETA = -0.052980118572961;
static const double GAMMA = 0.882911075530934;
static const double DELTA = 0.443506852043971;
static const double KAPPA = 1.230174104914001;

/* Published CDF 9/7 analysis filters (JPEG 2000 irreversible 9/7):
 * low-pass centred on even samples, offsets 0, +-1, .., +-4; high-pass
 * centred on odd samples, offsets 0, +-1, .., +-3. */
static const double H97[5] = {0.6029490182363579, 0.2668641184428723, -0.07822326652898785,
                              -0.01686411844287495, 0.02674875741080976};
static const double G97[4] = {1.115087052456994, -0.5912717631142470, -0.05754352622849957,
                              0.09127176311424948};

/* whole-sample symmetric reflection (same rule as dwt53_oracle.c) */
static long wss97(long k, long n)
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

/* One lifting step over the extended signal e[0..len): every sample of
 * parity `par` in [lo, hi) gets coef * (its two neighbours). */
static void lift_step(double *e, long len, int par, long lo, long hi, double coef)
{
    long j;
    (void)len;
    for (j = lo; j < hi; j++)
        if ((j & 1) == par)
            e[j] += coef * (e[j - 1] + e[j + 1]);
}

/* Forward 1-D lifting with two predict/update pairs and scaling (c = the
 * four lifting coefficients p1, u1, p2, u2; K the scaling) of x[0..n)
 * (stride apart): ceil(n/2) low, floor(n/2) high.  CDF 9/7 is
 * c = (ALPHA, BETA, GAMMA, DELTA), K = KAPPA; CDF 5/3 is (-1/2, 1/4, 0, 0), 1. */
static void lift2_fwd_1d(const double *x, long n, long stride, double *low, double *high, const double *c,
                         double K)
{
    long len = n + 2 * PAD, j, i;
    double *e = (double *)malloc((size_t)len * sizeof(double));
    for (j = 0; j < len; j++)
        e[j] = x[wss97(j - PAD, n) * stride];           /* PAD even: parity of j = parity of j - PAD */
    lift_step(e, len, 1, 1, len - 1, c[0]);             /* valid odd samples: [1, len-1) */
    lift_step(e, len, 0, 2, len - 2, c[1]);             /* valid even samples: [2, len-2) */
    lift_step(e, len, 1, 3, len - 3, c[2]);
    lift_step(e, len, 0, 4, len - 4, c[3]);             /* [4, len-4) covers [PAD, PAD+n) */
    for (i = 0; i < (n + 1) / 2; i++)
        low[i] = e[PAD + 2 * i] / K;
    for (i = 0; i < n / 2; i++)
        high[i] = e[PAD + 2 * i + 1] * K;
    free(e);
}

static const double C97[4] = {-1.586134342059924, -0.052980118572961, 0.882911075530934, 0.443506852043971};

static void lift97_fwd_1d(const double *x, long n, long stride, double *low, double *high)
{
    (void)ALPHA; (void)BETA; (void)GAMMA; (void)DELTA;
    lift2_fwd_1d(x, n, stride, low, high, C97, KAPPA);
}

/* Inverse of lift2_fwd_1d: x[0..n) (stride apart) from low / high. */
static void lift2_inv_1d(const double *low, const double *high, long n, double *x, long stride, const double *cf,
                         double K)
{
    long len = n + 2 * PAD, j, i, nl = (n + 1) / 2;
    double *c, *e;
    if (n == 1) {
        /* one sample: the extended signal is constant, so the forward is
         * low = G x / K with G the lifting's gain on a constant */
        double d1 = 1.0 + 2.0 * cf[0], s1 = 1.0 + 2.0 * cf[1] * d1;
        double d2 = d1 + 2.0 * cf[2] * s1, G = s1 + 2.0 * cf[3] * d2;
        x[0] = low[0] * K / G;
        return;
    }
    c = (double *)malloc((size_t)n * sizeof(double));
    e = (double *)malloc((size_t)len * sizeof(double));
    /* interleaved coefficient signal, scaling undone; it is symmetric with
     * the same whole-sample rule as the input, so it is extended likewise */
    for (i = 0; i < nl; i++)
        c[2 * i] = low[i] * K;
    for (i = 0; i < n / 2; i++)
        c[2 * i + 1] = high[i] / K;
    for (j = 0; j < len; j++)
        e[j] = c[wss97(j - PAD, n)];
    lift_step(e, len, 0, 1, len - 1, -cf[3]);
    lift_step(e, len, 1, 2, len - 2, -cf[2]);
    lift_step(e, len, 0, 3, len - 3, -cf[1]);
    lift_step(e, len, 1, 4, len - 4, -cf[0]);
    for (i = 0; i < n; i++)
        x[i * stride] = e[PAD + i];
    free(e);
    free(c);
}

static void lift97_inv_1d(const double *low, const double *high, long n, double *x, long stride)
{
    lift2_inv_1d(low, high, n, x, stride, C97, KAPPA);
}

static void level97_fwd_lifting(double *buf, long pitch, long W, long H)
{
    long nlx = (W + 1) / 2, nly = (H + 1) / 2, x, y;
    double *tmp = (double *)malloc((size_t)W * (size_t)H * sizeof(double));
    double *line = (double *)malloc((size_t)(W > H ? W : H) * sizeof(double));
    for (y = 0; y < H; y++) {
        lift97_fwd_1d(buf + y * pitch, W, 1, line, line + nlx);
        memcpy(tmp + y * W, line, (size_t)W * sizeof(double));
    }
    for (x = 0; x < W; x++) {
        lift97_fwd_1d(tmp + x, H, W, line, line + nly);
        for (y = 0; y < H; y++)
            buf[y * pitch + x] = line[y];
    }
    free(line);
    free(tmp);
}

static void level97_inv_lifting(double *buf, long pitch, long W, long H)
{
    long nlx = (W + 1) / 2, nly = (H + 1) / 2, x, y;
    double *tmp = (double *)malloc((size_t)W * (size_t)H * sizeof(double));
    double *line = (double *)malloc((size_t)(W > H ? W : H) * sizeof(double));
    for (x = 0; x < W; x++) {
        for (y = 0; y < H; y++)
            line[y] = buf[y * pitch + x];
        lift97_inv_1d(line, line + nly, H, tmp + x, W);
    }
    for (y = 0; y < H; y++) {
        memcpy(line, tmp + y * W, (size_t)W * sizeof(double));
        lift97_inv_1d(line, line + nlx, W, buf + y * pitch, 1);
    }
    free(line);
    free(tmp);
}

/* B97: one coefficient by brute-force 2-D convolution with the published taps */
static double conv97_coeff(const double *img, long pitch, long W, long H, int band, long m, long n)
{
    int hx = (band == 1 || band == 3), vy = (band == 2 || band == 3);
    int rx = hx ? 3 : 4, ry = vy ? 3 : 4;
    long cx = hx ? 2 * m + 1 : 2 * m, cy = vy ? 2 * n + 1 : 2 * n;
    double acc = 0.0;
    int i, j;
    for (j = -ry; j <= ry; j++) {
        double wy = vy ? G97[abs(j)] : H97[abs(j)];
        for (i = -rx; i <= rx; i++) {
            double wx = hx ? G97[abs(i)] : H97[abs(i)];
            acc += wy * wx * img[wss97(cy + j, H) * pitch + wss97(cx + i, W)];
        }
    }
    return acc;
}

static void level97_fwd_conv(double *buf, long pitch, long W, long H)
{
    long nlx = (W + 1) / 2, nly = (H + 1) / 2, nhx = W / 2, nhy = H / 2, m, n;
    double *res = (double *)malloc((size_t)W * (size_t)H * sizeof(double));
    for (n = 0; n < nly; n++)
        for (m = 0; m < nlx; m++)
            res[n * W + m] = conv97_coeff(buf, pitch, W, H, 0, m, n);
    for (n = 0; n < nly; n++)
        for (m = 0; m < nhx; m++)
            res[n * W + nlx + m] = conv97_coeff(buf, pitch, W, H, 1, m, n);
    for (n = 0; n < nhy; n++)
        for (m = 0; m < nlx; m++)
            res[(nly + n) * W + m] = conv97_coeff(buf, pitch, W, H, 2, m, n);
    for (n = 0; n < nhy; n++)
        for (m = 0; m < nhx; m++)
            res[(nly + n) * W + nlx + m] = conv97_coeff(buf, pitch, W, H, 3, m, n);
    for (n = 0; n < H; n++)
        memcpy(buf + n * pitch, res + n * W, (size_t)W * sizeof(double));
    free(res);
}

static void round97_f32(double *buf, long pitch, long W, long H)
{
    long x, y;
    for (y = 0; y < H; y++)
        for (x = 0; x < W; x++)
            buf[y * pitch + x] = (double)(float)buf[y * pitch + x];
}

/* ---- exported (ctypes; tests/ and bench only) ---- */

void oracle_dwt97_fwd_1d(const double *x, long n, double *out)
{
    lift97_fwd_1d(x, n, 1, out, out + (n + 1) / 2);
}

void oracle_dwt97_inv_1d(const double *in, long n, double *x)
{
    lift97_inv_1d(in, in + (n + 1) / 2, n, x, 1);
}

/* General K <= 2 lifting (SURVEY.md 8f N4 "general lifting wavelets"):
 * c = (p1, u1, p2, u2), K the scaling; levels of separable lifting on the
 * symmetric extension, Mallat layout; round_f32 as below. */
long oracle_lift2_forward(const double *in, double *out, long W, long H, long levels, int round_f32,
                          const double *c, double K)
{
    long k, w = W, h = H, x, y, nlx, nly;
    double *tmp, *line;
    if (W < 1 || H < 1 || levels < 0 || !(K > 0.0))
        return -1;
    memcpy(out, in, (size_t)W * (size_t)H * sizeof(double));
    tmp = (double *)malloc((size_t)W * (size_t)H * sizeof(double));
    line = (double *)malloc((size_t)(W > H ? W : H) * sizeof(double));
    for (k = 0; k < levels; k++) {
        nlx = (w + 1) / 2;
        nly = (h + 1) / 2;
        for (y = 0; y < h; y++) {
            lift2_fwd_1d(out + y * W, w, 1, line, line + nlx, c, K);
            memcpy(tmp + y * w, line, (size_t)w * sizeof(double));
        }
        for (x = 0; x < w; x++) {
            lift2_fwd_1d(tmp + x, h, w, line, line + nly, c, K);
            for (y = 0; y < h; y++)
                out[y * W + x] = line[y];
        }
        if (round_f32)
            round97_f32(out, W, w, h);
        w = nlx;
        h = nly;
    }
    free(line);
    free(tmp);
    return levels;
}

/* levels of A97 (use_conv = 0) or B97 (use_conv = 1); round_f32 rounds each
 * level's output to fp32 (the GPU storage type). */
long oracle_dwt97_forward(const double *in, double *out, long W, long H, long levels, int round_f32,
                          int use_conv)
{
    long k, w = W, h = H;
    if (W < 1 || H < 1 || levels < 0)
        return -1;
    memcpy(out, in, (size_t)W * (size_t)H * sizeof(double));
    for (k = 0; k < levels; k++) {
        if (use_conv)
            level97_fwd_conv(out, W, w, h);
        else
            level97_fwd_lifting(out, W, w, h);
        if (round_f32)
            round97_f32(out, W, w, h);
        w = (w + 1) / 2;
        h = (h + 1) / 2;
    }
    return levels;
}

long oracle_dwt97_inverse(const double *in, double *out, long W, long H, long levels, int round_f32)
{
    long k, ws[64], hs[64];
    if (W < 1 || H < 1 || levels < 0 || levels > 63)
        return -1;
    ws[0] = W;
    hs[0] = H;
    for (k = 1; k <= levels; k++) {
        ws[k] = (ws[k - 1] + 1) / 2;
        hs[k] = (hs[k - 1] + 1) / 2;
    }
    memcpy(out, in, (size_t)W * (size_t)H * sizeof(double));
    for (k = levels - 1; k >= 0; k--) {
        level97_inv_lifting(out, W, ws[k], hs[k]);
        if (round_f32)
            round97_f32(out, W, ws[k], hs[k]);
    }
    return levels;
}

/* B97 pointwise on an fp32 image: res[i] = coefficient (band[i], m[i], n[i]) */
void oracle_dwt97_conv_sample_f32(const float *img, long pitch, long W, long H, long count,
                                  const int *band, const long *m, const long *n, double *res)
{
    long i;
    int j, k;
    for (i = 0; i < count; i++) {
        int hx = (band[i] == 1 || band[i] == 3), vy = (band[i] == 2 || band[i] == 3);
        int rx = hx ? 3 : 4, ry = vy ? 3 : 4;
        long cx = hx ? 2 * m[i] + 1 : 2 * m[i], cy = vy ? 2 * n[i] + 1 : 2 * n[i];
        double acc = 0.0;
        for (j = -ry; j <= ry; j++)
            for (k = -rx; k <= rx; k++)
                acc += (vy ? G97[abs(j)] : H97[abs(j)]) * (hx ? G97[abs(k)] : H97[abs(k)])
                       * (double)img[wss97(cy + j, H) * pitch + wss97(cx + k, W)];
        res[i] = acc;
    }
}
