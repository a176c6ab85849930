// tail.cu -- the small last levels of a forward in ONE launch (SURVEY.md 8a
// row a7, the multi-level driver; BASELINE.json north_star "a multi-level
// driver recursing on LL").
//
// Levels of a few hundred KB are latency-bound: one dependent launch of a
// level kernel costs ~3.5-4 us whatever its size for the 5/3 kernel and 9-20 us
// for the K = 2 (CDF 9/7) kernel, whose warps walk a tile row by row through
// four lifting steps.  The tail kernel runs every such level
// in one launch of one or two CTAs per SM, all resident (the grid is clamped to
// the kernel's occupancy), with a grid barrier (release / acquire on a
// self-resetting counter) between levels.  Each thread owns quads and
// evaluates a quad's four coefficients pointwise from its neighbourhood of the
// whole-sample-symmetric extension: the 2-D analysis filters of Eq. (4)
// -- which the lifting steps of Eq. (5) reach exactly --
// as a row pass and a column pass:
//
//   LL = s_ll * h (x) h,  HL = s_d * g (x) h,  LH = s_d * h (x) g,  HH = s_hh * g (x) g
//
// with h the low-pass taps at even positions (radius R) and g the high-pass
// taps at odd positions (radius R - 1).  R = 2: the CDF 5/3 pair, taps written
// out (h = (-1/8, 1/4, 3/4, 1/4, -1/8), g = (-1/2, 1, -1/2)); every product
// and sum is exact in fp64 for these data, so the stored fp32 is bit for bit
// the level kernel's.  R = 4: any K <= 2 lifting pair (CDF 9/7, general
// lifting plans), taps derived on the host from the lifting coefficients by
// lifting unit impulses (tail_filter_from_lifting); the result differs from
// the lifting order only by fp64 rounding (<< the 1e-4 bar).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "dwt2_internal.h"

using namespace dwt2_detail;

namespace {

constexpr int TAIL_THREADS = 256;

struct TailArgs {
    TailLevelIO lv[MAX_TAIL];
    double h[9], g[7];                // R = 4 taps, index = offset + 4 (h) / + 3 (g)
    double sll, sd, shh;              // output scaling (R = 4)
    int nlev, count;
    unsigned int *bar;                // [0] barrier arrivals, [1] CTAs done (the last zeroes both)
};

__device__ __forceinline__ unsigned ld_relaxed(const unsigned int *p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void tail_barrier(unsigned int *bar, unsigned target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.release.gpu;" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while (ld_relaxed(bar) < target) {}
        asm volatile("fence.acquire.gpu;" ::: "memory");
    }
    __syncthreads();
}

// whole-sample symmetric reflection, any k (period 2 (n - 1), n >= 2)
__device__ __forceinline__ int wss_any(int k, int n)
{
    const int p = 2 * (n - 1);
    k %= p;
    if (k < 0) k += p;
    return k >= n ? p - k : k;
}

// one reflection when it suffices (|overhang| < n - 1), else the general form
__device__ __forceinline__ int wss_fast(int k, int n)
{
    const int r = k < 0 ? -k : (k >= n ? 2 * (n - 1) - k : k);
    return (r >= 0 && r < n) ? r : wss_any(k, n);
}

// reflection for k in [-2, n + 1], n >= 2 (radius-2 path)
__device__ __forceinline__ int wss2(int k, int n)
{
    k = k < 0 ? -k : k;
    return k >= n ? 2 * (n - 1) - k : k;
}

template <int R>
__global__ void __launch_bounds__(TAIL_THREADS) dwt_tail_kernel(const __grid_constant__ TailArgs ta)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int NT = 2 * R + 1;     // taps of h (g: NT - 2)
    const long long nthr = (long long)gridDim.x * TAIL_THREADS;
    const long long tid = (long long)blockIdx.x * TAIL_THREADS + threadIdx.x;
    for (int k = 0; k < ta.nlev; ++k) {
        if (k > 0) tail_barrier(ta.bar, unsigned(k) * gridDim.x);
        const TailLevelIO &L = ta.lv[k];
        const int W = L.W, H = L.H;
        const int Wq = (W + 1) >> 1, Hq = (H + 1) >> 1, Wh = W >> 1, Hh = H >> 1;
        const long long per_img = (long long)Wq * Hq;
        const long long total = per_img * ta.count;
        for (long long q = tid; q < total; q += nthr) {
            const int img = int(q / per_img);
            const int r = int(q - img * per_img);
            const int n = r / Wq, m = r - n * Wq;
            const float *x = L.in + img * L.in_img;
            int cx[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) cx[i] = R == 2 ? wss2(2 * m - R + i, W) : wss_fast(2 * m - R + i, W);
            double lo[NT], hi[NT];     // row passes: h at column 2m, g at column 2m + 1
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int y = R == 2 ? wss2(2 * n - R + j, H) : wss_fast(2 * n - R + j, H);
                const float *row = x + (long long)y * L.in_pitch;
                double v[NT];
#pragma unroll
                for (int i = 0; i < NT; ++i) v[i] = __ldcg(row + cx[i]);
                if (R == 2) {
                    lo[j] = fma(0.75, v[2], fma(0.25, v[1] + v[3], -0.125 * (v[0] + v[4])));
                    hi[j] = fma(-0.5, v[2] + v[4], v[3]);
                } else {
                    double s = 0.0, t = 0.0;
#pragma unroll
                    for (int i = 0; i < NT; ++i) s = fma(ta.h[i], v[i], s);
#pragma unroll
                    for (int i = 0; i < NT - 2; ++i) t = fma(ta.g[i], v[i + 2], t);
                    lo[j] = s;
                    hi[j] = t;
                }
            }
            double ll, lh, hl, hh;
            if (R == 2) {
                ll = fma(0.75, lo[2], fma(0.25, lo[1] + lo[3], -0.125 * (lo[0] + lo[4])));
                lh = fma(-0.5, lo[2] + lo[4], lo[3]);
                hl = fma(0.75, hi[2], fma(0.25, hi[1] + hi[3], -0.125 * (hi[0] + hi[4])));
                hh = fma(-0.5, hi[2] + hi[4], hi[3]);
            } else {
                ll = lh = hl = hh = 0.0;
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    ll = fma(ta.h[j], lo[j], ll);
                    hl = fma(ta.h[j], hi[j], hl);
                }
#pragma unroll
                for (int j = 0; j < NT - 2; ++j) {
                    lh = fma(ta.g[j], lo[j + 2], lh);
                    hh = fma(ta.g[j], hi[j + 2], hh);
                }
                ll *= ta.sll;
                hl *= ta.sd;
                lh *= ta.sd;
                hh *= ta.shh;
            }
            L.ll[img * L.ll_img + (long long)n * L.ll_pitch + m] = (float)ll;
            float *o = L.out + img * L.out_img;
            if (m < Wh) o[(long long)n * L.out_pitch + Wq + m] = (float)hl;
            if (n < Hh) {
                o[(long long)(Hq + n) * L.out_pitch + m] = (float)lh;
                if (m < Wh) o[(long long)(Hq + n) * L.out_pitch + Wq + m] = (float)hh;
            }
        }
    }
    // the last CTA out resets the barrier counters for the next launch
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(ta.bar + 1, 1u) == gridDim.x - 1) {
        atomicExch(ta.bar, 0u);
        atomicExch(ta.bar + 1, 0u);
    }
}

// ---- small single levels: one launch, one CTA per 32 x 8 quad block ------
//
// A level of at most a few MB (config 1: 512^2) is latency-bound on the level
// kernel, whose warps walk their tiles row by row through a TMA ring (a serial
// fp64 chain of ~3 us per 8-row stage).  Here a CTA loads the 19 x 67 input
// pixels its 32 x 8 quads depend on (rows 2 n0 - 2 .. 2 n0 + 16, columns
// 2 m0 - 2 .. 2 m0 + 64, whole-sample symmetric at the image edges) into
// shared memory in ONE round of independent coalesced loads, and every thread
// evaluates one quad pointwise with the exact 5 x 5 analysis filters of the
// radius-2 tail path (bit for bit the level kernel's values).  (Staging even
// and odd columns apart to avoid the 2-way bank conflicts of the window reads
// measured slower: 512^2 3.7 -> 4.1 us.)
constexpr int SQX = 32, SQY = 8;                         // quads per CTA
constexpr int STR = 2 * SQY + 3, STC = 2 * SQX + 3;      // staged rows / columns
constexpr int SN = (STR * STC + 255) / 256;              // staged floats per thread

__global__ void __launch_bounds__(256) dwt53_small_kernel(const __grid_constant__ TailLevelIO L, int nbx)
{
    __shared__ float t[STR][STC + 1];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int W = L.W, H = L.H;
    const int Wq = (W + 1) >> 1, Hq = (H + 1) >> 1, Wh = W >> 1, Hh = H >> 1;
    const int bx = blockIdx.x % nbx, by = blockIdx.x / nbx, img = blockIdx.y;
    const int m0 = bx * SQX, n0 = by * SQY;
    const float *x = L.in + img * L.in_img;
    float v[SN];
#pragma unroll
    for (int k = 0; k < SN; ++k) {                       // every load in flight at once
        const int i = threadIdx.x + 256 * k;
        const int r = i / STC, c = i - (i / STC) * STC;
        const int yy = 2 * n0 - 2 + r, xx = 2 * m0 - 2 + c;
        v[k] = (i < STR * STC && yy <= H + 1 && xx <= W + 1)
                   ? __ldg(x + (long long)wss2(yy, H) * L.in_pitch + wss2(xx, W)) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < SN; ++k) {
        const int i = threadIdx.x + 256 * k;
        if (i < STR * STC) t[i / STC][i - (i / STC) * STC] = v[k];
    }
    __syncthreads();
    const int tx = threadIdx.x & (SQX - 1), ty = threadIdx.x / SQX;
    const int m = m0 + tx, n = n0 + ty;
    if (m >= Wq || n >= Hq) return;
    double lo[5], hi[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const float *w = &t[2 * ty + j][2 * tx];
        const double v0 = w[0], v1 = w[1], v2 = w[2], v3 = w[3], v4 = w[4];
        lo[j] = fma(0.75, v2, fma(0.25, v1 + v3, -0.125 * (v0 + v4)));
        hi[j] = fma(-0.5, v2 + v4, v3);
    }
    const double ll = fma(0.75, lo[2], fma(0.25, lo[1] + lo[3], -0.125 * (lo[0] + lo[4])));
    const double lh = fma(-0.5, lo[2] + lo[4], lo[3]);
    const double hl = fma(0.75, hi[2], fma(0.25, hi[1] + hi[3], -0.125 * (hi[0] + hi[4])));
    const double hh = fma(-0.5, hi[2] + hi[4], hi[3]);
    L.ll[img * L.ll_img + (long long)n * L.ll_pitch + m] = (float)ll;
    float *o = L.out + img * L.out_img;
    if (m < Wh) o[(long long)n * L.out_pitch + Wq + m] = (float)hl;
    if (n < Hh) {
        o[(long long)(Hq + n) * L.out_pitch + m] = (float)lh;
        if (m < Wh) o[(long long)(Hq + n) * L.out_pitch + Wq + m] = (float)hh;
    }
}

// ---- small single levels of a K <= 2 lifting wavelet (radius-4 filters) ---
//
// The K = 2 level kernel walks a tile row by row through four lifting steps and
// four warm-up rows; a level of a few MB is a chain of such walks.  Here a CTA
// of 256 threads owns 32 x 8 quads: it stages the 23 x 71 input pixels they
// depend on (mirrored) in shared memory in one round of loads, runs the row
// pass once per staged row and quad column (the 9 low taps at column 2m, the 7
// high taps at 2m + 1, in fp64, into shared memory), then every thread runs the
// column pass of its quad and the 2-D scaling -- the tail kernel's radius-4
// evaluation, term for term, with each row pass shared by the quads above and
// below it.  Measured (scripts/r2/k2small_probe.py): a 1024^2 9/7 level 9.53 ->
// 8.72 us, the 9/7 config-4 pyramid 175.6 -> 174.4 us; from 2048^2 up it loses
// (15.2 -> 29.0 us: shared-memory and fp64 issue bound; staging the tile as fp64
// to save the conversions was slower still, 43 us with 16-byte-strided reads and
// 41.8 us with even / odd columns apart), so levels of <= 2^18 quads only.
constexpr int R4X = 32, R4Y = 8;
constexpr int R4R = 2 * R4Y + 7, R4C = 2 * R4X + 7;      // staged rows / columns
constexpr int R4N = (R4R * R4C + 255) / 256;

struct Small4Args {
    TailLevelIO L;
    double h[9], g[7];
    double sll, sd, shh;
    int nbx;
};

__global__ void __launch_bounds__(256) dwt_small4_kernel(const __grid_constant__ Small4Args A)
{
    __shared__ float t[R4R][R4C + 1];
    __shared__ double lo[R4R][R4X], hi[R4R][R4X];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const TailLevelIO &L = A.L;
    const int W = L.W, H = L.H;
    const int Wq = (W + 1) >> 1, Hq = (H + 1) >> 1, Wh = W >> 1, Hh = H >> 1;
    const int bx = blockIdx.x % A.nbx, by = blockIdx.x / A.nbx, img = blockIdx.y;
    const int m0 = bx * R4X, n0 = by * R4Y;
    const float *x = L.in + img * L.in_img;
    float v[R4N];
#pragma unroll
    for (int k = 0; k < R4N; ++k) {                      // every load in flight at once
        const int i = threadIdx.x + 256 * k;
        const int r = i / R4C, c = i - (i / R4C) * R4C;
        const int yy = 2 * n0 - 4 + r, xx = 2 * m0 - 4 + c;
        v[k] = (i < R4R * R4C && yy < H + 4 && xx < W + 4)
                   ? __ldg(x + (long long)wss_fast(yy, H) * L.in_pitch + wss_fast(xx, W)) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < R4N; ++k) {
        const int i = threadIdx.x + 256 * k;
        if (i < R4R * R4C) t[i / R4C][i - (i / R4C) * R4C] = v[k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < R4R * R4X; i += 256) {    // row passes
        const int r = i / R4X, q = i - (i / R4X) * R4X;
        const float *w = &t[r][2 * q];
        double s = 0.0, u = 0.0;
#pragma unroll
        for (int j = 0; j < 9; ++j) s = fma(A.h[j], (double)w[j], s);
#pragma unroll
        for (int j = 0; j < 7; ++j) u = fma(A.g[j], (double)w[j + 2], u);
        lo[r][q] = s;
        hi[r][q] = u;
    }
    __syncthreads();
    const int tx = threadIdx.x & (R4X - 1), ty = threadIdx.x / R4X;
    const int m = m0 + tx, n = n0 + ty;
    if (m >= Wq || n >= Hq) return;
    double ll = 0.0, hl = 0.0, lh = 0.0, hh = 0.0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        ll = fma(A.h[j], lo[2 * ty + j][tx], ll);
        hl = fma(A.h[j], hi[2 * ty + j][tx], hl);
    }
#pragma unroll
    for (int j = 0; j < 7; ++j) {
        lh = fma(A.g[j], lo[2 * ty + j + 2][tx], lh);
        hh = fma(A.g[j], hi[2 * ty + j + 2][tx], hh);
    }
    L.ll[img * L.ll_img + (long long)n * L.ll_pitch + m] = (float)(ll * A.sll);
    float *o = L.out + img * L.out_img;
    if (m < Wh) o[(long long)n * L.out_pitch + Wq + m] = (float)(hl * A.sd);
    if (n < Hh) {
        o[(long long)(Hq + n) * L.out_pitch + m] = (float)(lh * A.sd);
        if (m < Wh) o[(long long)(Hq + n) * L.out_pitch + Wq + m] = (float)(hh * A.shh);
    }
}

// ---- small single levels of an INVERSE ------------------------------------
//
// The inverse level kernels walk their tiles row by row too (the K = 2 inverse:
// ~10-13 us per small level of a 9/7 pyramid).  Here a CTA owns 32 x 8 output
// quads (64 x 16 pixels) and stages the (16 + 2R) x (64 + 2R) window of the
// INTERLEAVED coefficient field they depend on -- c(y, x) = LL / HL / LH / HH
// by the parities of (y, x), at whole-sample-symmetric mirrored positions (the
// coefficient field of a symmetric input is symmetric in the interleaved
// index; the parity of a position survives the mirror) -- in one round of
// loads, then synthesises separably in fp64: a horizontal pass per staged row
// and output column pair into shared memory, and each thread's vertical pass
// for its quad's 2 x 2 pixels:
//   x(p_y, p_x) = sum_q s_{q_y mod 2}[p_y - q_y] s_{q_x mod 2}[p_x - q_x] k(q) c(q)
// with s_0 / s_1 the low / high synthesis taps of the lifting pair (the inverse
// lifting applied to unit impulses, inv_filter_from_lifting) and k the undo of
// the forward scaling.  CDF 5/3: s_0 = (1/2, 1, 1/2), s_1 = (-1/8, -1/4, 3/4,
// -1/4, -1/8), dyadic -- every product and sum is exact in fp64, so the stored
// fp32 is bit for bit the inverse level kernel's.
constexpr int IVX = 32, IVY = 8;

struct SmallInvArgs {
    InvLevelIO L;
    double s0[9], s1[9];              // synthesis taps at offsets -4..4 (index offset + 4)
    double kll, kd, khh;
    int nbx;
};

template <int R>
__global__ void __launch_bounds__(256) dwt_small_inv_kernel(const __grid_constant__ SmallInvArgs A)
{
    constexpr int WS = 2 * R + 2;                          // coefficient rows / columns of one quad
    constexpr int SR = 2 * IVY + 2 * R, SC = 2 * IVX + 2 * R;
    constexpr int SN = (SR * SC + 255) / 256;
    __shared__ float t[SR][SC + 1];
    __shared__ double h0[SR][IVX], h1[SR][IVX];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const InvLevelIO &L = A.L;
    const int W = L.W, H = L.H;
    const int Wq = (W + 1) >> 1, Hq = (H + 1) >> 1;
    const int bx = blockIdx.x % A.nbx, by = blockIdx.x / A.nbx, img = blockIdx.y;
    const int m0 = bx * IVX, n0 = by * IVY;
    const int y0 = 2 * n0 - R, x0 = 2 * m0 - R;
    const float *llp = L.ll + img * L.ll_img;
    const float *dp = L.d + img * L.d_img;
    float v[SN];
#pragma unroll
    for (int k = 0; k < SN; ++k) {                       // every load in flight at once
        const int i = threadIdx.x + 256 * k;
        const int r = i / SC, c = i - (i / SC) * SC;
        float val = 0.f;
        if (i < SR * SC && y0 + r < H + R + 1 && x0 + c < W + R + 1) {
            const int y = wss_any(y0 + r, H), x = wss_any(x0 + c, W);
            const int ry = y >> 1, cx = x >> 1;
            const float *src = (!(y & 1) && !(x & 1)) ? llp + (long long)ry * L.ll_pitch + cx
                             : dp + (long long)((y & 1) ? Hq + ry : ry) * L.d_pitch + ((x & 1) ? Wq + cx : cx);
            val = __ldg(src);
        }
        v[k] = val;
    }
#pragma unroll
    for (int k = 0; k < SN; ++k) {
        const int i = threadIdx.x + 256 * k;
        if (i < SR * SC) t[i / SC][i - (i / SC) * SC] = v[k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < SR * IVX; i += 256) {    // horizontal synthesis
        const int r = i / IVX, q = i - (i / IVX) * IVX;
        const bool py = (y0 + r) & 1;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int j = 0; j < WS; ++j) {
            const int qpar = (R + j) & 1;                 // parity of column 2m - R + j
            const double k = (!py && !qpar) ? A.kll : (py && qpar) ? A.khh : A.kd;
            const double c = k * double(t[r][2 * q + j]);
            const double *sx = qpar ? A.s1 : A.s0;
            const int o0 = R - j;                          // 2m - (2m - R + j)
            if (o0 >= -4 && o0 <= 4) a0 = fma(sx[o0 + 4], c, a0);
            if (o0 + 1 >= -4 && o0 + 1 <= 4) a1 = fma(sx[o0 + 5], c, a1);
        }
        h0[r][q] = a0;
        h1[r][q] = a1;
    }
    __syncthreads();
    const int tx = threadIdx.x & (IVX - 1), ty = threadIdx.x / IVX;
    const int m = m0 + tx, n = n0 + ty;
    if (m >= Wq || n >= Hq) return;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int j = 0; j < WS; ++j) {
        const double *sy = ((R + j) & 1) ? A.s1 : A.s0;
        const int o0 = R - j;
        const double u0 = h0[2 * ty + j][tx], u1 = h1[2 * ty + j][tx];
        if (o0 >= -4 && o0 <= 4) {
            acc[0][0] = fma(sy[o0 + 4], u0, acc[0][0]);
            acc[0][1] = fma(sy[o0 + 4], u1, acc[0][1]);
        }
        if (o0 + 1 >= -4 && o0 + 1 <= 4) {
            acc[1][0] = fma(sy[o0 + 5], u0, acc[1][0]);
            acc[1][1] = fma(sy[o0 + 5], u1, acc[1][1]);
        }
    }
    float *o = L.out + img * L.out_img + (long long)(2 * n) * L.out_pitch + 2 * m;
    o[0] = (float)acc[0][0];
    if (2 * m + 1 < W) o[1] = (float)acc[0][1];
    if (2 * n + 1 < H) {
        o[L.out_pitch] = (float)acc[1][0];
        if (2 * m + 1 < W) o[L.out_pitch + 1] = (float)acc[1][1];
    }
}

template <int R>
int tail_resident()
{
    static int n = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dwt_tail_kernel<R>, TAIL_THREADS, 0) != cudaSuccess)
            n = 1;
        n = std::max(1, n);
    });
    cudaGetLastError();
    return n;
}

}  // namespace

namespace dwt2_detail {

TailFilter tail_filter_53()
{
    TailFilter f;
    memset(&f, 0, sizeof(f));
    f.radius = 2;
    f.sll = f.sd = f.shh = 1.0;
    return f;
}

TailFilter tail_filter_from_lifting(double c0, double c1, double c2, double c3, double K)
{
    // 1-D lifting of a unit impulse at position p of a long signal, far from
    // its ends: low[i] = h[p - 2 i], high[i] = g[p - 2 i - 1]
    //   d1 = x_odd + c0 (x_even[i] + x_even[i+1]),  s1 = x_even + c1 (d1[i-1] + d1[i]),
    //   d2 = d1 + c2 (s1[i] + s1[i+1]),             s2 = s1 + c3 (d2[i-1] + d2[i])
    TailFilter f;
    memset(&f, 0, sizeof(f));
    f.radius = 4;
    constexpr int N = 64, M = N / 2;
    for (int p = 30; p <= 31; ++p) {
        double x[N] = {0};
        x[p] = 1.0;
        double s[M], d[M];
        for (int i = 0; i < M; ++i) d[i] = x[2 * i + 1] + c0 * (x[2 * i] + (2 * i + 2 < N ? x[2 * i + 2] : 0.0));
        for (int i = 0; i < M; ++i) s[i] = x[2 * i] + c1 * ((i > 0 ? d[i - 1] : 0.0) + d[i]);
        for (int i = 0; i < M; ++i) d[i] = d[i] + c2 * (s[i] + (i + 1 < M ? s[i + 1] : 0.0));
        for (int i = 0; i < M; ++i) s[i] = s[i] + c3 * ((i > 0 ? d[i - 1] : 0.0) + d[i]);
        for (int i = 0; i < M; ++i) {
            const int jl = p - 2 * i, jh = p - 2 * i - 1;
            if (jl >= -4 && jl <= 4) f.h[jl + 4] = s[i];
            if (jh >= -3 && jh <= 3) f.g[jh + 3] = d[i];
        }
    }
    // 2-D scaling (JPEG 2000 normalisation, DESIGN.md C-B2): low / K and high * K per axis
    f.sll = 1.0 / (K * K);
    f.sd = 1.0;
    f.shh = K * K;
    return f;
}

int32_t launch_small_level(const TailLevelIO &lv, int count, cudaStream_t stream)
{
    const int Wq = (lv.W + 1) / 2, Hq = (lv.H + 1) / 2;
    const int nbx = (Wq + SQX - 1) / SQX, nby = (Hq + SQY - 1) / SQY;
    if ((long long)nbx * nby >= (1LL << 31) || count > 65535) return fail(DWT2_EINVAL);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nbx * nby, count);
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, dwt53_small_kernel, lv, nbx) != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

int32_t launch_small_level_r4(const TailLevelIO &lv, int count, const TailFilter &f, cudaStream_t stream)
{
    if (f.radius != 4) return fail(DWT2_EINVAL);
    const int Wq = (lv.W + 1) / 2, Hq = (lv.H + 1) / 2;
    Small4Args A;
    memset(&A, 0, sizeof(A));
    A.L = lv;
    memcpy(A.h, f.h, sizeof(A.h));
    memcpy(A.g, f.g, sizeof(A.g));
    A.sll = f.sll;
    A.sd = f.sd;
    A.shh = f.shh;
    A.nbx = (Wq + R4X - 1) / R4X;
    const int nby = (Hq + R4Y - 1) / R4Y;
    if ((long long)A.nbx * nby >= (1LL << 31) || count > 65535) return fail(DWT2_EINVAL);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(A.nbx * nby, count);
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, dwt_small4_kernel, A) != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

InvFilter inv_filter_from_lifting(double c0, double c1, double c2, double c3, double K)
{
    // inverse 1-D lifting of a unit coefficient at interleaved position q
    // (even: low, odd: high) of a long signal, far from its ends:
    //   s1 = s2 - c3 (d2[i-1] + d2[i]),  d1 = d2 - c2 (s1[i] + s1[i+1]),
    //   x_even = s1 - c1 (d1[i-1] + d1[i]),  x_odd = d1 - c0 (x_even[i] + x_even[i+1])
    InvFilter f;
    memset(&f, 0, sizeof(f));
    constexpr int N = 64, M = N / 2;
    for (int q = 30; q <= 31; ++q) {
        double sv[M] = {0}, d[M] = {0}, x[N];
        if (q % 2 == 0) sv[q / 2] = 1.0;
        else d[q / 2] = 1.0;
        for (int i = 0; i < M; ++i) sv[i] = sv[i] - c3 * ((i > 0 ? d[i - 1] : 0.0) + d[i]);
        for (int i = 0; i < M; ++i) d[i] = d[i] - c2 * (sv[i] + (i + 1 < M ? sv[i + 1] : 0.0));
        for (int i = 0; i < M; ++i) x[2 * i] = sv[i] - c1 * ((i > 0 ? d[i - 1] : 0.0) + d[i]);
        for (int i = 0; i < M; ++i) x[2 * i + 1] = d[i] - c0 * (x[2 * i] + (2 * i + 2 < N ? x[2 * i + 2] : 0.0));
        double *tap = q % 2 == 0 ? f.s0 : f.s1;
        int reach = 0;
        for (int p = 0; p < N; ++p) {
            const int off = p - q;
            if (off >= -4 && off <= 4) tap[off + 4] = x[p];
            else if (x[p] != 0.0) reach = 5;
            if (x[p] != 0.0) reach = std::max(reach, off < 0 ? -off : off);
        }
        f.radius = std::max(f.radius, reach);
    }
    f.radius = f.radius <= 2 ? 2 : (f.radius <= 4 ? 4 : 0);       // 0: taps beyond +-4 (unsupported)
    // undo the forward scaling (LL / K^2, HL and LH * 1, HH * K^2)
    f.kll = K * K;
    f.kd = 1.0;
    f.khh = 1.0 / (K * K);
    return f;
}

int32_t launch_small_inverse_level(const InvLevelIO &lv, int count, const InvFilter &f, cudaStream_t stream)
{
    if (f.radius != 2 && f.radius != 4) return fail(DWT2_EINVAL);
    const int Wq = (lv.W + 1) / 2, Hq = (lv.H + 1) / 2;
    SmallInvArgs A;
    memset(&A, 0, sizeof(A));
    A.L = lv;
    memcpy(A.s0, f.s0, sizeof(A.s0));
    memcpy(A.s1, f.s1, sizeof(A.s1));
    A.kll = f.kll;
    A.kd = f.kd;
    A.khh = f.khh;
    A.nbx = (Wq + IVX - 1) / IVX;
    const int nby = (Hq + IVY - 1) / IVY;
    if ((long long)A.nbx * nby >= (1LL << 31) || count > 65535) return fail(DWT2_EINVAL);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(A.nbx * nby, count);
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = f.radius == 2 ? cudaLaunchKernelEx(&cfg, dwt_small_inv_kernel<2>, A)
                                        : cudaLaunchKernelEx(&cfg, dwt_small_inv_kernel<4>, A);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

// Measured (scripts/r2/inv_small_probe.py, graph of 20 inverses; thresholds
// 0 / 2^16 / 2^18 / 2^20 quads): CDF 9/7 config 4 226.9 / 205.3 / 206.5 / 233.8 us;
// CDF 5/3 config 4 165.6 / 166.3 / 170.0 / 193.8 us (its ring kernel is fast on
// 16-byte-aligned levels), config 4b (odd widths: the plain-load kernel)
// 245.3 / 236.9 / 234.4 / 233.2 us; a cold single 1024^2 level is slower on the
// small kernel (5/3 7.2 -> 10.7 us).
bool small_inverse_level(const dwt2_plan *p, int k, int count)
{
    static const long long q53 = tuning_int("DWT2_INV_SMALL_QUADS", 1 << 16, 0, 1 << 30);
    static const long long q53_odd = tuning_int("DWT2_INV_SMALL_QUADS_ODD", 1 << 20, 0, 1 << 30);
    static const long long qk2 = tuning_int("DWT2_K2INV_SMALL_QUADS", 1 << 16, 0, 1 << 30);
    const long long quads = (long long)p->geom[k].Wq * p->geom[k].Hq * count;
    if (count > 65535) return false;                         // images go to gridDim.y
    if (p->wavelet != DWT2_WAVELET_CDF53) return quads <= qk2;
    return quads <= ((p->W % 4) != 0 ? q53_odd : q53);      // the Mallat pitch W: ring kernel iff 16-byte rows
}

int tail_start_levels(const dwt2_plan *p, int count, int first, int last, long long max_quads)
{
    int k = last + 1;
    while (k - 1 >= first && last - (k - 1) < MAX_TAIL &&
           (long long)p->geom[k - 1].Wq * p->geom[k - 1].Hq * count <= max_quads)
        --k;
    return k;
}

int32_t launch_tail_levels(const dwt2_plan *p, const TailLevelIO *lv, int n, int count, const TailFilter &f,
                           cudaStream_t stream)
{
    if (n < 1 || n > MAX_TAIL || (f.radius != 2 && f.radius != 4)) return fail(DWT2_EINVAL);
    TailArgs ta;
    memset(&ta, 0, sizeof(ta));
    ta.nlev = n;
    ta.count = count;
    long long most = 0;
    for (int k = 0; k < n; ++k) {
        ta.lv[k] = lv[k];
        most = std::max<long long>(most, (long long)((lv[k].W + 1) / 2) * ((lv[k].H + 1) / 2) * count);
    }
    memcpy(ta.h, f.h, sizeof(ta.h));
    memcpy(ta.g, f.g, sizeof(ta.g));
    ta.sll = f.sll;
    ta.sd = f.sd;
    ta.shh = f.shh;
    ta.bar = p->counters + 2 * QUEUE_TAIL;
    // every CTA must be resident at once (grid barrier): at most the occupancy
    const int resident = f.radius == 2 ? tail_resident<2>() : tail_resident<4>();
    static const int per_sm_knob = tuning_int("DWT2_TAIL_CTAS", 2, 1, 8);
    const int per_sm = std::min(resident, per_sm_knob);
    const long long want = (most + TAIL_THREADS - 1) / TAIL_THREADS;
    const int grid = int(std::max<long long>(1, std::min<long long>((long long)p->sms * per_sm, want)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(TAIL_THREADS);
    cfg.stream = stream;
    // cooperative: the grid barrier needs every CTA resident at once, which a
    // cooperative launch guarantees (or refuses) even next to other streams' work
    static const int coop = tuning_int("DWT2_TAIL_COOP", 1, 0, 1);
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop ? 2 : 1;
    const cudaError_t e = f.radius == 2 ? cudaLaunchKernelEx(&cfg, dwt_tail_kernel<2>, ta)
                                        : cudaLaunchKernelEx(&cfg, dwt_tail_kernel<4>, ta);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

}  // namespace dwt2_detail
