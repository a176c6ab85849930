// schemes.cu -- the paper's comparison schemes on B200, one kernel per step
// (section 4, Fig. 6).
//
// The paper's claim is about synchronisation: a scheme with fewer barrier-
// separated steps (`|`) is faster.  On a GPU the honest
// counterpart of a barrier between two steps that exchange data across the
// whole image is a kernel boundary, i.e. one more HBM round trip of the
// intermediate.  Each scheme below therefore runs each of its steps as its
// own kernel over the whole level:
//
//   SEP_LIFTING     Eq. (3): horizontal predict | vertical predict |
//                   horizontal update | vertical update           (4 steps)
//   SEP_CONV        Eq. (4): horizontal filter bank N^H | vertical
//                   filter bank N^V (5/3 taps, 1-D convolutions)   (2 steps)
//   NONSEP_LIFTING  Eq. (5): spatial predict | spatial update,
//                   literal 4x4 operators with PP* and UU*         (2 steps)
//   NONSEP_ADAPTED  Fig. 3: Eq. (5) with P = P0 + P1, U = U0 + U1;
//                   the constants P0 = -1/2, U0 = 1/4 applied separably and
//                   quad-locally, only P1 = -1/2 z, U1 = 1/4 z^-1 non-
//                   separably (18 instead of 24 MACs per quad)   (2 steps)
//   NONSEP_NAIVE    Eq. (5) fused into ONE kernel in the plain style of the
//                   others: one thread per quad, the predicted neighbours
//                   recomputed from the input   (1 step)
//
// and DWT2_SCHEME_FUSED is the product kernel of dwt2.cu (1 step, TMA ring,
// register carries, warp shuffles).  All kernels share one plain style
// (one thread per quad, fp64 in registers, fp32 between steps, every
// neighbour fetched through L1/L2) so that a comparison between them
// measures steps, not kernel engineering.
//
// Boundaries: whole-sample symmetric extension, applied in the PIXEL domain:
// a coefficient of parity p (0 = low, 1 = high) at quad index q sits at pixel
// 2q + p; an out-of-range neighbour is fetched at the mirrored pixel, which
// has the same parity.  Because the extended signal is symmetric, this gives
// exactly the quad-domain rules of the fused kernel (H[-1] := H[0],
// H[M] := H[M-1] for odd sizes, L[M] := L[M-1] for even sizes).
//
// Layouts: step 1 reads the interleaved level input; every intermediate is a
// Mallat buffer of the level (LL plane + HL / LH / HH at their offsets), so
// in-place steps (SEP_LIFTING steps 2-4, which read only the planes they do
// not write) work directly on the output, and out-of-place steps (the
// others, whose neighbour reads would race with their writes) go through the
// plan's work buffer.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "dwt2_internal.h"

using namespace dwt2_detail;

namespace {

// Whole-sample symmetric reflection of a pixel index (offsets are at most 2,
// and every level is at least 2 wide, so one reflection suffices).
__device__ __forceinline__ int wss(int k, int n)
{
    if (k < 0) k = -k;
    if (k > n - 1) k = 2 * (n - 1) - k;
    return k;
}

// Quad index of the coefficient of parity `par` at quad q, mirrored.
__device__ __forceinline__ int mq(int q, int par, int n) { return (wss(2 * q + par, n) - par) >> 1; }

struct Planes {                // one level's subbands: LL plane + Mallat detail buffer
    float *ll;
    long long ll_pitch, ll_img;
    float *d;                  // Mallat base: HL at (0, Wq), LH at (Hq, 0), HH at (Hq, Wq)
    long long d_pitch, d_img;
};

struct SArgs {
    const float *in;           // interleaved level input (step 1)
    long long in_pitch, in_img;
    Planes src, dst;
    int W, H;
};

// band 0 LL, 1 HL, 2 LH, 3 HH; (m, n) mirrored into the band's valid range
__device__ __forceinline__ long long band_off(const Planes &p, int W, int H, int band, int img, int m, int n)
{
    const int px = band & 1, py = band >> 1;
    const int Wq = (W + 1) >> 1, Hq = (H + 1) >> 1;
    const int mm = mq(m, px, W), nn = mq(n, py, H);
    if (band == 0) return (long long)img * p.ll_img + (long long)nn * p.ll_pitch + mm;
    return (long long)img * p.d_img + (long long)(nn + (py ? Hq : 0)) * p.d_pitch + mm + (px ? Wq : 0);
}

__device__ __forceinline__ double ldb(const Planes &p, int W, int H, int band, int img, int m, int n)
{
    const float *base = (band == 0) ? p.ll : p.d;
    return (double)__ldg(base + band_off(p, W, H, band, img, m, n));
}

__device__ __forceinline__ void stb(const Planes &p, int W, int H, int band, int img, int m, int n, double v)
{
    // only coefficients that exist: HL / HH need column 2m+1 < W, LH / HH row 2n+1 < H
    if ((band & 1) && 2 * m + 1 >= W) return;
    if ((band >> 1) && 2 * n + 1 >= H) return;
    float *base = (band == 0) ? p.ll : p.d;
    base[band_off(p, W, H, band, img, m, n)] = (float)v;
}

__device__ __forceinline__ double px(const SArgs &a, int img, int r, int c)
{
    return (double)__ldg(a.in + (long long)img * a.in_img + (long long)wss(r, a.H) * a.in_pitch + wss(c, a.W));
}

#define QUAD_PROLOGUE                                                          \
    const int m = blockIdx.x * blockDim.x + threadIdx.x;                       \
    const int n = blockIdx.y * blockDim.y + threadIdx.y;                       \
    const int img = blockIdx.z;                                                \
    if (m >= ((a.W + 1) >> 1) || n >= ((a.H + 1) >> 1)) return;

// ---- predicted values of quad (m, n) from the input (Eq. (5) right factor,
//      literal: HH' = d + P c + P* b + PP* a)
struct Pred { double a, hl, lh, hh; };

__device__ __forceinline__ Pred predict_literal(const SArgs &a, int img, int m, int n)
{
    const int x = 2 * m, y = 2 * n;
    const double A = px(a, img, y, x), B = px(a, img, y, x + 1), C = px(a, img, y + 1, x), D = px(a, img, y + 1, x + 1);
    const double Ar = px(a, img, y, x + 2), Ad = px(a, img, y + 2, x), Ard = px(a, img, y + 2, x + 2);
    const double Cr = px(a, img, y + 1, x + 2), Bd = px(a, img, y + 2, x + 1);
    Pred p;
    p.a = A;
    p.hl = B - 0.5 * (A + Ar);                                   // P
    p.lh = C - 0.5 * (A + Ad);                                   // P*
    p.hh = D - 0.5 * (C + Cr) - 0.5 * (B + Bd) + 0.25 * (A + Ar + Ad + Ard);   // P, P*, PP*
    return p;
}

// ---------------------------------------------------------------------------
// NONSEP_NAIVE: Eq. (5) in one kernel; the update's m-1 / n-1 neighbours are
// re-predicted from the input (quad indices mirrored through pixel parity:
// predicting quad -1 reads the mirrored pixels and yields H[-1] = H[0]).
// ---------------------------------------------------------------------------
__global__ void k_nonsep_naive(const SArgs a)
{
    QUAD_PROLOGUE
    const Pred c = predict_literal(a, img, m, n);
    const Pred l = predict_literal(a, img, m - 1, n);
    const Pred u = predict_literal(a, img, m, n - 1);
    const Pred ul = predict_literal(a, img, m - 1, n - 1);
    // the extended image is symmetric, so predicting a mirrored quad (m-1 = -1,
    // or the missing H column / row of an odd size) yields the mirrored values
    const double hl = c.hl, lh = c.lh, hh = c.hh, hh_l = l.hh, hh_u = u.hh;
    const double LL = c.a + 0.25 * (hl + l.hl) + 0.25 * (lh + u.lh) + 0.0625 * (hh + hh_l + hh_u + ul.hh);
    stb(a.dst, a.W, a.H, 0, img, m, n, LL);
    stb(a.dst, a.W, a.H, 1, img, m, n, hl + 0.25 * (hh + hh_u));
    stb(a.dst, a.W, a.H, 2, img, m, n, lh + 0.25 * (hh + hh_l));
    stb(a.dst, a.W, a.H, 3, img, m, n, hh);
}

// ---------------------------------------------------------------------------
// NONSEP_LIFTING: step 1 spatial predict -> work; step 2 spatial update
// ---------------------------------------------------------------------------
__global__ void k_nonsep_predict(const SArgs a)
{
    QUAD_PROLOGUE
    const Pred p = predict_literal(a, img, m, n);
    stb(a.dst, a.W, a.H, 0, img, m, n, p.a);
    stb(a.dst, a.W, a.H, 1, img, m, n, p.hl);
    stb(a.dst, a.W, a.H, 2, img, m, n, p.lh);
    stb(a.dst, a.W, a.H, 3, img, m, n, p.hh);
}

// Eq. (5) left factor, literal: LL = a + U HL' + U* LH' + UU* HH', HL = HL' +
// U* HH', LH = LH' + U HH'.  Reads are mirrored, so missing odd-size H values
// come out as their mirrors.
__global__ void k_nonsep_update(const SArgs a)
{
    QUAD_PROLOGUE
    const Planes &s = a.src;
    const double A = ldb(s, a.W, a.H, 0, img, m, n);
    const double hl = ldb(s, a.W, a.H, 1, img, m, n), hl_l = ldb(s, a.W, a.H, 1, img, m - 1, n);
    const double lh = ldb(s, a.W, a.H, 2, img, m, n), lh_u = ldb(s, a.W, a.H, 2, img, m, n - 1);
    const double hh = ldb(s, a.W, a.H, 3, img, m, n), hh_l = ldb(s, a.W, a.H, 3, img, m - 1, n);
    const double hh_u = ldb(s, a.W, a.H, 3, img, m, n - 1), hh_ul = ldb(s, a.W, a.H, 3, img, m - 1, n - 1);
    stb(a.dst, a.W, a.H, 0, img, m, n, A + 0.25 * (hl + hl_l) + 0.25 * (lh + lh_u) + 0.0625 * (hh + hh_l + hh_u + hh_ul));
    stb(a.dst, a.W, a.H, 1, img, m, n, hl + 0.25 * (hh + hh_u));
    stb(a.dst, a.W, a.H, 2, img, m, n, lh + 0.25 * (hh + hh_l));
    stb(a.dst, a.W, a.H, 3, img, m, n, hh);
}

// ---------------------------------------------------------------------------
// NONSEP_ADAPTED (Fig. 3): predict = C_V(P0*) C_H(P0) N(P1), update =
// C_V(U0*) C_H(U0) N(U1); N(.) is the non-separable part (neighbour reads),
// C_H / C_V the quad-local constant parts, applied after it within the step.
// ---------------------------------------------------------------------------
__global__ void k_adapted_predict(const SArgs a)
{
    QUAD_PROLOGUE
    const int x = 2 * m, y = 2 * n;
    const double A = px(a, img, y, x), B = px(a, img, y, x + 1), C = px(a, img, y + 1, x), D = px(a, img, y + 1, x + 1);
    const double Ar = px(a, img, y, x + 2), Ad = px(a, img, y + 2, x), Ard = px(a, img, y + 2, x + 2);
    const double Cr = px(a, img, y + 1, x + 2), Bd = px(a, img, y + 2, x + 1);
    // N(P1), P1 = -1/2 z_m: HL += P1 LL, LH += P1* LL, HH += P1 LH + P1* HL + P1 P1* LL
    double b = B - 0.5 * Ar;
    double c = C - 0.5 * Ad;
    double d = D - 0.5 * Cr - 0.5 * Bd + 0.25 * Ard;
    // C_H(P0), P0 = -1/2: HL += P0 LL, HH += P0 LH (quad-local)
    b = b - 0.5 * A;
    d = d - 0.5 * c;
    // C_V(P0*): LH += P0* LL, HH += P0* HL
    c = c - 0.5 * A;
    d = d - 0.5 * b;
    stb(a.dst, a.W, a.H, 0, img, m, n, A);
    stb(a.dst, a.W, a.H, 1, img, m, n, b);
    stb(a.dst, a.W, a.H, 2, img, m, n, c);
    stb(a.dst, a.W, a.H, 3, img, m, n, d);
}

__global__ void k_adapted_update(const SArgs a)
{
    QUAD_PROLOGUE
    const Planes &s = a.src;
    const double A = ldb(s, a.W, a.H, 0, img, m, n);
    const double hl = ldb(s, a.W, a.H, 1, img, m, n), hl_l = ldb(s, a.W, a.H, 1, img, m - 1, n);
    const double lh = ldb(s, a.W, a.H, 2, img, m, n), lh_u = ldb(s, a.W, a.H, 2, img, m, n - 1);
    const double hh = ldb(s, a.W, a.H, 3, img, m, n), hh_l = ldb(s, a.W, a.H, 3, img, m - 1, n);
    const double hh_u = ldb(s, a.W, a.H, 3, img, m, n - 1), hh_ul = ldb(s, a.W, a.H, 3, img, m - 1, n - 1);
    // N(U1), U1 = 1/4 z_m^-1: LL += U1 HL + U1* LH + U1 U1* HH, HL += U1* HH, LH += U1 HH
    double LL = A + 0.25 * hl_l + 0.25 * lh_u + 0.0625 * hh_ul;
    double HL = hl + 0.25 * hh_u;
    double LH = lh + 0.25 * hh_l;
    // C_H(U0), U0 = 1/4: LL += U0 HL, LH += U0 HH
    LL = LL + 0.25 * HL;
    LH = LH + 0.25 * hh;
    // C_V(U0*): LL += U0* LH, HL += U0* HH
    LL = LL + 0.25 * LH;
    HL = HL + 0.25 * hh;
    stb(a.dst, a.W, a.H, 0, img, m, n, LL);
    stb(a.dst, a.W, a.H, 1, img, m, n, HL);
    stb(a.dst, a.W, a.H, 2, img, m, n, LH);
    stb(a.dst, a.W, a.H, 3, img, m, n, hh);
}

// ---------------------------------------------------------------------------
// SEP_LIFTING (Eq. (3)): four 1-D lifting steps, each its own kernel
// ---------------------------------------------------------------------------
// step 1, horizontal predict (reads the input): HL = b + P a, HH = d + P c
__global__ void k_sep_hpredict(const SArgs a)
{
    QUAD_PROLOGUE
    const int x = 2 * m, y = 2 * n;
    const double A = px(a, img, y, x), B = px(a, img, y, x + 1), C = px(a, img, y + 1, x), D = px(a, img, y + 1, x + 1);
    const double Ar = px(a, img, y, x + 2), Cr = px(a, img, y + 1, x + 2);
    stb(a.dst, a.W, a.H, 0, img, m, n, A);
    stb(a.dst, a.W, a.H, 1, img, m, n, B - 0.5 * (A + Ar));
    stb(a.dst, a.W, a.H, 2, img, m, n, C);
    stb(a.dst, a.W, a.H, 3, img, m, n, D - 0.5 * (C + Cr));
}

// step 2, vertical predict (in place): LH += P* LL, HH += P* HL
__global__ void k_sep_vpredict(const SArgs a)
{
    QUAD_PROLOGUE
    if (2 * n + 1 >= a.H) return;                    // odd H: no LH / HH in the last quad row
    const Planes &s = a.dst;
    const double ll = ldb(s, a.W, a.H, 0, img, m, n), ll_d = ldb(s, a.W, a.H, 0, img, m, n + 1);
    stb(s, a.W, a.H, 2, img, m, n, ldb(s, a.W, a.H, 2, img, m, n) - 0.5 * (ll + ll_d));
    if (2 * m + 1 < a.W) {
        const double hl = ldb(s, a.W, a.H, 1, img, m, n), hl_d = ldb(s, a.W, a.H, 1, img, m, n + 1);
        stb(s, a.W, a.H, 3, img, m, n, ldb(s, a.W, a.H, 3, img, m, n) - 0.5 * (hl + hl_d));
    }
}

// step 3, horizontal update (in place): LL += U HL, LH += U HH
__global__ void k_sep_hupdate(const SArgs a)
{
    QUAD_PROLOGUE
    const Planes &s = a.dst;
    const double hl = ldb(s, a.W, a.H, 1, img, m, n), hl_l = ldb(s, a.W, a.H, 1, img, m - 1, n);
    stb(s, a.W, a.H, 0, img, m, n, ldb(s, a.W, a.H, 0, img, m, n) + 0.25 * (hl + hl_l));
    if (2 * n + 1 < a.H) {
        const double hh = ldb(s, a.W, a.H, 3, img, m, n), hh_l = ldb(s, a.W, a.H, 3, img, m - 1, n);
        stb(s, a.W, a.H, 2, img, m, n, ldb(s, a.W, a.H, 2, img, m, n) + 0.25 * (hh + hh_l));
    }
}

// step 4, vertical update (in place): LL += U* LH, HL += U* HH
__global__ void k_sep_vupdate(const SArgs a)
{
    QUAD_PROLOGUE
    const Planes &s = a.dst;
    const double lh = ldb(s, a.W, a.H, 2, img, m, n), lh_u = ldb(s, a.W, a.H, 2, img, m, n - 1);
    stb(s, a.W, a.H, 0, img, m, n, ldb(s, a.W, a.H, 0, img, m, n) + 0.25 * (lh + lh_u));
    if (2 * m + 1 < a.W) {
        const double hh = ldb(s, a.W, a.H, 3, img, m, n), hh_u = ldb(s, a.W, a.H, 3, img, m, n - 1);
        stb(s, a.W, a.H, 1, img, m, n, ldb(s, a.W, a.H, 1, img, m, n) + 0.25 * (hh + hh_u));
    }
}

// ---------------------------------------------------------------------------
// SEP_CONV (Eq. (4)): the whole 1-D transform of one axis as one
// convolution step.  Analysis taps of the 5/3 pair (Eq. (1) form of Eq. (2)):
// low h0 = (-1/8, 1/4, 3/4, 1/4, -1/8) around even samples, high
// g1 = (-1/2, 1, -1/2) around odd samples.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double h0(int k) { return k == 0 ? 0.75 : (k == 1 || k == -1) ? 0.25 : -0.125; }
__device__ __forceinline__ double g1(int k) { return k == 0 ? 1.0 : -0.5; }

// step 1, N^H (reads the input): rows 2n, 2n+1 filtered horizontally -> work
__global__ void k_conv_h(const SArgs a)
{
    QUAD_PROLOGUE
    const int x = 2 * m;
#pragma unroll
    for (int ry = 0; ry < 2; ++ry) {
        const int y = 2 * n + ry;
        if (y >= a.H) break;
        double lo = 0.0, hi = 0.0;
#pragma unroll
        for (int k = -2; k <= 2; ++k) lo += h0(k) * px(a, img, y, x + k);
#pragma unroll
        for (int k = -1; k <= 1; ++k) hi += g1(k) * px(a, img, y, x + 1 + k);
        stb(a.dst, a.W, a.H, 2 * ry, img, m, n, lo);
        stb(a.dst, a.W, a.H, 2 * ry + 1, img, m, n, hi);
    }
}

// row r of the horizontally filtered image, low (hpar 0) or high (hpar 1)
// half, at quad column m: even rows live in LL / HL, odd rows in LH / HH
__device__ __forceinline__ double hrow(const SArgs &a, int img, int r, int hpar, int m)
{
    const int rr = wss(r, a.H);
    return ldb(a.src, a.W, a.H, hpar + 2 * (rr & 1), img, m, rr >> 1);
}

// step 2, N^V (work -> output)
__global__ void k_conv_v(const SArgs a)
{
    QUAD_PROLOGUE
    const int y = 2 * n;
#pragma unroll
    for (int hpar = 0; hpar < 2; ++hpar) {
        if (hpar && 2 * m + 1 >= a.W) break;
        double lo = 0.0, hi = 0.0;
#pragma unroll
        for (int k = -2; k <= 2; ++k) lo += h0(k) * hrow(a, img, y + k, hpar, m);
#pragma unroll
        for (int k = -1; k <= 1; ++k) hi += g1(k) * hrow(a, img, y + 1 + k, hpar, m);
        stb(a.dst, a.W, a.H, hpar, img, m, n, lo);
        stb(a.dst, a.W, a.H, 2 + hpar, img, m, n, hi);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef void (*StepFn)(SArgs);

int32_t launch_step(StepFn fn, const SArgs &a, int count, cudaStream_t s)
{
    const int Wq = (a.W + 1) / 2, Hq = (a.H + 1) / 2;
    dim3 block(32, 8);
    dim3 grid((Wq + 31) / 32, (Hq + 7) / 8, count);
    fn<<<grid, block, 0, s>>>(a);
    if (cudaGetLastError() != cudaSuccess) return fail(DWT2_ECUDA);
    return DWT2_OK;
}

int32_t ensure_work(const dwt2_plan *p, size_t bytes)
{
    if (p->work && p->work_bytes >= bytes) return DWT2_OK;
    if (p->work) cudaFree(p->work);
    p->work = nullptr;
    p->work_bytes = 0;
    if (cudaMalloc(&p->work, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ENOMEM);
    }
    p->work_bytes = bytes;
    return DWT2_OK;
}

}  // namespace

extern "C" {

int32_t dwt2_forward_batched(const dwt2_plan *p, const float *in, float *out, int32_t count, int64_t in_stride,
                             int64_t out_stride, dwt2_stream_t stream);

int32_t dwt2_scheme_steps(int32_t scheme)
{
    switch (scheme) {
    case DWT2_SCHEME_FUSED: return 1;
    case DWT2_SCHEME_NONSEP_NAIVE: return 1;
    case DWT2_SCHEME_NONSEP_LIFTING: return 2;
    case DWT2_SCHEME_NONSEP_ADAPTED: return 2;
    case DWT2_SCHEME_SEP_CONV: return 2;
    case DWT2_SCHEME_SEP_LIFTING: return 4;
    case DWT2_SCHEME_FUSED_LITERAL: return 1;
    case DWT2_SCHEME_FUSED_ADAPTED: return 1;
    default: return fail(DWT2_EINVAL);
    }
}

int32_t dwt2_forward_scheme(const dwt2_plan *p, int32_t scheme, const float *in, float *out, int32_t count,
                            int64_t in_stride, int64_t out_stride, dwt2_stream_t stream)
{
    if (p && p->wavelet != DWT2_WAVELET_CDF53) return fail(DWT2_EUNSUPPORTED);
    if (scheme == DWT2_SCHEME_FUSED) return dwt2_forward_batched(p, in, out, count, in_stride, out_stride, stream);
    const long long img = (long long)(p ? p->W : 0) * (p ? p->H : 0);
    if (!p || !in || !out || p->strip || count < 1 || count > p->max_count || in_stride < img ||
        out_stride < img || !aligned(in, 4) || !aligned(out, 4) || dwt2_scheme_steps(scheme) < 0)
        return fail(DWT2_EINVAL);
    const size_t in_bytes = size_t((count - 1) * in_stride + img) * sizeof(float);
    const size_t out_bytes = size_t((count - 1) * out_stride + img) * sizeof(float);
    if (overlap(in, in_bytes, out, out_bytes) || !on_plan_device(p, in) || !on_plan_device(p, out))
        return fail(DWT2_EINVAL);
    if (scheme == DWT2_SCHEME_FUSED_LITERAL || scheme == DWT2_SCHEME_FUSED_ADAPTED) {
        int32_t r = forward_fused_variant(p, in, out, count, in_stride, out_stride,
                                          scheme == DWT2_SCHEME_FUSED_LITERAL ? 1 : 2,
                                          reinterpret_cast<cudaStream_t>(stream));
        if (r == DWT2_OK) g_last_error = DWT2_OK;
        return r;
    }
    const bool two_buffers = scheme != DWT2_SCHEME_SEP_LIFTING && scheme != DWT2_SCHEME_NONSEP_NAIVE;
    if (two_buffers) {
        int32_t r = ensure_work(p, size_t(count) * size_t(img) * sizeof(float));
        if (r != DWT2_OK) return r;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    for (int k = 0; k < p->levels; ++k) {
        const LevelGeom &g = p->geom[k];
        SArgs a;
        memset(&a, 0, sizeof(a));
        a.W = g.W;
        a.H = g.H;
        if (k == 0) {
            a.in = in;
            a.in_pitch = p->W;
            a.in_img = in_stride;
        } else {
            const int sidx = (k - 1) % 2;
            a.in = p->scratch[sidx];
            a.in_pitch = p->sc_pitch[sidx];
            a.in_img = p->sc_img_stride[sidx];
        }
        Planes fin;                               // the level's final subbands
        fin.d = out;
        fin.d_pitch = p->W;
        fin.d_img = out_stride;
        if (k == p->levels - 1) {
            fin.ll = out;
            fin.ll_pitch = p->W;
            fin.ll_img = out_stride;
        } else {
            const int sidx = k % 2;
            fin.ll = p->scratch[sidx];
            fin.ll_pitch = p->sc_pitch[sidx];
            fin.ll_img = p->sc_img_stride[sidx];
        }
        Planes wk;                                // intermediate (work buffer, Mallat of the level)
        wk.ll = wk.d = p->work;
        wk.ll_pitch = wk.d_pitch = g.W;
        wk.ll_img = wk.d_img = img;
        int32_t r = DWT2_OK;
        switch (scheme) {
        case DWT2_SCHEME_NONSEP_NAIVE:
            a.dst = fin;
            r = launch_step(k_nonsep_naive, a, count, s);
            break;
        case DWT2_SCHEME_NONSEP_LIFTING:
        case DWT2_SCHEME_NONSEP_ADAPTED: {
            const bool ad = scheme == DWT2_SCHEME_NONSEP_ADAPTED;
            a.dst = wk;
            r = launch_step(ad ? k_adapted_predict : k_nonsep_predict, a, count, s);
            if (r != DWT2_OK) break;
            a.src = wk;
            a.dst = fin;
            r = launch_step(ad ? k_adapted_update : k_nonsep_update, a, count, s);
            break;
        }
        case DWT2_SCHEME_SEP_CONV:
            a.dst = wk;
            r = launch_step(k_conv_h, a, count, s);
            if (r != DWT2_OK) break;
            a.src = wk;
            a.dst = fin;
            r = launch_step(k_conv_v, a, count, s);
            break;
        case DWT2_SCHEME_SEP_LIFTING:
            a.dst = fin;
            r = launch_step(k_sep_hpredict, a, count, s);
            if (r == DWT2_OK) r = launch_step(k_sep_vpredict, a, count, s);
            if (r == DWT2_OK) r = launch_step(k_sep_hupdate, a, count, s);
            if (r == DWT2_OK) r = launch_step(k_sep_vupdate, a, count, s);
            break;
        }
        if (r != DWT2_OK) return r;
    }
    g_last_error = DWT2_OK;
    return DWT2_OK;
}

}  // extern "C"
