// dwt97.cu -- B200 (sm_100a) forward 2-D CDF 9/7 DWT with the non-separable
// lifting scheme of arXiv:1708.07853 generalised to K = 2 lifting pairs
// ("the presented
// schemes are general and they are not limited to any particular wavelet").
//
// Eq. (5) with the pair (P_k, U_k) = (c_{2k} (1 + z),
// c_{2k+1} (1 + z^-1)) is applied for k = 1, 2 -- four spatial steps
// (predict 1 | update 1 | predict 2 | update 2) instead of the eight of the
// separable lifting scheme -- followed by the 2-D scaling of the subbands
// (LL / K^2, HL and LH * 1, HH * K^2).  CDF 9/7: (c0, c1, c2, c3) = (alpha,
// beta, gamma, delta) of Daubechies & Sweldens with JPEG 2000 normalisation
// (readings C-B1..C-B3).  The same kernel runs the CDF 5/3 pair as
// (-1/2, 1/4, 0, 0), K = 1 (a cross-check against the 5/3 path).
//
// One fused kernel per level, no intermediate ever leaves the registers:
// a warp owns a slab of 64 quad columns of which the middle 60 are output
// (lanes 1..30; lanes 0 and 31 carry the 2-quad halo each side that the four
// steps need) and walks DOWN it one quad row at a time.  Each spatial step
// reads its vertical neighbours from rows carried in registers (the predicts
// look one row ahead, the updates one row back, so the output lags the input
// by two quad rows) and its horizontal neighbours from the adjacent lane by
// shuffle.  The paper's synchronisation points `|` are
// warp shuffles.
//
// Boundaries: whole-sample symmetric extension applied to the PIXELS as they
// are loaded (every index mirrored), so every tile transforms the extended
// image and no quad-domain boundary rule is needed -- the same definition
// the oracle computes (oracle/dwt97_oracle.c, "transform of the symmetric
// extension").  fp32 in HBM, fp64 in registers.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "dwt2_internal.h"
#include "queue.cuh"

using namespace dwt2_detail;

namespace {

#ifndef DWT2_K2_QK
#define DWT2_K2_QK 2                       // measured: 4 quads per lane is not faster (fewer warps fit)
#endif
#ifndef DWT2_K2_MINB
#define DWT2_K2_MINB (DWT2_K2_QK == 4 ? 2 : 4)   // CTAs per SM the register budget is sized for
#endif
constexpr int KW = 4;                      // warps per CTA
constexpr int KT = KW * 32;
constexpr int QK = DWT2_K2_QK;             // quads per lane (2 or 4)
constexpr int SLABQ = 32 * QK;             // quad columns per warp
constexpr int OUTQ = 30 * QK;              // output quad columns per warp (lanes 1..30; lanes 0, 31: halo)
constexpr int RW = 2 * SLABQ;              // floats per staged pixel row (= 64 QK)
#ifndef DWT2_K2_DS
#define DWT2_K2_DS 5                      // measured: 5 > 4 > 6 > 8 > 2 (the row loop is unrolled DS times: i-cache)
#endif
constexpr int DS = DWT2_K2_DS;             // raw quad rows in flight per warp (shared-memory ring, cp.async)
#ifndef DWT2_K2_PEEL_ALL
#define DWT2_K2_PEEL_ALL 0                 // measurement builds: peel the warm-up rows on the ring path too
#endif
#ifndef DWT2_K2_DR
#define DWT2_K2_DR 1
#endif
constexpr int DR = DWT2_K2_DR;             // raw quad rows in flight per warp on the register path (edge slabs)
#ifndef DWT2_K2INV_DR
#define DWT2_K2INV_DR 2                    // the inverse's register path: 2 rows (measured: config 3 682 -> 697 Gpix/s)
#endif
constexpr int IDR = DWT2_K2INV_DR;
constexpr size_t K2_SMEM = size_t(KW) * DS * 2 * RW * sizeof(float);
static_assert(QK == 2 || QK == 4, "2 or 4 quads per lane");

__device__ __forceinline__ void cp_async16(float *dst, const float *src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct K2Args {
    const float *in;
    long long in_pitch, in_img;
    float *ll;                             // LL destination (scratch or out)
    long long ll_pitch, ll_img;
    float *hl, *lh, *hh;                   // detail subbands (Mallat positions in out)
    long long out_pitch, out_img;
    int W, H;
    int nslabs, tb, nblk, count;
    long long ntiles;
    FastDiv fd_img, fd_slabs;              // division by nblk * nslabs and by nslabs (ntiles < 2^31)
    double c0, c1, c2, c3;                 // lifting coefficients (predict, update, predict, update)
    double sll, sd, shh;                   // output scaling: LL, HL / LH (always 1, not applied), HH
    unsigned int *counter;                 // tile queue (queue.cuh)
    int nwarps;
    int slab_r, nedge;                     // edge-first order: edge slabs {0} u [slab_r, nslabs), nedge of them
                                           // per row (0: plain row-block-major order)
};

__device__ __forceinline__ int wssi(int k, int n);

// Queue index -> (image, row block, slab).  Edge-first order (nedge > 0): the
// tiles of the edge slabs of every row block come first -- they read through
// registers with mirrored indices and take longer, so they must not be the
// tail of the level -- then the interior tiles, row-block-major.
template <class Args>
__device__ __forceinline__ void k2_decode(const Args &a, int t, int &img, int &blk, int &slab)
{
    if (a.nedge > 0) {
        const int ne = a.nedge, ni = a.nslabs - a.nedge;
        const int edge_tiles = a.count * a.nblk * ne;
        if (t < edge_tiles) {
            img = t / (a.nblk * ne);
            const int r = t - img * a.nblk * ne;
            blk = r / ne;
            const int e = r - blk * ne;
            slab = e == 0 ? 0 : a.slab_r + e - 1;
        } else {
            const int u = t - edge_tiles;
            img = u / (a.nblk * ni);
            const int r = u - img * a.nblk * ni;
            blk = r / ni;
            slab = 1 + (r - blk * ni);
        }
        return;
    }
    img = fdiv(t, a.fd_img);
    const int rr = t - img * a.nblk * a.nslabs;
    blk = fdiv(rr, a.fd_slabs);
    slab = rr - blk * a.nslabs;
}

// The same reflection without the integer division when one mirror suffices
// (|overhang| < n - 1: every index of a slab or window of a level that is
// not tiny); the edge slabs of the K = 2 kernels call it once per pixel.
__device__ __forceinline__ int wssi_fast(int k, int n)
{
    const int r = k < 0 ? -k : (k >= n ? 2 * (n - 1) - k : k);
    return (r >= 0 && r < n) ? r : wssi(k, n);
}

__device__ __forceinline__ int wssi(int k, int n)
{
    // whole-sample symmetric reflection, any k (period 2 (n - 1))
    if (n == 1) return 0;
    const int p = 2 * (n - 1);
    k %= p;
    if (k < 0) k += p;
    return k >= n ? p - k : k;
}

// Raw quad row r (pixel rows 2r, 2r+1, mirrored) of the lane's QK quads:
// pixels x = xb .. xb + 2 QK - 1 with xb = 2 (m0 - QK) + 2 QK lane.
struct RawRow {
    float e[2 * QK], o[2 * QK];             // even row: a0 b0 a1 b1 ..; odd row: c0 d0 c1 d1 ..
};

template <bool VEC, bool EDGE>
__device__ __forceinline__ RawRow load_raw_row(const K2Args &a, const float *img, int r, int xb)
{
    int y0 = 2 * r, y1 = 2 * r + 1;
    if (y0 < 0 || y1 >= a.H) {                        // top / bottom rows: mirror
        y0 = wssi(y0, a.H);
        y1 = wssi(y1, a.H);
    }
    const float *p0 = img + (long long)y0 * a.in_pitch;
    const float *p1 = img + (long long)y1 * a.in_pitch;
    RawRow R;
    if (VEC && !EDGE) {
#pragma unroll
        for (int q = 0; q < QK / 2; ++q) {
            const float4 u = __ldg(reinterpret_cast<const float4 *>(p0 + xb) + q);
            const float4 v = __ldg(reinterpret_cast<const float4 *>(p1 + xb) + q);
            R.e[4 * q] = u.x; R.e[4 * q + 1] = u.y; R.e[4 * q + 2] = u.z; R.e[4 * q + 3] = u.w;
            R.o[4 * q] = v.x; R.o[4 * q + 1] = v.y; R.o[4 * q + 2] = v.z; R.o[4 * q + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 2 * QK; ++j) {
            const int x = EDGE ? wssi_fast(xb + j, a.W) : xb + j;
            R.e[j] = __ldg(p0 + x);
            R.o[j] = __ldg(p1 + x);
        }
    }
    return R;
}

// Register arithmetic type: fp64 (the product); -DDWT2_K2_F32 builds an fp32
// variant that exists to measure what the fp64 arithmetic costs.
#ifdef DWT2_K2_F32
typedef float k2r;
#else
typedef double k2r;
#endif

// carried state per quad (see the step comments in the kernel)
struct Carry2 {
    k2r a, c, d, hl1;        // raw a, c, d and predict-1 HL' of row r-1
    k2r hh1, lh1f;           // predict-1 HH' and update-1 LH of row r-2
    k2r A, hl2;              // update-1 LL and predict-2 HL' of row r-2
    k2r hh2, lh2f;           // predict-2 HH' and update-2 LH of row r-3
};

__device__ __forceinline__ k2r shr(k2r v) { return __shfl_down_sync(0xffffffffu, v, 1); }   // lane + 1
__device__ __forceinline__ k2r shl(k2r v) { return __shfl_up_sync(0xffffffffu, v, 1); }     // lane - 1

// horizontal neighbours of quad i of the lane: i + 1 (lane + 1's quad 0 for
// the last) and i - 1 (lane - 1's last quad for the first)
#define K2_RIGHT(x, i, nb) ((i) < QK - 1 ? (x)[(i) + 1] : (nb))
#define K2_LEFT(x, i, nb) ((i) > 0 ? (x)[(i) - 1] : (nb))

template <bool VEC, bool EDGE>
__device__ void k2_tile(const K2Args &a, float *wring, int img, int m0, int n0, int n1, int lane)
{
    // interior slabs with 16-byte rows: raw rows stream into a per-warp
    // shared-memory ring by cp.async (DS rows in flight, no registers held);
    // edge slabs (horizontal mirroring) load through registers
    // (measured: edge slabs through the ring too -- lanes outside the image
    // copying their pixels one by one from the mirrored columns -- are slower
    // than the register path: 8192^2 112.6 vs 105.8 us)
    constexpr bool ASYNC = VEC && !EDGE;
    constexpr int D = ASYNC ? DS : DR;
    const int Wq = (a.W + 1) >> 1, Wh = a.W >> 1, Hh = a.H >> 1;
    const float *in = a.in + (long long)img * a.in_img;
    const int xb = 2 * (m0 - QK) + 2 * QK * lane;
    Carry2 cy[QK];
#pragma unroll
    for (int i = 0; i < QK; ++i) cy[i] = Carry2{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const int r_first = n0 - 2, r_last = n1 + 1;
    RawRow reg[ASYNC ? 1 : D];
    auto issue = [&](int j, int r) {               // j: compile-time slot
        if (ASYNC) {
            int y0 = 2 * r, y1 = 2 * r + 1;
            if (y0 < 0 || y1 >= a.H) {
                y0 = wssi(y0, a.H);
                y1 = wssi(y1, a.H);
            }
            const float *r0 = in + (long long)y0 * a.in_pitch;
            const float *r1 = in + (long long)y1 * a.in_pitch;
            float *d0 = wring + (2 * j) * RW + 2 * QK * lane;
            float *d1 = wring + (2 * j + 1) * RW + 2 * QK * lane;
#pragma unroll
            for (int q = 0; q < QK / 2; ++q) {
                cp_async16(d0 + 4 * q, r0 + xb + 4 * q);
                cp_async16(d1 + 4 * q, r1 + xb + 4 * q);
            }
        } else {
            reg[ASYNC ? 0 : j] = load_raw_row<VEC, EDGE>(a, in, r, xb);
        }
    };
    // the row loop runs in whole groups of D rows (rows past r_last are
    // mirrored reads whose outputs are not stored): no early exit, so the
    // shuffles stay in provably convergent code
#pragma unroll
    for (int j = 0; j < D; ++j) {
        issue(j, r_first + j);
        if (ASYNC) cp_async_commit();
    }
    const int mo = m0 + QK * (lane - 1);              // first output quad of the lane (lanes 1..30)
    const bool out_lane = lane >= 1 && lane <= 30;
    // output cursors at row r - 2 of the walk, advanced one row per iteration
    float *cll = a.ll + (long long)img * a.ll_img + (long long)(r_first - 2) * a.ll_pitch + mo;
    const long long ob0 = (long long)img * a.out_img + (long long)(r_first - 2) * a.out_pitch + mo;
    float *chl = a.hl + ob0, *clh = a.lh + ob0, *chh = a.hh + ob0;
    // rows in groups of D so that every ring slot index is a compile-time
    // constant (a dynamic index would force the prefetched loads to land)
    // one walk row: ring slot j (compile-time), walk row r, warm-up phase ph
    // (r - r_first while < 4, else 4; a compile-time constant at every call)
    auto row = [&](const int j, const int r, const int ph) {
        RawRow R;
        if (ASYNC) {
            cp_async_wait<D - 1>();                    // row r's group (the oldest) has landed
#pragma unroll
            for (int q = 0; q < QK / 2; ++q) {
                const float4 u = *reinterpret_cast<const float4 *>(wring + (2 * j) * RW + 2 * QK * lane + 4 * q);
                const float4 v = *reinterpret_cast<const float4 *>(wring + (2 * j + 1) * RW + 2 * QK * lane + 4 * q);
                R.e[4 * q] = u.x; R.e[4 * q + 1] = u.y; R.e[4 * q + 2] = u.z; R.e[4 * q + 3] = u.w;
                R.o[4 * q] = v.x; R.o[4 * q + 1] = v.y; R.o[4 * q + 2] = v.z; R.o[4 * q + 3] = v.w;
            }
        } else {
            R = reg[ASYNC ? 0 : j];
        }
        if (!ASYNC) issue(j, r + D);
        k2r av[QK], bv[QK], cv[QK], dv[QK];
#pragma unroll
        for (int i = 0; i < QK; ++i) {
            av[i] = R.e[2 * i]; bv[i] = R.e[2 * i + 1];
            cv[i] = R.o[2 * i]; dv[i] = R.o[2 * i + 1];
        }
        // ---- predict 1, row r (same-row part): HL'1 = b + c0 (a + a[m+1])
        const k2r a_nb = shr(av[0]);
        k2r hl1[QK];
#pragma unroll
        for (int i = 0; i < QK; ++i) hl1[i] = fma(k2r(a.c0), av[i] + K2_RIGHT(av, i, a_nb), bv[i]);
        // warm-up: the first 4 rows of a tile only build the carries that
        // output row n0 needs, so step s runs from walk row r_first + s on
        // (1: predict-1 completion + LH1, 2: HL1 / LL1 / HL'2, 3: predict-2
        // completion + LH2, 4: HL2 / LL2).  The skipped values feed nothing
        // that is stored; the branch is warp-uniform.
        k2r lh1[QK], hh1[QK], C1[QK], A1[QK], B1[QK], hl2[QK], lh2[QK], hh2[QK], C2[QK];
#pragma unroll
        for (int i = 0; i < QK; ++i) {
            lh1[i] = hh1[i] = C1[i] = A1[i] = B1[i] = hl2[i] = lh2[i] = hh2[i] = C2[i] = k2r(0);
        }
        if (ph >= 1) {
        // ---- predict 1 completes row r-1: LH'1 = c + c0 (a + a[n+1]),
        //      HH'1 = d + c0 (c + c[m+1]) + c0 (HL'1 + HL'1[n+1])
        k2r cp_[QK];
#pragma unroll
        for (int i = 0; i < QK; ++i) cp_[i] = cy[i].c;
        const k2r c_nb = shr(cp_[0]);
#pragma unroll
        for (int i = 0; i < QK; ++i) {
            lh1[i] = fma(k2r(a.c0), cy[i].a + av[i], cy[i].c);
            hh1[i] = fma(k2r(a.c0), cy[i].hl1 + hl1[i], fma(k2r(a.c0), cy[i].c + K2_RIGHT(cp_, i, c_nb), cy[i].d));
        }
        // ---- update 1, row r-1: LH1 = LH'1 + c1 (HH'1 + HH'1[m-1]),
        //      HL1 = HL'1 + c1 (HH'1 + HH'1[n-1]),
        //      LL1 = a + c1 (HL'1 + HL'1[m-1]) + c1 (LH1 + LH1[n-1])
        const k2r hh1_l = shl(hh1[QK - 1]);
#pragma unroll
        for (int i = 0; i < QK; ++i) C1[i] = fma(k2r(a.c1), hh1[i] + K2_LEFT(hh1, i, hh1_l), lh1[i]);
        }
        if (ph >= 2) {
        k2r hlp[QK];
#pragma unroll
        for (int i = 0; i < QK; ++i) hlp[i] = cy[i].hl1;
        const k2r hl1p_l = shl(hlp[QK - 1]);
#pragma unroll
        for (int i = 0; i < QK; ++i) {
            B1[i] = fma(k2r(a.c1), hh1[i] + cy[i].hh1, cy[i].hl1);
            A1[i] = fma(k2r(a.c1), C1[i] + cy[i].lh1f, fma(k2r(a.c1), cy[i].hl1 + K2_LEFT(hlp, i, hl1p_l), cy[i].a));
        }
        // ---- predict 2 on the update-1 output, row r-1 (same-row part):
        //      HL'2 = HL1 + c2 (LL1 + LL1[m+1])
        const k2r A_nb = shr(A1[0]);
#pragma unroll
        for (int i = 0; i < QK; ++i) hl2[i] = fma(k2r(a.c2), A1[i] + K2_RIGHT(A1, i, A_nb), B1[i]);
        }
        if (ph >= 3) {
        // ---- predict 2 completes row r-2 (carried A, LH1 = lh1f, HH1 = hh1, HL'2):
        //      LH'2 = LH1 + c2 (LL1 + LL1[n+1]), HH'2 = HH1 + c2 (LH1 + LH1[m+1]) + c2 (HL'2 + HL'2[n+1])
        k2r lf[QK];
#pragma unroll
        for (int i = 0; i < QK; ++i) lf[i] = cy[i].lh1f;
        const k2r C_nb = shr(lf[0]);
#pragma unroll
        for (int i = 0; i < QK; ++i) {
            lh2[i] = fma(k2r(a.c2), cy[i].A + A1[i], cy[i].lh1f);
            hh2[i] = fma(k2r(a.c2), cy[i].hl2 + hl2[i], fma(k2r(a.c2), cy[i].lh1f + K2_RIGHT(lf, i, C_nb), cy[i].hh1));
        }
        // ---- update 2, row r-2
        const k2r hh2_l = shl(hh2[QK - 1]);
#pragma unroll
        for (int i = 0; i < QK; ++i) C2[i] = fma(k2r(a.c3), hh2[i] + K2_LEFT(hh2, i, hh2_l), lh2[i]);
        }
        k2r A2[QK], B2[QK];
        if (ph >= 4) {
        k2r h2p[QK];
#pragma unroll
        for (int i = 0; i < QK; ++i) h2p[i] = cy[i].hl2;
        const k2r hl2p_l = shl(h2p[QK - 1]);
#pragma unroll
        for (int i = 0; i < QK; ++i) {
            B2[i] = fma(k2r(a.c3), hh2[i] + cy[i].hh2, cy[i].hl2);
            A2[i] = fma(k2r(a.c3), C2[i] + cy[i].lh2f, fma(k2r(a.c3), cy[i].hl2 + K2_LEFT(h2p, i, hl2p_l), cy[i].A));
        }
        }
        // ---- store output row r-2 (scaled); ph < 4 only on warm-up rows (n < n0)
        const int n = r - 2;
        if (ph >= 4 && n >= n0 && n < n1 && out_lane) {
            float oLL[QK], oHL[QK], oLH[QK], oHH[QK];
#pragma unroll
            for (int i = 0; i < QK; ++i) {
                oLL[i] = (float)(A2[i] * a.sll);
                oHL[i] = (float)B2[i];          // HL, LH scaling: K / K = 1 (DESIGN.md C-B2)
                oLH[i] = (float)C2[i];
                oHH[i] = (float)(hh2[i] * a.shh);
            }
            const bool has_odd = n < Hh;
            if (VEC && !EDGE) {
                if (QK == 4) {
                    *reinterpret_cast<float4 *>(cll) = make_float4(oLL[0], oLL[1], oLL[2 % QK], oLL[3 % QK]);
                    __stcs(reinterpret_cast<float4 *>(chl), make_float4(oHL[0], oHL[1], oHL[2 % QK], oHL[3 % QK]));
                    if (has_odd) {
                        __stcs(reinterpret_cast<float4 *>(clh), make_float4(oLH[0], oLH[1], oLH[2 % QK], oLH[3 % QK]));
                        __stcs(reinterpret_cast<float4 *>(chh), make_float4(oHH[0], oHH[1], oHH[2 % QK], oHH[3 % QK]));
                    }
                } else {
                    *reinterpret_cast<float2 *>(cll) = make_float2(oLL[0], oLL[1]);
                    __stcs(reinterpret_cast<float2 *>(chl), make_float2(oHL[0], oHL[1]));
                    if (has_odd) {
                        __stcs(reinterpret_cast<float2 *>(clh), make_float2(oLH[0], oLH[1]));
                        __stcs(reinterpret_cast<float2 *>(chh), make_float2(oHH[0], oHH[1]));
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < QK; ++i) {
                    const int m = mo + i;
                    if (m < Wq) {
                        cll[i] = oLL[i];
                        if (has_odd) __stcs(clh + i, oLH[i]);
                    }
                    if (m < Wh) {
                        __stcs(chl + i, oHL[i]);
                        if (has_odd) __stcs(chh + i, oHH[i]);
                    }
                }
            }
        }
        cll += a.ll_pitch;
        chl += a.out_pitch;
        clh += a.out_pitch;
        chh += a.out_pitch;
        // ---- carries
#pragma unroll
        for (int i = 0; i < QK; ++i) {
            cy[i].hh2 = hh2[i];
            cy[i].lh2f = C2[i];
            cy[i].A = A1[i];
            cy[i].hl2 = hl2[i];
            cy[i].hh1 = hh1[i];
            cy[i].lh1f = C1[i];
            cy[i].a = av[i];
            cy[i].c = cv[i];
            cy[i].d = dv[i];
            cy[i].hl1 = hl1[i];
        }
        if (ASYNC) {
            // slot j is free again (its row was consumed above)
            if (r - j + D <= r_last) issue(j, r + D);    // the next group exists
            cp_async_commit();
        }
    };
    if (VEC && !DWT2_K2_PEEL_ALL) {
        // 16-byte rows (the ring path and its edge slabs): every row runs every
        // step.  Peeling the warm-up group measured slower here (8192^2 9/7
        // 389 -> 378 Gpix/s, 16384^2 unchanged: the extra copy of the D-row
        // body costs instruction-cache misses), and so did peeling only the
        // edge slabs' register path inside this kernel (config 4 389.6 -> 384.8)
        for (int rb = r_first; rb <= r_last; rb += D) {
#pragma unroll
            for (int j = 0; j < D; ++j) row(j, rb + j, 4);
        }
    } else {
        // unaligned rows (the register path on every slab): the warm-up rows
        // are peeled, their skipped steps fold away at compile time and the
        // steady-state body carries no phase test (a run-time phase test cost
        // 2-6 %; peeled: config 4b 9/7 287.3 -> 296.1 Gpix/s)
        constexpr int PEEL = (4 + D - 1) / D;
#pragma unroll
        for (int g = 0; g < PEEL; ++g) {
#pragma unroll
            for (int j = 0; j < D; ++j) row(j, r_first + g * D + j, g * D + j < 4 ? g * D + j : 4);
        }
        for (int rb = r_first + PEEL * D; rb <= r_last; rb += D) {
#pragma unroll
            for (int j = 0; j < D; ++j) row(j, rb + j, 4);
        }
    }
    if (ASYNC) cp_async_wait<0>();
}

__device__ __forceinline__ void pdl_wait97() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch97() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <bool VEC>
__global__ void __launch_bounds__(KT, DWT2_K2_MINB) dwt_k2_level_kernel(const __grid_constant__ K2Args a)
{
    pdl_launch97();
    pdl_wait97();
    extern __shared__ __align__(16) float k2_smem[];
    const int lane = threadIdx.x & 31;
    float *wring = k2_smem + (threadIdx.x >> 5) * (DS * 2 * RW);
    const int Wq = (a.W + 1) >> 1, Hq = (a.H + 1) >> 1;
    for (long long t = dwt2_queue_fetch(a.counter, a.ntiles, a.nwarps, lane); t < a.ntiles;
         t = dwt2_queue_fetch(a.counter, a.ntiles, a.nwarps, lane)) {
        int img, blk, slab;
        k2_decode(a, int(t), img, blk, slab);
        const int m0 = slab * OUTQ;
        const int n0 = blk * a.tb, n1 = min(n0 + a.tb, Hq);
        // pixel columns 2 (m0 - QK) .. 2 (m0 - QK + SLABQ) - 1 must lie inside the image for the
        // unmirrored path (and every output quad of the slab must exist)
        const bool edge = (m0 < QK) || (2 * (m0 - QK + SLABQ) > a.W) || (m0 + OUTQ > Wq);
        if (edge) k2_tile<VEC, true>(a, wring, img, m0, n0, n1, lane);
        else k2_tile<VEC, false>(a, wring, img, m0, n0, n1, lane);
    }
}

int k2_ctas_per_sm()
{
    static int per_sm = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int n = 0;
        if (cudaFuncSetAttribute(dwt_k2_level_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(K2_SMEM)) !=
                cudaSuccess ||
            cudaFuncSetAttribute(dwt_k2_level_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(K2_SMEM)) !=
                cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dwt_k2_level_kernel<true>, KT, K2_SMEM) != cudaSuccess || n < 1)
            n = 1;
        per_sm = n;
    });
    cudaGetLastError();
    return per_sm;
}

struct Wavelet2 {
    double c0, c1, c2, c3, K;
};

Wavelet2 wavelet_params(const dwt2_plan *p)
{
    const int wavelet = p->wavelet;
    if (wavelet == DWT2_WAVELET_LIFTING) return Wavelet2{p->lift[0], p->lift[1], p->lift[2], p->lift[3], p->lift[4]};
    if (wavelet == DWT2_WAVELET_CDF97)
        return Wavelet2{-1.586134342059924, -0.052980118572961, 0.882911075530934, 0.443506852043971,
                        1.230174104914001};
    return Wavelet2{-0.5, 0.25, 0.0, 0.0, 1.0};      // DWT2_WAVELET_CDF53_K2
}

int32_t launch_k2_level(const dwt2_plan *p, K2Args a, cudaStream_t s)
{
    const int Wq = (a.W + 1) / 2, Hq = (a.H + 1) / 2;
    a.nslabs = (Wq + OUTQ - 1) / OUTQ;
    const long long warps = (long long)p->sms * k2_ctas_per_sm() * KW;
    const long long slab_rows = (long long)a.count * a.nslabs * Hq;
    // ~32 tiles per resident warp through the queue, at least 16 rows each
    // (measured: 0.62 -> 0.77 of copy at 16384^2 from 4 to 16 tiles per warp,
    // 0.80 -> 0.86 from 16 to 32; the 4 warm-up rows per tile cost less than
    // the imbalance), scripts/sweeps/gpu_queue_tpw.sh, scripts/tile_probe.py
    static const int tpw = tuning_int("DWT2_K2_TPW", 32, 1, 1024);
    long long tb = slab_rows / (tpw * warps);
    static const int min_tb = tuning_int("DWT2_K2_MINTB", 16, 4, 512);
    tb = std::max<long long>(min_tb, std::min<long long>(512, tb)); // 4 warm-up rows per tile: >= 16 rows
    // levels with less than one minimum tile per resident warp: one tile per
    // warp of ceil(rows / warps) (>= 4) rows, so every warp takes part (a
    // small level is latency-bound: its time is one tile's row walk)
    static const int small_f = tuning_int("DWT2_K2_SMALLF", 1, 0, 64);
    if (slab_rows < (long long)min_tb * warps * small_f)
        tb = std::max<long long>(4, (slab_rows + warps - 1) / warps);
    a.tb = int(tb);
    a.nblk = int((Hq + tb - 1) / tb);
    a.ntiles = (long long)a.count * a.nblk * a.nslabs;
    a.fd_img = make_fastdiv(unsigned(a.nblk * a.nslabs));
    a.fd_slabs = make_fastdiv(unsigned(a.nslabs));
    // edge-first tile order (k2_decode): the edge slabs as the kernel classifies them
    static const int edge_first = tuning_int("DWT2_K2_EDGEFIRST", 1, 0, 1);
    a.nedge = 0;
    if (edge_first && a.nslabs >= 3) {
        int sr = a.nslabs;
        while (sr - 1 >= 1) {
            const int m0 = (sr - 1) * OUTQ;
            if ((2 * (m0 - QK + SLABQ) > a.W) || (m0 + OUTQ > Wq)) --sr;
            else break;
        }
        a.slab_r = sr;
        a.nedge = 1 + (a.nslabs - sr);
        if (a.nedge >= a.nslabs) a.nedge = 0;
    }
    if (a.ntiles >= (1LL << 31)) return fail(DWT2_EINVAL);
    const long long want = (a.ntiles + KW - 1) / KW;
    const int grid = int(std::max<long long>(1, std::min<long long>(want, warps / KW)));
    a.nwarps = grid * KW;
    const bool vec = aligned(a.in, 16) && a.in_pitch % 4 == 0 && (a.count == 1 || a.in_img % 4 == 0) &&
                     aligned(a.ll, 4 * QK) && aligned(a.hl, 4 * QK) && aligned(a.lh, 4 * QK) && aligned(a.hh, 4 * QK) &&
                     a.ll_pitch % QK == 0 && a.out_pitch % QK == 0 &&
                     (a.count == 1 || (a.ll_img % QK == 0 && a.out_img % QK == 0));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(KT);
    cfg.dynamicSmemBytes = K2_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = vec ? cudaLaunchKernelEx(&cfg, dwt_k2_level_kernel<true>, a)
                        : cudaLaunchKernelEx(&cfg, dwt_k2_level_kernel<false>, a);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

// ---------------------------------------------------------------------------
// Inverse of the K = 2 kernel (9/7 and general lifting wavelets): undo the
// scaling, then the four spatial steps in reverse (update 2, predict 2,
// update 1, predict 1), each Eq. (5) factor inverted by negating its
// polynomials.  Per quad row n loaded (after scaling: a2 = LL K^2, HL, LH,
// hh2 = HH / K^2):
//   undo U2, row n:    LH'2 = LH - c3 (hh2 + hh2[m-1]),  HL'2 = HL - c3 (hh2 + hh2[n-1]),
//                      LL1  = a2 - c3 (HL'2 + HL'2[m-1]) - c3 (LH + LH[n-1])
//   undo P2, row n-1:  HL1 = HL'2 - c2 (LL1 + LL1[m+1]),  LH1 = LH'2 - c2 (LL1 + LL1[n+1]),
//                      HH1 = hh2 - c2 (LH1 + LH1[m+1]) - c2 (HL'2 + HL'2[n+1])
//   undo U1, row n-1:  LH'1 = LH1 - c1 (HH1 + HH1[m-1]),  HL'1 = HL1 - c1 (HH1 + HH1[n-1]),
//                      a    = LL1 - c1 (HL'1 + HL'1[m-1]) - c1 (LH1 + LH1[n-1])
//   undo P1, row n-2:  b = HL'1 - c0 (a + a[m+1]),  c = LH'1 - c0 (a + a[n+1]),
//                      d = HH1 - c0 (c + c[m+1]) - c0 (HL'1 + HL'1[n+1])
// and pixel rows 2(n-2), 2(n-2)+1 are stored.  Boundaries: the coefficient
// field of a whole-sample-symmetric input is itself symmetric in the
// interleaved (pixel) index, so coefficients are fetched at mirrored pixel
// positions (a coefficient of parity p at quad q sits at pixel 2q + p), the
// same rule as the oracle's inverse (oracle/dwt97_oracle.c).
// ---------------------------------------------------------------------------
struct K2InvArgs {
    const float *ll, *hl, *lh, *hh;        // plane origins of image 0
    long long ll_pitch, ll_img, d_pitch, d_img;
    float *out;                            // reconstructed level input
    long long out_pitch, out_img;
    int W, H;
    int nslabs, tb, nblk, count;
    long long ntiles;
    FastDiv fd_img, fd_slabs;              // division by nblk * nslabs and by nslabs (ntiles < 2^31)
    double c0, c1, c2, c3, K2sq, invK2sq;  // K^2 and 1 / K^2
    int async;                             // 1: every plane 8-byte aligned with even pitches (cp.async ring)
    int vec_out;                           // 1: output 16-byte aligned with pitch % 4 == 0 (float4 stores)
    unsigned int *counter;                 // tile queue (queue.cuh)
    int nwarps;
    int slab_r, nedge;                     // edge-first tile order (k2_decode)
};

struct InvCarry {
    k2r hh2, lh, hl2p, lh2p, ll1;        // row n-1: scaled HH, input LH, HL'2, LH'2, LL1
    k2r hh1, lh1, a, hl1p, lh1p;         // row n-2: HH1, LH1, a, HL'1, LH'1
};

__device__ __forceinline__ int mqi(int q, int par, int n) { return (wssi_fast(2 * q + par, n) - par) >> 1; }

struct InvRaw {
    float LL[2], HL[2], LH[2], HH[2];
};

template <bool EDGE>
__device__ __forceinline__ InvRaw kinv_load(const K2InvArgs &a, int img, int n, int m0, int lane)
{
    const int nL = mqi(n, 0, a.H), nH = mqi(n, 1, a.H);
    const float *pll = a.ll + (long long)img * a.ll_img + (long long)nL * a.ll_pitch;
    const float *phl = a.hl + (long long)img * a.d_img + (long long)nL * a.d_pitch;
    const float *plh = a.lh + (long long)img * a.d_img + (long long)nH * a.d_pitch;
    const float *phh = a.hh + (long long)img * a.d_img + (long long)nH * a.d_pitch;
    const int m = m0 - 2 + 2 * lane;
    InvRaw R;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int mL = EDGE ? mqi(m + i, 0, a.W) : m + i;
        const int mH = EDGE ? mqi(m + i, 1, a.W) : m + i;
        R.LL[i] = __ldg(pll + mL);
        R.LH[i] = __ldg(plh + mL);
        R.HL[i] = __ldg(phl + mH);
        R.HH[i] = __ldg(phh + mH);
    }
    return R;
}

__device__ __forceinline__ void cp_async8(float *dst, const float *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src) : "memory");
}

#ifndef DWT2_K2INV_PEEL_ALL
#define DWT2_K2INV_PEEL_ALL 0              // measurement builds: peel the warm-up rows on the ring path too
#endif
#ifndef DWT2_K2INV_DS
#define DWT2_K2INV_DS 4
#endif
constexpr int IDSK = DWT2_K2INV_DS;            // quad rows in flight per warp (inverse ring)
constexpr size_t KINV_SMEM = size_t(KW) * IDSK * 4 * 64 * sizeof(float);

// Interior slabs with 8-byte aligned planes stream their rows through a
// per-warp shared-memory ring (cp.async, IDSK rows in flight); edge slabs
// (mirrored columns) or unaligned planes load through registers.
template <bool EDGE, bool ASYNC>
__device__ void kinv_tile(const K2InvArgs &a, float *ring, int img, int m0, int n0, int n1, int lane)
{
    constexpr int D = ASYNC ? IDSK : IDR;
    InvCarry cy[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) cy[i] = InvCarry{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const int r_first = n0 - 2, r_last = n1 + 1;
    const int mo = m0 + 2 * (lane - 1);
    const bool out_lane = lane >= 1 && lane <= 30;
    InvRaw reg[ASYNC ? 1 : D];
    auto issue = [&](int j, int n) {                 // j: compile-time slot
        if (ASYNC) {
            const int nL = mqi(n, 0, a.H), nH = mqi(n, 1, a.H);
            const int m = m0 - 2 + 2 * lane;
            float *st = ring + j * (4 * 64) + 2 * lane;
            cp_async8(st, a.ll + (long long)img * a.ll_img + (long long)nL * a.ll_pitch + m);
            cp_async8(st + 64, a.hl + (long long)img * a.d_img + (long long)nL * a.d_pitch + m);
            cp_async8(st + 128, a.lh + (long long)img * a.d_img + (long long)nH * a.d_pitch + m);
            cp_async8(st + 192, a.hh + (long long)img * a.d_img + (long long)nH * a.d_pitch + m);
        } else {
            reg[ASYNC ? 0 : j] = kinv_load<EDGE>(a, img, n, m0, lane);
        }
    };
#pragma unroll
    for (int j = 0; j < D; ++j) {
        issue(j, r_first + j);
        if (ASYNC) cp_async_commit();
    }
    // one walk row: ring slot j (compile-time), quad row n, warm-up phase ph
    // (n - r_first while < 4, else 4; a compile-time constant at every call)
    auto row = [&](const int j, const int n, const int ph) {
        InvRaw R;
        if (ASYNC) {
            cp_async_wait<D - 1>();
            const float *st = ring + j * (4 * 64) + 2 * lane;
            const float2 ll = *reinterpret_cast<const float2 *>(st);
            const float2 hl = *reinterpret_cast<const float2 *>(st + 64);
            const float2 lh = *reinterpret_cast<const float2 *>(st + 128);
            const float2 hh = *reinterpret_cast<const float2 *>(st + 192);
            R.LL[0] = ll.x; R.LL[1] = ll.y; R.HL[0] = hl.x; R.HL[1] = hl.y;
            R.LH[0] = lh.x; R.LH[1] = lh.y; R.HH[0] = hh.x; R.HH[1] = hh.y;
        } else {
            R = reg[ASYNC ? 0 : j];
            issue(j, n + D);
        }
        k2r LL[2], HL[2], LH[2], HH[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            LL[i] = R.LL[i]; HL[i] = R.HL[i]; LH[i] = R.LH[i]; HH[i] = R.HH[i];
        }
        // ---- scaling undone, undo U2 at row n
        k2r a2[2], hh2[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            a2[i] = LL[i] * k2r(a.K2sq);
            hh2[i] = HH[i] * k2r(a.invK2sq);
        }
        const k2r hh2_l = shl(hh2[1]);
        k2r lh2p[2], hl2p[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            lh2p[i] = fma(-k2r(a.c3), hh2[i] + (i == 0 ? hh2_l : hh2[0]), LH[i]);
            hl2p[i] = fma(-k2r(a.c3), hh2[i] + cy[i].hh2, HL[i]);
        }
        const k2r hl2p_l = shl(hl2p[1]);
        k2r ll1[2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
            ll1[i] = fma(-k2r(a.c3), LH[i] + cy[i].lh, fma(-k2r(a.c3), hl2p[i] + (i == 0 ? hl2p_l : hl2p[0]), a2[i]));
        // warm-up: the first 4 rows of a tile only build the carries that
        // output quad row n0 needs, so undo-P2 runs from walk row r_first + 2
        // on, undo-U1 from r_first + 3 and undo-P1 (the output) from r_first + 4;
        // the skipped values feed nothing that is stored (warp-uniform branches)
        k2r pll1[2], hl1[2], lh1[2], hh1[2], lh1p[2], hl1p[2], av[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            pll1[i] = cy[i].ll1;
            hl1[i] = lh1[i] = hh1[i] = lh1p[i] = hl1p[i] = av[i] = k2r(0);
        }
        if (ph >= 2) {
        // ---- undo P2 completes row n-1 (carried hl2p, lh2p, ll1, hh2 of row n-1)
        const k2r ll1_r = shr(pll1[0]);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            hl1[i] = fma(-k2r(a.c2), pll1[i] + (i == 0 ? pll1[1] : ll1_r), cy[i].hl2p);
            lh1[i] = fma(-k2r(a.c2), pll1[i] + ll1[i], cy[i].lh2p);
        }
        const k2r lh1_r = shr(lh1[0]);
#pragma unroll
        for (int i = 0; i < 2; ++i)
            hh1[i] = fma(-k2r(a.c2), cy[i].hl2p + hl2p[i], fma(-k2r(a.c2), lh1[i] + (i == 0 ? lh1[1] : lh1_r), cy[i].hh2));
        }
        if (ph >= 3) {
        // ---- undo U1, row n-1 (carried hh1, lh1 of row n-2)
        const k2r hh1_l = shl(hh1[1]);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            lh1p[i] = fma(-k2r(a.c1), hh1[i] + (i == 0 ? hh1_l : hh1[0]), lh1[i]);
            hl1p[i] = fma(-k2r(a.c1), hh1[i] + cy[i].hh1, hl1[i]);
        }
        const k2r hl1p_l = shl(hl1p[1]);
#pragma unroll
        for (int i = 0; i < 2; ++i)
            av[i] = fma(-k2r(a.c1), lh1[i] + cy[i].lh1, fma(-k2r(a.c1), hl1p[i] + (i == 0 ? hl1p_l : hl1p[0]), pll1[i]));
        }
        k2r pa[2], bo[2], co[2], dout[2];
        if (ph >= 4) {
        // ---- undo P1 completes row n-2 (carried a, hl1p, lh1p, hh1 of row n-2)
#pragma unroll
        for (int i = 0; i < 2; ++i) pa[i] = cy[i].a;
        const k2r a_r = shr(pa[0]);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            bo[i] = fma(-k2r(a.c0), pa[i] + (i == 0 ? pa[1] : a_r), cy[i].hl1p);
            co[i] = fma(-k2r(a.c0), pa[i] + av[i], cy[i].lh1p);
        }
        const k2r c_r = shr(co[0]);
#pragma unroll
        for (int i = 0; i < 2; ++i)
            dout[i] = fma(-k2r(a.c0), cy[i].hl1p + hl1p[i], fma(-k2r(a.c0), co[i] + (i == 0 ? co[1] : c_r), cy[i].hh1));
        }
        // ---- store pixel rows 2(n-2), 2(n-2)+1 (ph < 4 only on warm-up rows, q < n0)
        const int q = n - 2;
        if (ph >= 4 && q >= n0 && q < n1 && out_lane) {
            const int x = 2 * mo, y = 2 * q;
            float *r0 = a.out + (long long)img * a.out_img + (long long)y * a.out_pitch + x;
            float *r1 = r0 + a.out_pitch;
            const float e[4] = {(float)pa[0], (float)bo[0], (float)pa[1], (float)bo[1]};
            const float o[4] = {(float)co[0], (float)dout[0], (float)co[1], (float)dout[1]};
            const bool odd = y + 1 < a.H;
            if (!EDGE && a.vec_out) {
                __stcs(reinterpret_cast<float4 *>(r0), make_float4(e[0], e[1], e[2], e[3]));
                if (odd) __stcs(reinterpret_cast<float4 *>(r1), make_float4(o[0], o[1], o[2], o[3]));
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (x + j < a.W) {
                        __stcs(r0 + j, e[j]);
                        if (odd) __stcs(r1 + j, o[j]);
                    }
                }
            }
        }
        // ---- carries
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            cy[i].hh1 = hh1[i];
            cy[i].lh1 = lh1[i];
            cy[i].a = av[i];
            cy[i].hl1p = hl1p[i];
            cy[i].lh1p = lh1p[i];
            cy[i].hh2 = hh2[i];
            cy[i].lh = LH[i];
            cy[i].hl2p = hl2p[i];
            cy[i].lh2p = lh2p[i];
            cy[i].ll1 = ll1[i];
        }
        if (ASYNC) {
            if (n - j + D <= r_last) issue(j, n + D);  // slot j's row was consumed above
            cp_async_commit();
        }
    };
    if (ASYNC && !DWT2_K2INV_PEEL_ALL) {
        // every row runs every step (gating the warm-up rows at run time
        // measured neutral on the ring path: 9/7 inverse config 3 / 4 within 0.3 %)
        for (int rb = r_first; rb <= r_last; rb += D) {
#pragma unroll
            for (int j = 0; j < D; ++j) row(j, rb + j, 4);
        }
    } else {
        // register path (edge slabs, unaligned planes): the warm-up rows are
        // peeled and their skipped steps fold away at compile time (9/7
        // inverse config 4 325.5 -> 332.9 Gpix/s, 4b 240.0 -> 244.8, 3 691.5 -> 696.0)
        constexpr int PEEL = (4 + D - 1) / D;
#pragma unroll
        for (int g = 0; g < PEEL; ++g) {
#pragma unroll
            for (int j = 0; j < D; ++j) row(j, r_first + g * D + j, g * D + j < 4 ? g * D + j : 4);
        }
        for (int rb = r_first + PEEL * D; rb <= r_last; rb += D) {
#pragma unroll
            for (int j = 0; j < D; ++j) row(j, rb + j, 4);
        }
    }
    if (ASYNC) cp_async_wait<0>();
}

#ifndef DWT2_K2INV_MINB
#define DWT2_K2INV_MINB 5                  // measured: 5 > 4 (config 3 +2.7 %), 6 spills
#endif
__global__ void __launch_bounds__(KT, DWT2_K2INV_MINB) dwt_k2_inverse_kernel(const __grid_constant__ K2InvArgs a)
{
    extern __shared__ __align__(16) float kinv_smem[];
    pdl_launch97();
    pdl_wait97();
    const int lane = threadIdx.x & 31;
    float *ring = kinv_smem + (threadIdx.x >> 5) * (IDSK * 4 * 64);
    const int Wq = (a.W + 1) >> 1, Hq = (a.H + 1) >> 1;
    for (long long t = dwt2_queue_fetch(a.counter, a.ntiles, a.nwarps, lane); t < a.ntiles;
         t = dwt2_queue_fetch(a.counter, a.ntiles, a.nwarps, lane)) {
        int img, blk, slab;
        k2_decode(a, int(t), img, blk, slab);
        const int m0 = slab * OUTQ;
        const int n0 = blk * a.tb, n1 = min(n0 + a.tb, Hq);
        // coefficient columns m0 - 2 .. m0 + 61 must exist in every plane for the unmirrored path
        const bool edge = (m0 < 2) || (m0 + 62 > (a.W >> 1)) || (m0 + OUTQ > Wq);
        if (edge) kinv_tile<true, false>(a, ring, img, m0, n0, n1, lane);
        else if (a.async) kinv_tile<false, true>(a, ring, img, m0, n0, n1, lane);
        else kinv_tile<false, false>(a, ring, img, m0, n0, n1, lane);
    }
}

int32_t launch_k2_inverse_level(const dwt2_plan *p, K2InvArgs a, cudaStream_t s)
{
    static int per_sm = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int n = 0;
        if (cudaFuncSetAttribute(dwt_k2_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(KINV_SMEM)) !=
                cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dwt_k2_inverse_kernel, KT, KINV_SMEM) != cudaSuccess ||
            n < 1)
            n = 1;
        per_sm = n;
    });
    cudaGetLastError();
    const int Wq = (a.W + 1) / 2, Hq = (a.H + 1) / 2;
    a.nslabs = (Wq + OUTQ - 1) / OUTQ;
    const long long warps = (long long)p->sms * per_sm * KW;
    const long long slab_rows = (long long)a.count * a.nslabs * Hq;
    static const int tpw = tuning_int("DWT2_K2INV_TPW", 8, 1, 1024);
    long long tb = slab_rows / (tpw * warps);
    static const int min_tb = tuning_int("DWT2_K2INV_MINTB", 16, 4, 512);
    tb = std::max<long long>(min_tb, std::min<long long>(512, tb));
    // levels with >= 64 quad rows per warp: 32-row tiles (measured with the
    // edge-first order: 16384^2 0.821 -> 0.838, 8192^2 0.721 -> 0.729 of copy
    // against 20-row tiles; 48 rows: 0.855 / 0.685; smaller levels keep the
    // tpw-derived height)
    static const int tb_large = tuning_int("DWT2_K2INV_TB", 32, 0, 512);
    if (tb_large > 0 && slab_rows >= 64 * warps) tb = tb_large;
    // small levels: one short tile per warp (as the forward, launch_k2_level)
    static const int small_f = tuning_int("DWT2_K2INV_SMALLF", 1, 0, 64);
    if (slab_rows < (long long)min_tb * warps * small_f) tb = std::max<long long>(4, (slab_rows + warps - 1) / warps);
    a.tb = int(tb);
    a.nblk = int((Hq + tb - 1) / tb);
    a.ntiles = (long long)a.count * a.nblk * a.nslabs;
    a.fd_img = make_fastdiv(unsigned(a.nblk * a.nslabs));
    a.fd_slabs = make_fastdiv(unsigned(a.nslabs));
    // edge-first tile order (k2_decode): the edge slabs as the kernel classifies them
    static const int edge_first = tuning_int("DWT2_K2INV_EDGEFIRST", 1, 0, 1);
    a.nedge = 0;
    if (edge_first && a.nslabs >= 3) {
        int sr = a.nslabs;
        while (sr - 1 >= 1) {
            const int m0 = (sr - 1) * OUTQ;
            if ((m0 + 62 > (a.W >> 1)) || (m0 + OUTQ > Wq)) --sr;
            else break;
        }
        a.slab_r = sr;
        a.nedge = 1 + (a.nslabs - sr);
        if (a.nedge >= a.nslabs) a.nedge = 0;
    }
    if (a.ntiles >= (1LL << 31)) return fail(DWT2_EINVAL);
    const long long want = (a.ntiles + KW - 1) / KW;
    const int grid = int(std::max<long long>(1, std::min<long long>(want, warps / KW)));
    a.nwarps = grid * KW;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(KT);
    cfg.dynamicSmemBytes = KINV_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    a.async = aligned(a.ll, 8) && aligned(a.hl, 8) && aligned(a.lh, 8) && aligned(a.hh, 8) && a.ll_pitch % 2 == 0 &&
              a.d_pitch % 2 == 0 && (a.count == 1 || (a.ll_img % 2 == 0 && a.d_img % 2 == 0)) ? 1 : 0;
    a.vec_out = aligned(a.out, 16) && a.out_pitch % 4 == 0 && (a.count == 1 || a.out_img % 4 == 0) ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, dwt_k2_inverse_kernel, a) != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

}  // namespace

namespace dwt2_detail {

// All levels of the K = 2 lifting kernel (plans created with a wavelet other
// than DWT2_WAVELET_CDF53); buffer roles as run_levels in dwt2.cu.
int k2_tail_start(const dwt2_plan *p, int count)
{
    // levels of <= 2^12 quads (128^2 and below) in the tail launch; the 512^2 and
    // 256^2 levels run as separate small-level launches (tail.cu dwt_small4_kernel):
    // 9/7 config 4 174.2 -> 170.1 us against a 2^16 threshold (scripts/r2/gpu_k2tail2.sh)
    static const int k2_tail_quads = tuning_int("DWT2_K2_TAIL_QUADS", 1 << 12, 0, 1 << 30);
    return tail_start_levels(p, count, 0, p->levels - 1, k2_tail_quads);
}

int32_t run_levels_k2(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                      long long out_stride, cudaStream_t s)
{
    const Wavelet2 wv = wavelet_params(p);
    // the small last levels in one tail launch (tail.cu, radius-4 filters of the
    // lifting pair): the K = 2 kernel walks a tile row by row through four
    // lifting steps, ~9-20 us per dependent launch on a small level
    const int t0 = k2_tail_start(p, count);
    TailLevelIO tail[MAX_TAIL];
    for (int k = 0; k < p->levels; ++k) {
        const LevelGeom &g = p->geom[k];
        K2Args a;
        memset(&a, 0, sizeof(a));
        a.W = g.W;
        a.H = g.H;
        a.count = count;
        a.c0 = wv.c0; a.c1 = wv.c1; a.c2 = wv.c2; a.c3 = wv.c3;
        a.sll = 1.0 / (wv.K * wv.K);
        a.sd = 1.0;
        a.shh = wv.K * wv.K;
        if (k == 0) {
            a.in = in;
            a.in_pitch = p->W;
            a.in_img = in_stride;
        } else {
            const int si = (k - 1) % 2;
            a.in = p->scratch[si];
            a.in_pitch = p->sc_pitch[si];
            a.in_img = p->sc_img_stride[si];
        }
        a.hl = out + g.Wq;
        a.lh = out + (long long)g.Hq * p->W;
        a.hh = a.lh + g.Wq;
        a.out_pitch = p->W;
        a.out_img = out_stride;
        if (k == p->levels - 1) {
            a.ll = out;
            a.ll_pitch = p->W;
            a.ll_img = out_stride;
        } else {
            const int si = k % 2;
            a.ll = p->scratch[si];
            a.ll_pitch = p->sc_pitch[si];
            a.ll_img = p->sc_img_stride[si];
        }
        if (k >= t0) {
            tail[k - t0] = TailLevelIO{a.in, a.in_pitch, a.in_img, a.ll, a.ll_pitch, a.ll_img,
                                       out, a.out_pitch, a.out_img, a.W, a.H};
            continue;
        }
        // small levels: one launch of shared-memory-staged CTAs (tail.cu)
        static const long long k2_small = tuning_int("DWT2_K2_SMALL_QUADS", 1 << 18, 0, 1 << 30);
        if (count <= 65535 && (long long)g.Wq * g.Hq * count <= k2_small) {
            const TailLevelIO lv{a.in, a.in_pitch, a.in_img, a.ll, a.ll_pitch, a.ll_img,
                                 out, a.out_pitch, a.out_img, a.W, a.H};
            int32_t r = launch_small_level_r4(lv, count, tail_filter_from_lifting(wv.c0, wv.c1, wv.c2, wv.c3, wv.K), s);
            if (r != DWT2_OK) return r;
            continue;
        }
        a.counter = p->counters + 2 * (QUEUE_FORWARD + k);
        int32_t r = launch_k2_level(p, a, s);
        if (r != DWT2_OK) return r;
    }
    if (t0 < p->levels)
        return launch_tail_levels(p, tail, p->levels - t0, count,
                                  tail_filter_from_lifting(wv.c0, wv.c1, wv.c2, wv.c3, wv.K), s);
    return DWT2_OK;
}

// Inverse of all levels through the K = 2 kernel, coarsest first; buffer
// roles as run_inverse in inverse.cu.
int32_t run_inverse_k2(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                       long long out_stride, cudaStream_t s)
{
    const Wavelet2 wv = wavelet_params(p);
    for (int k = p->levels - 1; k >= 0; --k) {
        const LevelGeom &g = p->geom[k];
        K2InvArgs a;
        memset(&a, 0, sizeof(a));
        a.W = g.W;
        a.H = g.H;
        a.count = count;
        a.c0 = wv.c0; a.c1 = wv.c1; a.c2 = wv.c2; a.c3 = wv.c3;
        a.K2sq = wv.K * wv.K;
        a.invK2sq = 1.0 / (wv.K * wv.K);
        a.hl = in + g.Wq;
        a.lh = in + (long long)g.Hq * p->W;
        a.hh = a.lh + g.Wq;
        a.d_pitch = p->W;
        a.d_img = in_stride;
        if (k == p->levels - 1) {
            a.ll = in;
            a.ll_pitch = p->W;
            a.ll_img = in_stride;
        } else {
            const int si = k % 2;
            a.ll = p->scratch[si];
            a.ll_pitch = p->sc_pitch[si];
            a.ll_img = p->sc_img_stride[si];
        }
        if (k == 0) {
            a.out = out;
            a.out_pitch = p->W;
            a.out_img = out_stride;
        } else {
            const int si = (k - 1) % 2;
            a.out = p->scratch[si];
            a.out_pitch = p->sc_pitch[si];
            a.out_img = p->sc_img_stride[si];
        }
        a.counter = p->counters + 2 * (QUEUE_INVERSE + k);
        const InvFilter f = inv_filter_from_lifting(wv.c0, wv.c1, wv.c2, wv.c3, wv.K);
        if (f.radius != 0 && small_inverse_level(p, k, count)) {
            // a small level: shared-memory-staged pointwise synthesis (tail.cu)
            const InvLevelIO lv{a.ll, a.ll_pitch, a.ll_img, in, p->W, in_stride, a.out, a.out_pitch, a.out_img,
                                g.W, g.H};
            int32_t r = launch_small_inverse_level(lv, count, f, s);
            if (r != DWT2_OK) return r;
            continue;
        }
        int32_t r = launch_k2_inverse_level(p, a, s);
        if (r != DWT2_OK) return r;
    }
    return DWT2_OK;
}

}  // namespace dwt2_detail
