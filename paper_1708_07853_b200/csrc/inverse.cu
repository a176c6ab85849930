// inverse.cu -- B200 (sm_100a) inverse 2-D CDF 5/3 DWT: the non-separable
// lifting scheme of arXiv:1708.07853, Eq. (5), run
// backwards -- undo the spatial update, then undo the spatial predict -- in
// one fused kernel per level.
//
// Eq. (5) is [update] . [predict] with unit-diagonal triangular factors, so
// its inverse is [predict]^-1 . [update]^-1, each factor inverted by negating
// its off-diagonal polynomials.  Written per quad (m, n)
// with the subband coefficients (LL, HL, LH, HH) of the forward transform and
// the same separable grouping the forward kernel uses (dwt2.cu,
// predict_update):
//
//   undo update:   HH' = HH
//                  HL' = HL - 1/4 (HH + HH[n-1])            (HL = HL' + U* HH')
//                  LH' = LH - 1/4 (HH + HH[m-1])            (LH = LH' + U HH')
//                  a   = LL - 1/4 (HL' + HL'[m-1]) - 1/4 (LH + LH[n-1])
//   undo predict:  b   = HL' + 1/2 (a + a[m+1])             (HL' = b + P a)
//                  c   = LH' + 1/2 (a + a[n+1])             (LH' = c + P* a)
//                  d   = HH' + 1/2 (c + c[m+1]) + 1/2 (HL' + HL'[n+1])
//
// Boundaries (whole-sample symmetric extension, as the forward): H[-1] :=
// H[0] and, for odd sizes, H[M] := H[M-1] -- both realised by clamping the
// detail-plane indices of the raw loads -- and, for even sizes, L[M] :=
// L[M-1] (a and c of the missing right column / bottom row mirror the last
// ones), applied in registers.
//
// Work decomposition.  A warp owns a slab of 64 quad columns (2 quads per
// lane) and walks DOWN a tile of quad rows.  The n-1 neighbours are carried
// in registers, the m-1 / m+1 neighbours come from the adjacent lanes by
// shuffle; lane 0 and lane 31 evaluate the halo quads m0-1 and m0+64 from
// their own loads.  Row n is reconstructed (a, HL', LH') when it is loaded
// and the output pixel rows 2(n-1), 2(n-1)+1 are emitted one row later,
// when a[n] and HL'[n] are known.  fp32 in HBM, fp64 in registers.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "dwt2_internal.h"
#include "queue.cuh"

using namespace dwt2_detail;

namespace {

constexpr int IWARPS = 8;                  // warps per CTA
constexpr int ITHREADS = IWARPS * 32;
constexpr int IQ = 64;                     // quad columns per warp slab (2 per lane)

struct InvArgs {
    const float *ll, *hl, *lh, *hh;        // plane origins of image 0
    long long ll_pitch, ll_img;            // LL plane: row pitch, image stride (elements)
    long long d_pitch, d_img;              // HL / LH / HH planes (the Mallat buffer)
    float *out;                            // reconstructed level input, image 0
    long long out_pitch, out_img;
    int W, H;                              // reconstructed size
    int nslabs, nblk, tb, count;
    int nblk_a, tb_b, split;               // ring kernel, guided tiles: blocks < nblk_a are tb rows from 0,
                                           // the rest tb_b rows from quad row `split` (nblk_a = nblk: uniform)
    long long ntiles;
    FastDiv fd_img, fd_slabs;              // division by nblk * nslabs and by nslabs (ntiles < 2^31)
    const float *ll_lo, *ll_hi, *d_lo, *d_hi;   // allocation ranges of the LL / detail sources (ring loader)
    unsigned int *counter;                       // tile queue (queue.cuh)
    int nwarps;
};

// Raw coefficients of one quad row as one lane sees them: its 2 quads and,
// for the edge lanes, the halo quads m0-1 (HL, HH) and m0+64 (all four).
struct Raw {
    float LL[2], HL[2], LH[2], HH[2];
    float hlL, hhL;                        // quad m0-1
    float llR, hlR, lhR, hhR;              // quad m0+64
};

template <bool VEC, bool EDGE>
__device__ __forceinline__ Raw load_raw(const InvArgs &a, int img, int n, int m0, int lane)
{
    const int Wq = (a.W + 1) >> 1, Wh = a.W >> 1, Hh = a.H >> 1;
    const int nd = min(max(n, 0), Hh - 1);          // LH / HH rows: H[-1] := H[0], H[M] := H[M-1]
    const float *pll = a.ll + (long long)img * a.ll_img + (long long)n * a.ll_pitch;
    const float *phl = a.hl + (long long)img * a.d_img + (long long)n * a.d_pitch;
    const float *plh = a.lh + (long long)img * a.d_img + (long long)nd * a.d_pitch;
    const float *phh = a.hh + (long long)img * a.d_img + (long long)nd * a.d_pitch;
    const int m = m0 + 2 * lane;
    Raw r;
    if (!EDGE && VEC) {
        const float2 ll = __ldg(reinterpret_cast<const float2 *>(pll + m));
        const float2 hl = __ldg(reinterpret_cast<const float2 *>(phl + m));
        const float2 lh = __ldg(reinterpret_cast<const float2 *>(plh + m));
        const float2 hh = __ldg(reinterpret_cast<const float2 *>(phh + m));
        r.LL[0] = ll.x; r.LL[1] = ll.y; r.HL[0] = hl.x; r.HL[1] = hl.y;
        r.LH[0] = lh.x; r.LH[1] = lh.y; r.HH[0] = hh.x; r.HH[1] = hh.y;
    } else {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int mi = m + i;
            const int mL = EDGE ? min(mi, Wq - 1) : mi;                  // beyond the image: unused
            const int mH = EDGE ? min(max(mi, 0), Wh - 1) : mi;          // odd W: H[M] := H[M-1]
            r.LL[i] = __ldg(pll + mL);
            r.LH[i] = __ldg(plh + mL);
            r.HL[i] = __ldg(phl + mH);
            r.HH[i] = __ldg(phh + mH);
        }
    }
    r.hlL = r.hhL = 0.f;
    r.llR = r.hlR = r.lhR = r.hhR = 0.f;
    if (lane == 0) {
        const int mh = max(m0 - 1, 0);             // H[-1] := H[0]
        r.hlL = __ldg(phl + mh);
        r.hhL = __ldg(phh + mh);
    }
    if (lane == 31) {
        const int mr = m0 + IQ;
        const int mL = min(mr, Wq - 1), mH = min(mr, Wh - 1);
        r.llR = __ldg(pll + mL);
        r.lhR = __ldg(plh + mL);
        r.hlR = __ldg(phl + mH);
        r.hhR = __ldg(phh + mH);
    }
    return r;
}

// Reconstructed (undone update) values of one quad row.
struct Rec {
    double a[2], hlp[2], lhp[2], hh[2], lh[2];
    double aR, lhpR, hhR, lhR;           // right halo quad
    double hhL;                          // left halo quad (raw HH, carried for HL'[m-1])
};

__device__ __forceinline__ Rec undo_update(const Raw &r, const Rec &p, int lane)
{
    // p: the previous quad row (its raw HH / LH), for the n-1 neighbours
    Rec c;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        c.hh[i] = r.HH[i];
        c.lh[i] = r.LH[i];
        c.hlp[i] = fma(-0.25, c.hh[i] + p.hh[i], (double)r.HL[i]);
    }
    c.hhL = r.hhL;
    c.hhR = r.hhR;
    c.lhR = r.lhR;
    const double hlpL = fma(-0.25, c.hhL + p.hhL, (double)r.hlL);
    const double hlpR = fma(-0.25, c.hhR + p.hhR, (double)r.hlR);
    // m-1 neighbours of quad 0 (lane - 1's quad 1, or the halo quad)
    const double hlp_up = __shfl_up_sync(0xffffffffu, c.hlp[1], 1);
    const double hh_up = __shfl_up_sync(0xffffffffu, c.hh[1], 1);
    const double hlp_l = (lane == 0) ? hlpL : hlp_up;
    const double hh_l = (lane == 0) ? c.hhL : hh_up;
    c.lhp[0] = fma(-0.25, c.hh[0] + hh_l, (double)r.LH[0]);
    c.lhp[1] = fma(-0.25, c.hh[1] + c.hh[0], (double)r.LH[1]);
    c.lhpR = fma(-0.25, c.hhR + c.hh[1], (double)r.lhR);
    c.a[0] = fma(-0.25, c.lh[0] + p.lh[0], fma(-0.25, c.hlp[0] + hlp_l, (double)r.LL[0]));
    c.a[1] = fma(-0.25, c.lh[1] + p.lh[1], fma(-0.25, c.hlp[1] + c.hlp[0], (double)r.LL[1]));
    c.aR = fma(-0.25, c.lhR + p.lhR, fma(-0.25, hlpR + c.hlp[1], (double)r.llR));
    return c;
}

// Undo the predict of quad row n-1 (p) given row n (c; for the last row of
// an even-height image c == p, the mirror L[M] := L[M-1]) and store its two
// pixel rows (only the even one if has_odd_row is false).
template <bool VEC, bool EDGE>
__device__ __forceinline__ void undo_predict_store(const InvArgs &a, const Rec &p, const Rec &c, int img, int n,
                                                   int m0, int lane, bool has_odd_row)
{
    const int Wq = (a.W + 1) >> 1;
    const int m = m0 + 2 * lane;
    double cc[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) cc[i] = fma(0.5, p.a[i] + c.a[i], p.lhp[i]);
    const double ccR = fma(0.5, p.aR + c.aR, p.lhpR);
    const double a_dn = __shfl_down_sync(0xffffffffu, p.a[0], 1);
    const double c_dn = __shfl_down_sync(0xffffffffu, cc[0], 1);
    double ar[2] = {p.a[1], (lane == 31) ? p.aR : a_dn};
    double cr[2] = {cc[1], (lane == 31) ? ccR : c_dn};
    if (EDGE) {
        // even W: the right neighbour of the last quad column is itself (L[M] := L[M-1])
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (m + i == Wq - 1) {
                ar[i] = p.a[i];
                cr[i] = cc[i];
            }
    }
    float e[4], o[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        e[2 * i] = (float)p.a[i];
        e[2 * i + 1] = (float)fma(0.5, p.a[i] + ar[i], p.hlp[i]);
        o[2 * i] = (float)cc[i];
        o[2 * i + 1] = (float)fma(0.5, p.hlp[i] + c.hlp[i], fma(0.5, cc[i] + cr[i], p.hh[i]));
    }
    float *row0 = a.out + (long long)img * a.out_img + (long long)(2 * n) * a.out_pitch + 2 * m;
    float *row1 = row0 + a.out_pitch;
    const int x = 2 * m;
    if (!EDGE && VEC) {
        __stcs(reinterpret_cast<float4 *>(row0), make_float4(e[0], e[1], e[2], e[3]));
        if (has_odd_row) __stcs(reinterpret_cast<float4 *>(row1), make_float4(o[0], o[1], o[2], o[3]));
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (x + j < a.W) {
                __stcs(row0 + j, e[j]);
                if (has_odd_row) __stcs(row1 + j, o[j]);
            }
        }
    }
}

__device__ __forceinline__ void pdl_wait_inv() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_inv() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <bool VEC>
__global__ void __launch_bounds__(ITHREADS, 2) dwt53_inverse_level_kernel(const __grid_constant__ InvArgs a)
{
    pdl_launch_inv();
    pdl_wait_inv();
    const int lane = threadIdx.x & 31;
    const int Wq = (a.W + 1) >> 1, Hq = (a.H + 1) >> 1;
    for (long long t = dwt2_queue_fetch(a.counter, a.ntiles, a.nwarps, lane); t < a.ntiles;
         t = dwt2_queue_fetch(a.counter, a.ntiles, a.nwarps, lane)) {
        // tiles: image-major, then row block, then slab (adjacent slabs run together)
        const long long per_img = (long long)a.nblk * a.nslabs;
        const int img = fdiv(int(t), a.fd_img);
        const int r = int(t - (long long)img * per_img);
        const int blk = fdiv(r, a.fd_slabs);
        const int slab = r - blk * a.nslabs;
        const int m0 = slab * IQ;
        const int n0 = blk * a.tb, n1 = min(n0 + a.tb, Hq);
        const bool edge = (m0 == 0) || (m0 + IQ >= Wq);
        auto body = [&](auto edge_tag) {
            constexpr bool EG = decltype(edge_tag)::value;
            // the raw LH / HH of quad row n0-1 (mirrored at the top) seed the carry
            Rec prev;
            {
                const Raw r0 = load_raw<VEC, EG>(a, img, max(n0 - 1, 0), m0, lane);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    prev.hh[i] = r0.HH[i];
                    prev.lh[i] = r0.LH[i];
                }
                prev.hhL = r0.hhL;
                prev.hhR = r0.hhR;
                prev.lhR = r0.lhR;
            }
            Raw nxt = load_raw<VEC, EG>(a, img, n0, m0, lane);
            for (int n = n0; n < n1; ++n) {
                const Raw cur = nxt;
                if (n + 1 < Hq) nxt = load_raw<VEC, EG>(a, img, n + 1, m0, lane);   // prefetch
                const Rec rc = undo_update(cur, prev, lane);
                if (n > n0) undo_predict_store<VEC, EG>(a, prev, rc, img, n - 1, m0, lane, true);
                prev = rc;
            }
            // last quad row of the tile: needs row n1 (or the mirror at the bottom)
            if (n1 < Hq) {
                const Rec rc = undo_update(nxt, prev, lane);
                undo_predict_store<VEC, EG>(a, prev, rc, img, n1 - 1, m0, lane, true);
            } else {
                // even H: L[M] := L[M-1] (a, HL' of row Hq mirror row Hq-1);
                // odd H: the last quad row has no odd pixel row
                undo_predict_store<VEC, EG>(a, prev, prev, img, n1 - 1, m0, lane, (a.H & 1) == 0);
            }
        };
        if (edge) body(std::integral_constant<bool, true>());
        else body(std::integral_constant<bool, false>());
    }
}

// ---------------------------------------------------------------------------
// Ring variant (16-byte aligned planes and pitches): every warp streams its
// quad rows through a shared-memory ring by cp.async, IDS rows in flight, so
// the loads of later rows overlap the arithmetic of earlier ones.  A stage
// holds, per plane, the window of columns [m0 - 4, m0 + 68) (18 x 16 B).
// ---------------------------------------------------------------------------
constexpr int IRW = 4;                         // warps per CTA (ring kernel)
#ifndef DWT2_INV_MINB
#define DWT2_INV_MINB 4                        // resident CTAs per SM the register budget aims at
#endif
#ifndef DWT2_INV_DS
#define DWT2_INV_DS 4                          // measured with 4 CTAs per SM: 4 rows in flight > 3, 5 (> 6 at 3 CTAs)
#endif
constexpr int IDS = DWT2_INV_DS;               // quad rows in flight per warp
constexpr int IWIN = 72;                       // window floats per plane
constexpr int ISTAGE = 4 * IWIN;               // floats per stage
constexpr size_t IRING_SMEM = size_t(IRW) * IDS * ISTAGE * sizeof(float);

__device__ __forceinline__ void icp_async16(float *dst, const float *src, uint32_t nbytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void icp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void icp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Per-lane share of a stage: chunks c = lane, lane + 32, lane + 64 (< 72) of
// the 4 x 18 16-byte chunks; fixed for the whole kernel, so the plane
// selection is done once per tile (ChunkPlan) and a row costs one address
// update per chunk.
struct ChunkPlan {
    const float *src[3];        // chunk address at row 0 (image and column applied)
    int dst[3];                 // float offset in the stage
    int pl[3];                  // plane: 0 LL, 1 HL, 2 LH, 3 HH
};

__device__ __forceinline__ ChunkPlan chunk_plan(const InvArgs &a, int img, int m0, int lane)
{
    ChunkPlan P;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        const int c = min(lane + 32 * t, 71);
        const int pl = c / 18, k = c - pl * 18;
        const float *base = pl == 0 ? a.ll : pl == 1 ? a.hl : pl == 2 ? a.lh : a.hh;
        const long long img_off = (long long)img * (pl == 0 ? a.ll_img : a.d_img);
        P.src[t] = base + img_off + (m0 - 4 + 4 * k);
        P.dst[t] = pl * IWIN + 4 * k;
        P.pl[t] = pl;
    }
    return P;
}

// issue the 72 chunks of quad row n (4 planes x 18) into stage `st`.  Only
// edge slabs (first / last) can reach outside the buffers (columns left of
// plane 0 or past the last row's end): interior slabs skip the range check.
template <bool EDGE>
__device__ __forceinline__ void ring_issue(const InvArgs &a, const ChunkPlan &P, float *st, int n, int lane)
{
    const int nd = min(max(n, 0), (a.H >> 1) - 1);
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        if (t < 2 || lane < 8) {
            const float *src = P.src[t] + (long long)(P.pl[t] >= 2 ? nd : n) * (P.pl[t] == 0 ? a.ll_pitch : a.d_pitch);
            if (EDGE) {
                const float *lo = P.pl[t] == 0 ? a.ll_lo : a.d_lo, *hi = P.pl[t] == 0 ? a.ll_hi : a.d_hi;
                const uint32_t nb = (src >= lo && src + 4 <= hi) ? 16u : 0u;   // outside: zero fill
                icp_async16(st + P.dst[t], nb ? src : lo, nb);
            } else {
                icp_async16(st + P.dst[t], src, 16u);
            }
        }
    }
}

template <bool EDGE>
__device__ __forceinline__ Raw ring_read(const InvArgs &a, const float *st, int m0, int lane)
{
    const int Wq = (a.W + 1) >> 1, Wh = a.W >> 1;
    const int o = m0 - 4;                        // window column 0
    const int m = m0 + 2 * lane;
    Raw r;
    if (!EDGE) {
        const float2 ll = *reinterpret_cast<const float2 *>(st + 0 * IWIN + (m - o));
        const float2 hl = *reinterpret_cast<const float2 *>(st + 1 * IWIN + (m - o));
        const float2 lh = *reinterpret_cast<const float2 *>(st + 2 * IWIN + (m - o));
        const float2 hh = *reinterpret_cast<const float2 *>(st + 3 * IWIN + (m - o));
        r.LL[0] = ll.x; r.LL[1] = ll.y; r.HL[0] = hl.x; r.HL[1] = hl.y;
        r.LH[0] = lh.x; r.LH[1] = lh.y; r.HH[0] = hh.x; r.HH[1] = hh.y;
        r.hlL = st[1 * IWIN + (m0 - 1 - o)];
        r.hhL = st[3 * IWIN + (m0 - 1 - o)];
        r.llR = st[0 * IWIN + (m0 + IQ - o)];
        r.hlR = st[1 * IWIN + (m0 + IQ - o)];
        r.lhR = st[2 * IWIN + (m0 + IQ - o)];
        r.hhR = st[3 * IWIN + (m0 + IQ - o)];
    } else {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int mL = min(m + i, Wq - 1) - o, mH = min(max(m + i, 0), Wh - 1) - o;
            r.LL[i] = st[0 * IWIN + mL];
            r.LH[i] = st[2 * IWIN + mL];
            r.HL[i] = st[1 * IWIN + mH];
            r.HH[i] = st[3 * IWIN + mH];
        }
        const int mh = max(m0 - 1, 0) - o;
        r.hlL = st[1 * IWIN + mh];
        r.hhL = st[3 * IWIN + mh];
        const int mrL = min(m0 + IQ, Wq - 1) - o, mrH = min(m0 + IQ, Wh - 1) - o;
        r.llR = st[0 * IWIN + mrL];
        r.lhR = st[2 * IWIN + mrL];
        r.hlR = st[1 * IWIN + mrH];
        r.hhR = st[3 * IWIN + mrH];
    }
    return r;
}

template <bool EDGE>
__device__ __forceinline__ void ring_tile(const InvArgs &a, float *ring, int img, int m0, int n0, int n1, int lane)
{
    const int Hq = (a.H + 1) >> 1;
    const ChunkPlan P = chunk_plan(a, img, m0, lane);
    // load sequence: i = 0 -> row max(n0-1, 0) (seeds the n-1 carry), i >= 1 -> row n0 + i - 1
    const int T = 1 + (min(n1, Hq - 1) - n0 + 1);
    auto row_of = [&](int i) { return i == 0 ? max(n0 - 1, 0) : n0 + i - 1; };
#pragma unroll
    for (int j = 0; j < IDS; ++j) {
        if (j < T) ring_issue<EDGE>(a, P, ring + j * ISTAGE, row_of(j), lane);
        icp_commit();
    }
    Rec prev;
    for (int ib = 0; ib < T; ib += IDS) {
#pragma unroll
        for (int j = 0; j < IDS; ++j) {
            const int i = ib + j;
            if (i >= T) break;
            icp_wait<IDS - 1>();
            const Raw raw = ring_read<EDGE>(a, ring + j * ISTAGE, m0, lane);
            if (i == 0) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    prev.hh[q] = raw.HH[q];
                    prev.lh[q] = raw.LH[q];
                }
                prev.hhL = raw.hhL;
                prev.hhR = raw.hhR;
                prev.lhR = raw.lhR;
            } else {
                const int n = n0 + i - 1;
                const Rec rc = undo_update(raw, prev, lane);
                if (n > n0) undo_predict_store<true, EDGE>(a, prev, rc, img, n - 1, m0, lane, true);
                prev = rc;
            }
            // the stage's values are in registers (used above): refill it
            if (i + IDS < T) ring_issue<EDGE>(a, P, ring + j * ISTAGE, row_of(i + IDS), lane);
            icp_commit();
        }
    }
    icp_wait<0>();
    if (n1 == Hq) undo_predict_store<true, EDGE>(a, prev, prev, img, n1 - 1, m0, lane, (a.H & 1) == 0);
}

__global__ void __launch_bounds__(IRW * 32, DWT2_INV_MINB) dwt53_inverse_ring_kernel(const __grid_constant__ InvArgs a)
{
    extern __shared__ __align__(16) float iring_smem[];
    pdl_launch_inv();
    pdl_wait_inv();
    const int lane = threadIdx.x & 31;
    float *ring = iring_smem + (threadIdx.x >> 5) * (IDS * ISTAGE);
    const int Hq = (a.H + 1) >> 1;
    const long long per_img = (long long)a.nblk * a.nslabs;
    for (long long t = dwt2_queue_fetch(a.counter, a.ntiles, a.nwarps, lane); t < a.ntiles;
         t = dwt2_queue_fetch(a.counter, a.ntiles, a.nwarps, lane)) {
        const int img = fdiv(int(t), a.fd_img);
        const int r = int(t - (long long)img * per_img);
        const int blk = fdiv(r, a.fd_slabs);
        const int slab = r - blk * a.nslabs;
        const int m0 = slab * IQ;
        const int n0 = blk < a.nblk_a ? blk * a.tb : a.split + (blk - a.nblk_a) * a.tb_b;
        const int n1 = min(n0 + (blk < a.nblk_a ? a.tb : a.tb_b), blk < a.nblk_a ? min(a.split, Hq) : Hq);
        // interior: every plane's window [m0 - 4, m0 + 68) lies inside its row
        // (the narrowest planes, HL / HH, are Wh wide), so no clamping and no
        // range check of the cp.async sources
        if ((m0 == 0) || (m0 + IWIN - 4 > (a.W >> 1))) ring_tile<true>(a, ring, img, m0, n0, n1, lane);
        else ring_tile<false>(a, ring, img, m0, n0, n1, lane);
    }
}

int inverse_ring_ctas_per_sm()
{
    static int per_sm = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int n = 0;
        if (cudaFuncSetAttribute(dwt53_inverse_ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(IRING_SMEM)) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dwt53_inverse_ring_kernel, IRW * 32, IRING_SMEM) !=
                cudaSuccess || n < 1)
            n = 1;
        per_sm = n;
    });
    cudaGetLastError();
    return per_sm;
}

int inverse_ctas_per_sm()
{
    static int per_sm = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dwt53_inverse_level_kernel<true>, ITHREADS, 0) !=
                cudaSuccess || n < 1)
            n = 1;
        per_sm = n;
    });
    cudaGetLastError();
    return per_sm;
}

int32_t launch_inverse_level(const dwt2_plan *p, const InvArgs &base, cudaStream_t s)
{
    InvArgs a = base;
    const int Wq = (a.W + 1) / 2, Hq = (a.H + 1) / 2;
    a.nslabs = (Wq + IQ - 1) / IQ;
    // ring kernel: every plane row 16-byte aligned (cp.async chunks), float4 stores
    const bool ring = aligned(a.ll, 16) && aligned(a.hl, 16) && aligned(a.lh, 16) && aligned(a.hh, 16) &&
                      a.ll_pitch % 4 == 0 && a.d_pitch % 4 == 0 &&
                      (a.count == 1 || (a.ll_img % 4 == 0 && a.d_img % 4 == 0)) &&
                      aligned(a.out, 16) && a.out_pitch % 4 == 0 && (a.count == 1 || a.out_img % 4 == 0);
    if (ring) {
        const long long rwarps = (long long)p->sms * inverse_ring_ctas_per_sm() * IRW;
        const long long slab_rows = (long long)a.count * a.nslabs * Hq;
        // tiles per warp for the queue: 16 on large levels (balance), 4 on
        // mid-size ones (the seed row of a tile costs more there); measured,
        // scripts/sweeps/gpu_queue_tpw.sh
        static const int env_tpw = tuning_int("DWT2_INV_TPW", 0, 1, 1024);
        const int tpw = env_tpw > 0 ? env_tpw : (slab_rows >= 256 * rwarps ? 16 : 4);
        long long tb = slab_rows / (tpw * rwarps);
        tb = std::max<long long>(8, std::min<long long>(256, tb));
        // small levels (fewer than one 8-row tile per resident warp): one
        // short tile per warp, so every warp takes part
        static const int small_inv = tuning_int("DWT2_INV_SMALL", 1, 0, 1);
        if (small_inv && slab_rows < 8 * rwarps) tb = std::max<long long>(2, (slab_rows + rwarps - 1) / rwarps);
        // levels with >= 64 quad rows per warp: 20-row tiles (measured over
        // 8192^2 .. 16384^2 against 8, 12, 16, 24, 27..55-row tiles and the
        // guided split: 16384 x 8192 0.80 -> 0.88, 16384^2 0.89 -> 0.91,
        // 8192^2 0.81 -> 0.83 of copy); guided tiles below 64 rows per warp
        static const int env_tb = tuning_int("DWT2_INV_TB", 20, 0, 256);
        if (env_tpw <= 0 && env_tb > 0 && slab_rows >= 64 * rwarps) tb = env_tb;
        a.tb = int(tb);
        a.nblk = int((Hq + tb - 1) / tb);
        a.nblk_a = a.nblk;
        a.split = Hq;
        a.tb_b = a.tb;
        // guided tiles on mid-size levels (few tiles per warp): one large tile
        // per warp over ~70 % of the rows, then ~4 small tiles per warp (as
        // the forward kernel, dwt2.cu)
        static const int guided = tuning_int("DWT2_INV_GUIDED", 1, 0, 1);
        if (guided && a.count == 1 && slab_rows < 64 * rwarps && slab_rows >= 8 * rwarps) {
            const long long nba = std::max<long long>(1, rwarps / a.nslabs);
            static const int pct = tuning_int("DWT2_INV_GUIDED_A", 70, 10, 90);
            const long long tba = (pct * Hq / 100) / nba;
            if (tba >= 16) {
                a.tb = int(tba);
                a.nblk_a = int(nba);
                a.split = int(nba * tba);
                const long long rest = Hq - a.split;
                long long tbb = rest * a.nslabs / (4 * rwarps);
                tbb = std::max<long long>(8, std::min<long long>(256, tbb));
                a.tb_b = int(tbb);
                a.nblk = a.nblk_a + int((rest + tbb - 1) / tbb);
            }
        }
        a.ntiles = (long long)a.count * a.nblk * a.nslabs;
    a.fd_img = make_fastdiv(unsigned(a.nblk * a.nslabs));
    a.fd_slabs = make_fastdiv(unsigned(a.nslabs));
    if (a.ntiles >= (1LL << 31)) return fail(DWT2_EINVAL);
        const long long want = (a.ntiles + IRW - 1) / IRW;
        const int grid = int(std::max<long long>(1, std::min<long long>(want, rwarps / IRW)));
        a.nwarps = grid * IRW;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(IRW * 32);
        cfg.dynamicSmemBytes = IRING_SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, dwt53_inverse_ring_kernel, a) != cudaSuccess) {
            cudaGetLastError();
            return fail(DWT2_ECUDA);
        }
        return DWT2_OK;
    }
    const long long warps = (long long)p->sms * inverse_ctas_per_sm() * IWARPS;
    // tile height: ~8 tiles per resident warp, at least 8 quad rows (the
    // halo row re-read costs 1 / tb), at most 256
    long long slab_rows = (long long)a.count * a.nslabs * Hq;
    static const int ldg_tpw = tuning_int("DWT2_INV_LDG_TPW", 8, 1, 1024);
    long long tb = slab_rows / (ldg_tpw * warps);
    tb = std::max<long long>(8, std::min<long long>(256, tb));
    a.tb = int(tb);
    a.nblk = int((Hq + tb - 1) / tb);
    a.nblk_a = a.nblk;
    a.split = Hq;
    a.tb_b = a.tb;
    a.ntiles = (long long)a.count * a.nblk * a.nslabs;
    a.fd_img = make_fastdiv(unsigned(a.nblk * a.nslabs));
    a.fd_slabs = make_fastdiv(unsigned(a.nslabs));
    if (a.ntiles >= (1LL << 31)) return fail(DWT2_EINVAL);
    const long long want = (a.ntiles + IWARPS - 1) / IWARPS;
    const int grid = int(std::max<long long>(1, std::min<long long>(want, warps / IWARPS)));
    a.nwarps = grid * IWARPS;
    const bool vec = aligned(a.ll, 8) && aligned(a.hl, 8) && aligned(a.lh, 8) && aligned(a.hh, 8) &&
                     a.ll_pitch % 2 == 0 && a.d_pitch % 2 == 0 && (a.count == 1 || (a.ll_img % 2 == 0 && a.d_img % 2 == 0)) &&
                     aligned(a.out, 16) && a.out_pitch % 4 == 0 && (a.count == 1 || a.out_img % 4 == 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(ITHREADS);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = vec ? cudaLaunchKernelEx(&cfg, dwt53_inverse_level_kernel<true>, a)
                        : cudaLaunchKernelEx(&cfg, dwt53_inverse_level_kernel<false>, a);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

// Inverse of all levels: coarsest first.  Level k (0-based) reconstructs its
// input (geom[k]) from its LL (the coarsest level: `in` top-left; otherwise the
// output of level k+1) and its HL / LH / HH in the Mallat buffer `in`.
int32_t run_inverse(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                    long long out_stride, cudaStream_t s)
{
    for (int k = p->levels - 1; k >= 0; --k) {
        const LevelGeom &g = p->geom[k];
        InvArgs a;
        memset(&a, 0, sizeof(a));
        a.W = g.W;
        a.H = g.H;
        a.count = count;
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
            const int sidx = k % 2;                 // output of level k+1
            a.ll = p->scratch[sidx];
            a.ll_pitch = p->sc_pitch[sidx];
            a.ll_img = p->sc_img_stride[sidx];
        }
        if (k == 0) {
            a.out = out;
            a.out_pitch = p->W;
            a.out_img = out_stride;
        } else {
            const int sidx = (k - 1) % 2;
            a.out = p->scratch[sidx];
            a.out_pitch = p->sc_pitch[sidx];
            a.out_img = p->sc_img_stride[sidx];
        }
        a.d_lo = in;
        a.d_hi = in + (long long)(count - 1) * in_stride + (long long)p->W * p->H;
        if (k == p->levels - 1) {
            a.ll_lo = a.d_lo;
            a.ll_hi = a.d_hi;
        } else {
            const int sidx = k % 2;
            a.ll_lo = p->scratch[sidx];
            a.ll_hi = p->scratch[sidx] + (long long)count * p->sc_img_stride[sidx];
        }
        a.counter = p->counters + 2 * (QUEUE_INVERSE + k);
        if (small_inverse_level(p, k, count)) {
            // a small level: shared-memory-staged pointwise synthesis (tail.cu)
            static const InvFilter f53 = inv_filter_from_lifting(-0.5, 0.25, 0.0, 0.0, 1.0);
            const InvLevelIO lv{a.ll, a.ll_pitch, a.ll_img, in, p->W, in_stride, a.out, a.out_pitch, a.out_img,
                                g.W, g.H};
            int32_t r = launch_small_inverse_level(lv, count, f53, s);
            if (r != DWT2_OK) return r;
            continue;
        }
        int32_t r = launch_inverse_level(p, a, s);
        if (r != DWT2_OK) return r;
    }
    return DWT2_OK;
}

}  // namespace

extern "C" {

int32_t dwt2_inverse(const dwt2_plan *p, const float *in, float *out, dwt2_stream_t stream)
{
    if (!p || !in || !out || p->strip || !aligned(in, 4) || !aligned(out, 4)) return fail(DWT2_EINVAL);
    const size_t bytes = size_t(p->W) * p->H * sizeof(float);
    if (overlap(in, bytes, out, bytes) || !on_plan_device(p, in) || !on_plan_device(p, out))
        return fail(DWT2_EINVAL);
    const long long img = (long long)p->W * p->H;
    int32_t r = p->wavelet != DWT2_WAVELET_CDF53
                    ? run_inverse_k2(p, in, out, 1, img, img, reinterpret_cast<cudaStream_t>(stream))
                    : run_inverse(p, in, out, 1, img, img, reinterpret_cast<cudaStream_t>(stream));
    if (r != DWT2_OK) return r;
    g_last_error = DWT2_OK;
    return DWT2_OK;
}

int32_t dwt2_inverse_batched(const dwt2_plan *p, const float *in, float *out, int32_t count, int64_t in_stride,
                             int64_t out_stride, dwt2_stream_t stream)
{
    const long long img = (long long)(p ? p->W : 0) * (p ? p->H : 0);
    if (!p || !in || !out || p->strip || count < 1 || count > p->max_count || in_stride < img ||
        out_stride < img || !aligned(in, 4) || !aligned(out, 4))
        return fail(DWT2_EINVAL);
    const size_t in_bytes = size_t((count - 1) * in_stride + img) * sizeof(float);
    const size_t out_bytes = size_t((count - 1) * out_stride + img) * sizeof(float);
    if (overlap(in, in_bytes, out, out_bytes) || !on_plan_device(p, in) || !on_plan_device(p, out))
        return fail(DWT2_EINVAL);
    int32_t r = p->wavelet != DWT2_WAVELET_CDF53
                    ? run_inverse_k2(p, in, out, count, in_stride, out_stride, reinterpret_cast<cudaStream_t>(stream))
                    : run_inverse(p, in, out, count, in_stride, out_stride, reinterpret_cast<cudaStream_t>(stream));
    if (r != DWT2_OK) return r;
    g_last_error = DWT2_OK;
    return DWT2_OK;
}

}  // extern "C"
