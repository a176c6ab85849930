// dwt2.cu -- B200 (sm_100a) forward 2-D CDF 5/3 DWT with the non-separable
// lifting scheme of arXiv:1708.07853 (section 3, Eq. (5)).
//
// One fused kernel per decomposition level.  The paper's two spatial steps
// (predict, then update) and its single in-level synchronisation point `|`
// map onto one pass over HBM:
//
//   HBM --TMA--> per-warp smem ring (136-column slab + halo, R rows/stage)
//       --LDS.128--> registers: spatial predict (Eq. (5) right factor)
//       --warp shuffle (m-1 neighbour) + register carry (n-1 neighbour)-->
//       spatial update (Eq. (5) left factor) --> 4 subband stores (STG.64)
//
// so the `|` between predict and update costs a shuffle instead of a grid-wide
// barrier, and every level moves the algorithmic floor of 4 B read + 4 B
// written per pixel.  See DESIGN.md sections 5-6 for the layout and roofline.
//
// Work decomposition.  A warp owns a 128-pixel column slab (64 quads, 2 per
// lane) and walks DOWN it, row pair by row pair, carrying the predicted
// values of the previous quad row in registers.  A CTA is WARPS adjacent
// slabs (a 512-pixel "group") over the same quad rows, so the 8 halo columns
// its warps share are re-read from L2 at the same time.  The grid is
// persistent: the (image x group x quad-row) space is cut into one
// contiguous, balanced range per CTA, so every CTA finishes together and
// vertical halos (2 rows above, 1 below) are paid once per range.
//
// Arithmetic: fp32 in HBM, fp64 in registers.  Every CDF 5/3 coefficient is
// dyadic, so fp64 evaluation of fp32 inputs is exact in practice and the
// stored fp32 result is the correctly rounded exact value whatever the
// evaluation order (DESIGN.md section 5 / reading C-A13).
//
// Boundaries: whole-sample symmetric extension, applied in
// registers: mirrored raw samples on the right edge of even widths and on
// the bottom edge of even heights, mirrored predicted values (H[-1] = H[0],
// H[M] = H[M-1]) on the top/left edges and on odd right/bottom edges.

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>

#include "../../include/dwt2.h"

namespace {

// ---------------------------------------------------------------------------
// Tile geometry
// ---------------------------------------------------------------------------
constexpr int SLAB = 128;          // output pixel columns per warp (64 quads, 2 per lane)
constexpr int BOXW = 136;          // smem row: pixel columns [x0 - 4, x0 + 132)
constexpr int R = 16;              // rows per pipeline stage (one TMA box = BOXW x R)
constexpr int S = 3;               // stages per warp ring
constexpr int WARPS = 4;           // warps (adjacent slabs) per CTA
constexpr int THREADS = WARPS * 32;
constexpr int GROUP = WARPS * SLAB;                      // pixel columns per CTA
constexpr int STAGE_FLOATS = R * BOXW;                   // 2176 floats = 8704 B
constexpr int RING_FLOATS = S * STAGE_FLOATS;
constexpr size_t SMEM_BYTES = size_t(WARPS) * RING_FLOATS * sizeof(float) + size_t(WARPS) * S * 8;
constexpr int MIN_ROWS_PER_CTA = 8;                      // quad rows; below this, use fewer CTAs

static_assert((BOXW * 4) % 16 == 0, "TMA box inner extent must be a multiple of 16 bytes");
static_assert(BOXW >= SLAB + 5, "smem row must hold 2 halo columns left and 1 right");

// ---------------------------------------------------------------------------
// Kernel arguments (passed as a __grid_constant__ parameter; the TMA
// descriptor must be 64-byte aligned and live in param/const space)
// ---------------------------------------------------------------------------
struct alignas(64) LevelArgs {
    CUtensorMap tmap;                 // 3-D {W, in_rows, count}, box {BOXW, R, 1}
    const float *in;                  // generic loader: image 0, buffer row 0
    const float *in_end;              // one past the last element of the call's input
    long long in_pitch, in_img_stride;
    float *ll, *hl, *lh, *hh;         // subband bases for image 0, output row 0
    long long ll_pitch, ll_img_stride;
    long long out_pitch, out_img_stride;
    int W, H;                         // level input width, (global) height
    int in_row0, in_rows;             // global row of buffer row 0; rows present in the buffer
    int out_q0;                       // global quad row stored at output row 0
    int ngroups, count;
    int qa0, qa1, qb0, qb1;           // quad-row ranges [qa0, qa1) and [qb0, qb1)
    long long units;                  // count * ngroups * nq
};

// ---------------------------------------------------------------------------
// PTX helpers (mbarrier, TMA, cp.async, PDL)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int imin(int x, int y) { return x < y ? x : y; }
__host__ __device__ __forceinline__ long long imin64(long long x, long long y) { return x < y ? x : y; }

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ void tma_load_3d(float *dst, const CUtensorMap *map, int x, int y, int z,
                                            uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z),
          "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void cp_async_16(float *dst, const void *src, uint32_t src_bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes) : "memory");
}

__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void pdl_wait()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void pdl_launch_dependents()
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
// One smem row as seen by one lane, widened to fp64.
//   v0..v3: the lane's 4 pixels (quad columns mq0, mq0+1: a/b or c/d pairs)
//   l0, l1: the two pixels left of the slab (lane 0's halo quad)
//   r:      the pixel right of the lane (lane + 1's v0; lane 31 reads smem)
// ---------------------------------------------------------------------------
struct RowD {
    double v0, v1, v2, v3, l0, l1, r;
};

struct EdgeFlags {
    bool r_from_v2;    // even W, q1 is the last quad: x[W] := x[W-2]
    bool v2_from_v0;   // even W, q0 is the last quad: x[W] := x[W-2]
    bool odd_q0_last;  // odd W, q0 is the last quad (only a, c exist)
    bool odd_q1_last;  // odd W, q1 is the last quad
    bool left_edge;    // lane 0 of the slab at x = 0: H[-1] := H[0]
};

template <bool TMA>
__device__ __forceinline__ RowD load_row(const float *p, int lane, const EdgeFlags &ef)
{
    float f0, f1, f2, f3;
    if (TMA) {
        const float4 q = *reinterpret_cast<const float4 *>(p + 4 + 4 * lane);
        f0 = q.x; f1 = q.y; f2 = q.z; f3 = q.w;
    } else {
        f0 = p[4 + 4 * lane]; f1 = p[5 + 4 * lane]; f2 = p[6 + 4 * lane]; f3 = p[7 + 4 * lane];
    }
    const float fl0 = p[2], fl1 = p[3];                 // broadcast reads
    const float fr31 = p[4 + SLAB];                     // broadcast read
    const float fr = __shfl_down_sync(0xffffffffu, f0, 1);
    RowD d;
    d.v0 = f0; d.v1 = f1; d.v2 = f2; d.v3 = f3;
    d.l0 = fl0; d.l1 = fl1;
    d.r = (lane == 31) ? fr31 : fr;
    if (ef.r_from_v2) d.r = d.v2;
    if (ef.v2_from_v0) d.v2 = d.v0;
    return d;
}

// Spatial predict of Eq. (5) for one quad (a b / c d) with right (r), lower
// (dn) and lower-right (rdn) neighbours:
//   HL' = b + P a            = b - 1/2 (a + a[m+1])
//   LH' = c + P* a           = c - 1/2 (a + a[n+1])
//   HH' = d + P* b + P c + PP* a
//       = d - 1/2 (b + b[n+1]) - 1/2 (c + c[m+1]) + 1/4 (a + a[m+1] + a[n+1] + a[m+1,n+1])
struct Pred1 {
    double bp, cp, dp;
};

__device__ __forceinline__ Pred1 predict_quad(double a, double b, double c, double d, double ar, double cr,
                                              double adn, double bdn, double ardn)
{
    Pred1 p;
    const double sa = a + ar;
    p.bp = fma(-0.5, sa, b);
    p.cp = fma(-0.5, a + adn, c);
    double t = fma(-0.5, b + bdn, d);
    t = fma(-0.5, c + cr, t);
    p.dp = fma(0.25, sa + (adn + ardn), t);
    return p;
}

// Predicted values of the lane's two quads of quad row n plus the left
// neighbour's (m-1) HL' and HH' -- everything the update of row n reads
// from row n itself.
struct PredRow {
    double bp0, cp0, dp0, bp1, cp1, dp1, bl, dl;
};

__device__ __forceinline__ PredRow predict_row(const RowD &E, const RowD &O, const RowD &N, int lane,
                                               const EdgeFlags &ef)
{
    PredRow p;
    const Pred1 q0 = predict_quad(E.v0, E.v1, O.v0, O.v1, E.v2, O.v2, N.v0, N.v1, N.v2);
    const Pred1 q1 = predict_quad(E.v2, E.v3, O.v2, O.v3, E.r, O.r, N.v2, N.v3, N.r);
    p.bp0 = q0.bp; p.cp0 = q0.cp; p.dp0 = q0.dp;
    p.bp1 = q1.bp; p.cp1 = q1.cp; p.dp1 = q1.dp;
    // the single in-level synchronisation of Eq. (5): m-1 neighbours by shuffle
    double bl = __shfl_up_sync(0xffffffffu, q1.bp, 1);
    double dl = __shfl_up_sync(0xffffffffu, q1.dp, 1);
    if (lane == 0) {
        if (ef.left_edge) {            // H[-1] := H[0]
            bl = q0.bp;
            dl = q0.dp;
        } else {                       // recompute quad m0-1 from the smem halo
            const Pred1 h = predict_quad(E.l0, E.l1, O.l0, O.l1, E.v0, O.v0, N.l0, N.l1, N.v0);
            bl = h.bp;
            dl = h.dp;
        }
    }
    if (ef.odd_q0_last) {              // H[M] := H[M-1] for the last (L-only) column
        p.bp0 = bl;
        p.dp0 = dl;
    }
    if (ef.odd_q1_last) {
        p.bp1 = p.bp0;
        p.dp1 = p.dp0;
    }
    p.bl = bl;
    p.dl = dl;
    return p;
}

// Carried state of quad row n-1 (per lane quad): LH', HH' and the horizontal
// pair sum HH'(m) + HH'(m-1).
struct Carry {
    double cu0, du0, su0, cu1, du1, su1;
};

__device__ __forceinline__ void store2(float *p, float x, float y, bool v0, bool v1, bool vec, bool stream)
{
    if (v1) {
        if (vec) {
            if (stream) __stcs(reinterpret_cast<float2 *>(p), make_float2(x, y));
            else *reinterpret_cast<float2 *>(p) = make_float2(x, y);
        } else {
            if (stream) { __stcs(p, x); __stcs(p + 1, y); }
            else { p[0] = x; p[1] = y; }
        }
    } else if (v0) {
        if (stream) __stcs(p, x);
        else p[0] = x;
    }
}

// ---------------------------------------------------------------------------
// The fused level kernel
// ---------------------------------------------------------------------------
template <bool TMA, bool VEC>
__global__ void __launch_bounds__(THREADS)
dwt53_level_kernel(const __grid_constant__ LevelArgs a)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    float *ring = reinterpret_cast<float *>(smem_raw) + size_t(warp) * RING_FLOATS;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + size_t(WARPS) * RING_FLOATS * sizeof(float)) + warp * S;

    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], TMA ? 1u : 32u);
        fence_mbar_init();
    }
    __syncwarp();
    if (TMA && lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tmap)) : "memory");

    // Programmatic dependent launch: the next level may be scheduled now; it
    // waits (griddepcontrol.wait) for this grid's completion before touching
    // memory, exactly as this grid waits for its predecessor here.
    pdl_launch_dependents();
    pdl_wait();

    const int Wq = (a.W + 1) >> 1;          // L columns / LL width
    const int Wh = a.W >> 1;                // H columns
    const int Hh = a.H >> 1;
    const int lenA = a.qa1 - a.qa0;
    const int nq = lenA + (a.qb1 - a.qb0);
    const long long per_img = (long long)a.ngroups * nq;

    const long long u_begin = (a.units * blockIdx.x) / gridDim.x;
    const long long u_end = (a.units * (blockIdx.x + 1)) / gridDim.x;

    uint32_t stage_ctr = 0;                 // per-warp ring position (monotonic)

    for (long long u = u_begin; u < u_end;) {
        // ---- decode the segment: maximal run of units with equal (img, group, range)
        const int img = int(u / per_img);
        const long long rem = u - (long long)img * per_img;
        const int group = int(rem / nq);
        const int qi = int(rem - (long long)group * nq);
        const bool inA = qi < lenA;
        const int run_left = inA ? lenA - qi : nq - qi;
        const int seg_len = int(imin64(run_left, u_end - u));
        const int qa = inA ? a.qa0 + qi : a.qb0 + (qi - lenA);
        const int qb = qa + seg_len;
        u += seg_len;

        const int x0 = (group * WARPS + warp) * SLAB;
        if (x0 >= a.W) continue;            // warp-uniform: no pixels in this slab

        // ---- per-lane constants
        const int mq0 = (x0 >> 1) + 2 * lane;
        EdgeFlags ef;
        const bool evenW = (a.W & 1) == 0;
        ef.r_from_v2 = evenW && (mq0 + 1 == Wq - 1);
        ef.v2_from_v0 = evenW && (mq0 == Wq - 1);
        ef.odd_q0_last = !evenW && (mq0 == Wq - 1);
        ef.odd_q1_last = !evenW && (mq0 + 1 == Wq - 1);
        ef.left_edge = (x0 == 0) && (lane == 0);
        const bool L0 = mq0 < Wq, L1 = mq0 + 1 < Wq;
        const bool H0 = mq0 < Wh, H1 = mq0 + 1 < Wh;

        // ---- row stream: global rows [r_first, r_last]
        const bool top = (qa == 0);
        const int r_first = top ? 0 : 2 * qa - 2;
        const int r_last = imin(2 * qb, a.H - 1);
        const int nst = (r_last - r_first + R) / R;
        const uint32_t base = stage_ctr;
        stage_ctr += nst;

        const float *img_in = a.in + (long long)img * a.in_img_stride;

        auto issue = [&](int j) {
            const uint32_t k = base + j;
            const int slot = int(k % S);
            float *dst = ring + slot * STAGE_FLOATS;
            const int r0 = r_first + j * R;
            if (TMA) {
                if (lane == 0) {
                    fence_proxy_async();
                    mbar_arrive_expect_tx(&bars[slot], uint32_t(STAGE_FLOATS * sizeof(float)));
                    tma_load_3d(dst, &a.tmap, x0 - 4, r0 - a.in_row0, img, &bars[slot]);
                }
            } else {
                // 34 aligned 16-byte chunks per row cover [x0-4-delta, x0+132-delta)
                for (int idx = lane; idx < R * (BOXW / 4); idx += 32) {
                    const int rr = idx / (BOXW / 4);
                    const int c = idx - rr * (BOXW / 4);
                    const int br = r0 + rr - a.in_row0;
                    uint32_t nbytes = 0;     // 0: zero-fill, no global access
                    const char *src = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(a.in) & ~uintptr_t(15));
                    if (br >= 0 && br < a.in_rows) {
                        const float *rowp = img_in + (long long)br * a.in_pitch + (x0 - 4);
                        const uintptr_t al = reinterpret_cast<uintptr_t>(rowp) & ~uintptr_t(15);
                        const uintptr_t ch = al + uintptr_t(16) * c;
                        const uintptr_t lo = reinterpret_cast<uintptr_t>(a.in);
                        const uintptr_t hi = reinterpret_cast<uintptr_t>(a.in_end);
                        if (ch < hi && ch + 16 > lo) {
                            nbytes = uint32_t((hi - ch) < 16 ? (hi - ch) : 16);
                            src = reinterpret_cast<const char *>(ch);
                        }
                    }
                    cp_async_16(dst + rr * BOXW + 4 * c, src, nbytes);
                }
                cp_async_mbar_arrive(&bars[slot]);
            }
        };

        __syncwarp();                        // previous segment's reads of the ring are done
        for (int j = 0; j < imin(nst, S); ++j) issue(j);

        int waited = -1, released = 0;
        auto row_ptr = [&](int r) -> const float * {
            const int j = (r - r_first) / R;
            if (j > waited) {
                const uint32_t k = base + j;
                mbar_wait(&bars[k % S], (k / S) & 1u);
                waited = j;
            }
            const float *p = ring + int((base + j) % S) * STAGE_FLOATS + ((r - r_first) - j * R) * BOXW;
            if (!TMA) {
                const int br = r - a.in_row0;
                if (br >= 0 && br < a.in_rows) {
                    const float *rowp = img_in + (long long)br * a.in_pitch + (x0 - 4);
                    p += int((reinterpret_cast<uintptr_t>(rowp) >> 2) & 3);
                }
            }
            return p;
        };
        auto release_through = [&](int r) {  // every stage whose rows are all <= r is consumed
            const int done = (r - r_first + 1) / R;
            while (released < done) {
                if (released + S < nst) {
                    __syncwarp();
                    issue(released + S);
                }
                ++released;
            }
        };

        RowD E = load_row<TMA>(row_ptr(r_first), lane, ef);
        RowD O, N;
        Carry cy;
        int n0 = qa;
        if (!top) {
            // carry-in: predicted values of quad row qa-1 (rows 2qa-2 .. 2qa)
            O = load_row<TMA>(row_ptr(2 * qa - 1), lane, ef);
            N = load_row<TMA>(row_ptr(2 * qa), lane, ef);
            release_through(2 * qa);
            const PredRow p = predict_row(E, O, N, lane, ef);
            cy.cu0 = p.cp0; cy.du0 = p.dp0; cy.su0 = p.dp0 + p.dl;
            cy.cu1 = p.cp1; cy.du1 = p.dp1; cy.su1 = p.dp1 + p.dp0;
            E = N;
        }

        const long long oimg = (long long)img * a.out_img_stride;
        const long long limg = (long long)img * a.ll_img_stride;

        for (int n = n0; n < qb; ++n) {
            const bool has_odd = (2 * n + 1) <= a.H - 1;
            const bool has_next = (2 * n + 2) <= a.H - 1;
            PredRow p;
            double s0, s1;                   // HH'(m) + HH'(m-1) per lane quad
            if (has_odd) {
                O = load_row<TMA>(row_ptr(2 * n + 1), lane, ef);
                if (has_next) N = load_row<TMA>(row_ptr(2 * n + 2), lane, ef);
                else N = E;                  // even H: x[H] := x[H-2]
                release_through(has_next ? 2 * n + 2 : 2 * n + 1);
                p = predict_row(E, O, N, lane, ef);
                s0 = p.dp0 + p.dl;
                s1 = p.dp1 + p.dp0;
            } else {
                // odd H, last quad row: only row 2n exists.  HL' needs no
                // vertical neighbour; LH', HH' (and their m-1 sums) := their
                // values at n-1 (H[M] := H[M-1]).
                release_through(2 * n);
                p = predict_row(E, E, E, lane, ef);
                p.cp0 = cy.cu0; p.dp0 = cy.du0;
                p.cp1 = cy.cu1; p.dp1 = cy.du1;
                s0 = cy.su0;
                s1 = cy.su1;
            }
            if (n == 0) {                    // top edge: row -1 mirrors row 0
                cy.cu0 = p.cp0; cy.du0 = p.dp0; cy.su0 = s0;
                cy.cu1 = p.cp1; cy.du1 = p.dp1; cy.su1 = s1;
            }
            // spatial update (Eq. (5) left factor)
            //   LL = a + U HL' + U* LH' + UU* HH'
            //   HL = HL' + U* HH';  LH = LH' + U HH';  HH = HH'
            const double A0 = E.v0 + 0.25 * (p.bp0 + p.bl) + 0.25 * (p.cp0 + cy.cu0) + 0.0625 * (s0 + cy.su0);
            const double A1 = E.v2 + 0.25 * (p.bp1 + p.bp0) + 0.25 * (p.cp1 + cy.cu1) + 0.0625 * (s1 + cy.su1);
            const double B0 = fma(0.25, p.dp0 + cy.du0, p.bp0);
            const double B1 = fma(0.25, p.dp1 + cy.du1, p.bp1);
            const double C0 = fma(0.25, s0, p.cp0);
            const double C1 = fma(0.25, s1, p.cp1);

            const int orow = n - a.out_q0;
            float *pll = a.ll + limg + (long long)orow * a.ll_pitch + mq0;
            float *phl = a.hl + oimg + (long long)orow * a.out_pitch + mq0;
            store2(pll, __double2float_rn(A0), __double2float_rn(A1), L0, L1, VEC, false);
            store2(phl, __double2float_rn(B0), __double2float_rn(B1), H0, H1, VEC, true);
            if (n < Hh) {
                float *plh = a.lh + oimg + (long long)orow * a.out_pitch + mq0;
                float *phh = a.hh + oimg + (long long)orow * a.out_pitch + mq0;
                store2(plh, __double2float_rn(C0), __double2float_rn(C1), L0, L1, VEC, true);
                store2(phh, __double2float_rn(p.dp0), __double2float_rn(p.dp1), H0, H1, VEC, true);
            }

            cy.cu0 = p.cp0; cy.du0 = p.dp0; cy.su0 = s0;
            cy.cu1 = p.cp1; cy.du1 = p.dp1; cy.su1 = s1;
            E = N;
        }
        release_through(r_last);             // (all stages are waited for by now)
    }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
thread_local int32_t g_last_error = DWT2_OK;

int32_t fail(int32_t code)
{
    g_last_error = code;
    return code;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

struct LevelGeom {
    int W, H;            // level input size
    int Wq, Hq;          // LL size
};

typedef void (*KernelFn)(LevelArgs);

KernelFn kernel_for(bool tma, bool vec)
{
    if (tma) return vec ? dwt53_level_kernel<true, true> : dwt53_level_kernel<true, false>;
    return vec ? dwt53_level_kernel<false, true> : dwt53_level_kernel<false, false>;
}

bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }

}  // namespace

struct dwt2_plan {
    int W, H, levels, max_count;
    int device;
    // strip plans
    bool strip;
    int Hg, row_begin, row_end, ghost_top, ghost_bot;
    // geometry and scratch
    LevelGeom geom[32];
    float *scratch[2];
    long long sc_pitch[2], sc_img_stride[2];
    size_t scratch_bytes;
    int max_ctas;
    // host e2e staging
    mutable float *d_in, *d_out;
    mutable cudaStream_t s_h2d, s_d2h;
    mutable cudaEvent_t ev[64];
};

namespace {

struct LaunchIO {
    const float *in;
    long long in_pitch, in_img_stride;
    int in_row0, in_rows;
    const float *in_end;
    float *ll;
    long long ll_pitch, ll_img_stride;
    float *out;               // Mallat base of this level (subbands at offsets)
    long long out_pitch, out_img_stride;
    int out_q0, hq_local;     // strip-local quad row 0, LL rows present in out (LH offset)
    int count;
};

int32_t launch_level(const dwt2_plan *p, int W, int H, const LaunchIO &io, int qa0, int qa1, int qb0, int qb1,
                     cudaStream_t stream)
{
    LevelArgs a;
    memset(&a, 0, sizeof(a));
    const int Wq = (W + 1) / 2;
    a.in = io.in;
    a.in_end = io.in_end;
    a.in_pitch = io.in_pitch;
    a.in_img_stride = io.in_img_stride;
    a.ll = io.ll;
    a.ll_pitch = io.ll_pitch;
    a.ll_img_stride = io.ll_img_stride;
    a.hl = io.out + Wq;
    a.lh = io.out + (long long)io.hq_local * io.out_pitch;
    a.hh = a.lh + Wq;
    a.out_pitch = io.out_pitch;
    a.out_img_stride = io.out_img_stride;
    a.W = W;
    a.H = H;
    a.in_row0 = io.in_row0;
    a.in_rows = io.in_rows;
    a.out_q0 = io.out_q0;
    a.ngroups = (W + GROUP - 1) / GROUP;
    a.count = io.count;
    a.qa0 = qa0; a.qa1 = qa1; a.qb0 = qb0; a.qb1 = qb1;
    const int nq = (qa1 - qa0) + (qb1 - qb0);
    a.units = (long long)io.count * a.ngroups * nq;
    if (a.units == 0) return DWT2_OK;

    const bool tma = aligned(io.in, 16) && (io.in_pitch * 4) % 16 == 0 &&
                     (io.count == 1 || (io.in_img_stride * 4) % 16 == 0);
    const bool vec = aligned(a.ll, 8) && aligned(a.hl, 8) && aligned(a.lh, 8) && aligned(a.hh, 8) &&
                     io.ll_pitch % 2 == 0 && io.out_pitch % 2 == 0 &&
                     (io.count == 1 || (io.ll_img_stride % 2 == 0 && io.out_img_stride % 2 == 0));
    if (tma) {
        PFN_cuTensorMapEncodeTiled_v12000 enc = get_encode();
        if (!enc) return fail(DWT2_ECUDA);
        cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)io.in_rows, (cuuint64_t)io.count};
        long long img_bytes = io.count > 1 ? io.in_img_stride * 4 : round_up(io.in_pitch * 4 * io.in_rows, 16);
        cuuint64_t strides[2] = {(cuuint64_t)(io.in_pitch * 4), (cuuint64_t)img_bytes};
        cuuint32_t box[3] = {(cuuint32_t)BOXW, (cuuint32_t)R, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = enc(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(io.in), dims, strides,
                         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(DWT2_ECUDA);
    }

    const long long max_units_ctas = (a.units + MIN_ROWS_PER_CTA - 1) / MIN_ROWS_PER_CTA;
    const int grid = int(std::max<long long>(1, std::min<long long>(p->max_ctas, max_units_ctas)));

    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel_for(tma, vec), a);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

int32_t configure_kernels(int *max_ctas)
{
    static int cached = 0;
    static std::once_flag once;
    static int32_t status = DWT2_OK;
    std::call_once(once, [] {
        KernelFn fns[4] = {kernel_for(true, true), kernel_for(true, false), kernel_for(false, true),
                           kernel_for(false, false)};
        int dev = 0, sms = 0, per_sm = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
            status = DWT2_ECUDA;
            return;
        }
        for (KernelFn f : fns) {
            if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES)) !=
                cudaSuccess) {
                status = DWT2_ECUDA;
                return;
            }
        }
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[0], THREADS, SMEM_BYTES) != cudaSuccess ||
            per_sm < 1) {
            status = DWT2_ECUDA;
            return;
        }
        cached = sms * per_sm;
    });
    cudaGetLastError();
    *max_ctas = cached;
    return status;
}

dwt2_plan *make_plan(int W, int H, int levels, int boundary, int max_count, bool strip, int Hg, int rb, int re)
{
    if (boundary != DWT2_BOUNDARY_SYMMETRIC) {
        g_last_error = DWT2_EUNSUPPORTED;
        return nullptr;
    }
    if (W < 2 || H < 1 || levels < 1 || levels > 30 || max_count < 1) {
        g_last_error = DWT2_EINVAL;
        return nullptr;
    }
    int dev = 0;
    cudaDeviceProp prop;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
        cudaGetLastError();
        g_last_error = DWT2_ECUDA;
        return nullptr;
    }
    if (prop.major != 10) {
        g_last_error = DWT2_EUNSUPPORTED;
        return nullptr;
    }
    dwt2_plan *p = new (std::nothrow) dwt2_plan;
    if (!p) {
        g_last_error = DWT2_ENOMEM;
        return nullptr;
    }
    memset(p, 0, sizeof(*p));
    p->W = W;
    p->H = H;
    p->levels = levels;
    p->max_count = max_count;
    p->device = dev;
    p->strip = strip;
    p->Hg = Hg;
    p->row_begin = rb;
    p->row_end = re;
    p->ghost_top = (strip && rb > 0) ? 2 : 0;
    p->ghost_bot = (strip && re < Hg) ? 1 : 0;
    int w = W, h = H;
    for (int k = 0; k < levels; ++k) {
        if (w < 2 || h < 2) {
            delete p;
            g_last_error = DWT2_EINVAL;
            return nullptr;
        }
        p->geom[k] = LevelGeom{w, h, (w + 1) / 2, (h + 1) / 2};
        w = (w + 1) / 2;
        h = (h + 1) / 2;
    }
    int32_t st = configure_kernels(&p->max_ctas);
    if (st != DWT2_OK) {
        delete p;
        g_last_error = st;
        return nullptr;
    }
    // LL scratch: level k (1-based, k < levels) writes LL_k to scratch[(k-1) % 2]
    for (int s = 0; s < 2; ++s) {
        if (levels >= s + 2) {
            const LevelGeom &g = p->geom[s];  // LL of level s+1
            p->sc_pitch[s] = round_up(g.Wq, 32);
            p->sc_img_stride[s] = p->sc_pitch[s] * g.Hq;
            size_t bytes = size_t(p->sc_img_stride[s]) * max_count * sizeof(float);
            if (cudaMalloc(&p->scratch[s], bytes) != cudaSuccess) {
                cudaGetLastError();
                if (p->scratch[0]) cudaFree(p->scratch[0]);
                delete p;
                g_last_error = DWT2_ENOMEM;
                return nullptr;
            }
            p->scratch_bytes += bytes;
        }
    }
    g_last_error = DWT2_OK;
    return p;
}

bool overlap(const void *a, size_t an, const void *b, size_t bn)
{
    const char *x = static_cast<const char *>(a), *y = static_cast<const char *>(b);
    return x < y + bn && y < x + an;
}

bool on_plan_device(const dwt2_plan *p, const void *ptr)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) && at.device == p->device;
}

// Forward of levels [first, last] for `count` images.  Level 1 reads `in`.
// Level-1 quad rows may be restricted to [q1a, q1b) (host pipelining).
int32_t run_levels(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                   long long out_stride, int first, int last, int q1a, int q1b, cudaStream_t s)
{
    for (int k = first; k <= last; ++k) {
        const LevelGeom &g = p->geom[k];
        LaunchIO io;
        memset(&io, 0, sizeof(io));
        io.count = count;
        if (k == 0) {
            io.in = in;
            io.in_pitch = p->W;
            io.in_img_stride = in_stride;
            io.in_rows = p->H;
            io.in_end = in + (long long)(count - 1) * in_stride + (long long)p->W * p->H;
        } else {
            const int s = (k - 1) % 2;
            io.in = p->scratch[s];
            io.in_pitch = p->sc_pitch[s];
            io.in_img_stride = p->sc_img_stride[s];
            io.in_rows = g.H;
            io.in_end = io.in + (long long)(count - 1) * io.in_img_stride + io.in_pitch * g.H;
        }
        io.in_row0 = 0;
        io.out = out;
        io.out_pitch = p->W;
        io.out_img_stride = out_stride;
        io.out_q0 = 0;
        io.hq_local = g.Hq;
        if (k == p->levels - 1) {
            io.ll = out;
            io.ll_pitch = p->W;
            io.ll_img_stride = out_stride;
        } else {
            const int s = k % 2;
            io.ll = p->scratch[s];
            io.ll_pitch = p->sc_pitch[s];
            io.ll_img_stride = p->sc_img_stride[s];
        }
        int qa = 0, qb = g.Hq;
        if (k == 0) {
            qa = q1a;
            qb = q1b;
        }
        int32_t r = launch_level(p, g.W, g.H, io, qa, qb, 0, 0, s);
        if (r != DWT2_OK) return r;
    }
    return DWT2_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

dwt2_plan *dwt2_plan_create(int32_t width, int32_t height, int32_t levels, int32_t boundary)
{
    return make_plan(width, height, levels, boundary, 1, false, height, 0, height);
}

dwt2_plan *dwt2_plan_create_batched(int32_t width, int32_t height, int32_t levels, int32_t boundary,
                                    int32_t max_count)
{
    return make_plan(width, height, levels, boundary, max_count, false, height, 0, height);
}

dwt2_plan *dwt2_plan_create_strip(int32_t width, int32_t global_height, int32_t row_begin, int32_t row_end,
                                  int32_t boundary)
{
    if (global_height < 2 || row_begin < 0 || row_begin >= row_end || row_end > global_height ||
        (row_begin & 1) || ((row_end & 1) && row_end != global_height)) {
        g_last_error = DWT2_EINVAL;
        return nullptr;
    }
    // geometry is validated on the full image (every level input >= 2 x 2)
    dwt2_plan *p = make_plan(width, global_height, 1, boundary, 1, true, global_height, row_begin, row_end);
    return p;
}

int32_t dwt2_forward(const dwt2_plan *p, const float *in, float *out, dwt2_stream_t stream)
{
    if (!p || !in || !out || p->strip || !aligned(in, 4) || !aligned(out, 4)) return fail(DWT2_EINVAL);
    const size_t bytes = size_t(p->W) * p->H * sizeof(float);
    if (overlap(in, bytes, out, bytes) || !on_plan_device(p, in) || !on_plan_device(p, out))
        return fail(DWT2_EINVAL);
    int32_t r = run_levels(p, in, out, 1, (long long)p->W * p->H, (long long)p->W * p->H, 0, p->levels - 1, 0,
                           p->geom[0].Hq, reinterpret_cast<cudaStream_t>(stream));
    if (r != DWT2_OK) return r;
    g_last_error = DWT2_OK;
    return DWT2_OK;
}

int32_t dwt2_forward_batched(const dwt2_plan *p, const float *in, float *out, int32_t count, int64_t in_stride,
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
    int32_t r = run_levels(p, in, out, count, in_stride, out_stride, 0, p->levels - 1, 0, p->geom[0].Hq,
                           reinterpret_cast<cudaStream_t>(stream));
    if (r != DWT2_OK) return r;
    g_last_error = DWT2_OK;
    return DWT2_OK;
}

int32_t dwt2_forward_strip(const dwt2_plan *p, const float *in, float *out, int32_t part, dwt2_stream_t stream)
{
    if (!p || !in || !out || !p->strip || part < 0 || part > 2 || !aligned(in, 4) || !aligned(out, 4))
        return fail(DWT2_EINVAL);
    const int hl = p->row_end - p->row_begin;
    const int in_rows = hl + p->ghost_top + p->ghost_bot;
    const size_t in_bytes = size_t(p->W) * in_rows * sizeof(float);
    const size_t out_bytes = size_t(p->W) * hl * sizeof(float);
    if (overlap(in, in_bytes, out, out_bytes) || !on_plan_device(p, in) || !on_plan_device(p, out))
        return fail(DWT2_EINVAL);
    const int qs = p->row_begin / 2, qe = (p->row_end + 1) / 2;
    LaunchIO io;
    memset(&io, 0, sizeof(io));
    io.count = 1;
    io.in = in;
    io.in_pitch = p->W;
    io.in_img_stride = (long long)p->W * in_rows;
    io.in_row0 = p->row_begin - p->ghost_top;
    io.in_rows = in_rows;
    io.in_end = in + (long long)p->W * in_rows;
    io.out = out;
    io.out_pitch = p->W;
    io.out_img_stride = (long long)p->W * hl;
    io.out_q0 = qs;
    io.hq_local = qe - qs;
    io.ll = out;
    io.ll_pitch = p->W;
    io.ll_img_stride = io.out_img_stride;
    const int ia = qs + (p->ghost_top ? 1 : 0), ib = qe - (p->ghost_bot ? 1 : 0);
    int a0, a1, b0 = 0, b1 = 0;
    if (part == DWT2_STRIP_ALL) {
        a0 = qs; a1 = qe;
    } else if (part == DWT2_STRIP_INTERIOR) {
        a0 = ia; a1 = std::max(ia, ib);
    } else {
        // boundary rows: [qs, ia) and [max(ib, ia), qe)
        a0 = qs; a1 = ia;
        b0 = std::max(ib, ia); b1 = qe;
        if (b0 < a1) b0 = a1;
    }
    int32_t r = launch_level(p, p->W, p->Hg, io, a0, a1, b0, b1, reinterpret_cast<cudaStream_t>(stream));
    if (r != DWT2_OK) return r;
    g_last_error = DWT2_OK;
    return DWT2_OK;
}

int32_t dwt2_forward_host(const dwt2_plan *p, const float *host_in, float *host_out, dwt2_stream_t stream)
{
    if (!p || !host_in || !host_out || p->strip || p->max_count != 1) return fail(DWT2_EINVAL);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const long long npx = (long long)p->W * p->H;
    if (!p->d_in) {
        if (cudaMalloc(&p->d_in, npx * sizeof(float)) != cudaSuccess ||
            cudaMalloc(&p->d_out, npx * sizeof(float)) != cudaSuccess) {
            cudaGetLastError();
            if (p->d_in) cudaFree(p->d_in);
            p->d_in = p->d_out = nullptr;
            return fail(DWT2_ENOMEM);
        }
        if (cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking) != cudaSuccess)
            return fail(DWT2_ECUDA);
        for (int i = 0; i < 64; ++i)
            if (cudaEventCreateWithFlags(&p->ev[i], cudaEventDisableTiming) != cudaSuccess) return fail(DWT2_ECUDA);
    }
    // Pipeline over NB row bands of level 1: H2D(band b) -> kernel on the
    // quad rows whose inputs have all arrived -> D2H of finished output rows.
    const LevelGeom &g = p->geom[0];
    const int NB = std::min(16, std::max(1, g.Hq / 64));
    const size_t rowb = size_t(p->W) * sizeof(float);
    cudaEvent_t *ev_in = p->ev, *ev_k = p->ev + 16, *ev_done = p->ev + 32;
    if (cudaEventRecord(ev_done[0], s) != cudaSuccess) return fail(DWT2_ECUDA);   // order after prior work
    if (cudaStreamWaitEvent(p->s_h2d, ev_done[0], 0) != cudaSuccess) return fail(DWT2_ECUDA);
    int q_done = 0;
    for (int b = 0; b < NB; ++b) {
        const int r0 = int((long long)p->H * b / NB), r1 = int((long long)p->H * (b + 1) / NB);
        if (cudaMemcpyAsync(p->d_in + (long long)r0 * p->W, host_in + (long long)r0 * p->W, rowb * (r1 - r0),
                            cudaMemcpyHostToDevice, p->s_h2d) != cudaSuccess)
            return fail(DWT2_ECUDA);
        cudaEventRecord(ev_in[b], p->s_h2d);
        cudaStreamWaitEvent(s, ev_in[b], 0);
        // quad rows n with all of rows 2n-2 .. 2n+2 (clipped to the image) present: 2n+2 <= r1-1
        const int ready = (r1 >= 3) ? (r1 - 3) / 2 + 1 : 0;   // 2n + 2 <= r1 - 1
        int qe = (b == NB - 1) ? g.Hq : std::max(q_done, std::min(g.Hq, ready));
        if (qe > q_done) {
            int32_t r = run_levels(p, p->d_in, p->d_out, 1, npx, npx, 0, 0, q_done, qe, s);
            if (r != DWT2_OK) return r;
            cudaEventRecord(ev_k[b], s);
            if (p->levels == 1) {
                // finished rows: LL|HL rows [q_done, qe) and LH|HH rows Hq + [q_done, min(qe, H/2))
                cudaStreamWaitEvent(p->s_d2h, ev_k[b], 0);
                cudaMemcpyAsync(host_out + (long long)q_done * p->W, p->d_out + (long long)q_done * p->W,
                                rowb * (qe - q_done), cudaMemcpyDeviceToHost, p->s_d2h);
                const int h0 = std::min(q_done, p->H / 2), h1 = std::min(qe, p->H / 2);
                if (h1 > h0)
                    cudaMemcpyAsync(host_out + (long long)(g.Hq + h0) * p->W, p->d_out + (long long)(g.Hq + h0) * p->W,
                                    rowb * (h1 - h0), cudaMemcpyDeviceToHost, p->s_d2h);
            } else {
                // level-1 LH|HH rows are final at once; the top half waits for the coarser levels
                const int h0 = std::min(q_done, p->H / 2), h1 = std::min(qe, p->H / 2);
                if (h1 > h0) {
                    cudaStreamWaitEvent(p->s_d2h, ev_k[b], 0);
                    cudaMemcpyAsync(host_out + (long long)(g.Hq + h0) * p->W, p->d_out + (long long)(g.Hq + h0) * p->W,
                                    rowb * (h1 - h0), cudaMemcpyDeviceToHost, p->s_d2h);
                }
            }
            q_done = qe;
        }
    }
    if (p->levels > 1) {
        int32_t r = run_levels(p, p->d_in, p->d_out, 1, npx, npx, 1, p->levels - 1, 0, 0, s);
        if (r != DWT2_OK) return r;
        cudaEventRecord(ev_done[1], s);
        cudaStreamWaitEvent(p->s_d2h, ev_done[1], 0);
        cudaMemcpyAsync(host_out, p->d_out, rowb * g.Hq, cudaMemcpyDeviceToHost, p->s_d2h);
    }
    cudaEventRecord(ev_done[2], p->s_d2h);
    cudaStreamWaitEvent(s, ev_done[2], 0);
    if (cudaStreamSynchronize(s) != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    if (cudaGetLastError() != cudaSuccess) return fail(DWT2_ECUDA);
    g_last_error = DWT2_OK;
    return DWT2_OK;
}

void dwt2_destroy(dwt2_plan *p)
{
    if (!p) return;
    for (int s = 0; s < 2; ++s)
        if (p->scratch[s]) cudaFree(p->scratch[s]);
    if (p->d_in) {
        cudaFree(p->d_in);
        cudaFree(p->d_out);
        cudaStreamDestroy(p->s_h2d);
        cudaStreamDestroy(p->s_d2h);
        for (int i = 0; i < 64; ++i) cudaEventDestroy(p->ev[i]);
    }
    cudaGetLastError();
    delete p;
}

int32_t dwt2_plan_info(const dwt2_plan *p, dwt2_plan_info_t *info)
{
    if (!p || !info) return fail(DWT2_EINVAL);
    memset(info, 0, sizeof(*info));
    info->width = p->W;
    info->height = p->strip ? (p->row_end - p->row_begin) : p->H;
    info->levels = p->levels;
    info->max_count = p->max_count;
    info->launches_per_forward = p->levels;
    int tma = 0;
    long long bytes = 0;
    for (int k = 0; k < p->levels; ++k) {
        const LevelGeom &g = p->geom[k];
        // level 1 reads the caller's buffer: TMA iff its rows are 16-byte aligned
        if (k > 0 || (p->W % 4) == 0) ++tma;
        bytes += 8LL * g.W * (p->strip ? (p->row_end - p->row_begin) : g.H);
    }
    info->tma_levels = tma;
    info->algorithmic_bytes = bytes;
    info->scratch_bytes = (int64_t)p->scratch_bytes;
    return DWT2_OK;
}

int32_t dwt2_last_error(void) { return g_last_error; }

const char *dwt2_error_string(int32_t code)
{
    switch (code) {
    case DWT2_OK: return "ok";
    case DWT2_EINVAL: return "invalid argument";
    case DWT2_ENOMEM: return "out of memory";
    case DWT2_ECUDA: return "CUDA error";
    case DWT2_EUNSUPPORTED: return "unsupported (boundary mode or device)";
    default: return "unknown error";
    }
}

const char *dwt2_version(void) { return "dwt2-b200 0.1 sm_100a (non-separable lifting, CDF 5/3)"; }

}  // extern "C"
