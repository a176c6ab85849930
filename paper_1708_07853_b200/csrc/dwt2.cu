// dwt2.cu -- B200 (sm_100a) forward 2-D CDF 5/3 DWT with the non-separable
// lifting scheme of arXiv:1708.07853 (section 3, Eq. (5)).
//
// One fused kernel per decomposition level.  The paper's two spatial steps
// (predict, then update) and its single in-level synchronisation point `|`
// map onto one pass over HBM:
//
//   HBM --TMA--> per-warp smem ring (136-column slab + halo, R rows/stage;
//                row pitches that are not a multiple of 16 bytes: row-grouped
//                tensor maps, see grp_row)
//       --LDS.128--> registers: spatial predict (Eq. (5) right factor)
//       --warp shuffle (m-1 neighbour) + register carry (n-1 neighbour)-->
//       spatial update (Eq. (5) left factor) --> 4 subband stores (STG.64)
//
// so the `|` between predict and update costs a shuffle instead of a grid-wide
// barrier, and every level moves the algorithmic floor of 4 B read + 4 B
// written per pixel.  See DESIGN.md sections 5-6 for the layout and roofline.
//
// Work decomposition.  A warp owns a 128-pixel column slab (64 quads, 2 per
// lane) and walks DOWN a tile of tb quad rows, row pair by row pair,
// carrying the predicted values of the previous quad row in registers.  The
// grid is persistent (4 warps per CTA, 4 CTAs per SM); warps are independent
// and take tiles from a self-resetting atomic queue in row-block-major order
// (horizontally adjacent tiles run together and share their halo columns in
// L2), prefetching the next tile's stages while finishing the current one.
// The queue exists because SMs differ by up to 1.5x in throughput under full
// HBM load; mid-size levels use guided tiles (one large tile per warp, then
// small ones) and small levels one static tile per warp (see tile_policy and
// launch_level).
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
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <type_traits>

#include "dwt2_internal.h"

using namespace dwt2_detail;

namespace {

// ---------------------------------------------------------------------------
// Tile geometry
//
// A warp owns a column slab of SLAB = 64 QPL pixels: lane l holds the 2 QPL
// pixel columns starting at x0 + 2 QPL l, i.e. QPL quads.  Its smem ring
// holds, per row, the slab plus the 5/3 halo (2 columns left, 1 right),
// staged by NBOX 2-D TMA boxes of 136 x BOXH floats (a TMA box extent is at
// most 256 elements; a 544-byte inner extent keeps every row 16-B aligned):
//   QPL = 2: one box,  columns [x0 - 4, x0 + 132)
//   QPL = 4: two boxes, columns [x0 - 8, x0 + 128) and [x0 + 128, x0 + 264)
// ---------------------------------------------------------------------------
#ifndef DWT2_QPL
#define DWT2_QPL 2
#endif
#ifndef DWT2_PAIRS
#define DWT2_PAIRS 4
#endif
#ifndef DWT2_STAGES
#define DWT2_STAGES 2
#endif
#ifndef DWT2_WARPS
#define DWT2_WARPS 4
#endif
#ifndef DWT2_MINB
#define DWT2_MINB 4
#endif
#ifndef DWT2_MIN_TPW
#define DWT2_MIN_TPW 6                // below this many tiles per warp: one static tile per warp (c2 sweep)
#endif
#ifndef DWT2_TPW
#define DWT2_TPW 32                 // target tiles per warp on large levels (measured optimum)
#endif
#ifndef DWT2_FORCE_GENERIC                  // probes only: the generic (bulk-copy) loader everywhere
#define DWT2_FORCE_GENERIC 0
#endif
#ifndef DWT2_SCALAR_LDS                    // probes only: scalar smem loads on the TMA path
#define DWT2_SCALAR_LDS 0
#endif
#ifndef DWT2_GRP_NOFIX                     // probes only
#define DWT2_GRP_NOFIX 0
#endif
#ifndef DWT2_NO_GRP                        // probes only: no row-grouped TMA (bulk-copy loader instead)
#define DWT2_NO_GRP 0
#endif
#ifndef DWT2_PROBE_NOWAIT                  // probes only (WRONG results): levels >= 2 skip griddepcontrol.wait at entry
#define DWT2_PROBE_NOWAIT 0                 // (they wait at exit), to bound what overlapping a level's drain with
#endif                                      // the next level's start could save
#ifndef DWT2_FORCE_SCALAR                   // probes only: scalar subband stores everywhere
#define DWT2_FORCE_SCALAR 0
#endif
#ifndef DWT2_L2_PROMOTION
#define DWT2_L2_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_NONE
#endif
constexpr int QPL = DWT2_QPL;               // quads per lane (2 or 4)
constexpr int SLAB = 64 * QPL;              // output pixel columns per warp
constexpr int NBOX = QPL / 2;               // TMA boxes per stage
constexpr int BOXW = 136;                   // box inner extent (floats)
constexpr int BOX0 = (QPL == 2) ? -4 : -8;  // column of box 0 relative to x0
constexpr int BOX1 = 128;                   // column of box 1 relative to x0 (QPL = 4)
constexpr int PAIRS = DWT2_PAIRS;           // row pairs (quad rows) per pipeline stage
constexpr int ROWS = 2 * PAIRS;             // new rows per stage
constexpr int BOXH = ROWS + 1;              // a stage holds rows [r, r + ROWS + 1): its first (even)
                                            // row is also the last row of the previous stage, so
                                            // an (odd, even) row pair never straddles two stages
constexpr int S = DWT2_STAGES;              // stages per warp ring
constexpr int WARPS = DWT2_WARPS;           // warps per CTA (independent; packing only)
constexpr int THREADS = WARPS * 32;
constexpr int MIN_TILE_ROWS = 11;           // min quad rows per tile (sweep: 11 > 7, 15 on 4096^2 and 8192^2)
constexpr int MAX_TILE_ROWS = 127;
constexpr int MAX_COUNTERS = QUEUE_SLOTS;    // work-queue counter pairs (slots: dwt2_internal.h)

// smem row pitch: TMA writes a box densely (136); the cp.async loader keeps
// every row's 16-byte alignment shift delta (0..3 floats), hence 4 more.
template <bool TMA> struct Lay {
    static constexpr int RP = TMA ? BOXW : BOXW + 4;
    static constexpr int SUB = (BOXH * RP + 31) / 32 * 32;       // one box; TMA dst is 128-B aligned
};
template <bool TMA, int NS = S> struct Ring {
    static constexpr int STAGE = NBOX * Lay<TMA>::SUB;          // floats per stage
    static constexpr int FLOATS = NS * STAGE;                   // floats per warp ring
    static constexpr size_t SMEM = size_t(WARPS) * FLOATS * sizeof(float) + size_t(WARPS) * NS * 8;
};
// Large levels run a 3-stage ring (3 CTAs per SM by shared memory): measured
// 16384^2 805.5 -> 811.7 Gpix/s (0.982 -> 0.990 of copy); mid-size levels keep
// 2 stages and 4 CTAs per SM (3 stages there: config 2 616 -> 589, config 4 474 -> 463)
constexpr int S_LARGE = 3;

static_assert((Ring<true>::STAGE * 4) % 128 == 0 && (Ring<false>::STAGE * 4) % 128 == 0,
              "every ring slot must be 128-byte aligned for TMA");
static_assert(BOXH <= 256, "TMA box extent limit");
static_assert(QPL == 2 || QPL == 4, "2 or 4 quads per lane");

// smem offsets (floats, from a row of box 0) of what a lane reads
template <bool TMA>
__device__ __forceinline__ int lane_offset(int lane)
{
    if (QPL == 2) return 4 + 4 * lane;
    return lane < 16 ? 8 + 8 * lane : Lay<TMA>::SUB + 8 * (lane - 16);
}
constexpr int HALO_OFF = (QPL == 2) ? 2 : 6;                    // columns x0-2, x0-1
template <bool TMA>
__device__ __forceinline__ constexpr int right_offset() { return (QPL == 2) ? 132 : Lay<TMA>::SUB + 128; }

// ---------------------------------------------------------------------------
// Kernel arguments (a __grid_constant__ parameter: the TMA descriptor must be
// 64-byte aligned and live in param space)
// ---------------------------------------------------------------------------
struct alignas(64) LevelArgs {
    CUtensorMap tmap;                 // 3-D {W, in_rows, count}, box {BOXW, BOXH, 1}
                                      // (GRP: row groups {G P, flat_rows / G, 1}, box {BOXWG, ceil(BOXH / G), 1})
    CUtensorMap tmap_b;               // GRP only: the same groups, box {BOXWG, floor(BOXH / G), 1}
    const float *in;                  // generic loader: image 0, buffer row 0
    const float *in_end;              // one past the last element of the call's input
    long long in_pitch, in_img_stride;
    float *ll, *hl, *lh, *hh;         // subband bases for image 0, output row 0
    long long ll_pitch, ll_img_stride;
    long long out_pitch, out_img_stride;
    unsigned int *counter;            // [0] tile counter, [1] finished-warp counter (self-resetting)
    int W, H;                         // level input width, (global) height
    int in_row0, in_rows;             // global row of buffer row 0; rows present in the buffer
    int out_q0;                       // global quad row stored at output row 0
    int nslabs, count;
    FastDiv fd_slabs, fd_img;         // division by nslabs and by nblk * nslabs
    int unroll_first;                 // 1: a tile's first stage (carry-in pair) on the unrolled path
    int qa0, qa1, qb0, qb1;           // quad-row ranges [qa0, qa1) and [qb0, qb1)
    int tb;                           // quad rows per tile (range A)
    int tb_b;                         // quad rows per tile (range B)
    int nblk_a, nblk;                 // row blocks in range A, in A and B
    int ntiles;                       // count * nblk * nslabs
    int nwarps;                       // warps in the grid
    int static_tiles;                 // 1: tile w -> warp w, no work queue
    int glog;                         // GRP: log2 G, G = rows per 16-byte-aligned row group (2 or 4)
    long long grp_rows;               // GRP: flat rows covered by whole groups (G floor(flat_rows / G))
    long long flat_rows;              // GRP: count * in_rows
    int rev;                          // 1: images and quad rows in reverse order (tile t -> mirrored rows)
    int rsum;                         // rev: qa0 + the end of the level's quad rows (mirror q -> rsum - q)
    int nowait;                       // DWT2_PROBE_NOWAIT builds only
    int peer;                         // peer strip launch (peer.cu): publish pb.level's ready flag at entry
    int pb_ctas;                      // the last pb_ctas CTAs of the grid take the boundary role
    PeerBoundaryArgs pb;
};

// Row-grouped TMA (GRP) for row pitches that are not a multiple of 16 bytes:
// G consecutive rows (G = 2 if the pitch is 8 mod 16 bytes, else 4) span a
// multiple of 16 bytes, so the input is a 2-D tensor of row GROUPS {G P
// floats, flat_rows / G} whose row stride TMA accepts, and row r of the
// buffer is group r / G at inner offset (r mod G) P.  A stage's BOXH rows
// then come as G boxes, box k holding the rows r0 + k, r0 + k + G, ...; smem
// keeps them in that order: stage row `off` lives at smem offset grp_row(off).
// A tiled TMA load faults (illegal instruction, measured) unless its inner
// start coordinate is 16-byte aligned, so each box starts at the column
// aligned down from x0 - 4 and is BOXWG = BOXW + 4 wide; row class c sits
// shifted by (c P) mod 4 floats, which the consumer adds (scalar smem loads).
constexpr int BOXWG = BOXW + 4;
// TMA writes each box at a 128-byte-aligned smem address, so class k starts
// at a multiple of 32 floats: the first BOXH mod G classes hold
// ceil(BOXH / G) rows, the others floor(BOXH / G).
__host__ __device__ constexpr int grp_class_floats(int rows) { return (rows * BOXWG + 31) / 32 * 32; }
__host__ __device__ constexpr int grp_stage_floats(int glog)
{
    return (BOXH & ((1 << glog) - 1)) * grp_class_floats((BOXH + (1 << glog) - 1) >> glog) +
           ((1 << glog) - (BOXH & ((1 << glog) - 1))) * grp_class_floats(BOXH >> glog);
}
constexpr int SUBG = grp_stage_floats(1) > grp_stage_floats(2) ? grp_stage_floats(1) : grp_stage_floats(2);
// smem offset (floats) of stage row `off` in the row-grouped layout
template <int GG>
__device__ __forceinline__ int grp_row(int off)
{
    constexpr int rem = BOXH % GG;
    constexpr int ca = grp_class_floats((BOXH + GG - 1) / GG), cb = grp_class_floats(BOXH / GG);
    const int k = off & (GG - 1);
    return (k < rem ? k * ca : rem * ca + (k - rem) * cb) + (off / GG) * BOXWG;
}
template <bool TMA, int GG, int NS = S> struct RingG {
    static constexpr int STAGE = GG > 1 ? SUBG : Ring<TMA>::STAGE;
    static constexpr int FLOATS = NS * STAGE;
    static constexpr size_t SMEM = size_t(WARPS) * FLOATS * sizeof(float) + size_t(WARPS) * NS * 8;
};
static_assert((SUBG * 4) % 128 == 0, "GRP stage slots must stay 128-byte aligned");

// ---------------------------------------------------------------------------
// PTX helpers (mbarrier, TMA, cp.async, PDL)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int imin(int x, int y) { return x < y ? x : y; }
__host__ __device__ __forceinline__ int imax(int x, int y) { return x > y ? x : y; }

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

__device__ __forceinline__ void tma_load_3d(float *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar)
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

// 1-D bulk copy global -> shared (16-byte granules), completing on an mbarrier
__device__ __forceinline__ void bulk_copy_g2s(float *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
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

#ifdef DWT2_PROF
__device__ unsigned long long g_prof[4];   // cycles waiting for stages, cycles working, stages, tiles
__device__ unsigned long long g_cta[4096][4];   // per CTA: entry, work start, work end (globaltimer ns), smid

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// Register arithmetic type.  The product is fp64; the
// fp32 build (-DDWT2_F32MATH) exists only to measure what the arithmetic
// costs and is never shipped.
#if defined(DWT2_F32MATH)
typedef float real;
#define R_(x) x##f
#else
typedef double real;
#define R_(x) x
#endif

__device__ __forceinline__ float to_f32(real x) { return (float)x; }   // round to nearest even

// ---------------------------------------------------------------------------
// Tiles and the work queue.
//
// Tile t covers quad rows [qa, qb) (<= tb of them) of one slab of one image.
// Tiles are ordered image-major, then row block, then slab, so the tiles
// that warps fetch at about the same time are horizontally adjacent and
// share their halo columns through L2.  Warps take tiles from a global
// atomic counter (dynamic load balancing: a B200 runs some SMs' CTAs up to
// 1.5x slower than others' under full HBM load; static partitions wait for
// the slowest).  The counter resets itself: the last warp to find the queue
// empty zeroes it for the next launch, which cannot start its own fetches
// before this grid completes (stream order / griddepcontrol.wait).
// ---------------------------------------------------------------------------
struct Tile {
    int img, x0, qa, qb;
};

__device__ __forceinline__ Tile decode_tile(const LevelArgs &a, int t)
{
    Tile T;
    const int per_img = a.nblk * a.nslabs;
    T.img = fdiv(t, a.fd_img);
    const int r = t - T.img * per_img;
    const int blk = fdiv(r, a.fd_slabs);
    const int slab = r - blk * a.nslabs;
    T.x0 = slab * SLAB;
    if (blk < a.nblk_a) {
        T.qa = a.qa0 + blk * a.tb;
        T.qb = imin(T.qa + a.tb, a.qa1);
    } else {
        T.qa = a.qb0 + (blk - a.nblk_a) * a.tb_b;
        T.qb = imin(T.qa + a.tb_b, a.qb1);
    }
    if (a.rev) {
        const int qa = T.qa;
        T.qa = a.rsum - T.qb;
        T.qb = a.rsum - qa;
        T.img = a.count - 1 - T.img;
    }
    return T;
}

__device__ __forceinline__ int fetch_tile(const LevelArgs &a, int lane, bool &first)
{
    if (a.static_tiles) {
        const int t = first ? int(blockIdx.x * WARPS + (threadIdx.x >> 5)) : a.ntiles;
        first = false;
        return t < a.ntiles ? t : -1;
    }
    int t = 0;
    if (lane == 0) {
        t = int(atomicAdd(a.counter, 1u));
        if (t >= a.ntiles) {
            // queue drained for this warp; the last warp resets both counters
            if (atomicAdd(a.counter + 1, 1u) == unsigned(a.nwarps - 1)) {
                atomicExch(a.counter, 0u);
                atomicExch(a.counter + 1, 0u);
            }
        }
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    return t < a.ntiles ? t : -1;
}

// Row stream of a tile.  r_first = 0 at the image top, else 2 qa - 2.  Stage
// j holds rows [r_first + ROWS j, r_first + ROWS j + BOXH); pair k = rows
// (r_first + 2k + 1, r_first + 2k + 2) lies in stage k / PAIRS at offsets
// (2 (k % PAIRS) + 1, 2 (k % PAIRS) + 2) and yields the predicted values of
// quad row n_first + k (n_first = 0 at the top, else qa - 1).
__device__ __forceinline__ int tile_stages(const Tile &T)
{
    const int n_first = (T.qa == 0) ? 0 : T.qa - 1;
    return (T.qb - n_first + PAIRS - 1) / PAIRS;
}

__device__ __forceinline__ int tile_row0(const Tile &T) { return (T.qa == 0) ? 0 : 2 * T.qa - 2; }

// ---------------------------------------------------------------------------
// One smem row as seen by one lane, widened to the register type.
//   v[0 .. 2 QPL): the lane's pixels = QPL quads (a,b / c,d pairs)
//   r:             the pixel right of the lane (lane + 1's v[0]; lane 31 reads smem)
//   l0, l1:        the 2 pixels left of the slab (feed lane 0's halo quad)
//   bp[i], bh:     even rows only: HL' = b - 1/2 (a + a[m+1]) of every quad
//                  and of the halo quad (the horizontal predict, reused by
//                  the vertical predict of the quad row above)
// ---------------------------------------------------------------------------
struct RowD {
    real v[2 * QPL];
    real r, l0, l1;
    real bp[QPL], bh;
};

struct EdgeFlags {
    int last;          // index 0..QPL-1 of the image's last quad in this lane, else -1
    bool evenW;
    bool left_edge;    // lane 0 of the slab at x = 0: H[-1] := H[0]
};

template <bool TMA, bool EDGE>
__device__ __forceinline__ RowD load_row(const float *p, int lane, const EdgeFlags &ef, bool even_row)
{
    float f[2 * QPL];
    const float *q = p + lane_offset<TMA>(lane);
    if (TMA && !DWT2_SCALAR_LDS) {
#pragma unroll
        for (int i = 0; i < QPL / 2; ++i) {
            const float4 t = *reinterpret_cast<const float4 *>(q + 4 * i);
            f[4 * i] = t.x; f[4 * i + 1] = t.y; f[4 * i + 2] = t.z; f[4 * i + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 2 * QPL; ++i) f[i] = q[i];
    }
    const float fl0 = p[HALO_OFF], fl1 = p[HALO_OFF + 1];       // broadcast
    const float fr31 = p[right_offset<TMA>()];                  // broadcast
    const float fr = __shfl_down_sync(0xffffffffu, f[0], 1);
    RowD d;
#pragma unroll
    for (int i = 0; i < 2 * QPL; ++i) d.v[i] = f[i];
    d.r = (lane == 31) ? fr31 : fr;
    d.l0 = fl0;
    d.l1 = fl1;
    if (EDGE && ef.evenW) {
        // even W: the last quad's right neighbour column W is x[W-2] (WSS)
#pragma unroll
        for (int i = 0; i < QPL - 1; ++i)
            if (ef.last == i) d.v[2 * i + 2] = d.v[2 * i];
        if (ef.last == QPL - 1) d.r = d.v[2 * QPL - 2];
    }
    if (even_row) {
        // horizontal predict HL' = b + P a = b - 1/2 (a + a[m+1])
#pragma unroll
        for (int i = 0; i < QPL; ++i) {
            const real ar = (i < QPL - 1) ? d.v[2 * i + 2] : d.r;
            d.bp[i] = fma(R_(-0.5), d.v[2 * i] + ar, d.v[2 * i + 1]);
        }
        d.bh = fma(R_(-0.5), d.l0 + d.v[0], d.l1);
    }
    return d;
}

// Spatial predict and spatial update of Eq. (5) for quad row n.
//
// Predict (Eq. (5) right factor), per quad with E = row 2n, O = row 2n+1,
// N = row 2n+2:
//   HL' = b + P a                        (E.bp, computed with the row)
//   LH' = c + P* a       = c - 1/2 (a + a[n+1])
//   HH' = d + P c + P* b + PP* a = d - 1/2 (c + c[m+1]) - 1/2 (HL' + HL'[n+1])
// (PP* a + P* b = P* (b + P a) = P* HL', so the 4-term PP* stencil is
// evaluated through HL', which is exact in the fp64 register arithmetic.)
//
// Update (Eq. (5) left factor) through the same factorisation:
//   LH  = LH' + U HH'                     = LH' + 1/4 (HH' + HH'[m-1])
//   HL  = HL' + U* HH'                    = HL' + 1/4 (HH' + HH'[n-1])
//   LL  = a + U HL' + U* LH' + UU* HH'    = (a + 1/4 (HL' + HL'[m-1])) + 1/4 (LH + LH[n-1])
//   HH  = HH'
// The m-1 neighbours of the lane's first quad come from lane - 1 by
// shuffle (the single in-level synchronisation `|` of the paper), lane 0
// computes the halo quad m0-1 itself; the n-1 neighbours are carried in
// registers from the previous quad row (Carry).
struct Carry {
    real lh[QPL], hh[QPL];            // LH and HH' of quad row n-1
    real lhp[QPL];                    // LH' of quad row n-1 (literal / adapted arithmetic only)
    real hh_halo;                     // HH' of the halo quad m0-1 at n-1 (lane 0)
};

// Arithmetic of the spatial steps (the same operators, evaluated three ways;
// all exact in the fp64 registers for these data, so bit-identical results):
//   AR_GROUPED  separable grouping, 16 DP ops per quad (the product path)
//   AR_LITERAL  Eq. (5) as printed: PP* and UU* as 4-term stencils, 24 MACs
//   AR_ADAPTED  Fig. 3: P = P0 + P1, U = U0 + U1, non-separable N(P1), N(U1)
//               then the quad-local constants C_H, C_V (18 MACs)
enum { AR_GROUPED = 0, AR_LITERAL = 1, AR_ADAPTED = 2 };

struct Out {
    float A[QPL], B[QPL], C[QPL], D[QPL];
};

// Returns the outputs of quad row n; updates the carry to row n.
// missing_odd: odd H, n is the last quad row (row 2n+1 does not exist):
// LH', HH' := their values at n-1 (H[M] := H[M-1]).
template <bool EDGE, int AR>
__device__ __forceinline__ Out predict_update_literal(const RowD &E, const RowD &O, const RowD &N, Carry &cy,
                                                      int lane, const EdgeFlags &ef, bool carry_in, bool missing_odd)
{
    // Eq. (5) literally (AR_LITERAL) or in the adapted form of Fig. 3
    // (AR_ADAPTED).  Same boundary rules as the grouped path: raw samples
    // mirrored in load_row (even right / bottom edges), predicted values
    // mirrored here (H[-1] := H[0] left / top, H[M] := H[M-1] odd edges).
    real cp[QPL], dp[QPL], bp[QPL];
#pragma unroll
    for (int i = 0; i < QPL; ++i) {
        const real a = E.v[2 * i], b = E.v[2 * i + 1], c = O.v[2 * i], d = O.v[2 * i + 1];
        const real ar = (i < QPL - 1) ? E.v[2 * i + 2] : E.r;
        const real cr = (i < QPL - 1) ? O.v[2 * i + 2] : O.r;
        const real ad = N.v[2 * i], bd = N.v[2 * i + 1];
        const real ard = (i < QPL - 1) ? N.v[2 * i + 2] : N.r;
        if (AR == AR_LITERAL) {
            bp[i] = fma(R_(-0.5), a + ar, b);                                     // HL' = b + P a
            cp[i] = fma(R_(-0.5), a + ad, c);                                     // LH' = c + P* a
            dp[i] = fma(R_(0.25), (a + ar) + (ad + ard),                          // HH' = d + P c + P* b + PP* a
                        fma(R_(-0.5), b + bd, fma(R_(-0.5), c + cr, d)));
        } else {
            const real b1 = fma(R_(-0.5), ar, b);                                 // N(P1): HL += P1 LL
            const real c1 = fma(R_(-0.5), ad, c);                                 //        LH += P1* LL
            const real d1 = fma(R_(0.25), ard, fma(R_(-0.5), bd, fma(R_(-0.5), cr, d)));
            const real b2 = fma(R_(-0.5), a, b1);                                 // C_H(P0)
            const real d2 = fma(R_(-0.5), c1, d1);
            cp[i] = fma(R_(-0.5), a, c1);                                         // C_V(P0*)
            dp[i] = fma(R_(-0.5), b2, d2);
            bp[i] = b2;
        }
    }
    // halo quad m0 - 1 (columns x0-2, x0-1), literal form for both variants
    real hbp = fma(R_(-0.5), E.l0 + E.v[0], E.l1);
    real hdp = fma(R_(0.25), (E.l0 + E.v[0]) + (N.l0 + N.v[0]),
                   fma(R_(-0.5), E.l1 + N.l1, fma(R_(-0.5), O.l0 + O.v[0], O.l1)));
    if (missing_odd) {
#pragma unroll
        for (int i = 0; i < QPL; ++i) {
            dp[i] = cy.hh[i];
            cp[i] = cy.lhp[i];
        }
        hdp = cy.hh_halo;
    }
    // n-1 neighbours (carry) and their m-1 neighbours, captured before the carry moves on
    real hu[QPL], lpu[QPL];
#pragma unroll
    for (int i = 0; i < QPL; ++i) {
        hu[i] = cy.hh[i];
        lpu[i] = cy.lhp[i];
    }
    real hu_halo = cy.hh_halo;
    if (carry_in) {            // the first pair of a tile: row n-1 is this row (or the top mirror)
#pragma unroll
        for (int i = 0; i < QPL; ++i) {
            hu[i] = dp[i];
            lpu[i] = cp[i];
        }
        hu_halo = hdp;
    }
    const real bl_sh = __shfl_up_sync(0xffffffffu, bp[QPL - 1], 1);
    const real dl_sh = __shfl_up_sync(0xffffffffu, dp[QPL - 1], 1);
    const real dul_sh = __shfl_up_sync(0xffffffffu, hu[QPL - 1], 1);
    real bl = (lane == 0) ? hbp : bl_sh;
    real dl = (lane == 0) ? hdp : dl_sh;
    real dul = (lane == 0) ? hu_halo : dul_sh;
    if (EDGE) {
        if (ef.left_edge) {            // H[-1] := H[0]
            bl = bp[0];
            dl = dp[0];
            dul = hu[0];
        }
        if (!ef.evenW) {
#pragma unroll
            for (int i = 0; i < QPL; ++i) {
                if (ef.last == i) {
                    bp[i] = (i == 0) ? bl : bp[i - 1];
                    dp[i] = (i == 0) ? dl : dp[i - 1];
                }
            }
            if (carry_in) {    // the mirrored last column's HH' is row n-1's too
#pragma unroll
                for (int i = 0; i < QPL; ++i) hu[i] = dp[i];
            }
        }
    }
    Out o;
#pragma unroll
    for (int i = 0; i < QPL; ++i) {
        const real a = E.v[2 * i];
        const real hll = (i == 0) ? bl : bp[i - 1];          // HL'[m-1]
        const real hhl = (i == 0) ? dl : dp[i - 1];          // HH'[m-1]
        const real hhul = (i == 0) ? dul : hu[i - 1];        // HH'[m-1, n-1]
        real A, B, C;
        if (AR == AR_LITERAL) {
            // LL = a + U HL' + U* LH' + UU* HH',  HL = HL' + U* HH',  LH = LH' + U HH'
            A = fma(R_(0.0625), (dp[i] + hhl) + (hu[i] + hhul),
                    fma(R_(0.25), cp[i] + lpu[i], fma(R_(0.25), bp[i] + hll, a)));
            B = fma(R_(0.25), dp[i] + hu[i], bp[i]);
            C = fma(R_(0.25), dp[i] + hhl, cp[i]);
        } else {
            // N(U1): LL += U1 HL + U1* LH + U1 U1* HH, HL += U1* HH, LH += U1 HH
            const real ll1 = fma(R_(0.0625), hhul, fma(R_(0.25), lpu[i], fma(R_(0.25), hll, a)));
            const real hl1 = fma(R_(0.25), hu[i], bp[i]);
            const real lh1 = fma(R_(0.25), hhl, cp[i]);
            const real ll2 = fma(R_(0.25), hl1, ll1);        // C_H(U0): LL += U0 HL, LH += U0 HH
            C = fma(R_(0.25), dp[i], lh1);
            A = fma(R_(0.25), C, ll2);                       // C_V(U0*): LL += U0* LH, HL += U0* HH
            B = fma(R_(0.25), dp[i], hl1);
        }
        o.A[i] = to_f32(A);
        o.B[i] = to_f32(B);
        o.C[i] = to_f32(C);
        o.D[i] = to_f32(dp[i]);
        cy.lh[i] = C;
        cy.hh[i] = dp[i];
        cy.lhp[i] = cp[i];
    }
    cy.hh_halo = hdp;
    return o;
}

template <bool EDGE, int AR = AR_GROUPED>
__device__ __forceinline__ Out predict_update(const RowD &E, const RowD &O, const RowD &N, Carry &cy, int lane,
                                              const EdgeFlags &ef, bool carry_in, bool missing_odd)
{
    if (AR != AR_GROUPED) return predict_update_literal<EDGE, AR>(E, O, N, cy, lane, ef, carry_in, missing_odd);
    real cp[QPL], dp[QPL], bp[QPL];
#pragma unroll
    for (int i = 0; i < QPL; ++i) {
        bp[i] = E.bp[i];
        const real c = O.v[2 * i], d = O.v[2 * i + 1];
        const real cr = (i < QPL - 1) ? O.v[2 * i + 2] : O.r;
        cp[i] = fma(R_(-0.5), E.v[2 * i] + N.v[2 * i], c);
        dp[i] = fma(R_(-0.5), E.bp[i] + N.bp[i], fma(R_(-0.5), c + cr, d));
    }
    // halo quad m0 - 1 (columns x0-2, x0-1): every lane computes it (a
    // masked warp instruction costs the same pipe time); lane 0 keeps it
    real hdp = fma(R_(-0.5), E.bh + N.bh, fma(R_(-0.5), O.l0 + O.v[0], O.l1));
    if (missing_odd) {
#pragma unroll
        for (int i = 0; i < QPL; ++i) dp[i] = cy.hh[i];
        hdp = cy.hh_halo;
    }
    const real bl_sh = __shfl_up_sync(0xffffffffu, bp[QPL - 1], 1);
    const real dl_sh = __shfl_up_sync(0xffffffffu, dp[QPL - 1], 1);
    real bl = (lane == 0) ? E.bh : bl_sh;
    real dl = (lane == 0) ? hdp : dl_sh;
    if (EDGE) {
        if (ef.left_edge) {            // H[-1] := H[0]
            bl = bp[0];
            dl = dp[0];
        }
        if (!ef.evenW) {
            // odd W: the last column is L-only; H[M] := H[M-1]
#pragma unroll
            for (int i = 0; i < QPL; ++i) {
                if (ef.last == i) {
                    bp[i] = (i == 0) ? bl : bp[i - 1];
                    dp[i] = (i == 0) ? dl : dp[i - 1];
                }
            }
        }
    }
    Out o;
    real lh[QPL];
#pragma unroll
    for (int i = 0; i < QPL; ++i) {
        const real dleft = (i == 0) ? dl : dp[i - 1];
        lh[i] = missing_odd ? cy.lh[i] : fma(R_(0.25), dp[i] + dleft, cp[i]);
    }
    cy.hh_halo = hdp;
    if (carry_in) {
#pragma unroll
        for (int i = 0; i < QPL; ++i) {
            cy.lh[i] = lh[i];
            cy.hh[i] = dp[i];
        }
    }
#pragma unroll
    for (int i = 0; i < QPL; ++i) {
        const real bleft = (i == 0) ? bl : bp[i - 1];
        const real a1 = fma(R_(0.25), bp[i] + bleft, E.v[2 * i]);
        o.A[i] = to_f32(fma(R_(0.25), lh[i] + cy.lh[i], a1));
        o.B[i] = to_f32(fma(R_(0.25), dp[i] + cy.hh[i], bp[i]));
        o.C[i] = to_f32(lh[i]);
        o.D[i] = to_f32(dp[i]);
        cy.lh[i] = lh[i];
        cy.hh[i] = dp[i];
    }
    return o;
}

// Stores QPL consecutive coefficients of one subband row; n valid (0..QPL).
template <bool VEC, bool EDGE>
__device__ __forceinline__ void storeq(float *p, const float (&x)[QPL], int n, bool stream)
{
    if (VEC && (!EDGE || n == QPL)) {
        if (QPL == 4) {
            const float4 v = make_float4(x[0], x[1], x[2 % QPL], x[3 % QPL]);
            if (stream) __stcs(reinterpret_cast<float4 *>(p), v);
            else *reinterpret_cast<float4 *>(p) = v;
        } else {
            const float2 v = make_float2(x[0], x[1]);
            if (stream) __stcs(reinterpret_cast<float2 *>(p), v);
            else *reinterpret_cast<float2 *>(p) = v;
        }
    } else {
#pragma unroll
        for (int i = 0; i < QPL; ++i) {
            if (!EDGE || i < n) {
                if (stream) __stcs(p + i, x[i]);
                else p[i] = x[i];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// The fused level kernel: a persistent grid of independent warps; each warp
// streams tiles from the work queue through its own TMA ring (producer and
// consumer in one warp, prefetching across tile boundaries).
// ---------------------------------------------------------------------------
template <bool TMA, bool VEC, int AR, int GG, int NS = S, bool PEER = false>
__global__ void __launch_bounds__(THREADS, NS == 2 ? DWT2_MINB : 3)
dwt53_level_kernel(const __grid_constant__ LevelArgs a)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr bool GRP = GG > 1;            // row-grouped TMA, G = GG rows per group
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    float *ring = reinterpret_cast<float *>(smem_raw) + size_t(warp) * RingG<TMA, GG, NS>::FLOATS;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + size_t(WARPS) * RingG<TMA, GG, NS>::FLOATS * sizeof(float)) +
                     warp * NS;

    if (lane == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1u);     // one arrive.expect_tx per stage
        fence_mbar_init();
    }
    __syncwarp();
    if (TMA && lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tmap)) : "memory");
    if (GG > 1 && lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tmap_b)) : "memory");

    // Programmatic dependent launch: the next level may be scheduled now; it
    // waits (griddepcontrol.wait) for this grid's completion before touching
    // memory, exactly as this grid waits for its predecessor here.
#ifdef DWT2_PROF
    const unsigned long long t_entry = gtimer();
#endif
    pdl_launch_dependents();
    if (!DWT2_PROBE_NOWAIT || !a.nowait) pdl_wait();
    // peer strip launch (peer.cu): every earlier launch of this rank's step is
    // complete, so this level's input rows are final -- tell the neighbours;
    // in a fused launch the CTAs past the level's own grid compute the strip's
    // boundary quad rows from the neighbours' memory
    // (a separate instantiation: the hooks cost the other launches measurably --
    // config 5's 2048^2 x 256 batch 1737 -> 1808 us with them compiled in)
    if constexpr (PEER) {
    if (a.peer && blockIdx.x == 0 && threadIdx.x == 0) peer_publish(a.pb.flags, a.pb.level);
    if (a.pb_ctas > 0 && int(blockIdx.x) >= int(gridDim.x) - a.pb_ctas) {
        const int c = int(blockIdx.x) - (int(gridDim.x) - a.pb_ctas);
        peer_boundary_role(a.pb, c % a.pb.nbx, c / a.pb.nbx, reinterpret_cast<float *>(smem_raw));
        __syncthreads();
        if (threadIdx.x == 0) peer_exit(a.pb);
        return;
    }
    }
#ifdef DWT2_PROF
    if (threadIdx.x == 0 && blockIdx.x < 4096) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_cta[blockIdx.x][0] = t_entry;
        g_cta[blockIdx.x][1] = gtimer();
        g_cta[blockIdx.x][3] = smid;
    }
    const long long t_work = clock64();
    long long t_wait = 0;
#endif

    const int Wq = (a.W + 1) >> 1;
    const int Wh = a.W >> 1;
    const int Hq = (a.H + 1) >> 1;
    const int Hh = a.H >> 1;

    // ---- producer state: the tile whose stages are being issued
    Tile pt;
    bool first_fetch = true;
    int pt_id = fetch_tile(a, lane, first_fetch);
    int pt_j = 0, pt_nst = 0;
    if (pt_id >= 0) {
        pt = decode_tile(a, pt_id);
        pt_nst = tile_stages(pt);
    }
    // tile ids handed from producer to consumer, in order (warp-private smem
    // would do too; NS + 1 entries suffice because the producer is at most NS
    // stages -- hence at most NS tiles -- ahead)
    int tq[NS + 1];
#pragma unroll
    for (int i = 0; i <= NS; ++i) tq[i] = -1;
    int tq_head = 0, tq_tail = 0;      // consumer pops at head, producer pushes at tail
    if (pt_id >= 0) {
        tq[0] = pt_id;
        tq_tail = 1;
    }
    uint32_t prod_seq = 0, cons_seq = 0;

    auto issue_next = [&]() {
        // issue the next stage of the global stage sequence (if any)
        if (pt_id < 0) return;
        if (pt_j == pt_nst) {
            pt_id = fetch_tile(a, lane, first_fetch);
            if (pt_id < 0) return;
            pt = decode_tile(a, pt_id);
            pt_nst = tile_stages(pt);
            pt_j = 0;
#pragma unroll
            for (int i = 0; i <= NS; ++i)
                if (i == tq_tail % (NS + 1)) tq[i] = pt_id;
            ++tq_tail;
        }
        const int slot = int(prod_seq % NS);
        float *dst = ring + slot * RingG<TMA, GG, NS>::STAGE;
        const int r0 = tile_row0(pt) + pt_j * ROWS;
        if (GRP) {
            // G boxes per column box, one per row class (see grp_row).  Rows
            // before the buffer or past its whole groups are zero-filled by
            // TMA; the latter (< G rows at the very end of the buffer) are then
            // copied by the warp once the stage has landed -- once per call.
            constexpr int G = GG;
            const long long fr0 = (long long)pt.img * a.in_rows + (r0 - a.in_row0);
            if (lane == 0) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&bars[slot], uint32_t(NBOX * BOXH * BOXWG * sizeof(float)));
#pragma unroll
                for (int k = 0; k < G; ++k) {
                    const long long fr = fr0 + k;
                    const int g = int(fr >> (G == 2 ? 1 : 2));              // floor(fr / G), also for fr < 0
                    const int cls = int(fr) & (G - 1);
                    const int xk = (cls * int(a.in_pitch) + pt.x0 + BOX0) & ~3;     // 16-byte-aligned start
                    tma_load_3d(dst + grp_row<G>(k), k < BOXH % G ? &a.tmap : &a.tmap_b, xk, g, 0, &bars[slot]);
                }
            }
            if (!DWT2_GRP_NOFIX && fr0 + BOXH > a.grp_rows && fr0 < a.flat_rows) {
                mbar_wait(&bars[slot], (prod_seq / NS) & 1u);
                for (int off = 0; off < BOXH; ++off) {
                    const long long fr = fr0 + off;
                    if (fr < a.grp_rows || fr >= a.flat_rows) continue;
                    const float *src = a.in + fr * a.in_pitch;
                    const int c0 = pt.x0 + BOX0 - ((int(fr & (G - 1)) * int(a.in_pitch)) & 3);
                    float *d = dst + grp_row<G>(off);
                    for (int c = lane; c < BOXWG; c += 32)
                        if (c0 + c >= 0 && c0 + c < a.W) d[c] = src[c0 + c];
                }
                fence_proxy_async();       // before TMA refills this slot
                __syncwarp();
            }
        } else if (TMA) {
            if (lane == 0) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&bars[slot], uint32_t(NBOX * BOXH * BOXW * sizeof(float)));
                tma_load_3d(dst, &a.tmap, pt.x0 + BOX0, r0 - a.in_row0, pt.img, &bars[slot]);
                if (NBOX == 2)
                    tma_load_3d(dst + Lay<TMA>::SUB, &a.tmap, pt.x0 + BOX1, r0 - a.in_row0, pt.img, &bars[slot]);
            }
        } else {
            // Unaligned rows the row-grouped loader does not take (a base
            // pointer that is not 16-byte aligned, batched images with gaps,
            // the literal / adapted arithmetic variants):
            // one 1-D bulk copy per box row (cp.async.bulk, 16-byte granules)
            // of the 140 floats from the row's 16-byte-aligned address at or
            // below column x0 + BOX0 (the consumer re-derives the shift).  Lane
            // i < NBOX * BOXH copies row i.  The bulk copies stay inside the
            // 16-byte-aligned part [lo16, hi16) of the buffer [in, in_end); the
            // row's lane copies the < 16-byte head [in, lo16) and tail
            // [hi16, in_end) with plain loads before lane 0's arrive (bytes left
            // of `in` are never read: they lie left of the image).  Rows outside
            // the buffer are not copied.
            const float *img_in = a.in + (long long)pt.img * a.in_img_stride;
            const uintptr_t lo = reinterpret_cast<uintptr_t>(a.in);
            const uintptr_t hi = reinterpret_cast<uintptr_t>(a.in_end);
            const uintptr_t lo16 = (lo + 15) & ~uintptr_t(15);     // bulk copies stay inside [lo16, hi16)
            const uintptr_t hi16 = hi & ~uintptr_t(15);
            uint32_t my_bytes = 0;
            uintptr_t my_src = 0;
            float *my_dst = nullptr;
            if (lane < NBOX * BOXH) {
                const int bx = lane / BOXH, rr = lane - bx * BOXH;
                const int br = r0 + rr - a.in_row0;
                if (br >= 0 && br < a.in_rows) {
                    const float *rowp = img_in + (long long)br * a.in_pitch + (pt.x0 + (bx ? BOX1 : BOX0));
                    uintptr_t st = reinterpret_cast<uintptr_t>(rowp) & ~uintptr_t(15);
                    uintptr_t en = st + 4 * Lay<false>::RP;
                    float *d = dst + bx * Lay<false>::SUB + rr * Lay<false>::RP;
                    if (st < lo16) {                // at the buffer start: [lo, lo16) by plain loads
                        for (uintptr_t q = (st > lo ? st : lo); q < lo16 && q < en; q += 4)
                            d[(q - st) / 4] = *reinterpret_cast<const float *>(q);
                        d += (lo16 - st) / 4;
                        st = lo16;
                    }
                    if (en > hi16) en = hi16;       // the < 16-byte tail: lane 0 below
                    if (en > st) {
                        my_bytes = uint32_t(en - st);
                        my_src = st;
                        my_dst = d;
                    }
                    if (hi > hi16 && reinterpret_cast<uintptr_t>(rowp) + 4 * Lay<false>::RP > hi16 &&
                        reinterpret_cast<uintptr_t>(rowp) < hi) {
                        // this row reaches into the unaligned tail of the buffer
                        const uintptr_t st0 = reinterpret_cast<uintptr_t>(rowp) & ~uintptr_t(15);
                        float *dt = dst + bx * Lay<false>::SUB + rr * Lay<false>::RP + (hi16 - st0) / 4;
                        const float *tail = reinterpret_cast<const float *>(hi16);
                        const uintptr_t room = Lay<false>::RP - (hi16 - st0) / 4;    // stay inside the smem row
                        const uintptr_t nt = (hi - hi16) / 4 < room ? (hi - hi16) / 4 : room;
                        for (uintptr_t k = 0; k < nt; ++k) dt[k] = tail[k];
                    }
                }
            }
            // total bytes of the stage (warp sum), posted by lane 0 with its arrival
            uint32_t total = my_bytes;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
            // plain smem stores of the tail must be visible to the async proxy / consumers
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive_expect_tx(&bars[slot], total);
            if (my_bytes) bulk_copy_g2s(my_dst, reinterpret_cast<const void *>(my_src), my_bytes, &bars[slot]);
        }
        ++pt_j;
        ++prod_seq;
    };

    // prologue: fill the ring
    for (int i = 0; i < NS; ++i) issue_next();

    // ---- consumer: tiles in the order the producer fetched them
    while (tq_head < tq_tail) {
        int t_id = -1;
#pragma unroll
        for (int i = 0; i <= NS; ++i)
            if (i == tq_head % (NS + 1)) t_id = tq[i];
        ++tq_head;
        const Tile T = decode_tile(a, t_id);
        const int x0 = T.x0;
        const int img = T.img;
        const bool edge = (x0 == 0) || ((x0 >> 1) + SLAB / 2 >= Wq - 1);

        const int mq0 = (x0 >> 1) + QPL * lane;
        EdgeFlags ef;
        ef.evenW = (a.W & 1) == 0;
        ef.last = (Wq - 1 - mq0 >= 0 && Wq - 1 - mq0 < QPL) ? Wq - 1 - mq0 : -1;
        ef.left_edge = (x0 == 0) && (lane == 0);
        const int nL = imax(0, imin(QPL, Wq - mq0));
        const int nH = imax(0, imin(QPL, Wh - mq0));

        const bool top = (T.qa == 0);
        const int r_first = tile_row0(T);
        const int n_first = top ? 0 : T.qa - 1;
        const int npairs = T.qb - n_first;
        const bool bottom = (T.qb == Hq);
        const int nst = tile_stages(T);
        const float *img_in = a.in + (long long)img * a.in_img_stride;

        // output cursors (all subbands advance one row per quad row)
        const int orow = T.qa - a.out_q0;
        float *pll = a.ll + (long long)img * a.ll_img_stride + (long long)orow * a.ll_pitch + mq0;
        const long long ob = (long long)img * a.out_img_stride + (long long)orow * a.out_pitch + mq0;
        float *phl = a.hl + ob, *plh = a.lh + ob, *phh = a.hh + ob;

        Carry cy;
        RowD E;
        for (int j = 0; j < nst; ++j) {
            const uint32_t k = cons_seq++;
            const float *slot = ring + int(k % NS) * RingG<TMA, GG, NS>::STAGE;
#ifdef DWT2_PROF
            const long long tw = clock64();
#endif
            mbar_wait(&bars[k % NS], (k / NS) & 1u);
#ifdef DWT2_PROF
            t_wait += clock64() - tw;
#endif
            // GRP: buffer row class of stage row 0 (the shift of row `off` is
            // ((cls0 + off) mod G) P mod 4 floats)
            const int cls0 = GRP ? (int)(((long long)img * a.in_rows + (r_first + j * ROWS - a.in_row0)) & (GG - 1)) : 0;
            const int p4 = int(a.in_pitch & 3);
            auto rowp = [&](int off) -> const float * {
                const float *p = slot + (GRP ? grp_row<GG>(off) : off * Lay<TMA>::RP);
                if (GRP) p += (((cls0 + off) & (GG - 1)) * p4) & 3;
                if (!TMA) {
                    const int br = r_first + j * ROWS + off - a.in_row0;
                    if (br >= 0 && br < a.in_rows) {
                        const float *g = img_in + (long long)br * a.in_pitch + (x0 + BOX0);
                        p += int((reinterpret_cast<uintptr_t>(g) >> 2) & 3);
                    }
                }
                return p;
            };
            auto body = [&](auto edge_tag) {
                constexpr bool EG = decltype(edge_tag)::value;
                if (j == 0) E = load_row<TMA && !GRP, EG>(rowp(0), lane, ef, true);
                const int k0 = j * PAIRS;
                const int kend = imin(k0 + PAIRS, npairs);
                const bool has_special_end = bottom && (kend == npairs);
                if ((j > 0 || (!top && a.unroll_first)) && kend - k0 == PAIRS && !has_special_end) {
                    // steady state: PAIRS regular pairs, fully unrolled; the first
                    // stage of a tile below the top starts with its carry-in pair
                    // (quad row qa - 1: carries only, nothing stored)
                    const bool cin0 = (j == 0);
#pragma unroll
                    for (int i = 0; i < PAIRS; ++i) {
                        const RowD O = load_row<TMA && !GRP, EG>(rowp(2 * i + 1), lane, ef, false);
                        const RowD N = load_row<TMA && !GRP, EG>(rowp(2 * i + 2), lane, ef, true);
                        const bool cin = (i == 0) && cin0;
                        const Out o = predict_update<EG, AR>(E, O, N, cy, lane, ef, cin, false);
                        if (cin) {
                            E = N;
                            continue;
                        }
                        storeq<VEC, EG>(pll, o.A, nL, false);
                        storeq<VEC, EG>(phl, o.B, nH, true);
                        storeq<VEC, EG>(plh, o.C, nL, true);
                        storeq<VEC, EG>(phh, o.D, nH, true);
                        pll += a.ll_pitch; phl += a.out_pitch; plh += a.out_pitch; phh += a.out_pitch;
                        E = N;
                    }
                } else {
                    for (int kk = k0; kk < kend; ++kk) {
                        const int i = kk - k0;
                        const int n = n_first + kk;
                        const bool last = bottom && (kk == npairs - 1);
                        const bool has_odd = !last || (2 * n + 1 <= a.H - 1);
                        const bool has_next = !last || (2 * n + 2 <= a.H - 1);
                        RowD O, N;
                        if (has_odd) {
                            O = load_row<TMA && !GRP, EG>(rowp(2 * i + 1), lane, ef, false);
                            N = has_next ? load_row<TMA && !GRP, EG>(rowp(2 * i + 2), lane, ef, true)
                                         : E;        // even H: x[H] := x[H-2]
                        } else {
                            O = E;                   // odd H: row 2n+1 is missing
                            N = E;
                        }
                        // carry-in pair: quad row qa-1 (or row -1 mirroring row 0 at the top)
                        const bool cin = (kk == 0);
                        const Out o = predict_update<EG, AR>(E, O, N, cy, lane, ef, cin, !has_odd);
                        if (!(cin && !top)) {
                            storeq<VEC, true>(pll, o.A, nL, false);
                            storeq<VEC, true>(phl, o.B, nH, true);
                            if (n < Hh) {
                                storeq<VEC, true>(plh, o.C, nL, true);
                                storeq<VEC, true>(phh, o.D, nH, true);
                            }
                            pll += a.ll_pitch; phl += a.out_pitch; plh += a.out_pitch; phh += a.out_pitch;
                        }
                        E = N;
                    }
                }
            };
            if (edge) body(std::integral_constant<bool, true>());
            else body(std::integral_constant<bool, false>());
            // stage consumed: its slot takes the next stage of the sequence
            __syncwarp();
            issue_next();
        }
    }
    if (DWT2_PROBE_NOWAIT && a.nowait) pdl_wait();
#ifdef DWT2_PROF
    if (lane == 0) {
        atomicAdd(&g_prof[0], (unsigned long long)t_wait);
        atomicAdd(&g_prof[1], (unsigned long long)(clock64() - t_work));
        atomicAdd(&g_prof[2], (unsigned long long)cons_seq);
    }
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_cta[blockIdx.x][2] = gtimer();
#endif
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
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

typedef void (*KernelFn)(LevelArgs);

// the 3-stage product kernel of large levels (3-D TMA loader, grouped arithmetic)
// peer strip launches (peer.cu; their buffers always take the 3-D TMA loader)
KernelFn kernel_peer(bool large, bool vec)
{
    if (large)
        return vec ? dwt53_level_kernel<true, true, AR_GROUPED, 1, S_LARGE, true>
                   : dwt53_level_kernel<true, false, AR_GROUPED, 1, S_LARGE, true>;
    return vec ? dwt53_level_kernel<true, true, AR_GROUPED, 1, S, true> : dwt53_level_kernel<true, false, AR_GROUPED, 1, S, true>;
}

// the 3-stage row-grouped kernel of large levels with pitches that are not a multiple of 16 bytes
KernelFn kernel_large_grp(bool vec, int gg)
{
    if (gg == 2) return vec ? dwt53_level_kernel<true, true, AR_GROUPED, 2, S_LARGE> : dwt53_level_kernel<true, false, AR_GROUPED, 2, S_LARGE>;
    return vec ? dwt53_level_kernel<true, true, AR_GROUPED, 4, S_LARGE> : dwt53_level_kernel<true, false, AR_GROUPED, 4, S_LARGE>;
}

KernelFn kernel_large(bool vec)
{
    return vec ? dwt53_level_kernel<true, true, AR_GROUPED, 1, S_LARGE> : dwt53_level_kernel<true, false, AR_GROUPED, 1, S_LARGE>;
}

template <int AR>
KernelFn kernel_for_ar(bool tma, bool vec)
{
    if (tma) return vec ? dwt53_level_kernel<true, true, AR, 1> : dwt53_level_kernel<true, false, AR, 1>;
    return vec ? dwt53_level_kernel<false, true, AR, 1> : dwt53_level_kernel<false, false, AR, 1>;
}

// grp: the row-grouped TMA loader (product arithmetic only; the literal /
// adapted variants keep the bulk-copy loader for such pitches)
KernelFn kernel_for(bool tma, bool vec, int ar = AR_GROUPED, int gg = 1)
{
    if (gg == 2) return vec ? dwt53_level_kernel<true, true, AR_GROUPED, 2> : dwt53_level_kernel<true, false, AR_GROUPED, 2>;
    if (gg == 4) return vec ? dwt53_level_kernel<true, true, AR_GROUPED, 4> : dwt53_level_kernel<true, false, AR_GROUPED, 4>;
    if (ar == AR_LITERAL) return kernel_for_ar<AR_LITERAL>(tma, vec);
    if (ar == AR_ADAPTED) return kernel_for_ar<AR_ADAPTED>(tma, vec);
    return kernel_for_ar<AR_GROUPED>(tma, vec);
}

}  // namespace


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
    const PeerBoundaryArgs *peer;   // fused peer strip launch (else null) and its boundary-role CTAs
    int peer_ctas;
};

// Tile-size policy of the work queue (measured on B200).
// A -DDWT2_TUNING build reads DWT2_TPW, DWT2_MIN_TB, ... from the environment
// for sweeps (tuning_int, read once per process); the product build does not.
struct TilePolicy {
    int tpw;       // target tiles per warp on large levels
    int min_tb;    // minimum quad rows per tile
    int min_tpw;   // below this many tiles per warp: one tile per warp, no queue
    int guided;    // mid-size levels: large tiles first, small ones last (DWT2_GUIDED=0 disables)
    int guided_a;  // percent of the rows in the large (one per warp) tiles
    int guided_b;  // small tiles per warp for the rest
    int tb_large;  // tile height of large levels (0: off)
    int large_tpw; // a level is large from this many tiles per warp at tb_large
};

const TilePolicy &tile_policy()
{
    static TilePolicy pol;
    static std::once_flag once;
    std::call_once(once, [] {
        pol.tpw = tuning_int("DWT2_TPW", DWT2_TPW, 1, 1024);
        pol.min_tb = tuning_int("DWT2_MIN_TB", MIN_TILE_ROWS, PAIRS - 1, MAX_TILE_ROWS);
        pol.min_tpw = tuning_int("DWT2_MIN_TPW", DWT2_MIN_TPW, 1, 1024);
        pol.guided = tuning_int("DWT2_GUIDED", 1, 0, 1);
        pol.guided_a = tuning_int("DWT2_GUIDED_A", 60, 10, 90);   // cold-cache sweep: 55-60 > 70 > 80 on 4096^2 .. 16384 x 2048
        pol.guided_b = tuning_int("DWT2_GUIDED_B", 4, 1, 64);
        pol.tb_large = tuning_int("DWT2_TB_LARGE", 15, 0, MAX_TILE_ROWS);
        pol.large_tpw = tuning_int("DWT2_LARGE_TPW", 9, 1, 1024);
    });
    return pol;
}

int32_t launch_level(const dwt2_plan *p, int level, int W, int H, const LaunchIO &io, int qa0, int qa1, int qb0,
                     int qb1, cudaStream_t stream, int queue = 0, int ar = AR_GROUPED)
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
    a.nslabs = (W + SLAB - 1) / SLAB;
    a.count = io.count;
    a.qa0 = qa0; a.qa1 = qa1; a.qb0 = qb0; a.qb1 = qb1;
    a.nowait = (DWT2_PROBE_NOWAIT && level >= 1 && queue == 0) ? 1 : 0;
    if (io.peer) {
        a.peer = 1;
        a.pb = *io.peer;
        a.pb_ctas = io.peer_ctas;
    }
    const int lenA = qa1 - qa0, lenB = qb1 - qb0;
    const long long slab_rows = (long long)io.count * a.nslabs * (lenA + lenB);
    if (slab_rows == 0) return io.peer ? fail(DWT2_EINVAL) : DWT2_OK;      // peer.cu launches no empty level

    const bool tma = !DWT2_FORCE_GENERIC && aligned(io.in, 16) && (io.in_pitch * 4) % 16 == 0 &&
                     (io.count == 1 || (io.in_img_stride * 4) % 16 == 0);
    // other pitches: row-grouped TMA when the images are contiguous rows of
    // one 16-byte-aligned buffer, else the bulk-copy loader
    const int glog = (io.in_pitch % 4 == 0) ? 0 : (io.in_pitch % 2 == 0 ? 1 : 2);
    const long long flat_rows = (long long)io.count * io.in_rows;
    const bool grp = !tma && !DWT2_FORCE_GENERIC && !DWT2_NO_GRP && NBOX == 1 && ar == AR_GROUPED && aligned(io.in, 16) &&
                     (io.count == 1 || io.in_img_stride == io.in_pitch * io.in_rows) &&
                     (io.in_pitch << glog) < (1LL << 30) && (flat_rows >> glog) >= 1 &&
                     io.in + flat_rows * io.in_pitch <= io.in_end;
    const int va = (QPL == 4) ? 16 : 8;        // subband store width in bytes
    const bool vec = !DWT2_FORCE_SCALAR && aligned(a.ll, va) && aligned(a.hl, va) && aligned(a.lh, va) && aligned(a.hh, va) &&
                     io.ll_pitch % QPL == 0 && io.out_pitch % QPL == 0 &&
                     (io.count == 1 || (io.ll_img_stride % QPL == 0 && io.out_img_stride % QPL == 0));
    if (level < 0 || level >= MAX_LEVELS) return fail(DWT2_EINVAL);
    dwt2_plan::TmapCache &tc = p->tcache[level];
    a.glog = grp ? glog : 0;
    a.flat_rows = flat_rows;
    a.grp_rows = grp ? (flat_rows >> glog) << glog : 0;
    if ((tma || grp) && tc.in == io.in && tc.pitch == io.in_pitch && tc.stride == io.in_img_stride && tc.W == W &&
        tc.rows == io.in_rows && tc.count == io.count && tc.grp == grp) {
        a.tmap = tc.map;                      // same input tensor as the last launch of this level
        a.tmap_b = tc.map_b;
    } else if (grp) {
        PFN_cuTensorMapEncodeTiled_v12000 enc = get_encode();
        if (!enc) return fail(DWT2_ECUDA);
        const int G = 1 << glog;
        cuuint64_t dims[3] = {(cuuint64_t)(io.in_pitch * G), (cuuint64_t)(flat_rows >> glog), 1};
        cuuint64_t strides[2] = {(cuuint64_t)(io.in_pitch * G * 4), (cuuint64_t)(io.in_pitch * G * 4)};
        cuuint32_t estr[3] = {1, 1, 1};
        for (int m = 0; m < 2; ++m) {
            const int h = m == 0 ? (BOXH + G - 1) / G : BOXH / G;
            cuuint32_t box[3] = {(cuuint32_t)BOXWG, (cuuint32_t)h, 1};
            CUresult r = enc(m == 0 ? &a.tmap : &a.tmap_b, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                             const_cast<float *>(io.in), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, DWT2_L2_PROMOTION, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(DWT2_ECUDA);
        }
        tc.in = io.in; tc.pitch = io.in_pitch; tc.stride = io.in_img_stride;
        tc.W = W; tc.rows = io.in_rows; tc.count = io.count; tc.grp = true;
        tc.map = a.tmap;
        tc.map_b = a.tmap_b;
    } else if (tma) {
        PFN_cuTensorMapEncodeTiled_v12000 enc = get_encode();
        if (!enc) return fail(DWT2_ECUDA);
        cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)io.in_rows, (cuuint64_t)io.count};
        long long img_bytes = io.count > 1 ? io.in_img_stride * 4 : round_up(io.in_pitch * 4 * io.in_rows, 16);
        cuuint64_t strides[2] = {(cuuint64_t)(io.in_pitch * 4), (cuuint64_t)img_bytes};
        cuuint32_t box[3] = {(cuuint32_t)BOXW, (cuuint32_t)BOXH, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = enc(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(io.in), dims, strides,
                         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         DWT2_L2_PROMOTION, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(DWT2_ECUDA);
        tc.in = io.in; tc.pitch = io.in_pitch; tc.stride = io.in_img_stride;
        tc.W = W; tc.rows = io.in_rows; tc.count = io.count; tc.grp = false;
        tc.map = a.tmap;
    }

    // Grid of independent warps, each streaming tiles of tb quad rows x one
    // slab.  Large levels: a persistent grid pulls ~4 tiles per warp from the
    // work queue (load balance).  Small levels (at most one tile per resident
    // warp): tile w goes to warp w, no queue.  tb + 1 pairs (incl. the
    // carry-in pair) fill whole stages.
    const int max_ctas = p->max_ctas[tma || grp ? 1 : 0];
    const long long warps_full = (long long)max_ctas * WARPS;
    const TilePolicy &pol = tile_policy();
    long long tb = slab_rows / ((long long)pol.tpw * warps_full);
    const bool large = pol.tb_large > 0 && slab_rows >= (long long)pol.large_tpw * pol.tb_large * warps_full;
    static const int use_s3 = tuning_int("DWT2_LARGE_S3", 1, 0, 1);
    const bool s3 = use_s3 && large && tma && ar == AR_GROUPED;      // the 3-stage kernel (S_LARGE)
    static const int use_s3g = tuning_int("DWT2_LARGE_S3G", 1, 0, 1);
    const bool s3g = use_s3 && use_s3g && large && grp && ar == AR_GROUPED && p->max_ctas[3] > 0;   // its GRP form
    if (large) {
        // large levels (>= large_tpw tiles per warp at tb_large quad rows):
        // tb_large, measured best from 16384 x 6144 up -- 16384 x 8192 (a
        // config-3 strip at G = 2): 0.82 -> 0.96 of copy against 11-row
        // tiles; config 5's batch: 571 -> 602 Gpix/s against 55-row ones;
        // 16384^2 unchanged (tpw already gave 15).  Smaller levels keep the
        // rules below (8192^2: 11-row tiles 0.93, 15-row 0.88).
        tb = pol.tb_large;
    }
    if (tb < pol.min_tb) {
        // fewer than tpw tiles per warp even at the minimum tile height: keep
        // the minimum height (queue balancing) while that still gives every
        // warp at least min_tpw tiles, else one tile per warp (small levels)
        tb = pol.min_tb;
        if (slab_rows / (tb * warps_full) < pol.min_tpw) tb = (slab_rows + warps_full - 1) / warps_full;
    }
    tb = std::max<long long>(PAIRS - 1, std::min<long long>(MAX_TILE_ROWS, tb));
    tb = std::max<long long>(PAIRS - 1, (tb + 1 + PAIRS - 1) / PAIRS * PAIRS - 1);
    a.tb = int(tb);
    a.tb_b = int(tb);
    a.nblk_a = (lenA + a.tb - 1) / a.tb;
    a.nblk = a.nblk_a + (lenB + a.tb - 1) / a.tb;
    // Guided tiles for mid-size levels (few tiles per warp): one large tile
    // per warp over ~60 % of the rows first, then the rest as ~4 small tiles
    // per warp from the queue, so warps on slower SMs (a 1.5x spread of SM
    // throughput under full HBM load) do not set the kernel's length, while
    // most rows still pay the carry-in row of a large tile only.
    static const int guided_max_tpw = tuning_int("DWT2_GUIDED_MAXTPW", 8, 1, 1024);
    if (pol.guided && io.count == 1 && lenB == 0 && slab_rows >= 16LL * warps_full &&
        slab_rows / ((long long)a.tb * warps_full) < guided_max_tpw) {
        const long long nblk_a = std::max<long long>(1, warps_full / a.nslabs);
        long long tb_a = (pol.guided_a * lenA / 100) / nblk_a;
        tb_a = (tb_a + 1) / PAIRS * PAIRS - 1;                       // tb + 1 whole stages, rounded down
        if (tb_a >= 2 * PAIRS - 1 && nblk_a * tb_a < lenA) {
            const long long rows_a = nblk_a * tb_a, rest = lenA - rows_a;     // rest > 0
            long long tb_b = rest * a.nslabs / ((long long)pol.guided_b * warps_full);
            static const int min_b = tuning_int("DWT2_GUIDED_MINB", 2, 1, 16);
            tb_b = std::max<long long>(min_b * PAIRS - 1, (tb_b + 1 + PAIRS - 1) / PAIRS * PAIRS - 1);
            a.tb = int(tb_a);
            a.tb_b = int(std::min<long long>(tb_b, MAX_TILE_ROWS));
            a.qa1 = int(qa0 + rows_a);
            a.qb0 = a.qa1;
            a.qb1 = qa1;
            a.nblk_a = int(nblk_a);
            a.nblk = a.nblk_a + int((rest + a.tb_b - 1) / a.tb_b);
        }
    }
    const long long ntiles = (long long)io.count * a.nblk * a.nslabs;
    if (ntiles >= (1LL << 31)) return fail(DWT2_EINVAL);
    a.ntiles = int(ntiles);
    a.fd_slabs = make_fastdiv(unsigned(a.nslabs));
    a.fd_img = make_fastdiv(unsigned(a.nblk * a.nslabs));
    const long long want_ctas = (ntiles + WARPS - 1) / WARPS;
    const int grid = int(std::max<long long>(1, std::min<long long>(s3 ? p->max_ctas[2] : s3g ? p->max_ctas[3] : max_ctas,
                                                                    want_ctas)));
    a.nwarps = grid * WARPS;
    a.static_tiles = ntiles <= a.nwarps ? 1 : 0;
    // the first stage of a tile on the unrolled path: measured faster on
    // guided (mid-size) levels, one-tile-per-warp levels and on the
    // row-grouped loader (4096^2 0.79 -> 0.85, 16384 x 2048 0.85 -> 0.87,
    // 2048^2 0.55 -> 0.60, 8193^2 0.85 -> 0.87, 4095 x 3001 0.60 -> 0.68) but
    // slower on large 3-D TMA levels (8192^2 0.94 -> 0.83, 16384^2 0.98 ->
    // 0.97), for reasons not established; DWT2_UNROLL_FIRST=0/1 forces it (tuning builds)
    static const int env_uf = tuning_int("DWT2_UNROLL_FIRST", -1, 0, 1);
    a.unroll_first = env_uf >= 0 ? env_uf : ((a.tb_b != a.tb || a.qb1 > a.qb0 || grp || a.static_tiles) ? 1 : 0);
    a.counter = p->counters + 2 * ((queue ? QUEUE_STRIP_BOUNDARY : QUEUE_FORWARD) + level);
    // reverse order on every other level of a pyramid: level k + 1 then starts
    // on the LL rows level k wrote last, still in L2 (config 4: level 2 reads
    // 64 -> 53 MB from DRAM, the step 142.8 -> 141.3 us; scripts/r2/gpu_rev.sh)
    static const int rev_mode = tuning_int("DWT2_REV", 1, 0, 1);
    if (rev_mode && (level & 1) && (lenB == 0 || qb0 == qa1)) {
        a.rev = 1;
        a.rsum = qa0 + (lenB ? qb1 : qa1);
    }

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid + a.pb_ctas);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = grp ? (s3g ? RingG<true, 2, S_LARGE>::SMEM : RingG<true, 2>::SMEM)
                               : s3 ? Ring<true, S_LARGE>::SMEM : tma ? Ring<true>::SMEM : Ring<false>::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    KernelFn fn = s3 ? kernel_large(vec) : s3g ? kernel_large_grp(vec, 1 << glog)
                                          : kernel_for(tma || grp, vec, ar, grp ? 1 << glog : 1);
    if (io.peer) {
        if (!tma || ar != AR_GROUPED) return fail(DWT2_EINVAL);        // peer.cu buffers are TMA-aligned
        fn = kernel_peer(s3, vec);
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

int32_t configure_kernels(int *max_ctas)
{
    static int cached[4] = {0, 0, 0, 0};
    static std::once_flag once;
    static int32_t status = DWT2_OK;
    std::call_once(once, [] {
        KernelFn fns[4] = {kernel_for(true, true), kernel_for(true, false), kernel_for(false, true),
                           kernel_for(false, false)};
        for (int ar = AR_LITERAL; ar <= AR_ADAPTED; ++ar)
            for (int t = 0; t < 4; ++t) {
                const size_t smem = t < 2 ? Ring<true>::SMEM : Ring<false>::SMEM;
                if (cudaFuncSetAttribute(kernel_for(t < 2, (t & 1) == 0, ar), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem)) != cudaSuccess) {
                    status = DWT2_ECUDA;
                    return;
                }
            }
        for (int v = 0; v < 4; ++v)
            if (cudaFuncSetAttribute(kernel_for(true, (v & 1) == 0, AR_GROUPED, v < 2 ? 2 : 4),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(RingG<true, 2>::SMEM)) != cudaSuccess) {
                status = DWT2_ECUDA;
                return;
            }
        int dev = 0, sms = 0, per_sm = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
            status = DWT2_ECUDA;
            return;
        }
        for (int i = 0; i < 4; ++i) {
            const size_t smem = i < 2 ? Ring<true>::SMEM : Ring<false>::SMEM;
            if (cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) {
                status = DWT2_ECUDA;
                return;
            }
        }
        for (int t = 0; t < 2; ++t) {   // t = 1: TMA kernels
            const size_t smem = t ? Ring<true>::SMEM : Ring<false>::SMEM;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[t ? 0 : 2], THREADS, smem) != cudaSuccess ||
                per_sm < 1) {
                status = DWT2_ECUDA;
                return;
            }
            cached[t] = sms * per_sm;
        }
        for (int v = 0; v < 2; ++v)
            if (cudaFuncSetAttribute(kernel_large(v == 0), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(Ring<true, S_LARGE>::SMEM)) != cudaSuccess ||
                cudaFuncSetAttribute(kernel_peer(true, v == 0), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(Ring<true, S_LARGE>::SMEM)) != cudaSuccess ||
                cudaFuncSetAttribute(kernel_peer(false, v == 0), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(Ring<true>::SMEM)) != cudaSuccess) {
                status = DWT2_ECUDA;
                return;
            }
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_large(true), THREADS,
                                                          Ring<true, S_LARGE>::SMEM) != cudaSuccess || per_sm < 1) {
            status = DWT2_ECUDA;
            return;
        }
        cached[2] = sms * per_sm;
        for (int v = 0; v < 4; ++v)
            if (cudaFuncSetAttribute(kernel_large_grp((v & 1) == 0, v < 2 ? 2 : 4), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(RingG<true, 2, S_LARGE>::SMEM)) != cudaSuccess) {
                status = DWT2_ECUDA;
                return;
            }
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_large_grp(true, 4), THREADS,
                                                          RingG<true, 2, S_LARGE>::SMEM) != cudaSuccess || per_sm < 1) {
            status = DWT2_ECUDA;
            return;
        }
        cached[3] = sms * per_sm;
    });
    cudaGetLastError();
    max_ctas[0] = cached[0];
    max_ctas[1] = cached[1];
    max_ctas[2] = cached[2];
    max_ctas[3] = cached[3];
    return status;
}

dwt2_plan *make_plan(int W, int H, int levels, int boundary, int max_count, bool strip, int Hg, int rb, int re,
                     int wavelet = DWT2_WAVELET_CDF53)
{
    if (wavelet < DWT2_WAVELET_CDF53 || wavelet > DWT2_WAVELET_LIFTING || (strip && wavelet != DWT2_WAVELET_CDF53)) {
        g_last_error = wavelet < 0 || wavelet > DWT2_WAVELET_LIFTING ? DWT2_EINVAL : DWT2_EUNSUPPORTED;
        return nullptr;
    }
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
    p->wavelet = wavelet;
    p->device = dev;
    p->sms = prop.multiProcessorCount;
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
    int32_t st = configure_kernels(p->max_ctas);
    if (st != DWT2_OK) {
        delete p;
        g_last_error = st;
        return nullptr;
    }
    // work-queue counters (zeroed once; every launch leaves them zeroed)
    const size_t cbytes = sizeof(unsigned int) * 2 * MAX_COUNTERS;
    if (cudaMalloc(&p->counters, cbytes) != cudaSuccess || cudaMemset(p->counters, 0, cbytes) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        cudaGetLastError();
        if (p->counters) cudaFree(p->counters);
        delete p;
        g_last_error = DWT2_ENOMEM;
        return nullptr;
    }
    p->scratch_bytes += cbytes;
    // LL scratch: level k (1-based, k < levels) writes LL_k to scratch[(k-1) % 2]
    for (int s = 0; s < 2; ++s) {
        if (!strip && levels >= s + 2) {   // strip plans: the caller owns every level's buffers
            const LevelGeom &g = p->geom[s];  // LL of level s+1
            p->sc_pitch[s] = round_up(g.Wq, 32);
            p->sc_img_stride[s] = p->sc_pitch[s] * g.Hq;
            size_t bytes = size_t(p->sc_img_stride[s]) * max_count * sizeof(float);
            if (cudaMalloc(&p->scratch[s], bytes) != cudaSuccess) {
                cudaGetLastError();
                if (p->scratch[0]) cudaFree(p->scratch[0]);
                cudaFree(p->counters);
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

}  // namespace

namespace dwt2_detail {

thread_local int32_t g_last_error = DWT2_OK;

// Checked on every call (no cache: a freed and re-used address must not pass
// on the strength of an earlier check).
bool on_plan_device(const dwt2_plan *p, const void *ptr)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) && at.device == p->device;
}

}  // namespace dwt2_detail

namespace {

// The small last levels of a forward as one tail launch (tail.cu).
int32_t launch_tail(const dwt2_plan *p, int first, int n, const LaunchIO *ios, cudaStream_t stream)
{
    TailLevelIO lv[MAX_TAIL];
    for (int k = 0; k < n; ++k) {
        const LevelGeom &g = p->geom[first + k];
        const LaunchIO &io = ios[k];
        lv[k] = TailLevelIO{io.in, io.in_pitch, io.in_img_stride, io.ll, io.ll_pitch, io.ll_img_stride,
                            io.out, io.out_pitch, io.out_img_stride, g.W, g.H};
    }
    return launch_tail_levels(p, lv, n, ios[0].count, tail_filter_53(), stream);
}

// First level of [first, last] that starts the tail launch (last + 1: none).
int tail_start(const dwt2_plan *p, int count, int first, int last)
{
    // measured (config 4): levels of <= 256^2 input (16384 quads) 141.2 -> 140.5 us; adding the
    // 512^2 level changes nothing, adding 1024^2 is slower (145.4); a 512^2 one-level image (config 1)
    // is faster on the level kernel (3.9 vs 4.4 us per call)
    static const int tail_quads = tuning_int("DWT2_TAIL_QUADS", 1 << 14, 0, 1 << 30);
    return tail_start_levels(p, count, first, last, tail_quads);
}

// Launch geometry of level k of a forward of `count` images: level 0 reads
// `in`, level k >= 1 the LL scratch of level k-1; the last level's LL goes to
// `out`, the others' to scratch (ping-pong).
LaunchIO level_io(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                  long long out_stride, int k)
{
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
    return io;
}

// Levels that run on the small-level kernel (tail.cu launch_small_level) when
// they are not in the tail launch.  Measured (scripts/r2/small_probe.py, graph
// of 20 calls): a single 512^2 level 4.05 -> 3.74 us (2^16 quads), 1024^2
// 5.34 -> 5.87 us (slower from a cold input); inside a pyramid, where a
// level's input is the LL just written (in L2), the 1024^2 level pays too:
// config 4 139.3 -> 137.7 us, 4b 150.7 -> 148.9 with levels of <= 2^18 quads.
bool small_level(const dwt2_plan *p, int k, int count)
{
    static const long long small_first = tuning_int("DWT2_SMALL_QUADS", 1 << 16, 0, 1 << 30);
    static const long long small_ll = tuning_int("DWT2_SMALL_QUADS_LL", 1 << 18, 0, 1 << 30);
    return count <= 65535 &&          // images go to gridDim.y
           (long long)p->geom[k].Wq * p->geom[k].Hq * count <= (k == 0 ? small_first : small_ll);
}

// Forward of levels [first, last] for `count` images.  Level 1 reads `in`.
// Level-1 quad rows may be restricted to [q1a, q1b) (host pipelining).  The
// small last levels (tail_start) run as one tail launch, the others one
// level-kernel launch each.
int32_t run_levels(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                   long long out_stride, int first, int last, int q1a, int q1b, cudaStream_t s, int ar = AR_GROUPED)
{
    const bool restricted0 = (first == 0) && (q1a != 0 || q1b != p->geom[0].Hq);
    const int t0 = (ar == AR_GROUPED) ? std::max(tail_start(p, count, first, last), first + (restricted0 ? 1 : 0))
                                      : last + 1;
    for (int k = first; k <= last; ++k) {
        if (k == t0) {
            LaunchIO tios[MAX_TAIL];
            for (int j = 0; j <= last - k; ++j) tios[j] = level_io(p, in, out, count, in_stride, out_stride, k + j);
            return launch_tail(p, k, last - k + 1, tios, s);
        }
        const LevelGeom &g = p->geom[k];
        const LaunchIO io = level_io(p, in, out, count, in_stride, out_stride, k);
        int qa = 0, qb = g.Hq;
        if (k == 0) {
            qa = q1a;
            qb = q1b;
        }
        // small levels (whole level, product arithmetic): the shared-memory
        // tiled pointwise kernel (tail.cu) instead of the row-walking level kernel
        if (ar == AR_GROUPED && qa == 0 && qb == g.Hq && small_level(p, k, count)) {
            const TailLevelIO lv{io.in, io.in_pitch, io.in_img_stride, io.ll, io.ll_pitch, io.ll_img_stride,
                                 io.out, io.out_pitch, io.out_img_stride, g.W, g.H};
            int32_t r = launch_small_level(lv, count, s);
            if (r != DWT2_OK) return r;
            continue;
        }
        int32_t r = launch_level(p, k, g.W, g.H, io, qa, qb, 0, 0, s, 0, ar);
        if (r != DWT2_OK) return r;
    }
    return DWT2_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

// Measurement builds only (-DDWT2_PROF): per-CTA timestamps; not in dwt2.h.
int32_t dwt2_debug_cta(unsigned long long *out, int32_t n)
{
#ifdef DWT2_PROF
    return cudaMemcpyFromSymbol(out, g_cta, sizeof(unsigned long long) * 4 * n) == cudaSuccess ? DWT2_OK : DWT2_ECUDA;
#else
    (void)out; (void)n;
    return DWT2_EUNSUPPORTED;
#endif
}

// Measurement builds only (-DDWT2_PROF): per-warp cycle counters; not in dwt2.h.
int32_t dwt2_debug_prof(unsigned long long *out4, int32_t reset)
{
#ifdef DWT2_PROF
    if (cudaMemcpyFromSymbol(out4, g_prof, sizeof(unsigned long long) * 4) != cudaSuccess) return DWT2_ECUDA;
    if (reset) {
        unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    }
    return DWT2_OK;
#else
    (void)out4; (void)reset;
    return DWT2_EUNSUPPORTED;
#endif
}

dwt2_plan *dwt2_plan_create(int32_t width, int32_t height, int32_t levels, int32_t boundary)
{
    return make_plan(width, height, levels, boundary, 1, false, height, 0, height);
}

dwt2_plan *dwt2_plan_create_ex(int32_t width, int32_t height, int32_t levels, int32_t boundary, int32_t wavelet,
                               int32_t max_count)
{
    return make_plan(width, height, levels, boundary, max_count, false, height, 0, height, wavelet);
}

dwt2_plan *dwt2_plan_create_lifting(int32_t width, int32_t height, int32_t levels, int32_t boundary,
                                    const double *coeffs, double K, int32_t max_count)
{
    if (!coeffs || !(K > 0.0) || !std::isfinite(K)) {
        g_last_error = DWT2_EINVAL;
        return nullptr;
    }
    for (int i = 0; i < 4; ++i)
        if (!std::isfinite(coeffs[i])) {
            g_last_error = DWT2_EINVAL;
            return nullptr;
        }
    dwt2_plan *p = make_plan(width, height, levels, boundary, max_count, false, height, 0, height,
                             DWT2_WAVELET_LIFTING);
    if (!p) return nullptr;
    for (int i = 0; i < 4; ++i) p->lift[i] = coeffs[i];
    p->lift[4] = K;
    return p;
}

dwt2_plan *dwt2_plan_create_batched(int32_t width, int32_t height, int32_t levels, int32_t boundary,
                                    int32_t max_count)
{
    return make_plan(width, height, levels, boundary, max_count, false, height, 0, height);
}

int32_t dwt2_forward(const dwt2_plan *p, const float *in, float *out, dwt2_stream_t stream)
{
    if (!p || !in || !out || p->strip || !aligned(in, 4) || !aligned(out, 4)) return fail(DWT2_EINVAL);
    const size_t bytes = size_t(p->W) * p->H * sizeof(float);
    if (overlap(in, bytes, out, bytes) || !on_plan_device(p, in) || !on_plan_device(p, out))
        return fail(DWT2_EINVAL);
    if (p->wavelet != DWT2_WAVELET_CDF53) {
        int32_t r = run_levels_k2(p, in, out, 1, (long long)p->W * p->H, (long long)p->W * p->H,
                                  reinterpret_cast<cudaStream_t>(stream));
        if (r == DWT2_OK) g_last_error = DWT2_OK;
        return r;
    }
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
    if (p->wavelet != DWT2_WAVELET_CDF53) {
        int32_t r = run_levels_k2(p, in, out, count, in_stride, out_stride, reinterpret_cast<cudaStream_t>(stream));
        if (r == DWT2_OK) g_last_error = DWT2_OK;
        return r;
    }
    int32_t r = run_levels(p, in, out, count, in_stride, out_stride, 0, p->levels - 1, 0, p->geom[0].Hq,
                           reinterpret_cast<cudaStream_t>(stream));
    if (r != DWT2_OK) return r;
    g_last_error = DWT2_OK;
    return DWT2_OK;
}

dwt2_plan *dwt2_plan_create_strip_levels(int32_t width, int32_t global_height, int32_t row_begin, int32_t row_end,
                                         int32_t levels, int32_t boundary)
{
    if (levels < 1 || levels > 30 || global_height < 2 || row_begin < 0 || row_begin >= row_end ||
        row_end > global_height) {
        g_last_error = DWT2_EINVAL;
        return nullptr;
    }
    const long long unit = 1LL << levels;
    if ((row_begin % unit) != 0 || ((row_end % unit) != 0 && row_end != global_height)) {
        g_last_error = DWT2_EINVAL;
        return nullptr;
    }
    // geometry is validated on the full image (every level input >= 2 x 2)
    dwt2_plan *p = make_plan(width, global_height, levels, boundary, 1, true, global_height, row_begin, row_end);
    if (!p) return nullptr;
    // every level's strip must hold >= 2 rows (the halo messages send 2 rows)
    for (int k = 0; k < levels; ++k) {
        dwt2_strip_level_t L;
        dwt2_strip_level_info(p, k, &L);
        if (L.row_end - L.row_begin < 2) {
            dwt2_destroy(p);
            g_last_error = DWT2_EINVAL;
            return nullptr;
        }
    }
    return p;
}

dwt2_plan *dwt2_plan_create_strip(int32_t width, int32_t global_height, int32_t row_begin, int32_t row_end,
                                  int32_t boundary)
{
    return dwt2_plan_create_strip_levels(width, global_height, row_begin, row_end, 1, boundary);
}

int32_t dwt2_strip_level_info(const dwt2_plan *p, int32_t level, dwt2_strip_level_t *info)
{
    if (!p || !info || !p->strip || level < 0 || level >= p->levels) return fail(DWT2_EINVAL);
    // rows [rb_k, re_k) of level k's input: rb_k = row_begin / 2^k, re_k = ceil(re_{k-1} / 2)
    int rb = p->row_begin, re = p->row_end;
    for (int k = 0; k < level; ++k) {
        rb >>= 1;
        re = (re + 1) >> 1;
    }
    const LevelGeom &g = p->geom[level];
    info->width = g.W;
    info->global_height = g.H;
    info->row_begin = rb;
    info->row_end = re;
    info->ghost_top = rb > 0 ? 2 : 0;
    info->ghost_bot = re < g.H ? 1 : 0;
    return DWT2_OK;
}

}  // extern "C"

namespace dwt2_detail {

int32_t strip_level_launch(const dwt2_plan *p, int level, const float *in, long long in_pitch, float *ll_out,
                           long long ll_pitch, float *out, int part, cudaStream_t stream,
                           const PeerBoundaryArgs *peer, int peer_ctas)
{
    dwt2_strip_level_t L;
    if (!p || !in || !out || !p->strip || part < 0 || part > 2 || !aligned(in, 4) || !aligned(out, 4) ||
        dwt2_strip_level_info(p, level, &L) != DWT2_OK || in_pitch < L.width)
        return fail(DWT2_EINVAL);
    const bool last = level == p->levels - 1;
    if (!last && (!ll_out || !aligned(ll_out, 4) || ll_pitch < (L.width + 1) / 2)) return fail(DWT2_EINVAL);
    const int rows = L.row_end - L.row_begin;
    const int in_rows = rows + L.ghost_top + L.ghost_bot;
    const int hloc0 = p->row_end - p->row_begin;          // strip-local pyramid: W x hloc0, pitch W
    const size_t in_bytes = size_t(in_pitch) * in_rows * sizeof(float);
    const size_t out_bytes = size_t(p->W) * hloc0 * sizeof(float);
    if (overlap(in, in_bytes, out, out_bytes) || !on_plan_device(p, in) || !on_plan_device(p, out))
        return fail(DWT2_EINVAL);
    if (!last) {
        const size_t ll_bytes = size_t(ll_pitch) * ((rows + 1) / 2) * sizeof(float);
        if (overlap(in, in_bytes, ll_out, ll_bytes) || overlap(out, out_bytes, ll_out, ll_bytes) ||
            !on_plan_device(p, ll_out))
            return fail(DWT2_EINVAL);
    }
    const int qs = L.row_begin / 2, qe = (L.row_end + 1) / 2;
    LaunchIO io;
    memset(&io, 0, sizeof(io));
    io.count = 1;
    io.in = in;
    io.in_pitch = in_pitch;
    io.in_img_stride = (long long)in_pitch * in_rows;
    io.in_row0 = L.row_begin - L.ghost_top;
    io.in_rows = in_rows;
    io.in_end = in + (long long)in_pitch * in_rows;
    io.out = out;
    io.out_pitch = p->W;
    io.out_img_stride = (long long)p->W * hloc0;
    io.out_q0 = qs;
    io.hq_local = qe - qs;
    if (last) {
        io.ll = out;
        io.ll_pitch = p->W;
    } else {
        io.ll = ll_out;
        io.ll_pitch = ll_pitch;
    }
    io.ll_img_stride = io.ll_pitch * (qe - qs);
    io.peer = peer;
    io.peer_ctas = peer_ctas;
    const int ia = qs + (L.ghost_top ? 1 : 0), ib = qe - (L.ghost_bot ? 1 : 0);
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
    // BOUNDARY launches use their own work-queue counters, so they may run on
    // another stream concurrently with the INTERIOR launch of the same level
    int32_t r = launch_level(p, level, L.width, L.global_height, io, a0, a1, b0, b1, stream,
                             part == DWT2_STRIP_BOUNDARY ? 1 : 0);
    if (r != DWT2_OK) return r;
    g_last_error = DWT2_OK;
    return DWT2_OK;
}

int level_kernel_threads() { return THREADS; }

// a boundary-role CTA of a fused peer launch stages 5 rows of 2 THREADS + 4 floats in the ring's smem
static_assert(5 * (2 * THREADS + 4) * sizeof(float) <= Ring<false>::SMEM, "boundary role tile exceeds the ring");

}  // namespace dwt2_detail

extern "C" {

int32_t dwt2_forward_strip_level(const dwt2_plan *p, int32_t level, const float *in, int64_t in_pitch,
                                 float *ll_out, int64_t ll_pitch, float *out, int32_t part, dwt2_stream_t stream)
{
    return strip_level_launch(p, level, in, in_pitch, ll_out, ll_pitch, out, part,
                              reinterpret_cast<cudaStream_t>(stream));
}

int32_t dwt2_forward_strip(const dwt2_plan *p, const float *in, float *out, int32_t part, dwt2_stream_t stream)
{
    if (!p || !p->strip || p->levels != 1) return fail(DWT2_EINVAL);
    return dwt2_forward_strip_level(p, 0, in, p->W, nullptr, 0, out, part, stream);
}

}  // extern "C"

namespace {

// Releases whatever host_staging_create acquired (any subset) and marks the
// plan as having no staging (d_in == nullptr).
void host_staging_release(const dwt2_plan *p)
{
    if (p->d_in) cudaFree(p->d_in);
    if (p->d_out) cudaFree(p->d_out);
    if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
    if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
    for (int i = 0; i < 132; ++i)
        if (p->ev[i]) cudaEventDestroy(p->ev[i]);
    p->d_in = p->d_out = nullptr;
    p->s_h2d = p->s_d2h = nullptr;
    for (int i = 0; i < 132; ++i) p->ev[i] = nullptr;
    cudaGetLastError();
}

// All-or-nothing: device staging buffers, the copy streams and the events of
// dwt2_forward_host.  On failure nothing stays allocated and d_in stays null.
int32_t host_staging_create(const dwt2_plan *p, long long npx)
{
    int32_t code = DWT2_OK;
    if (cudaMalloc(&p->d_in, npx * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&p->d_out, npx * sizeof(float)) != cudaSuccess)
        code = DWT2_ENOMEM;
    else if (cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
             cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking) != cudaSuccess)
        code = DWT2_ECUDA;
    for (int i = 0; code == DWT2_OK && i < 132; ++i)
        if (cudaEventCreateWithFlags(&p->ev[i], cudaEventDisableTiming) != cudaSuccess) code = DWT2_ECUDA;
    if (code != DWT2_OK) host_staging_release(p);
    return code;
}

}  // namespace

extern "C" {

int32_t dwt2_forward_host(const dwt2_plan *p, const float *host_in, float *host_out, dwt2_stream_t stream)
{
    if (!p || !host_in || !host_out || p->strip || p->max_count != 1) return fail(DWT2_EINVAL);
    if (p->wavelet != DWT2_WAVELET_CDF53) return fail(DWT2_EUNSUPPORTED);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const long long npx = (long long)p->W * p->H;
    if (!p->d_in) {
        int32_t st = host_staging_create(p, npx);
        if (st != DWT2_OK) return fail(st);
    }
    // Pipeline over NB row bands of level 1: H2D(band b) -> kernel on the
    // quad rows whose inputs have all arrived -> D2H of finished output rows.
    const LevelGeom &g = p->geom[0];
    static const int max_bands = tuning_int("DWT2_HOST_BANDS", 16, 1, 64);   // 16 = 32: 11.5 Gpix/s at config 3 (PCIe-bound)
    const int NB = std::min(max_bands, std::max(1, g.Hq / 64));
    const size_t rowb = size_t(p->W) * sizeof(float);
    cudaEvent_t *ev_in = p->ev, *ev_k = p->ev + 64, *ev_done = p->ev + 128;
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
                // level-1 LH|HH rows and the HL part of the LL|HL rows are final
                // at once; only the LL quadrant waits for the coarser levels
                cudaStreamWaitEvent(p->s_d2h, ev_k[b], 0);
                const size_t hlb = size_t(p->W - g.Wq) * sizeof(float);
                if (hlb > 0)
                    cudaMemcpy2DAsync(host_out + (long long)q_done * p->W + g.Wq, rowb,
                                      p->d_out + (long long)q_done * p->W + g.Wq, rowb, hlb, qe - q_done,
                                      cudaMemcpyDeviceToHost, p->s_d2h);
                const int h0 = std::min(q_done, p->H / 2), h1 = std::min(qe, p->H / 2);
                if (h1 > h0)
                    cudaMemcpyAsync(host_out + (long long)(g.Hq + h0) * p->W, p->d_out + (long long)(g.Hq + h0) * p->W,
                                    rowb * (h1 - h0), cudaMemcpyDeviceToHost, p->s_d2h);
            }
            q_done = qe;
        }
    }
    if (p->levels > 1) {
        int32_t r = run_levels(p, p->d_in, p->d_out, 1, npx, npx, 1, p->levels - 1, 0, 0, s);
        if (r != DWT2_OK) return r;
        cudaEventRecord(ev_done[1], s);
        cudaStreamWaitEvent(p->s_d2h, ev_done[1], 0);
        // the level-1 LL quadrant, now the Mallat pyramid of the coarser levels
        cudaMemcpy2DAsync(host_out, rowb, p->d_out, rowb, size_t(g.Wq) * sizeof(float), g.Hq,
                          cudaMemcpyDeviceToHost, p->s_d2h);
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
    if (p->counters) cudaFree(p->counters);
    for (int s = 0; s < 2; ++s)
        if (p->scratch[s]) cudaFree(p->scratch[s]);
    if (p->work) cudaFree(p->work);
    host_staging_release(p);
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
    if (!p->strip) {
        // the small last levels run as one tail launch (run_levels, run_levels_k2)
        const int t0 = p->wavelet == DWT2_WAVELET_CDF53 ? tail_start(p, p->max_count, 0, p->levels - 1)
                                                        : k2_tail_start(p, p->max_count);
        if (t0 < p->levels) info->launches_per_forward = t0 + 1;
    }
    int tma = 0;
    long long bytes = 0;
    const int t0 = p->strip ? p->levels
                            : (p->wavelet == DWT2_WAVELET_CDF53 ? tail_start(p, p->max_count, 0, p->levels - 1)
                                                                 : k2_tail_start(p, p->max_count));
    for (int k = 0; k < p->levels; ++k) {
        const LevelGeom &g = p->geom[k];
        // level kernel levels (not the tail launch, not the small-level kernel);
        // level 1 reads the caller's buffer: TMA iff its rows are 16-byte aligned
        const bool level_kernel = k < t0 && (p->strip || p->wavelet != DWT2_WAVELET_CDF53 ||
                                             !small_level(p, k, p->max_count));
        if (level_kernel && p->wavelet == DWT2_WAVELET_CDF53 && (k > 0 || (p->W % 4) == 0)) ++tma;
        long long rows = g.H;
        if (p->strip) {
            dwt2_strip_level_t L;
            dwt2_strip_level_info(p, k, &L);
            rows = L.row_end - L.row_begin;
        }
        bytes += 8LL * g.W * rows;
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
    case DWT2_ETIMEOUT: return "peer flag wait timed out";
    default: return "unknown error";
    }
}

const char *dwt2_version(void) { return "dwt2-b200 0.1 sm_100a (non-separable lifting, CDF 5/3)"; }

}  // extern "C"

namespace dwt2_detail {

int32_t forward_fused_variant(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                              long long out_stride, int variant, cudaStream_t s)
{
    return run_levels(p, in, out, count, in_stride, out_stride, 0, p->levels - 1, 0, p->geom[0].Hq, s,
                      variant == 1 ? AR_LITERAL : AR_ADAPTED);
}

}  // namespace dwt2_detail
