// dwt2_internal.h -- state shared by the translation units behind the C ABI
// of include/dwt2.h (forward level kernel: dwt2.cu; inverse: inverse.cu;
// kernel-per-step scheme variants: schemes.cu).  Not installed, not part of
// the ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "../../include/dwt2.h"

namespace dwt2_detail {

constexpr int MAX_LEVELS = 32;

// Work-queue counter pairs in dwt2_plan::counters (each level kernel's
// self-resetting tile queue, see queue.cuh), by slot base + level:
constexpr int QUEUE_FORWARD = 0;                  // forward level kernels (5/3 or K = 2)
constexpr int QUEUE_STRIP_BOUNDARY = MAX_LEVELS;  // strip BOUNDARY launches (may overlap INTERIOR)
constexpr int QUEUE_INVERSE = 2 * MAX_LEVELS;     // inverse level kernels
constexpr int QUEUE_TAIL = 3 * MAX_LEVELS;        // tail kernel: [0] grid-barrier arrivals, [1] CTAs done
constexpr int QUEUE_SLOTS = 3 * MAX_LEVELS + 1;

// Division by a launch-constant divisor without the integer-divide sequence
// (decode_tile runs twice per tile; ncu had its two divisions at 3.5 % of the
// kernel's instructions): q = (umulhi(n, mul) + n) >> shift for n < 2^31
// (Granlund & Montgomery's round-up multiplier; d = 1: mul = shift = 0).
struct FastDiv {
    unsigned mul, shift;
};

inline FastDiv make_fastdiv(unsigned d)
{
    FastDiv f{0u, 0u};
    if (d > 1) {
        unsigned sh = 0;
        while ((1ull << sh) < d) ++sh;
        f.shift = sh;
        f.mul = unsigned(((1ull << 32) * ((1ull << sh) - d)) / d + 1);
    }
    return f;
}

__device__ __forceinline__ int fdiv(int n, FastDiv f)
{
    return int((__umulhi(unsigned(n), f.mul) + unsigned(n)) >> f.shift);
}

// Tile-policy knobs for measurement sweeps.  Only a -DDWT2_TUNING build
// (build/variants, _build.build_variant) reads them from the environment, and
// only inside [lo, hi]; the product library always uses the measured defaults,
// so its performance does not depend on the caller's environment.
inline int tuning_int(const char *name, int dflt, int lo, int hi)
{
#ifdef DWT2_TUNING
    if (const char *v = getenv(name)) {
        const int x = atoi(v);
        if (x >= lo && x <= hi) return x;
    }
#endif
    (void)name; (void)lo; (void)hi;
    return dflt;
}

struct LevelGeom {
    int W, H;            // level input size
    int Wq, Hq;          // LL size: ceil(W / 2) x ceil(H / 2)
};

extern thread_local int32_t g_last_error;

inline int32_t fail(int32_t code)
{
    g_last_error = code;
    return code;
}

inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

inline long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }

inline bool overlap(const void *a, size_t an, const void *b, size_t bn)
{
    const char *x = static_cast<const char *>(a), *y = static_cast<const char *>(b);
    return x < y + bn && y < x + an;
}

}  // namespace dwt2_detail

struct dwt2_plan {
    int W, H, levels, max_count;
    int wavelet;              // DWT2_WAVELET_*: CDF53 runs the fused 5/3 kernel (dwt2.cu), others dwt97.cu
    double lift[5];           // DWT2_WAVELET_LIFTING: p1, u1, p2, u2, K
    int device;
    // strip plans
    bool strip;
    int Hg, row_begin, row_end, ghost_top, ghost_bot;
    // geometry and scratch: level k (0-based) has input geom[k]; the LL of
    // level k < levels-1 lives in scratch[k % 2] (pitch sc_pitch, per-image
    // stride sc_img_stride).  The inverse reuses the same buffers: the
    // reconstructed input of level k >= 1 goes to scratch[(k - 1) % 2].
    dwt2_detail::LevelGeom geom[dwt2_detail::MAX_LEVELS];
    float *scratch[2];
    long long sc_pitch[2], sc_img_stride[2];
    size_t scratch_bytes;
    int max_ctas[4];          // resident CTAs of the forward kernels: [0] cp.async, [1] TMA, [2] TMA 3-stage (large
                              // levels), [3] row-grouped TMA 3-stage (large levels of pitches not a multiple of 16 B)
    int sms;                  // multiprocessors of the plan's device
    unsigned int *counters;   // per level: tile queue + finished-warp counter (device, self-resetting)
    // host-side caches (the API serialises calls on one plan)
    struct TmapCache {
        const float *in;
        long long pitch, stride;
        int W, rows, count;
        bool grp;                           // map / map_b: row-grouped maps (dwt2.cu, GRP loader)
        CUtensorMap map, map_b;
    };
    mutable TmapCache tcache[dwt2_detail::MAX_LEVELS];
    // scheme variants (schemes.cu): one full-size work buffer, allocated lazily
    mutable float *work;
    mutable size_t work_bytes;
    // host e2e staging
    mutable float *d_in, *d_out;
    mutable cudaStream_t s_h2d, s_d2h;
    mutable cudaEvent_t ev[132];      // host e2e: 64 band-arrived, 64 band-done, 4 sync
};

namespace dwt2_detail {

// ---- peer strip contexts (peer.cu): flag block layout (uint32 words)
constexpr int PEER_EPOCH = 0;        // the rank's step epoch (advanced by the first launch of level 0)
constexpr int PEER_DONE = 1;         // epoch whose last level has finished reading the neighbours
constexpr int PEER_ERR = 2;          // nonzero: a flag wait timed out
constexpr int PEER_CTR = 3;          // boundary-role CTAs of the current launch that finished (self-resetting)
constexpr int PEER_READY = 8;        // + k: epoch whose level-k input rows are final
constexpr int PEER_FLAG_WORDS = PEER_READY + MAX_LEVELS;

// The boundary quad rows of one level of a peer strip (the first and / or the
// last quad row of the strip, whose 5 x 5 windows reach into the neighbours'
// rows), computed by boundary-role CTAs: the CTAs past the level kernel's own
// grid in a fused launch, or the whole grid of peer.cu's boundary kernel.
struct PeerBoundaryArgs {
    const float *own;                 // global row rb of this rank (level k)
    const float *up;                  // global row rb - 2 in the rank above (null: none)
    const float *dn;                  // global row re in the rank below (null: none)
    long long own_pitch, up_pitch, dn_pitch;
    const unsigned int *up_flags, *dn_flags;
    unsigned int *flags;              // this rank's flag block
    float *ll;                        // LL row of quad row qs
    float *hl, *lh, *hh;              // subband rows of quad row qs (strip-local output)
    long long ll_pitch, out_pitch;
    long long timeout_ns;
    int W, H, rb, re, qs;
    int n0, n1;                       // the boundary quad rows (global)
    int nbx;                          // boundary-role CTAs per boundary quad row
    int nroles;                       // boundary-role CTAs of the launch
    int level, last;                  // last: the strip's last level (publishes done)
    int quiesce;                      // last level: wait until the neighbours are done reading this rank
};

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long peer_gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned peer_ld_acquire_sys(const unsigned int *p)
{
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void peer_st_release_sys(unsigned int *p, unsigned v)
{
#ifdef DWT2_PEER_FENCE_GPU      // probe builds only: device-scope release (ranks on one GPU)
    asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else
    asm volatile("fence.acq_rel.sys;\n\tst.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}

// Publish "level `level` input rows of this rank are final for the current
// epoch": one thread of the first launch of the level, after
// griddepcontrol.wait (every earlier launch of the rank's step has completed
// and its writes are visible; the system-scope release carries them to a peer
// GPU that acquires the flag over NVLink).  The first publish of level 0 in a
// step (epoch == done) advances the epoch; publishing again is a no-op.
static __device__ __noinline__ void peer_publish(unsigned int *f, int level)
{
    volatile unsigned int *vf = f;
    unsigned e = vf[PEER_EPOCH];
    if (level == 0 && e == vf[PEER_DONE]) vf[PEER_EPOCH] = ++e;
    peer_st_release_sys(f + PEER_READY + level, e);
}

// spin until *f >= e (epochs compared modulo 2^32); latches PEER_ERR and gives
// up after timeout_ns (no hang if a neighbour never arrives)
static __device__ __noinline__ void peer_wait_epoch(const unsigned int *f, unsigned e, const PeerBoundaryArgs &a)
{
    const unsigned long long t0 = peer_gtime();
    while (int(peer_ld_acquire_sys(f) - e) < 0) {
        if ((long long)(peer_gtime() - t0) > a.timeout_ns) {
            atomicExch(a.flags + PEER_ERR, 1u);
            return;
        }
        __nanosleep(100);
    }
}

// this step's epoch: once the level-0 publish of the step has run, epoch =
// done + 1 (a boundary-role CTA of level 0 may start before the CTA that
// publishes; it waits for it)
static __device__ __noinline__ unsigned peer_epoch(const PeerBoundaryArgs &a)
{
    volatile const unsigned int *vf = a.flags;
    const unsigned long long t0 = peer_gtime();
    unsigned e;
    while ((e = vf[PEER_EPOCH]) != vf[PEER_DONE] + 1u) {
        if ((long long)(peer_gtime() - t0) > a.timeout_ns) {
            atomicExch(a.flags + PEER_ERR, 1u);
            break;
        }
        __nanosleep(100);
    }
    return e;
}

// whole-sample symmetric reflection for k in [-2, n + 1], n >= 2
__device__ __forceinline__ int peer_wss2(int k, int n)
{
    k = k < 0 ? -k : k;
    return k >= n ? 2 * (n - 1) - k : k;
}

// One boundary-role CTA: blockDim.x quads of boundary quad row (by ? n1 : n0)
// from quad bx * blockDim.x.  tile: 5 x (2 blockDim.x + 4) floats of smem.
// Waits (thread 0) for the neighbours' level-k ready flags, stages the 5 input
// rows -- the neighbours' from their memory -- and evaluates the 2-D analysis
// filters pointwise: h = (-1/8, 1/4, 3/4, 1/4, -1/8) at even, g = (-1/2, 1, -1/2)
// at odd positions, row pass then column pass in fp64 (Eq. (4), PAPER.md
// L160-171, which the lifting steps of Eq. (5) reach exactly: every product and
// sum here is exact for fp32 data, so the stored fp32 is the level kernel's).
static __device__ __noinline__ void peer_boundary_role(const PeerBoundaryArgs &a, int bx, int by, float *tile)
{
    const int nt = blockDim.x, cols = 2 * nt + 4;
    if (threadIdx.x == 0) {
        const unsigned e = peer_epoch(a);
        if (a.up_flags) peer_wait_epoch(a.up_flags + PEER_READY + a.level, e, a);
        if (a.dn_flags) peer_wait_epoch(a.dn_flags + PEER_READY + a.level, e, a);
    }
    __syncthreads();
    const int n = by == 0 ? a.n0 : a.n1;
    const int W = a.W, H = a.H;
    const int Wq = (W + 1) >> 1, Wh = W >> 1, Hh = H >> 1;
    const int m0 = bx * nt;
    const int c0 = 2 * m0 - 2;
    // every load of the thread in flight at once (one memory round trip; a
    // load / smem-store loop paid one round trip per element: ~10 us per CTA)
    float v[5][3];                        // cols <= 3 nt for nt >= 4
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int y = peer_wss2(2 * n - 2 + j, H);
        const float *row = y < a.rb ? a.up + (long long)(y - (a.rb - 2)) * a.up_pitch
                         : y >= a.re ? a.dn + (long long)(y - a.re) * a.dn_pitch
                                     : a.own + (long long)(y - a.rb) * a.own_pitch;
#pragma unroll
        for (int it = 0; it < 3; ++it) {
            const int i = threadIdx.x + it * nt, x = c0 + i;
            v[j][it] = (i < cols && x <= W + 1) ? __ldcg(row + peer_wss2(x, W)) : 0.f;
        }
    }
#pragma unroll
    for (int j = 0; j < 5; ++j)
#pragma unroll
        for (int it = 0; it < 3; ++it) {
            const int i = threadIdx.x + it * nt;
            if (i < cols) tile[j * cols + i] = v[j][it];
        }
    __syncthreads();
    const int m = m0 + threadIdx.x;
    if (m < Wq) {
        double lo[5], hi[5];              // row passes: h at column 2m, g at column 2m + 1
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const float *v = tile + j * cols + 2 * threadIdx.x;
            const double v0 = v[0], v1 = v[1], v2 = v[2], v3 = v[3], v4 = v[4];
            lo[j] = fma(0.75, v2, fma(0.25, v1 + v3, -0.125 * (v0 + v4)));
            hi[j] = fma(-0.5, v2 + v4, v3);
        }
        const double ll = fma(0.75, lo[2], fma(0.25, lo[1] + lo[3], -0.125 * (lo[0] + lo[4])));
        const double lh = fma(-0.5, lo[2] + lo[4], lo[3]);
        const double hl = fma(0.75, hi[2], fma(0.25, hi[1] + hi[3], -0.125 * (hi[0] + hi[4])));
        const double hh = fma(-0.5, hi[2] + hi[4], hi[3]);
        const long long r = n - a.qs;
        a.ll[r * a.ll_pitch + m] = (float)ll;
        if (m < Wh) a.hl[r * a.out_pitch + m] = (float)hl;
        if (n < Hh) {
            a.lh[r * a.out_pitch + m] = (float)lh;
            if (m < Wh) a.hh[r * a.out_pitch + m] = (float)hh;
        }
    }
}

// A boundary-role CTA has finished (all its stores and neighbour reads, after
// a __syncthreads; one thread).  On the strip's last level the last role CTA
// of the launch publishes done = epoch and, for concurrent ranks, waits until
// both neighbours are done reading this rank's buffers.
static __device__ __noinline__ void peer_exit(const PeerBoundaryArgs &a)
{
    if (!a.last) return;
    __threadfence();
    if (atomicAdd(a.flags + PEER_CTR, 1u) + 1u != unsigned(a.nroles)) return;
    atomicExch(a.flags + PEER_CTR, 0u);
    __threadfence();
    const unsigned e = *reinterpret_cast<volatile unsigned int *>(a.flags + PEER_EPOCH);
    peer_st_release_sys(a.flags + PEER_DONE, e);
    if (a.quiesce) {
        if (a.up_flags) peer_wait_epoch(a.up_flags + PEER_DONE, e, a);
        if (a.dn_flags) peer_wait_epoch(a.dn_flags + PEER_DONE, e, a);
    }
}
#endif

// threads per CTA of the level kernel (quads of a boundary-role CTA in a fused launch)
int level_kernel_threads();

// dwt2_forward_strip_level; with `peer` (peer.cu) the level kernel publishes
// the level's ready flag at entry and its grid gets peer_ctas more CTAs in the
// boundary role
int32_t strip_level_launch(const dwt2_plan *p, int level, const float *in, long long in_pitch, float *ll_out,
                           long long ll_pitch, float *out, int part, cudaStream_t stream,
                           const PeerBoundaryArgs *peer = nullptr, int peer_ctas = 0);

// ---- tail kernel (tail.cu): the small last levels of a forward in one launch
constexpr int MAX_TAIL = 16;

struct TailLevelIO {
    const float *in;
    long long in_pitch, in_img;       // level input rows and images (floats)
    float *ll;
    long long ll_pitch, ll_img;       // LL destination
    float *out;
    long long out_pitch, out_img;     // Mallat base of this level's HL / LH / HH
    int W, H;                         // level input size (each >= 2)
};

struct TailFilter {
    int radius;                       // 2: CDF 5/3 (exact path); 4: K <= 2 lifting filters below
    double h[9], g[7];                // low taps at offsets -4..4, high taps at -3..3 (radius 4)
    double sll, sd, shh;              // output scaling (radius 4)
};

TailFilter tail_filter_53();
TailFilter tail_filter_from_lifting(double c0, double c1, double c2, double c3, double K);
// first level of [first, last] from which every level has <= max_quads quads over `count` images
int tail_start_levels(const dwt2_plan *p, int count, int first, int last, long long max_quads);
int32_t launch_tail_levels(const dwt2_plan *p, const TailLevelIO *lv, int n, int count, const TailFilter &f,
                           cudaStream_t stream);
// one small level of an inverse (tail.cu): the reconstructed W x H level input
// `out` from the level's LL plane and its HL / LH / HH in the Mallat buffer d
struct InvLevelIO {
    const float *ll;
    long long ll_pitch, ll_img;
    const float *d;                   // the Mallat pyramid (level subbands at their Mallat offsets)
    long long d_pitch, d_img;
    float *out;
    long long out_pitch, out_img;
    int W, H;                         // reconstructed size (each >= 2)
};
struct InvFilter {
    int radius;                       // 2: CDF 5/3 (dyadic taps: exact), 4: K <= 2 lifting pairs; 0: unsupported
    double s0[9], s1[9];              // low / high synthesis taps at offsets -4..4
    double kll, kd, khh;              // undo of the forward scaling
};
InvFilter inv_filter_from_lifting(double c0, double c1, double c2, double c3, double K);
int32_t launch_small_inverse_level(const InvLevelIO &lv, int count, const InvFilter &f, cudaStream_t stream);
// levels of an inverse that run on launch_small_inverse_level
bool small_inverse_level(const dwt2_plan *p, int k, int count);

// one small CDF 5/3 level in one launch of shared-memory-tiled pointwise CTAs (tail.cu)
int32_t launch_small_level(const TailLevelIO &lv, int count, cudaStream_t stream);
// one small level of a K <= 2 lifting wavelet (radius-4 filters f) in one launch (tail.cu)
int32_t launch_small_level_r4(const TailLevelIO &lv, int count, const TailFilter &f, cudaStream_t stream);

// true if ptr is device (or managed) memory of the plan's device
bool on_plan_device(const dwt2_plan *p, const void *ptr);

// forward of `count` images with the literal (variant 1) or adapted (2)
// arithmetic of the fused 5/3 kernel (dwt2.cu; schemes FUSED_LITERAL / _ADAPTED)
int32_t forward_fused_variant(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                              long long out_stride, int variant, cudaStream_t s);

// inverse of all levels through the K = 2 lifting kernel (dwt97.cu)
int32_t run_inverse_k2(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                       long long out_stride, cudaStream_t s);

// first level of a K = 2 forward that runs in the tail launch (levels: none)
int k2_tail_start(const dwt2_plan *p, int count);

// all levels through the K = 2 lifting kernel (dwt97.cu)
int32_t run_levels_k2(const dwt2_plan *p, const float *in, float *out, int count, long long in_stride,
                      long long out_stride, cudaStream_t s);

}  // namespace dwt2_detail
