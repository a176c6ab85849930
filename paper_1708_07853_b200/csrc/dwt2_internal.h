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
    int max_ctas[3];          // resident CTAs of the forward kernels: [0] cp.async, [1] TMA, [2] TMA 3-stage (large levels)
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
constexpr int PEER_EPOCH = 0;        // the rank's step epoch (advanced by the level-0 INTERIOR launch)
constexpr int PEER_DONE = 1;         // epoch whose last-level BOUNDARY launch has finished reading the neighbours
constexpr int PEER_ERR = 2;          // nonzero: a flag wait timed out
constexpr int PEER_CTR = 3;          // BOUNDARY CTAs finished (last level; self-resetting)
constexpr int PEER_READY = 8;        // + k: epoch whose level-k input rows are final
constexpr int PEER_FLAG_WORDS = PEER_READY + MAX_LEVELS;

#ifdef __CUDACC__
// Publish "level `level` input rows of this rank are final for the current
// epoch" (one thread, after griddepcontrol.wait: every earlier launch of the
// rank's step has completed and its writes are visible).  Level 0 advances
// the epoch.  The system-scope fence makes those writes visible to a peer GPU
// that acquires the flag over NVLink before it reads the rows.
__device__ __forceinline__ void peer_publish_ready(unsigned int *f, int level)
{
    volatile unsigned int *vf = f;
    unsigned e = vf[PEER_EPOCH];
    if (level == 0) vf[PEER_EPOCH] = ++e;
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f + PEER_READY + level), "r"(e) : "memory");
}
#endif

// a one-thread launch of peer_publish_ready (strips whose INTERIOR part is empty)
int32_t launch_peer_publish(unsigned int *flags, int level, cudaStream_t stream);

// dwt2_forward_strip_level with an optional peer flag block (peer.cu INTERIOR parts)
int32_t strip_level_launch(const dwt2_plan *p, int level, const float *in, long long in_pitch, float *ll_out,
                           long long ll_pitch, float *out, int part, cudaStream_t stream, unsigned int *peer_flags);

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
