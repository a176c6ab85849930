/*
 * dwt2.h -- C ABI of the B200-native forward 2-D CDF 5/3 DWT computed with
 * the non-separable lifting scheme of arXiv:1708.07853.
 *
 * Operation (section 3, Eq. (5)): one decomposition level
 * maps every 2x2 quad (a, b, c, d) = (x[2n][2m], x[2n][2m+1], x[2n+1][2m],
 * x[2n+1][2m+1]) to the four subband coefficients (LL, HL, LH, HH) by a
 * spatial predict followed by a spatial update,
 *
 *   predict  [1 0 0 0; P 1 0 0; P* 0 1 0; PP* P* P 1]
 *   update   [1 U U* UU*; 0 1 0 U*; 0 0 1 U; 0 0 0 1]
 *
 * with the CDF 5/3 lifting pair P = -1/2 (1 + z), U = 1/4 (1 + z^-1)
 * (coefficients SPEC.md L145).  In exact arithmetic the result
 * is the separable 2-D CDF 5/3 transform (tensor product of
 * 1-D transforms).  Boundaries: whole-sample symmetric extension (the paper
 * is silent).  Multi-level: the transform recurses on LL,
 * W_{k+1} = ceil(W_k / 2), H_{k+1} = ceil(H_k / 2) (BASELINE.json north_star).
 *
 * Layouts.  Images are fp32, row-major.  The output is the Mallat pyramid
 * (SPEC.md L358-366): level k writes, inside the W x H output with the
 * caller's row pitch,
 *     HL_k -> rows [0, ceil(H_k/2)),   cols [ceil(W_k/2), W_k)
 *     LH_k -> rows [ceil(H_k/2), H_k), cols [0, ceil(W_k/2))
 *     HH_k -> rows [ceil(H_k/2), H_k), cols [ceil(W_k/2), W_k)
 * and the last level's LL goes to rows [0, ceil(H_L/2)), cols
 * [0, ceil(W_L/2)).  HL is the horizontal high band (odd column, even row).
 *
 * Arithmetic: fp32 in HBM, fp64 in registers.  For
 * integer-valued inputs in [0, 255] the result is bit-exact at every level
 * that fits the fp32 mantissa (levels 1-2); otherwise every level's output is
 * the correctly rounded fp32 value of the exact level result.
 *
 * Execution: every call is asynchronous on the given CUDA stream (pass a
 * cudaStream_t; NULL = legacy default stream).  No host synchronisation, no
 * device allocation and no retained pointers inside dwt2_forward*, except
 * dwt2_forward_host (see there).  Concurrent calls that share one plan must
 * be serialised by the caller (the plan owns its LL scratch); distinct plans
 * are independent.  A plan is bound to the CUDA device current at creation.
 *
 * Errors: functions returning int32_t return DWT2_OK (0) or a negative code;
 * plan constructors return NULL and set a thread-local code readable with
 * dwt2_last_error().  Asynchronous kernel faults surface at the caller's next
 * synchronisation, as for any CUDA launch.
 */
#ifndef DWT2_H
#define DWT2_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque CUDA stream handle, ABI-identical to cudaStream_t. */
typedef struct CUstream_st *dwt2_stream_t;

typedef struct dwt2_plan dwt2_plan;

enum {
    DWT2_OK = 0,
    DWT2_EINVAL = -1,      /* bad argument: null, overlap, size, alignment, wrong device */
    DWT2_ENOMEM = -2,      /* device or pinned host allocation failed */
    DWT2_ECUDA = -3,       /* a CUDA runtime / driver call or a launch failed */
    DWT2_EUNSUPPORTED = -4 /* boundary mode other than SYMMETRIC, or device is not sm_100 */
};

enum { DWT2_BOUNDARY_SYMMETRIC = 0 }; /* whole-sample symmetric extension */

/* Wavelets (dwt2_plan_create_ex).  The paper evaluates CDF 5/3
 * and states the schemes are general (L39, L365-367). */
enum {
    DWT2_WAVELET_CDF53 = 0,    /* CDF 5/3, the fused non-separable kernel (the product path) */
    DWT2_WAVELET_CDF97 = 1,    /* CDF 9/7: Eq. (5) for K = 2 lifting pairs + scaling, one fused kernel per
                                  level; constants of Daubechies & Sweldens, JPEG 2000 normalisation
                                  (low / K, high * K; DESIGN.md C-B1..C-B3) */
    DWT2_WAVELET_CDF53_K2 = 2, /* CDF 5/3 through the K = 2 kernel (second pair = 0, K = 1): a cross-check */
    DWT2_WAVELET_LIFTING = 3   /* any wavelet of <= 2 symmetric lifting pairs (dwt2_plan_create_lifting) */
};

enum {                         /* dwt2_forward_strip `part` */
    DWT2_STRIP_ALL = 0,        /* every quad row of the strip */
    DWT2_STRIP_INTERIOR = 1,   /* quad rows that read no ghost row */
    DWT2_STRIP_BOUNDARY = 2,   /* the first and the last quad row (read ghost rows) */
    DWT2_STRIP_PUBLISH = 3     /* peer strips only: publish the level's ready flag (dwt2_peer_strip_level) */
};

/* Plan for a single W x H image, `levels` levels (1 <= levels, and every
 * level's input at least 2 x 2).  boundary must be DWT2_BOUNDARY_SYMMETRIC.
 * Allocates and owns the LL scratch of levels >= 2 on the current device.
 * Returns NULL on error (dwt2_last_error()). */
dwt2_plan *dwt2_plan_create(int32_t width, int32_t height, int32_t levels, int32_t boundary);

/* General plan: `wavelet` (DWT2_WAVELET_*), up to max_count images per
 * batched call.  Plans of a wavelet other than CDF53 support dwt2_forward and
 * dwt2_forward_batched only (others return DWT2_EUNSUPPORTED); their
 * arithmetic is fp64 in registers, fp32 in memory, so results match the
 * fp64 definition within fp32 rounding of each level's output. */
dwt2_plan *dwt2_plan_create_ex(int32_t width, int32_t height, int32_t levels, int32_t boundary, int32_t wavelet,
                               int32_t max_count);

/* Plan for a general lifting wavelet (SURVEY.md 8f N4 "general lifting
 * wavelets"): at most two predict / update pairs of the symmetric 2-tap form
 * of Eq. (2) and a scaling,
 *     predict k:  d[i] += p_k (s[i] + s[i+1])      (P = p_k (1 + z))
 *     update  k:  s[i] += u_k (d[i-1] + d[i])      (U = u_k (1 + z^-1))
 *     scaling:    low = s / K, high = d * K,
 * coeffs = {p1, u1, p2, u2} (host array, copied), K > 0 and finite; unused
 * pairs are 0.  Evaluated by the non-separable K = 2 kernel (dwt97.cu) as
 * DWT2_WAVELET_LIFTING; supports what DWT2_WAVELET_CDF97 plans support. */
dwt2_plan *dwt2_plan_create_lifting(int32_t width, int32_t height, int32_t levels, int32_t boundary,
                                    const double *coeffs, double K, int32_t max_count);

/* As dwt2_plan_create, with scratch for up to max_count images per
 * dwt2_forward_batched call (BASELINE.json config 5). */
dwt2_plan *dwt2_plan_create_batched(int32_t width, int32_t height, int32_t levels,
                                    int32_t boundary, int32_t max_count);

/* One-level plan for the row strip [row_begin, row_end) of a width x
 * global_height image (the paper's row bands, SPEC.md
 * L313-318).  row_begin must be even; row_end must be even or equal to
 * global_height; 0 <= row_begin < row_end <= global_height.
 * Input rows present in the `in` buffer of dwt2_forward_strip:
 *   2 ghost rows above the strip if row_begin > 0 (rows row_begin-2, -1),
 *   the strip rows, then 1 ghost row below if row_end < global_height.
 * Output: the strip-local Mallat layout of W x (row_end - row_begin): the
 * strip's quad rows of LL | HL over LH | HH. */
dwt2_plan *dwt2_plan_create_strip(int32_t width, int32_t global_height, int32_t row_begin,
                                  int32_t row_end, int32_t boundary);

/* Multi-level strip plan: `levels` levels of the row
 * strip [row_begin, row_end) of a width x global_height image, one halo
 * exchange per level.  row_begin must be a multiple of 2^levels, row_end a
 * multiple of 2^levels or equal to global_height, and every level's strip
 * must keep >= 2 rows.  Level k (0-based) transforms rows [rb_k, re_k) of
 * the level-k input (the LL of level k-1), rb_k = row_begin / 2^k,
 * re_k = ceil(re_{k-1} / 2); see dwt2_strip_level_info.  The plan owns no
 * image buffers: the caller provides each level's ghost-padded input.
 * dwt2_plan_create_strip is this with levels = 1. */
dwt2_plan *dwt2_plan_create_strip_levels(int32_t width, int32_t global_height, int32_t row_begin,
                                         int32_t row_end, int32_t levels, int32_t boundary);

/* Geometry of level k of a strip plan: the level's global input size
 * (width x global_height), the strip's rows [row_begin, row_end) of it, and
 * the ghost rows its input buffer carries (2 above unless row_begin == 0,
 * 1 below unless row_end == global_height). */
typedef struct {
    int32_t width, global_height, row_begin, row_end, ghost_top, ghost_bot;
} dwt2_strip_level_t;

int32_t dwt2_strip_level_info(const dwt2_plan *plan, int32_t level, dwt2_strip_level_t *info);

/* Level k of a multi-level strip plan.
 * in:     device, (ghost_top + rows + ghost_bot) x in_pitch fp32 (rows =
 *         row_end - row_begin of level k; in_pitch >= the level width),
 *         the ghost rows already filled (neighbour strips or exchange).
 * ll_out: device, where the level's LL rows go ((rows + 1) / 2 rows, pitch
 *         ll_pitch): the first owned row of level k+1's input buffer.
 *         Ignored (may be NULL) for the last level, whose LL goes to out.
 * out:    device, the strip-local Mallat pyramid: W x (row_end - row_begin)
 *         of level 0, pitch W; level k writes its subband rows where a
 *         Mallat pyramid of that W x h image puts level k.
 * part:   as dwt2_forward_strip.
 * in, out and ll_out must not overlap. */
int32_t dwt2_forward_strip_level(const dwt2_plan *plan, int32_t level, const float *in, int64_t in_pitch,
                                 float *ll_out, int64_t ll_pitch, float *out, int32_t part,
                                 dwt2_stream_t stream);

/* Forward transform of one image.
 * in:  device pointer, W x H fp32, row pitch W elements, caller-owned,
 *      read-only, 4-byte aligned.
 * out: device pointer, W x H fp32 Mallat pyramid, row pitch W, caller-owned.
 * in and out must not overlap (no in-place transform).
 * Performance only (results are identical on every path): a 16-byte-aligned
 * `in` is read by TMA -- 3-D tensor maps when W is a multiple of 4, row-group
 * tensor maps (2 or 4 rows per tensor row) otherwise; an `in` that is only
 * 4-byte aligned, or batched images with gaps between them, take a 1-D
 * bulk-copy loader; an even ceil(W/2) with 8-byte-aligned subband rows gets
 * vector stores.  Launches: one per level, except that the small last levels
 * (at most 16384 quads each over all images for CDF 5/3, 65536 for the K = 2
 * wavelets) run together in ONE tail launch (dwt2_plan_info reports the
 * count).
 * Returns DWT2_OK, DWT2_EINVAL or DWT2_ECUDA. */
int32_t dwt2_forward(const dwt2_plan *plan, const float *in, float *out, dwt2_stream_t stream);

/* Forward transform of `count` images of the plan's size (count <= the
 * plan's max_count).  Image i is read at in + i * in_stride and written at
 * out + i * out_stride (element strides, >= W * H).  One launch per level
 * (or the tail launch, see dwt2_forward) covers all images. */
int32_t dwt2_forward_batched(const dwt2_plan *plan, const float *in, float *out, int32_t count,
                             int64_t in_stride, int64_t out_stride, dwt2_stream_t stream);

/* Forward transform of a one-level strip plan (see dwt2_plan_create_strip for the
 * `in` / `out` layouts).  part selects all quad rows, only the interior ones
 * (which read no ghost row, so they may run while the ghost rows are still in
 * flight) or only the two boundary quad rows.  A BOUNDARY call may run on
 * another stream concurrently with the INTERIOR call of the same level (they
 * write disjoint rows and use separate work queues); other calls on one plan
 * must be serialised. */
int32_t dwt2_forward_strip(const dwt2_plan *plan, const float *in, float *out, int32_t part,
                           dwt2_stream_t stream);

/* ---- Row strips with the halo exchange fused into the level launch --------
 *
 * The paper's synchronisation point between cores is the exchange of the
 * samples a step needs from its neighbours (section 3; the
 * row bands of SPEC.md L313-318).  A peer strip context replaces the message
 * exchange of dwt2_forward_strip_level (ghost rows copied by NCCL before the
 * BOUNDARY launch) with device-side PEER READS: boundary-role CTAs, appended
 * to the level kernel's own launch, wait on the neighbour's level-k ready
 * flag and load the 2 rows above / 1 row below straight from the
 * neighbour's buffer (NVLink peer memory mapped through CUDA IPC, or the same
 * device for ranks emulated in one process) while the interior tiles run.
 * No host call sits between the levels, so a whole step is a stream-ordered
 * sequence of ONE launch per level (CUDA-graph capturable).
 *
 * Synchronisation (flags in the context's own device memory, epochs counted
 * on the device): the first launch of level k publishes ready[k] = e once it
 * runs (after griddepcontrol.wait: the rank's earlier launches are complete,
 * so the level's input rows are final -- written by level k-1, or by the
 * caller before the step for k = 0); the first level-0 launch of a step
 * advances the epoch e.  A boundary quad row of level k waits until each
 * neighbour's ready[k] >= e, then reads the neighbour's rows.  The boundary
 * CTAs of the last level publish done = e and, in DWT2_PEER_RANKS mode, wait
 * until each neighbour's done >= e, so when a step has completed on a rank's
 * stream no neighbour still reads that rank's buffers: the caller may then
 * rewrite the level-0 rows, and the next step may overwrite every level.  A
 * wait that exceeds the context's timeout gives up (the step's output is then
 * invalid) and latches DWT2_ETIMEOUT, reported by dwt2_peer_strip_status. */

enum {
    DWT2_PEER_RANKS = 0,       /* one rank per GPU (or process), running concurrently */
    DWT2_PEER_SEQUENTIAL = 1   /* every rank in one process and one stream (1-GPU emulation): per level,
                                  every rank's PUBLISH then every rank's ALL, or every rank's INTERIOR then
                                  every rank's BOUNDARY -- a wait is then always met by an earlier launch;
                                  no end-of-step wait; dwt2_peer_strip_forward is rejected */
};

enum { DWT2_ETIMEOUT = -5 };   /* a peer flag wait timed out (dwt2_peer_strip_status) */

typedef struct dwt2_peer_strip dwt2_peer_strip;

/* What a neighbour needs to map a context: plain bytes, safe to send through
 * any host channel (the Python binding uses torch.distributed all_gather). */
typedef struct {
    uint8_t ipc_handle[64];    /* cudaIpcMemHandle_t of the context's single device allocation */
    uint64_t base;             /* that allocation's address in the exporting process */
    int64_t pid;               /* exporting process: the same process maps `base` directly */
    int32_t device;            /* CUDA ordinal in the exporting process */
    int32_t width, global_height, levels;
    int32_t row_begin, row_end;            /* level-0 strip rows */
    int32_t timeout_ms;
    int32_t reserved;
    int64_t owned_off[32];     /* byte offset (from base) of level k's first owned row */
    int64_t pitch[32];         /* level k's row pitch, floats */
    int64_t flags_off;         /* byte offset of the flag block */
} dwt2_peer_desc_t;

/* Allocates, on the plan's device, every level's ghost-padded input buffer of
 * the multi-level strip plan `plan` (dwt2_plan_create_strip_levels; row
 * pitches rounded up to 4 floats) and the flag block, in ONE cudaMalloc
 * (exportable through CUDA IPC).  The context keeps a pointer to `plan`,
 * which must outlive it.  timeout_ms bounds every flag wait (<= 0: 10000).
 * Returns NULL on error (dwt2_last_error()). */
dwt2_peer_strip *dwt2_peer_strip_create(const dwt2_plan *plan, int32_t timeout_ms);

/* Level k's owned rows in the context: *owned = the first owned row (device),
 * *pitch in floats.  Level 0's owned rows are where the caller writes the
 * strip's pixels (row_end - row_begin rows of `width` floats) before a step. */
int32_t dwt2_peer_strip_buffer(const dwt2_peer_strip *ctx, int32_t level, float **owned, int64_t *pitch);

/* Fills *desc for the neighbours of this rank. */
int32_t dwt2_peer_strip_export(const dwt2_peer_strip *ctx, dwt2_peer_desc_t *desc);

/* Maps the neighbours: `above` is the rank owning the rows just above
 * row_begin (NULL iff row_begin == 0), `below` the rank owning the rows from
 * row_end (NULL iff row_end == global_height).  Their geometry must match
 * (same width, height, levels; above->row_end == row_begin, below->row_begin
 * == row_end), else DWT2_EINVAL.  Descriptors of another process are opened
 * with cudaIpcOpenMemHandle (peer access over NVLink); those of this process
 * are used directly.  mode: DWT2_PEER_RANKS or DWT2_PEER_SEQUENTIAL.  Call
 * once, before the first step; DWT2_ECUDA if a mapping fails. */
int32_t dwt2_peer_strip_connect(dwt2_peer_strip *ctx, const dwt2_peer_desc_t *above,
                                const dwt2_peer_desc_t *below, int32_t mode);

/* Level k of a step, on `stream`, after level k-1:
 *   DWT2_STRIP_ALL       ONE launch: the fused level kernel on the interior
 *                        quad rows plus boundary-role CTAs that wait for the
 *                        neighbours and compute the first / last quad row from
 *                        their rows in peer memory (the step's form);
 *   DWT2_STRIP_INTERIOR  the level kernel on the interior quad rows only, then
 *   DWT2_STRIP_BOUNDARY  the boundary quad rows in a launch of their own.
 *   DWT2_STRIP_PUBLISH   only publishes ready[k] (a 1-thread launch): the
 *                        sequential emulation issues it for every rank before
 *                        the ranks' ALL launches of the level.
 * For one level use ALL, or INTERIOR then BOUNDARY.  out: the strip-local
 * Mallat pyramid (W x (row_end - row_begin), pitch W, device), as
 * dwt2_forward_strip_level writes it.  A rank without neighbours runs every
 * quad row in one level launch (BOUNDARY is then a no-op). */
int32_t dwt2_peer_strip_level(dwt2_peer_strip *ctx, int32_t level, int32_t part, float *out,
                              dwt2_stream_t stream);

/* A whole step: one DWT2_STRIP_ALL launch per level (no host
 * synchronisation; capturable in a CUDA graph).  DWT2_PEER_RANKS mode only. */
int32_t dwt2_peer_strip_forward(dwt2_peer_strip *ctx, float *out, dwt2_stream_t stream);

/* DWT2_OK, or DWT2_ETIMEOUT once any flag wait of this context has timed out
 * (reads device memory: synchronises with the device). */
int32_t dwt2_peer_strip_status(const dwt2_peer_strip *ctx);

/* Unmaps the neighbours and frees the context (no step may be in flight, on
 * this rank or on a neighbour reading it).  NULL is a no-op. */
void dwt2_peer_strip_destroy(dwt2_peer_strip *ctx);

/* End-to-end call on HOST buffers: host_in (W x H fp32) is copied to the
 * device, transformed, and the Mallat result copied back to host_out, all on
 * `stream`; returns after the stream has drained (the only synchronising
 * call).  The copies are chunked by row bands and overlapped with the level-1
 * kernel (copy engine H2D || kernel || D2H).  Pinned (page-locked) host
 * buffers are required for full speed; pageable buffers work but serialise.
 * The first call allocates device staging (2 x W x H fp32) owned by the plan.
 * Single-image plans only. */
int32_t dwt2_forward_host(const dwt2_plan *plan, const float *host_in, float *host_out,
                          dwt2_stream_t stream);

/* Inverse transform of one image: the Mallat pyramid
 * `in` (W x H fp32, pitch W, as dwt2_forward writes it) is reconstructed
 * into the W x H image `out`, coarsest level first.  Each level undoes the
 * spatial update, then the spatial predict of Eq. (5) (
 * steps reversed and negated) in one fused kernel, with the
 * same whole-sample symmetric extension as the forward.  fp64 in registers,
 * every level's reconstruction stored as fp32 (intermediate levels in the
 * plan's scratch).  Same ownership, overlap and stream rules as
 * dwt2_forward; strip plans are rejected (DWT2_EINVAL).  For integer-valued
 * inputs in [0, 255] and <= 2 levels, dwt2_inverse(dwt2_forward(x)) == x bit
 * for bit. */
int32_t dwt2_inverse(const dwt2_plan *plan, const float *in, float *out, dwt2_stream_t stream);

/* Batched inverse: `count` pyramids, element strides as in
 * dwt2_forward_batched.  One launch per level covers all images. */
int32_t dwt2_inverse_batched(const dwt2_plan *plan, const float *in, float *out, int32_t count,
                             int64_t in_stride, int64_t out_stride, dwt2_stream_t stream);

/* Schemes of the paper, for the comparison of SURVEY.md 8f row N1 (PAPER.md
 * section 4, Fig. 6): the same transform computed with one kernel per
 * barrier-separated step of each scheme (a step boundary that exchanges
 * data across the image is a kernel boundary, i.e. an HBM round trip), and
 * the fused single-step kernel with the literal and the adapted arithmetic
 * (the paper's operation-count trade-off at a fixed number of steps). */
enum {
    DWT2_SCHEME_FUSED = 0,          /* Eq. (5) fused into one kernel per level (the product path) */
    DWT2_SCHEME_NONSEP_NAIVE = 1,   /* Eq. (5), one plain kernel, predicted neighbours recomputed */
    DWT2_SCHEME_NONSEP_LIFTING = 2, /* Eq. (5): spatial predict | spatial update (2 kernels) */
    DWT2_SCHEME_NONSEP_ADAPTED = 3, /* Fig. 3: Eq. (5) with the constants P0, U0 split off (2 kernels) */
    DWT2_SCHEME_SEP_CONV = 4,       /* Eq. (4): horizontal | vertical filter bank (2 kernels) */
    DWT2_SCHEME_SEP_LIFTING = 5,    /* Eq. (3): 4 separable lifting steps (4 kernels) */
    DWT2_SCHEME_FUSED_LITERAL = 6,  /* the fused kernel with Eq. (5)'s operators as printed (24 MACs / quad) */
    DWT2_SCHEME_FUSED_ADAPTED = 7   /* the fused kernel with Fig. 3's adapted arithmetic (18 MACs / quad) */
};

/* Kernel launches (barrier-separated steps) per level of a scheme, or
 * DWT2_EINVAL for an unknown scheme. */
int32_t dwt2_scheme_steps(int32_t scheme);

/* Forward transform of `count` images (strides as in dwt2_forward_batched)
 * with the given scheme.  Same result as dwt2_forward up to fp32 rounding of
 * the intermediates between steps (bit-exact for integer-valued inputs at
 * <= 2 levels).  The 2-step schemes (except NONSEP_NAIVE and SEP_LIFTING,
 * which work in place on `out`) use a plan-owned work buffer of count x W x H
 * fp32, allocated on first use (so the first call is not capture-safe).
 * DWT2_SCHEME_FUSED is dwt2_forward_batched. */
int32_t dwt2_forward_scheme(const dwt2_plan *plan, int32_t scheme, const float *in, float *out, int32_t count,
                            int64_t in_stride, int64_t out_stride, dwt2_stream_t stream);

/* Frees the plan and its device memory (cudaFree synchronises the device).
 * NULL is a no-op.  No work using the plan may be in flight. */
void dwt2_destroy(dwt2_plan *plan);

/* Static facts of a plan, for benchmarks and tests. */
typedef struct {
    int32_t width, height, levels, max_count;
    int32_t launches_per_forward;    /* kernel launches one dwt2_forward issues */
    int32_t tma_levels;              /* levels served by the TMA-staged kernel */
    int64_t algorithmic_bytes;       /* 8 B x sum_k W_k H_k (one image) */
    int64_t scratch_bytes;           /* device bytes owned by the plan */
} dwt2_plan_info_t;

int32_t dwt2_plan_info(const dwt2_plan *plan, dwt2_plan_info_t *info);

/* Thread-local code of the last failing call in this thread (0 if none). */
int32_t dwt2_last_error(void);

/* Static description of a code; never NULL. */
const char *dwt2_error_string(int32_t code);

/* Library version string, e.g. "dwt2-b200 0.1 sm_100a". */
const char *dwt2_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DWT2_H */
