// peer.cu -- row strips with the halo exchange fused into the boundary kernel
// (include/dwt2.h "peer strip context").
//
// The paper's multi-core mapping synchronises cores at the exchange of the
// samples a step needs from a neighbouring band (section 3).
// On an NVSwitch node the neighbour's rows are one NVLink load away, so the
// exchange is not a message: the BOUNDARY kernel of level k acquires the
// neighbour's level-k ready flag and reads the 2 rows above / 1 row below
// straight from the neighbour's buffer (CUDA IPC mapping; ranks emulated in
// one process share the device).  The INTERIOR launch of the level (the fused
// TMA level kernel of dwt2.cu, unchanged apart from publishing the flag at
// entry) needs no neighbour row and never waits.
//
// The boundary quad rows are computed pointwise with the 2-D analysis
// filters that the lifting steps of Eq. (5) reach exactly (PAPER.md
// L160-171, Eq. (4)): h = (-1/8, 1/4, 3/4, 1/4, -1/8) on even positions,
// g = (-1/2, 1, -1/2) on odd ones, a row pass and a column pass in fp64
// (every product and partial sum of these dyadic taps with fp32 data is
// exact, so the stored fp32 equals the level kernel's; tail.cu uses the same
// evaluation).  A CTA stages the 5 input rows of 256 quads in shared memory
// (coalesced loads: peer memory is read once per element).
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>

#include "dwt2_internal.h"

using namespace dwt2_detail;

struct dwt2_peer_strip {
    const dwt2_plan *plan;
    int device, levels, timeout_ms, mode;
    char *base;                                   // the single device allocation
    size_t bytes;
    long long buf_off[MAX_LEVELS];                // level k's ghost-padded buffer (the level kernel's `in`)
    long long own_off[MAX_LEVELS];                // level k's first owned row
    long long pitch[MAX_LEVELS];                  // floats
    dwt2_strip_level_t info[MAX_LEVELS];
    long long flags_off;
    bool connected;
    const char *nb_base[2];                       // neighbours' allocations in this process ([0] above, [1] below)
    bool nb_mapped[2];                            // opened with cudaIpcOpenMemHandle (close on destroy)
    dwt2_peer_desc_t nb[2];

    unsigned int *flags() const { return reinterpret_cast<unsigned int *>(base + flags_off); }
};

namespace {

constexpr int PB_THREADS = 256;                   // quads per CTA
constexpr int PB_COLS = 2 * PB_THREADS + 4;       // staged columns 2 m0 - 2 .. 2 m0 + 2 PB_THREADS + 1

struct PeerBoundaryArgs {
    const float *own;                 // global row rb of this rank (level k)
    const float *up;                  // global row rb - 2 in the rank above (null: none)
    const float *dn;                  // global row re in the rank below (null: none)
    long long own_pitch, up_pitch, dn_pitch;
    const unsigned int *up_flags, *dn_flags;
    unsigned int *flags;
    float *ll;                        // LL row of quad row qs
    float *hl, *lh, *hh;              // subband rows of quad row qs (strip-local output)
    long long ll_pitch, out_pitch;
    long long timeout_ns;
    int W, H, rb, re, qs;
    int n0, n1;                       // the boundary quad rows (global); blockIdx.y selects
    int level, last, quiesce;
};

__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned int *p)
{
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// spin until *f >= e (epochs compared modulo 2^32); false after timeout_ns
__device__ bool wait_epoch(const unsigned int *f, unsigned e, long long timeout_ns)
{
    const unsigned long long t0 = gtime();
    while (int(ld_acquire_sys(f) - e) < 0) {
        if ((long long)(gtime() - t0) > timeout_ns) return false;
        __nanosleep(100);
    }
    return true;
}

// whole-sample symmetric reflection for k in [-2, n + 1], n >= 2
__device__ __forceinline__ int wss2(int k, int n)
{
    k = k < 0 ? -k : k;
    return k >= n ? 2 * (n - 1) - k : k;
}

__global__ void __launch_bounds__(1) peer_publish_kernel(unsigned int *flags, int level)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    peer_publish_ready(flags, level);
}

__global__ void __launch_bounds__(PB_THREADS) peer_boundary_kernel(const __grid_constant__ PeerBoundaryArgs a)
{
    __shared__ float tile[5][PB_COLS];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const unsigned e = *reinterpret_cast<volatile unsigned int *>(a.flags + PEER_EPOCH);
    if (threadIdx.x == 0) {
        bool ok = true;
        if (a.up_flags) ok = wait_epoch(a.up_flags + PEER_READY + a.level, e, a.timeout_ns) && ok;
        if (a.dn_flags) ok = wait_epoch(a.dn_flags + PEER_READY + a.level, e, a.timeout_ns) && ok;
        if (!ok) atomicExch(a.flags + PEER_ERR, 1u);
    }
    __syncthreads();

    const int n = blockIdx.y == 0 ? a.n0 : a.n1;
    const int W = a.W, H = a.H;
    const int Wq = (W + 1) >> 1, Wh = W >> 1, Hh = H >> 1;
    const int m0 = blockIdx.x * PB_THREADS;
    const int c0 = 2 * m0 - 2;
    // stage input rows 2n-2 .. 2n+2 (mirrored at the image edges; rows outside
    // [rb, re) come from the neighbours' memory), columns c0 .. c0 + PB_COLS - 1
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int y = wss2(2 * n - 2 + j, H);
        const float *row = y < a.rb ? a.up + (long long)(y - (a.rb - 2)) * a.up_pitch
                         : y >= a.re ? a.dn + (long long)(y - a.re) * a.dn_pitch
                                     : a.own + (long long)(y - a.rb) * a.own_pitch;
        for (int i = threadIdx.x; i < PB_COLS; i += PB_THREADS) {
            const int x = c0 + i;
            if (x <= W + 1) tile[j][i] = __ldcg(row + wss2(x, W));
        }
    }
    __syncthreads();

    const int m = m0 + threadIdx.x;
    if (m < Wq) {
        double lo[5], hi[5];              // row passes: h at column 2m, g at column 2m + 1
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const float *v = &tile[j][2 * threadIdx.x];
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

    if (a.last) {
        // the last CTA to finish publishes done = e (no CTA of this rank reads a
        // neighbour any more this step) and, for concurrent ranks, waits until
        // the neighbours are done reading this rank's buffers
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned total = gridDim.x * gridDim.y;
            if (atomicAdd(a.flags + PEER_CTR, 1u) == total - 1) {
                atomicExch(a.flags + PEER_CTR, 0u);
                __threadfence_system();
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.flags + PEER_DONE), "r"(e) : "memory");
                if (a.quiesce) {
                    bool ok = true;
                    if (a.up_flags) ok = wait_epoch(a.up_flags + PEER_DONE, e, a.timeout_ns) && ok;
                    if (a.dn_flags) ok = wait_epoch(a.dn_flags + PEER_DONE, e, a.timeout_ns) && ok;
                    if (!ok) atomicExch(a.flags + PEER_ERR, 1u);
                }
            }
        }
    }
}

cudaLaunchAttribute pdl_attr()
{
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = 1;
    return at;
}

void level_rows(int rb0, int re0, int k, int *rb, int *re)
{
    int b = rb0, e = re0;
    for (int i = 0; i < k; ++i) {
        b >>= 1;
        e = (e + 1) >> 1;
    }
    *rb = b;
    *re = e;
}

bool same_geometry(const dwt2_peer_strip *c, const dwt2_peer_desc_t *d)
{
    const dwt2_plan *p = c->plan;
    return d->width == p->W && d->global_height == p->Hg && d->levels == p->levels && d->device >= 0;
}

}  // namespace

namespace dwt2_detail {

int32_t launch_peer_publish(unsigned int *flags, int level, cudaStream_t stream)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(1);
    cfg.stream = stream;
    cudaLaunchAttribute at = pdl_attr();
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, peer_publish_kernel, flags, level) != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

}  // namespace dwt2_detail

extern "C" {

dwt2_peer_strip *dwt2_peer_strip_create(const dwt2_plan *p, int32_t timeout_ms)
{
    if (!p || !p->strip || p->levels < 1 || p->levels > MAX_LEVELS || p->wavelet != DWT2_WAVELET_CDF53) {
        g_last_error = DWT2_EINVAL;
        return nullptr;
    }
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev != p->device) {
        cudaGetLastError();
        g_last_error = DWT2_EINVAL;
        return nullptr;
    }
    dwt2_peer_strip *c = new (std::nothrow) dwt2_peer_strip;
    if (!c) {
        g_last_error = DWT2_ENOMEM;
        return nullptr;
    }
    memset(c, 0, sizeof(*c));
    c->plan = p;
    c->device = dev;
    c->levels = p->levels;
    c->timeout_ms = timeout_ms > 0 ? timeout_ms : 10000;
    long long off = 0;
    for (int k = 0; k < p->levels; ++k) {
        dwt2_strip_level_t &L = c->info[k];
        dwt2_strip_level_info(p, k, &L);
        const long long pitch = round_up(L.width, 4);          // 16-byte rows: the TMA-staged loader
        const long long rows = L.ghost_top + (L.row_end - L.row_begin) + L.ghost_bot;
        c->pitch[k] = pitch;
        c->buf_off[k] = off;
        c->own_off[k] = off + (long long)L.ghost_top * pitch * (long long)sizeof(float);
        off = round_up(off + rows * pitch * (long long)sizeof(float), 256);
    }
    c->flags_off = off;
    c->bytes = size_t(off + 256);
    if (cudaMalloc(&c->base, c->bytes) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        g_last_error = DWT2_ENOMEM;
        return nullptr;
    }
    if (cudaMemset(c->base, 0, c->bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        cudaGetLastError();
        cudaFree(c->base);
        delete c;
        g_last_error = DWT2_ECUDA;
        return nullptr;
    }
    g_last_error = DWT2_OK;
    return c;
}

int32_t dwt2_peer_strip_buffer(const dwt2_peer_strip *c, int32_t level, float **owned, int64_t *pitch)
{
    if (!c || !owned || !pitch || level < 0 || level >= c->levels) return fail(DWT2_EINVAL);
    *owned = reinterpret_cast<float *>(c->base + c->own_off[level]);
    *pitch = c->pitch[level];
    return DWT2_OK;
}

int32_t dwt2_peer_strip_export(const dwt2_peer_strip *c, dwt2_peer_desc_t *d)
{
    if (!c || !d) return fail(DWT2_EINVAL);
    memset(d, 0, sizeof(*d));
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, c->base) == cudaSuccess) {
        static_assert(sizeof(h) <= sizeof(d->ipc_handle), "IPC handle size");
        memcpy(d->ipc_handle, &h, sizeof(h));
    } else {
        cudaGetLastError();             // no IPC here: the descriptor still serves this process
    }
    d->base = reinterpret_cast<uint64_t>(c->base);
    d->pid = (int64_t)getpid();
    d->device = c->device;
    d->width = c->plan->W;
    d->global_height = c->plan->Hg;
    d->levels = c->levels;
    d->row_begin = c->plan->row_begin;
    d->row_end = c->plan->row_end;
    d->timeout_ms = c->timeout_ms;
    for (int k = 0; k < c->levels; ++k) {
        d->owned_off[k] = c->own_off[k];
        d->pitch[k] = c->pitch[k];
    }
    d->flags_off = c->flags_off;
    return DWT2_OK;
}

int32_t dwt2_peer_strip_connect(dwt2_peer_strip *c, const dwt2_peer_desc_t *above, const dwt2_peer_desc_t *below,
                                int32_t mode)
{
    if (!c || c->connected || (mode != DWT2_PEER_RANKS && mode != DWT2_PEER_SEQUENTIAL)) return fail(DWT2_EINVAL);
    const dwt2_plan *p = c->plan;
    if ((above != nullptr) != (p->row_begin > 0) || (below != nullptr) != (p->row_end < p->Hg)) return fail(DWT2_EINVAL);
    if (above && (!same_geometry(c, above) || above->row_end != p->row_begin || above->row_begin >= above->row_end))
        return fail(DWT2_EINVAL);
    if (below && (!same_geometry(c, below) || below->row_begin != p->row_end || below->row_begin >= below->row_end))
        return fail(DWT2_EINVAL);
    const dwt2_peer_desc_t *nb[2] = {above, below};
    for (int s = 0; s < 2; ++s) {
        if (!nb[s]) continue;
        c->nb[s] = *nb[s];
        if (nb[s]->pid == (int64_t)getpid()) {
            c->nb_base[s] = reinterpret_cast<const char *>(nb[s]->base);
        } else {
            cudaIpcMemHandle_t h;
            memcpy(&h, nb[s]->ipc_handle, sizeof(h));
            void *ptr = nullptr;
            if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                if (s == 1 && c->nb_mapped[0]) cudaIpcCloseMemHandle(const_cast<char *>(c->nb_base[0]));
                c->nb_base[0] = c->nb_base[1] = nullptr;
                c->nb_mapped[0] = c->nb_mapped[1] = false;
                return fail(DWT2_ECUDA);
            }
            c->nb_base[s] = static_cast<const char *>(ptr);
            c->nb_mapped[s] = true;
        }
    }
    c->mode = mode;
    c->connected = true;
    return DWT2_OK;
}

int32_t dwt2_peer_strip_level(dwt2_peer_strip *c, int32_t level, int32_t part, float *out, dwt2_stream_t stream)
{
    if (!c || !c->connected || level < 0 || level >= c->levels || !out || !aligned(out, 4) ||
        (part != DWT2_STRIP_INTERIOR && part != DWT2_STRIP_BOUNDARY))
        return fail(DWT2_EINVAL);
    const dwt2_plan *p = c->plan;
    const size_t out_bytes = size_t(p->W) * (p->row_end - p->row_begin) * sizeof(float);
    if (overlap(out, out_bytes, c->base, c->bytes) || !on_plan_device(p, out)) return fail(DWT2_EINVAL);
    const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const dwt2_strip_level_t &L = c->info[level];
    const bool last = level == c->levels - 1;
    float *ll_out = last ? nullptr : reinterpret_cast<float *>(c->base + c->own_off[level + 1]);
    const long long ll_pitch = last ? 0 : c->pitch[level + 1];
    if (part == DWT2_STRIP_INTERIOR) {
        const float *in = reinterpret_cast<const float *>(c->base + c->buf_off[level]);
        const bool alone = L.ghost_top == 0 && L.ghost_bot == 0;      // no neighbour: nothing to publish
        return strip_level_launch(p, level, in, c->pitch[level], ll_out, ll_pitch, out, DWT2_STRIP_INTERIOR, s,
                                  alone ? nullptr : c->flags());
    }
    if (L.ghost_top == 0 && L.ghost_bot == 0) return DWT2_OK;
    // the boundary quad rows: [qs, ia) and [max(ib, ia), qe) (dwt2_forward_strip_level)
    const int qs = L.row_begin / 2, qe = (L.row_end + 1) / 2;
    const int ia = qs + (L.ghost_top ? 1 : 0), ib = qe - (L.ghost_bot ? 1 : 0);
    int rows[2], nr = 0;
    if (ia > qs) rows[nr++] = qs;
    if (L.ghost_bot && std::max(ib, ia) < qe && !(nr == 1 && rows[0] == qe - 1)) rows[nr++] = qe - 1;
    PeerBoundaryArgs a;
    memset(&a, 0, sizeof(a));
    a.own = reinterpret_cast<const float *>(c->base + c->own_off[level]);
    a.own_pitch = c->pitch[level];
    if (L.ghost_top) {
        const dwt2_peer_desc_t &d = c->nb[0];
        int rb, re;
        level_rows(d.row_begin, d.row_end, level, &rb, &re);
        a.up = reinterpret_cast<const float *>(c->nb_base[0] + d.owned_off[level]) + (long long)(re - rb - 2) * d.pitch[level];
        a.up_pitch = d.pitch[level];
        a.up_flags = reinterpret_cast<const unsigned int *>(c->nb_base[0] + d.flags_off);
    }
    if (L.ghost_bot) {
        const dwt2_peer_desc_t &d = c->nb[1];
        a.dn = reinterpret_cast<const float *>(c->nb_base[1] + d.owned_off[level]);
        a.dn_pitch = d.pitch[level];
        a.dn_flags = reinterpret_cast<const unsigned int *>(c->nb_base[1] + d.flags_off);
    }
    a.flags = c->flags();
    // output bases as the level kernel computes them (dwt2.cu launch_level)
    const int Wq = (L.width + 1) / 2;
    const int hq_local = qe - qs;
    const int hloc0 = p->row_end - p->row_begin;
    (void)hloc0;
    float *mallat = out;                            // level k's subbands start at row 0 of the strip pyramid
    a.ll = last ? out : ll_out;
    a.ll_pitch = last ? p->W : ll_pitch;
    a.hl = mallat + Wq;
    a.lh = mallat + (long long)hq_local * p->W;
    a.hh = a.lh + Wq;
    a.out_pitch = p->W;
    a.timeout_ns = (long long)c->timeout_ms * 1000000LL;
    a.W = L.width;
    a.H = L.global_height;
    a.rb = L.row_begin;
    a.re = L.row_end;
    a.qs = qs;
    a.n0 = rows[0];
    a.n1 = nr > 1 ? rows[1] : rows[0];
    a.level = level;
    a.last = last ? 1 : 0;
    a.quiesce = c->mode == DWT2_PEER_RANKS ? 1 : 0;

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((Wq + PB_THREADS - 1) / PB_THREADS, nr);
    cfg.blockDim = dim3(PB_THREADS);
    cfg.stream = s;
    cudaLaunchAttribute at = pdl_attr();
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, peer_boundary_kernel, a) != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return DWT2_OK;
}

int32_t dwt2_peer_strip_forward(dwt2_peer_strip *c, float *out, dwt2_stream_t stream)
{
    if (!c || !c->connected || c->mode != DWT2_PEER_RANKS) return fail(DWT2_EINVAL);
    for (int k = 0; k < c->levels; ++k) {
        int32_t r = dwt2_peer_strip_level(c, k, DWT2_STRIP_INTERIOR, out, stream);
        if (r == DWT2_OK) r = dwt2_peer_strip_level(c, k, DWT2_STRIP_BOUNDARY, out, stream);
        if (r != DWT2_OK) return r;
    }
    return DWT2_OK;
}

int32_t dwt2_peer_strip_status(const dwt2_peer_strip *c)
{
    if (!c) return fail(DWT2_EINVAL);
    unsigned int err = 0;
    if (cudaMemcpy(&err, c->flags() + PEER_ERR, sizeof(err), cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return fail(DWT2_ECUDA);
    }
    return err ? fail(DWT2_ETIMEOUT) : DWT2_OK;
}

void dwt2_peer_strip_destroy(dwt2_peer_strip *c)
{
    if (!c) return;
    for (int s = 0; s < 2; ++s)
        if (c->nb_mapped[s]) cudaIpcCloseMemHandle(const_cast<char *>(c->nb_base[s]));
    cudaFree(c->base);
    cudaGetLastError();
    delete c;
}

}  // extern "C"
