// peer.cu -- row strips with the halo exchange fused into the level launch
// (include/dwt2.h "peer strip context").
//
// The paper's multi-core mapping synchronises cores at the exchange of the
// samples a step needs from a neighbouring band (section 3).
// On an NVSwitch node the neighbour's rows are one NVLink load away, so the
// exchange is not a message: boundary-role CTAs acquire the neighbour's
// level-k ready flag and read the 2 rows above / 1 row below straight from the
// neighbour's buffer (CUDA IPC mapping; ranks emulated in one process share the
// device).  In a whole step (DWT2_STRIP_ALL) those CTAs ride in the level
// kernel's own launch (dwt2.cu: the CTAs past its grid take the boundary role),
// so a level is ONE launch and the exchange overlaps the interior tiles; the
// first launch of a level publishes its ready flag at entry (dwt2_internal.h
// peer_publish).
//
// The boundary quad rows are computed pointwise with the 2-D analysis filters
// that the lifting steps of Eq. (5) reach exactly (Eq. (4);
// dwt2_internal.h peer_boundary_role), bit for bit the level kernel's values.
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

constexpr int PB_THREADS = 256;                   // quads per CTA of the standalone boundary kernel

__global__ void __launch_bounds__(1) peer_publish_kernel(unsigned int *flags, int level)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    peer_publish(flags, level);
}

__global__ void __launch_bounds__(PB_THREADS) peer_boundary_kernel(const __grid_constant__ PeerBoundaryArgs a)
{
    __shared__ float tile[5 * (2 * PB_THREADS + 4)];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) peer_publish(a.flags, a.level);
    peer_boundary_role(a, blockIdx.x, blockIdx.y, tile);
    __syncthreads();
    if (threadIdx.x == 0) peer_exit(a);
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

// the boundary quad rows of level k and their arguments (returns their count, 0: none)
int boundary_args(const dwt2_peer_strip *c, int level, float *out, PeerBoundaryArgs *a)
{
    const dwt2_plan *p = c->plan;
    const dwt2_strip_level_t &L = c->info[level];
    const bool last = level == c->levels - 1;
    // [qs, ia) and [max(ib, ia), qe), as dwt2_forward_strip_level splits a level
    const int qs = L.row_begin / 2, qe = (L.row_end + 1) / 2;
    const int ia = qs + (L.ghost_top ? 1 : 0), ib = qe - (L.ghost_bot ? 1 : 0);
    int rows[2], nr = 0;
    if (ia > qs) rows[nr++] = qs;
    if (std::max(ib, ia) < qe) rows[nr++] = qe - 1;
    memset(a, 0, sizeof(*a));
    if (nr == 0) return 0;
    a->own = reinterpret_cast<const float *>(c->base + c->own_off[level]);
    a->own_pitch = c->pitch[level];
    if (L.ghost_top) {
        const dwt2_peer_desc_t &d = c->nb[0];
        int rb, re;
        level_rows(d.row_begin, d.row_end, level, &rb, &re);
        a->up = reinterpret_cast<const float *>(c->nb_base[0] + d.owned_off[level]) + (long long)(re - rb - 2) * d.pitch[level];
        a->up_pitch = d.pitch[level];
        a->up_flags = reinterpret_cast<const unsigned int *>(c->nb_base[0] + d.flags_off);
    }
    if (L.ghost_bot) {
        const dwt2_peer_desc_t &d = c->nb[1];
        a->dn = reinterpret_cast<const float *>(c->nb_base[1] + d.owned_off[level]);
        a->dn_pitch = d.pitch[level];
        a->dn_flags = reinterpret_cast<const unsigned int *>(c->nb_base[1] + d.flags_off);
    }
    a->flags = c->flags();
    // output bases as the level kernel's (dwt2.cu launch_level): level k's
    // subbands start at row 0 of the strip-local pyramid (pitch W)
    const int Wq = (L.width + 1) / 2;
    a->ll = last ? out : reinterpret_cast<float *>(c->base + c->own_off[level + 1]);
    a->ll_pitch = last ? p->W : c->pitch[level + 1];
    a->hl = out + Wq;
    a->lh = out + (long long)(qe - qs) * p->W;
    a->hh = a->lh + Wq;
    a->out_pitch = p->W;
    a->timeout_ns = (long long)c->timeout_ms * 1000000LL;
    a->W = L.width;
    a->H = L.global_height;
    a->rb = L.row_begin;
    a->re = L.row_end;
    a->qs = qs;
    a->n0 = rows[0];
    a->n1 = rows[nr - 1];
    a->level = level;
    a->last = last ? 1 : 0;
    a->quiesce = c->mode == DWT2_PEER_RANKS ? 1 : 0;
    return nr;
}

int32_t launch_boundary(const PeerBoundaryArgs &a, int nr, cudaStream_t s)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.nbx, nr);
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

}  // namespace

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
        part < DWT2_STRIP_ALL || part > DWT2_STRIP_PUBLISH)
        return fail(DWT2_EINVAL);
    const dwt2_plan *p = c->plan;
    const size_t out_bytes = size_t(p->W) * (p->row_end - p->row_begin) * sizeof(float);
    if (overlap(out, out_bytes, c->base, c->bytes) || !on_plan_device(p, out)) return fail(DWT2_EINVAL);
    const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const dwt2_strip_level_t &L = c->info[level];
    const bool last = level == c->levels - 1;
    const float *in = reinterpret_cast<const float *>(c->base + c->buf_off[level]);
    float *ll_out = last ? nullptr : reinterpret_cast<float *>(c->base + c->own_off[level + 1]);
    const long long ll_pitch = last ? 0 : c->pitch[level + 1];
    PeerBoundaryArgs a;
    const int nr = boundary_args(c, level, out, &a);
    if (nr == 0) {
        // no neighbour: the whole strip in one level launch, nothing to publish
        if (part == DWT2_STRIP_BOUNDARY || part == DWT2_STRIP_PUBLISH) return DWT2_OK;
        return strip_level_launch(p, level, in, c->pitch[level], ll_out, ll_pitch, out, DWT2_STRIP_ALL, s);
    }
    const int qs = L.row_begin / 2, qe = (L.row_end + 1) / 2;
    const int interior = (qe - (L.ghost_bot ? 1 : 0)) - (qs + (L.ghost_top ? 1 : 0));
    if (part == DWT2_STRIP_PUBLISH || (part == DWT2_STRIP_INTERIOR && interior <= 0)) {
        // (an INTERIOR part without interior quad rows still publishes the level)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(1);
        cfg.stream = s;
        cudaLaunchAttribute at = pdl_attr();
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, peer_publish_kernel, c->flags(), (int)level) != cudaSuccess) {
            cudaGetLastError();
            return fail(DWT2_ECUDA);
        }
        return DWT2_OK;
    }
    if (part == DWT2_STRIP_INTERIOR)        // publishes the level at entry, no boundary-role CTAs
        return strip_level_launch(p, level, in, c->pitch[level], ll_out, ll_pitch, out, DWT2_STRIP_INTERIOR, s, &a, 0);
    if (part == DWT2_STRIP_BOUNDARY || interior <= 0) {
        a.nbx = ((L.width + 1) / 2 + PB_THREADS - 1) / PB_THREADS;
        a.nroles = a.nbx * nr;
        return launch_boundary(a, nr, s);
    }
    // ALL: ONE launch -- the level kernel on the interior quad rows plus
    // boundary-role CTAs (level_kernel_threads() quads each) past its own grid
    const int threads = level_kernel_threads();
    a.nbx = ((L.width + 1) / 2 + threads - 1) / threads;
    a.nroles = a.nbx * nr;
    return strip_level_launch(p, level, in, c->pitch[level], ll_out, ll_pitch, out, DWT2_STRIP_INTERIOR, s, &a,
                              a.nroles);
}

int32_t dwt2_peer_strip_forward(dwt2_peer_strip *c, float *out, dwt2_stream_t stream)
{
    if (!c || !c->connected || c->mode != DWT2_PEER_RANKS) return fail(DWT2_EINVAL);
    int32_t r = DWT2_OK;
    for (int k = 0; k < c->levels && r == DWT2_OK; ++k) r = dwt2_peer_strip_level(c, k, DWT2_STRIP_ALL, out, stream);
    return r;
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
