// tail.cu -- the last, tiny levels of a forward 5/3 pyramid in ONE launch.
//
// Every level of the multi-level driver is one kernel launch; on B200 a
// dependent launch costs ~3.5-4 us whatever the level's size (measured:
// scripts/launch_floor.py, scripts/level_costs.py -- config 4's levels 6-8,
// 256^2 .. 64^2, take 11.6 us for 0.7 MB of data).  Levels whose input has
// at most TAIL_MAX_PX pixels therefore run here, all of them in one launch
// of one thread-block cluster: one thread per quad (the Eq. (5) predict and
// update written out per quad, its m-1 / n-1 neighbours re-predicted from
// the input, as the one-kernel NONSEP_NAIVE scheme of schemes.cu), and a
// cluster barrier (release / acquire at cluster scope) between levels so
// that level k+1 reads the LL level k wrote.  Loads bypass L1 (ld.global.cg):
// a level's input was written by other CTAs of the cluster.
//
// Arithmetic: fp64 registers, fp32 stores, the same operators as the level
// kernel (Eq. (5)), with whole-sample symmetric extension
// applied to pixel indices (schemes.cu: a coefficient of parity p at quad q
// sits at pixel 2q + p, an out-of-range neighbour is read at the mirrored
// pixel).  Every stored value is the correctly rounded fp32 of the exact
// result, so the tail is bit-identical to the per-level kernels (tests).

#include <cuda_runtime.h>

#include <cstring>

#include "dwt2_internal.h"

using namespace dwt2_detail;

namespace {

#ifndef DWT2_TAIL_CTAS
#define DWT2_TAIL_CTAS 16
#endif
constexpr int TAIL_CTAS = DWT2_TAIL_CTAS;   // one cluster (16: non-portable size, allowed below)
constexpr int TAIL_THREADS = 1024;

struct TailLevel {
    const float *in;                  // level input, image 0
    long long in_pitch, in_img;
    float *ll;                        // LL destination (scratch, or `out` for the last level)
    long long ll_pitch, ll_img;
    float *hl, *lh, *hh;              // detail subbands (Mallat positions in `out`)
    long long out_pitch, out_img;
    int W, H;
};

struct TailArgs {
    TailLevel lv[TAIL_MAX_LEVELS];
    int nlev, count;
};

__device__ __forceinline__ int wss_t(int k, int n)
{
    if (k < 0) k = -k;
    if (k > n - 1) k = 2 * (n - 1) - k;
    return k;
}

__device__ __forceinline__ double px_t(const TailLevel &L, int img, int r, int c)
{
    return (double)__ldcg(L.in + (long long)img * L.in_img + (long long)wss_t(r, L.H) * L.in_pitch + wss_t(c, L.W));
}

struct PredT {
    double a, hl, lh, hh;
};

// predicted values of quad (m, n) (Eq. (5) right factor)
__device__ __forceinline__ PredT predict_t(const TailLevel &L, int img, int m, int n)
{
    const int x = 2 * m, y = 2 * n;
    const double A = px_t(L, img, y, x), B = px_t(L, img, y, x + 1), C = px_t(L, img, y + 1, x);
    const double D = px_t(L, img, y + 1, x + 1), Ar = px_t(L, img, y, x + 2), Ad = px_t(L, img, y + 2, x);
    const double Ard = px_t(L, img, y + 2, x + 2), Cr = px_t(L, img, y + 1, x + 2), Bd = px_t(L, img, y + 2, x + 1);
    PredT p;
    p.a = A;
    p.hl = B - 0.5 * (A + Ar);
    p.lh = C - 0.5 * (A + Ad);
    p.hh = D - 0.5 * (C + Cr) - 0.5 * (B + Bd) + 0.25 * (A + Ar + Ad + Ard);
    return p;
}

__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(TAIL_THREADS) dwt53_tail_kernel(const __grid_constant__ TailArgs a)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nthreads = gridDim.x * blockDim.x;
    for (int k = 0; k < a.nlev; ++k) {
        const TailLevel &L = a.lv[k];
        const int Wq = (L.W + 1) >> 1, Hq = (L.H + 1) >> 1, Wh = L.W >> 1, Hh = L.H >> 1;
        const long long nq = (long long)Wq * Hq;
        for (long long q = tid; q < nq * a.count; q += nthreads) {
            const int img = int(q / nq);
            const int r = int(q - (long long)img * nq);
            const int n = r / Wq, m = r - n * Wq;
            // the update's neighbours: predicted values at m-1, n-1 and (m-1, n-1);
            // predicting an out-of-range quad (m-1 = -1) or the missing H column /
            // row of an odd size reads the mirrored pixels, so it yields the
            // mirrored values (H[-1] = H[0], H[M] = H[M-1]) by itself
            const PredT c = predict_t(L, img, m, n);
            const PredT l = predict_t(L, img, m - 1, n);
            const PredT u = predict_t(L, img, m, n - 1);
            const PredT ul = predict_t(L, img, m - 1, n - 1);
            const double hl = c.hl, lh = c.lh, hh = c.hh;
            const double LL = c.a + 0.25 * (hl + l.hl) + 0.25 * (lh + u.lh) + 0.0625 * (hh + l.hh + u.hh + ul.hh);
            const float oLL = (float)LL;
            const float oHL = (float)(hl + 0.25 * (hh + u.hh));
            const float oLH = (float)(lh + 0.25 * (hh + l.hh));
            const float oHH = (float)hh;
            L.ll[(long long)img * L.ll_img + (long long)n * L.ll_pitch + m] = oLL;
            const long long ob = (long long)img * L.out_img + (long long)n * L.out_pitch + m;
            if (m < Wh) L.hl[ob] = oHL;
            if (n < Hh) {
                L.lh[ob] = oLH;
                if (m < Wh) L.hh[ob] = oHH;
            }
        }
        if (k + 1 < a.nlev) cluster_sync_all();       // level k's LL is level k+1's input
    }
}

}  // namespace

namespace dwt2_detail {

// Levels [first, levels) of plan p in one cluster launch; DWT2_EUNSUPPORTED
// if the launch configuration is refused (the caller then runs them one by one).
int32_t run_tail(const dwt2_plan *p, const float *in_level0, float *out, int count, long long in_stride,
                 long long out_stride, int first, cudaStream_t s)
{
    TailArgs a;
    memset(&a, 0, sizeof(a));
    a.count = count;
    a.nlev = p->levels - first;
    if (a.nlev < 1 || a.nlev > TAIL_MAX_LEVELS) return DWT2_EUNSUPPORTED;
    for (int k = first; k < p->levels; ++k) {
        const LevelGeom &g = p->geom[k];
        TailLevel &L = a.lv[k - first];
        L.W = g.W;
        L.H = g.H;
        if (k == 0) {
            L.in = in_level0;
            L.in_pitch = p->W;
            L.in_img = in_stride;
        } else {
            const int si = (k - 1) % 2;
            L.in = p->scratch[si];
            L.in_pitch = p->sc_pitch[si];
            L.in_img = p->sc_img_stride[si];
        }
        if (k == p->levels - 1) {
            L.ll = out;
            L.ll_pitch = p->W;
            L.ll_img = out_stride;
        } else {
            const int si = k % 2;
            L.ll = p->scratch[si];
            L.ll_pitch = p->sc_pitch[si];
            L.ll_img = p->sc_img_stride[si];
        }
        L.hl = out + g.Wq;
        L.lh = out + (long long)g.Hq * p->W;
        L.hh = L.lh + g.Wq;
        L.out_pitch = p->W;
        L.out_img = out_stride;
    }
    static const bool attr_ok = [] {
        const bool ok = TAIL_CTAS <= 8 ||
                        cudaFuncSetAttribute(dwt53_tail_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                            cudaSuccess;
        cudaGetLastError();
        return ok;
    }();
    if (!attr_ok) return DWT2_EUNSUPPORTED;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(TAIL_CTAS);
    cfg.blockDim = dim3(TAIL_THREADS);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = TAIL_CTAS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, dwt53_tail_kernel, a) != cudaSuccess) {
        cudaGetLastError();
        return DWT2_EUNSUPPORTED;
    }
    return DWT2_OK;
}

}  // namespace dwt2_detail
