// ccl_api.cu -- the extern "C" boundary of libccl_b200.so (include/ccl.h).
// Argument checks run on the host before any CUDA call.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <new>

#include "ccl.h"
#include "ccl_internal.cuh"

namespace cclb {

Geometry make_geometry(int H, int W) { return make_geometry_batch(1, H, W); }

Geometry make_geometry_batch(int B, int IH, int W) {
    Geometry g;
    const int H = B * IH;
    g.H = H;
    g.W = W;
    g.IH = IH;
    g.tpi = (IH + TH - 1) / TH;
    g.WW = (W + 31) / 32;
    g.nTx = (W + TW - 1) / TW;
    g.nTy = B * g.tpi;
    g.nT = g.nTx * g.nTy;
    g.nseg = H * g.nTx;
    const int tw = W < TW ? W : TW, th = IH < TH ? IH : TH;
    g.maxrun = (tw + 1) / 2;
    g.capc = ((th + 1) / 2) * g.maxrun;
    g.capb = 2 * g.maxrun + th;
    g.capw = (g.capc + 31) / 32;
    g.aligned = (W % 16) == 0;
    g.row0 = 0;
    g.thr = 0;
    return g;
}

enum {
    A_BM, A_RUNCOMP, A_COMPNODE, A_NRLAB, A_TLB, A_TBITS, A_TWPRE, A_GPARENT, A_GKEY, A_GNODECOMP, A_GNODELAB,
    A_EDGEROW, A_TOP, A_BOT, A_LEFT, A_RIGHT, A_META, A_SEGCNT, A_SEGOFF, A_SCANSTATE, A_TICKET, A_ROWEXCL, A_K1OVER, A_STATS, A_COUNT
};

void workspace_layout(const Geometry &g, size_t offs[], size_t *total) {
    const size_t nT = (size_t)g.nT, H = (size_t)g.H;
    const size_t sz[A_COUNT] = {
        H * g.WW * 4,                   // bm
        H * g.nTx * g.maxrun * 2,       // runcomp
        nT * g.capc * 4,                // compnode
        nT * g.capc * 4,                // nrlab
        nT * TH * 4,                    // tlb
        nT * g.capw * 4,                // tbits
        nT * g.capw * 4,                // twpre
        nT * g.capb * 4,                // gparent
        nT * g.capb * 8,                // gkey
        nT * g.capb * 4,                // gnodecomp
        nT * g.capb * 4,                // gnodelab
        nT * 2 * WPR * 4,               // edgerow
        nT * g.maxrun * 4,              // topnode
        nT * g.maxrun * 4,              // botnode
        (size_t)g.nTx * H * 4,          // leftnode
        (size_t)g.nTx * H * 4,          // rightnode
        nT * META * 4,                  // meta
        (size_t)g.nseg * 4,             // segcnt
        (size_t)g.nseg * 4,             // segoff
        (size_t)g.nTy * 8,              // scanstate
        16,                             // ticket
        (size_t)g.nTy * 4,              // rowexcl
        (nT + 1) * 4,                   // k1over + its count
        STAT_COUNT * 8,                 // stats
    };
    size_t o = 0;
    for (int i = 0; i < A_COUNT; i++) {
        offs[i] = o;
        o += (sz[i] + 255) & ~(size_t)255;
    }
    *total = o;
}

Workspace workspace_bind(const Geometry &g, void *base) {
    size_t offs[A_COUNT], total;
    workspace_layout(g, offs, &total);
    char *b = static_cast<char *>(base);
    Workspace w;
    w.bm = reinterpret_cast<uint32_t *>(b + offs[A_BM]);
    w.runcomp = reinterpret_cast<uint16_t *>(b + offs[A_RUNCOMP]);
    w.compnode = reinterpret_cast<int32_t *>(b + offs[A_COMPNODE]);
    w.nrlab = reinterpret_cast<int32_t *>(b + offs[A_NRLAB]);
    w.tlb = reinterpret_cast<int32_t *>(b + offs[A_TLB]);
    w.tbits = reinterpret_cast<uint32_t *>(b + offs[A_TBITS]);
    w.twpre = reinterpret_cast<int32_t *>(b + offs[A_TWPRE]);
    w.gparent = reinterpret_cast<int32_t *>(b + offs[A_GPARENT]);
    w.gkey = reinterpret_cast<int64_t *>(b + offs[A_GKEY]);
    w.gnodecomp = reinterpret_cast<int32_t *>(b + offs[A_GNODECOMP]);
    w.gnodelab = reinterpret_cast<int32_t *>(b + offs[A_GNODELAB]);
    w.edgerow = reinterpret_cast<uint32_t *>(b + offs[A_EDGEROW]);
    w.topnode = reinterpret_cast<int32_t *>(b + offs[A_TOP]);
    w.botnode = reinterpret_cast<int32_t *>(b + offs[A_BOT]);
    w.leftnode = reinterpret_cast<int32_t *>(b + offs[A_LEFT]);
    w.rightnode = reinterpret_cast<int32_t *>(b + offs[A_RIGHT]);
    w.meta = reinterpret_cast<int32_t *>(b + offs[A_META]);
    w.segcnt = reinterpret_cast<int32_t *>(b + offs[A_SEGCNT]);
    w.segoff = reinterpret_cast<int32_t *>(b + offs[A_SEGOFF]);
    w.scanstate = reinterpret_cast<unsigned long long *>(b + offs[A_SCANSTATE]);
    w.ticket = reinterpret_cast<int32_t *>(b + offs[A_TICKET]);
    w.rowexcl = reinterpret_cast<int32_t *>(b + offs[A_ROWEXCL]);
    w.k1over = reinterpret_cast<int32_t *>(b + offs[A_K1OVER]);
    w.k1over_n = w.k1over + g.nT;
    w.stats = reinterpret_cast<unsigned long long *>(b + offs[A_STATS]);
    w.xlab = nullptr;
    w.boff = nullptr;
    return w;
}

// Test hook (ccl_debug_set(5, seed)): fresh workspaces are filled with
// pseudo-random words instead of whatever the allocation held, so tests can
// check that no kernel decodes workspace it has not written in this call.
static uint32_t g_poison = 0;
__global__ void k_poison(uint32_t *p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 0x9E3779B9u ^ seed;
        h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
        p[i] = h;
    }
}
cudaError_t workspace_poison(void *mem, size_t bytes, cudaStream_t s) {
    if (!g_poison) return cudaSuccess;
    k_poison<<<1184, 256, 0, s>>>(static_cast<uint32_t *>(mem), bytes / 4, g_poison);
    return cudaGetLastError();
}

cudaError_t workspace_init(const Workspace &ws, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(ws.k1over_n, 0, sizeof(int32_t), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(ws.stats, 0, STAT_COUNT * sizeof(unsigned long long), stream);
    return e;
}

}  // namespace cclb

using namespace cclb;

struct ccl_plan_st {
    Geometry g;
    int32_t *hint = nullptr;  // mapped pinned host word: K1's last hand-over count
    void *ws_mem = nullptr;
    size_t ws_bytes = 0;
    Workspace ws;
    // ccl_plan_label_host_async: two staging slots, three internal streams
    // (H2D, compute, D2H) and per-slot events, so step i+1's H2D and kernels
    // overlap step i's D2H
    bool host_init = false;
    cudaStream_t s_h2d = nullptr, s_cmp = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_cmp[2] = {}, ev_d2h[2] = {};
    uint8_t *a_img[2] = {};
    int32_t *a_lab[2] = {}, *a_n[2] = {};
    int slot = 0;
    // ordering of the plan's pipelines across the async host path and the
    // device path (one workspace): the stream of the last device-path call,
    // and an event after it once the host pipe exists
    cudaStream_t last_dev_stream = nullptr;
    bool dev_called = false, dev_pending = false;
    cudaEvent_t ev_dev = nullptr;
    int prof_sets = 0;             // profiling ring size (0 = off)
    cudaEvent_t *ev = nullptr;     // prof_sets * (K_COUNT + 1) events
    long long prof_calls = 0;      // profiled calls since the ring was (re)armed
};

static void free_events(ccl_plan p) {
    if (p->ev) {
        for (int i = 0; i < p->prof_sets * (K_COUNT + 1); i++)
            if (p->ev[i]) cudaEventDestroy(p->ev[i]);
        delete[] p->ev;
    }
    p->ev = nullptr;
    p->prof_sets = 0;
    p->prof_calls = 0;
}

static ccl_status check_shape(int H, int W) {
    if (H < 1 || W < 1) return CCL_INVALID_ARGUMENT;
    if ((int64_t)H * (int64_t)W > (int64_t)INT32_MAX) return CCL_TOO_LARGE;
    return CCL_OK;
}

static ccl_status check_buffers(const void *img, const void *labels, const void *n, int H, int W) {
    if (!img || !labels || !n) return CCL_INVALID_ARGUMENT;
    const char *a = static_cast<const char *>(img);
    const char *l = static_cast<const char *>(labels);
    const size_t nb = (size_t)H * (size_t)W;
    if (a < l + nb * 4 && l < a + nb) return CCL_INVALID_ARGUMENT;  // labels alias img
    return CCL_OK;
}

extern "C" {

const char *ccl_status_string(ccl_status s) {
    switch (s) {
        case CCL_OK: return "CCL_OK";
        case CCL_INVALID_ARGUMENT: return "CCL_INVALID_ARGUMENT";
        case CCL_TOO_LARGE: return "CCL_TOO_LARGE";
        case CCL_CUDA_ERROR: return "CCL_CUDA_ERROR";
        case CCL_NCCL_ERROR: return "CCL_NCCL_ERROR";
        case CCL_OUT_OF_MEMORY: return "CCL_OUT_OF_MEMORY";
    }
    return "CCL_UNKNOWN_STATUS";
}

const char *ccl_version(void) { return "0.1.0"; }

ccl_status ccl_label(const uint8_t *img, int H, int W, int32_t *labels, int32_t *n_components,
                     ccl_stream_t stream) {
    return ccl_label_threshold(img, H, W, 0, labels, n_components, stream);
}

static ccl_status label_oneshot(const uint8_t *img, int B, int H, int W, int threshold, int32_t *labels,
                                int32_t *n_components, ccl_stream_t stream);

ccl_status ccl_label_threshold(const uint8_t *img, int H, int W, int threshold, int32_t *labels,
                               int32_t *n_components, ccl_stream_t stream) {
    return label_oneshot(img, 1, H, W, threshold, labels, n_components, stream);
}

ccl_status ccl_label_batch(const uint8_t *imgs, int B, int H, int W, int32_t *labels,
                           int32_t *n_components, ccl_stream_t stream) {
    return label_oneshot(imgs, B, H, W, 0, labels, n_components, stream);
}

static ccl_status label_oneshot(const uint8_t *img, int B, int H, int W, int threshold, int32_t *labels,
                                int32_t *n_components, ccl_stream_t stream) {
    if (B < 1) return CCL_INVALID_ARGUMENT;
    ccl_status st = check_shape(H, W);
    if (st != CCL_OK) return st;
    if ((int64_t)B * H > INT32_MAX || (st = check_shape(B * H, W)) != CCL_OK) return CCL_TOO_LARGE;
    if (threshold < 0 || threshold > 255) return CCL_INVALID_ARGUMENT;
    if ((st = check_buffers(img, labels, n_components, B * H, W)) != CCL_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Geometry g = make_geometry_batch(B, H, W);
    g.thr = threshold;
    size_t offs[32], total;
    workspace_layout(g, offs, &total);
    void *mem = nullptr;
    cudaError_t e = cudaMallocAsync(&mem, total, s);
    if (e == cudaErrorMemoryAllocation) return CCL_OUT_OF_MEMORY;
    if (e != cudaSuccess) return CCL_CUDA_ERROR;
    Workspace ws = workspace_bind(g, mem);
    e = workspace_poison(mem, total, s);
    if (e == cudaSuccess) e = workspace_init(ws, s);
    if (e == cudaSuccess) e = run_pipeline(g, ws, img, labels, n_components, s, nullptr);
    cudaError_t e2 = cudaFreeAsync(mem, s);
    if (e != cudaSuccess || e2 != cudaSuccess) return CCL_CUDA_ERROR;
    return CCL_OK;
}

ccl_status ccl_plan_create(int H, int W, ccl_plan *plan_out) {
    return ccl_plan_create_batch(1, H, W, plan_out);
}

ccl_status ccl_plan_create_batch(int B, int H, int W, ccl_plan *plan_out) {
    if (!plan_out) return CCL_INVALID_ARGUMENT;
    *plan_out = nullptr;
    if (B < 1) return CCL_INVALID_ARGUMENT;
    ccl_status st = check_shape(H, W);
    if (st != CCL_OK) return st;
    if ((int64_t)B * H > INT32_MAX || check_shape(B * H, W) != CCL_OK) return CCL_TOO_LARGE;
    ccl_plan p = new (std::nothrow) ccl_plan_st;
    if (!p) return CCL_OUT_OF_MEMORY;
    p->g = make_geometry_batch(B, H, W);
    size_t offs[32];
    workspace_layout(p->g, offs, &p->ws_bytes);
    cudaError_t e = cudaMalloc(&p->ws_mem, p->ws_bytes);
    if (e != cudaSuccess) {
        delete p;
        return e == cudaErrorMemoryAllocation ? CCL_OUT_OF_MEMORY : CCL_CUDA_ERROR;
    }
    p->ws = workspace_bind(p->g, p->ws_mem);
    // the hand-over hint word (see Workspace::k1hint_dev)
    int32_t *hint = nullptr, *hint_dev = nullptr;
    if (cudaHostAlloc(&hint, sizeof(int32_t), cudaHostAllocMapped) == cudaSuccess) {
        *hint = -1;
        if (cudaHostGetDevicePointer(reinterpret_cast<void **>(&hint_dev), hint, 0) == cudaSuccess) {
            p->hint = hint;
            p->ws.k1hint_dev = hint_dev;
            p->ws.k1hint_host = hint;
        } else {
            cudaFreeHost(hint);
        }
    }
    cudaGetLastError();  // (no hint: the full hand-over grid every call)
    if (workspace_poison(p->ws_mem, p->ws_bytes, 0) != cudaSuccess || workspace_init(p->ws, 0) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        cudaFree(p->ws_mem);
        if (p->hint) cudaFreeHost(p->hint);
        delete p;
        return CCL_CUDA_ERROR;
    }
    *plan_out = p;
    return CCL_OK;
}

static void free_host_pipe(ccl_plan p) {
    if (!p->host_init) return;
    for (cudaStream_t s : {p->s_h2d, p->s_cmp, p->s_d2h})
        if (s) cudaStreamSynchronize(s);
    for (int k = 0; k < 2; k++) {
        for (cudaEvent_t e : {p->ev_h2d[k], p->ev_cmp[k], p->ev_d2h[k]})
            if (e) cudaEventDestroy(e);
        if (p->a_img[k]) cudaFree(p->a_img[k]);
        if (p->a_lab[k]) cudaFree(p->a_lab[k]);
        if (p->a_n[k]) cudaFree(p->a_n[k]);
    }
    for (cudaStream_t s : {p->s_h2d, p->s_cmp, p->s_d2h})
        if (s) cudaStreamDestroy(s);
    if (p->ev_dev) cudaEventDestroy(p->ev_dev);
    p->host_init = false;
}

static cudaError_t init_host_pipe(ccl_plan p) {
    if (p->host_init) return cudaSuccess;
    p->host_init = true;  // (free_host_pipe releases whatever was made)
    const size_t n = (size_t)p->g.H * (size_t)p->g.W;
    const size_t nn = sizeof(int32_t) * (size_t)(p->g.nTy / p->g.tpi);
    cudaError_t e;
    for (cudaStream_t *s : {&p->s_h2d, &p->s_cmp, &p->s_d2h})
        if ((e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&p->ev_dev, cudaEventDisableTiming)) != cudaSuccess) return e;
    if (p->dev_called) {  // device-path calls made before the pipe existed
        if ((e = cudaEventRecord(p->ev_dev, p->last_dev_stream)) != cudaSuccess) return e;
        p->dev_pending = true;
    }
    for (int k = 0; k < 2; k++) {
        for (cudaEvent_t *ev : {&p->ev_h2d[k], &p->ev_cmp[k], &p->ev_d2h[k]})
            if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaMalloc(&p->a_img[k], n)) != cudaSuccess || (e = cudaMalloc(&p->a_lab[k], n * 4)) != cudaSuccess ||
            (e = cudaMalloc(&p->a_n[k], nn)) != cudaSuccess)
            return e;
    }
    return cudaSuccess;
}

ccl_status ccl_plan_destroy(ccl_plan p) {
    if (!p) return CCL_INVALID_ARGUMENT;
    free_host_pipe(p);
    cudaError_t e = cudaSuccess;
    if (p->ws_mem) e = cudaFree(p->ws_mem);
    if (p->hint) cudaFreeHost(p->hint);
    free_events(p);
    delete p;
    return e == cudaSuccess ? CCL_OK : CCL_CUDA_ERROR;
}

ccl_status ccl_plan_set_threshold(ccl_plan p, int threshold) {
    if (!p || threshold < 0 || threshold > 255) return CCL_INVALID_ARGUMENT;
    p->g.thr = threshold;
    return CCL_OK;
}

ccl_status ccl_plan_workspace_bytes(ccl_plan p, uint64_t *bytes) {
    if (!p || !bytes) return CCL_INVALID_ARGUMENT;
    *bytes = p->ws_bytes;
    return CCL_OK;
}

ccl_status ccl_plan_label(ccl_plan p, const uint8_t *img, int32_t *labels, int32_t *n_components,
                          ccl_stream_t stream) {
    if (!p) return CCL_INVALID_ARGUMENT;
    ccl_status st = check_buffers(img, labels, n_components, p->g.H, p->g.W);
    if (st != CCL_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaEvent_t *ev = nullptr;
    if (p->prof_sets > 0) {
        ev = p->ev + (p->prof_calls % p->prof_sets) * (K_COUNT + 1);
        p->prof_calls++;
    }
    cudaError_t e = cudaSuccess;
    if (p->host_init) {  // after the async host path's last kernels (same workspace)
        e = cudaStreamWaitEvent(s, p->ev_cmp[p->slot ^ 1], 0);
    }
    if (e == cudaSuccess) e = run_pipeline(p->g, p->ws, img, labels, n_components, s, ev);
    if (e == cudaSuccess && p->host_init) {
        e = cudaEventRecord(p->ev_dev, s);
        p->dev_pending = true;
    }
    p->dev_called = true;
    p->last_dev_stream = s;
    return e == cudaSuccess ? CCL_OK : CCL_CUDA_ERROR;
}

ccl_status ccl_plan_label_host_async(ccl_plan p, const uint8_t *h_img, int32_t *h_labels,
                                     int32_t *h_n_components, ccl_stream_t stream) {
    if (!p || !h_img || !h_labels || !h_n_components) return CCL_INVALID_ARGUMENT;
    const size_t n = (size_t)p->g.H * (size_t)p->g.W;
    const size_t nn = sizeof(int32_t) * (size_t)(p->g.nTy / p->g.tpi);
    cudaError_t e = init_host_pipe(p);
    if (e != cudaSuccess) {
        free_host_pipe(p);
        return e == cudaErrorMemoryAllocation ? CCL_OUT_OF_MEMORY : CCL_CUDA_ERROR;
    }
    const int k = p->slot;
    p->slot ^= 1;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
#define CKA(x)                                   \
    do {                                         \
        if ((x) != cudaSuccess) return CCL_CUDA_ERROR; \
    } while (0)
    // H2D into slot k once the kernels of the call before last are done with it
    CKA(cudaStreamWaitEvent(p->s_h2d, p->ev_cmp[k], 0));
    CKA(cudaMemcpyAsync(p->a_img[k], h_img, n, cudaMemcpyHostToDevice, p->s_h2d));
    CKA(cudaEventRecord(p->ev_h2d[k], p->s_h2d));
    // kernels: after this call's H2D and after the D2H that last read slot k
    CKA(cudaStreamWaitEvent(p->s_cmp, p->ev_h2d[k], 0));
    CKA(cudaStreamWaitEvent(p->s_cmp, p->ev_d2h[k], 0));
    if (p->dev_pending) {  // a device-path call since the last async call
        CKA(cudaStreamWaitEvent(p->s_cmp, p->ev_dev, 0));
        p->dev_pending = false;
    }
    cudaEvent_t *ev = nullptr;
    if (p->prof_sets > 0) {
        ev = p->ev + (p->prof_calls % p->prof_sets) * (K_COUNT + 1);
        p->prof_calls++;
    }
    CKA(run_pipeline(p->g, p->ws, p->a_img[k], p->a_lab[k], p->a_n[k], p->s_cmp, ev));
    CKA(cudaEventRecord(p->ev_cmp[k], p->s_cmp));
    // D2H of the labels and N, then the caller's stream waits for it
    CKA(cudaStreamWaitEvent(p->s_d2h, p->ev_cmp[k], 0));
    CKA(cudaMemcpyAsync(h_labels, p->a_lab[k], n * 4, cudaMemcpyDeviceToHost, p->s_d2h));
    CKA(cudaMemcpyAsync(h_n_components, p->a_n[k], nn, cudaMemcpyDeviceToHost, p->s_d2h));
    CKA(cudaEventRecord(p->ev_d2h[k], p->s_d2h));
    CKA(cudaStreamWaitEvent(s, p->ev_d2h[k], 0));
#undef CKA
    return CCL_OK;
}

ccl_status ccl_plan_label_host(ccl_plan p, const uint8_t *h_img, int32_t *h_labels,
                               int32_t *h_n_components, ccl_stream_t stream) {
    ccl_status st = ccl_plan_label_host_async(p, h_img, h_labels, h_n_components, stream);
    if (st != CCL_OK) return st;
    return cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? CCL_OK : CCL_CUDA_ERROR;
}

ccl_status ccl_plan_set_profiling(ccl_plan p, int nsets) {
    if (!p || nsets < 0) return CCL_INVALID_ARGUMENT;
    free_events(p);
    if (nsets == 0) return CCL_OK;
    p->ev = new (std::nothrow) cudaEvent_t[(size_t)nsets * (K_COUNT + 1)]();
    if (!p->ev) return CCL_OUT_OF_MEMORY;
    p->prof_sets = nsets;
    for (int i = 0; i < nsets * (K_COUNT + 1); i++)
        if (cudaEventCreate(&p->ev[i]) != cudaSuccess) return CCL_CUDA_ERROR;
    return CCL_OK;
}

ccl_status ccl_plan_kernel_times(ccl_plan p, const char **names, float *ms, int cap, int *count) {
    if (!p || !count) return CCL_INVALID_ARGUMENT;
    *count = K_COUNT;
    if (p->prof_sets == 0 || p->prof_calls == 0) return CCL_INVALID_ARGUMENT;
    const int nset = (int)(p->prof_calls < p->prof_sets ? p->prof_calls : p->prof_sets);
    for (int i = 0; i < K_COUNT && i < cap; i++) {
        if (names) names[i] = kKernelNames[i];
        if (!ms) continue;
        double acc = 0;
        for (int k = 0; k < nset; k++) {
            cudaEvent_t *e = p->ev + (size_t)k * (K_COUNT + 1);
            if (cudaEventSynchronize(e[i + 1]) != cudaSuccess) return CCL_CUDA_ERROR;
            float t = 0;
            if (cudaEventElapsedTime(&t, e[i], e[i + 1]) != cudaSuccess) return CCL_CUDA_ERROR;
            acc += t;
        }
        ms[i] = (float)(acc / nset);
    }
    return CCL_OK;
}

ccl_status ccl_plan_counters(ccl_plan p, uint64_t *out, int cap, int *count) {
    if (!p || !count) return CCL_INVALID_ARGUMENT;
    *count = STAT_COUNT;
    if (!out || cap <= 0) return CCL_OK;
    unsigned long long h[STAT_COUNT];
    if (cudaMemcpy(h, p->ws.stats, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return CCL_CUDA_ERROR;
    for (int i = 0; i < STAT_COUNT && i < cap; i++) out[i] = h[i];
    return CCL_OK;
}

}  // extern "C"

// Development hook (not part of include/ccl.h): base pointer and byte offsets
// of the plan's workspace arrays, in Workspace declaration order.
extern "C" int ccl_debug_workspace(ccl_plan p, void **base, uint64_t *offs, int cap) {
    if (!p || !base || !offs) return CCL_INVALID_ARGUMENT;
    size_t o[32], total;
    workspace_layout(p->g, o, &total);
    *base = p->ws_mem;
    for (int i = 0; i < A_COUNT && i < cap; i++) offs[i] = o[i];
    return A_COUNT;
}

namespace cclb { extern int g_k1_stop, g_k1_exper, g_no_small, g_no_wide; }
extern "C" int ccl_debug_set(int key, int value) {
    if (key == 1) { cclb::g_k1_stop = value; return 0; }
    if (key == 2) { cclb::g_k1_exper = value; return 0; }
    if (key == 3) { cclb::g_no_small = value; return 0; }
    if (key == 4) { cclb::g_no_wide = value; return 0; }
    if (key == 5) { cclb::g_poison = (uint32_t)value; return 0; }
    return 1;
}
