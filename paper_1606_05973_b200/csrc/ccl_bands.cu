// ccl_bands.cu -- one image as contiguous row bands (multi-GPU), the B200
// analogue of PARemSP's row chunks: every band is labelled
// locally with keys that carry its global row offset (PARemSP's per-thread
// label base, "count <- start x col"); the boundary rows of
// all bands are all-gathered and every rank resolves the small cross-band
// equivalence graph on its GPU (PARemSP's boundary merge);
// per-band root counts are all-gathered (with the band-local labels of the
// boundary roots) so each band numbers its labels after the earlier bands.  Everything stays on the device and on the stream: no
// host synchronization inside a call.
//
// Protocol per band (the same code drives NCCL ranks and the single-GPU
// "virtual bands" mode, which only differs in how the two all-gathers move
// bytes):
//   A  tile labeling + tile-edge merge of the band; per pixel of its first and
//      last row the band-local root key and node (2W "slots"), and for every
//      slot the first slot of the same band-local component
//   X1 all-gather of slot keys and representatives
//   B  every rank: union-find over all nb*2W slots (band-local components,
//      8-adjacency across every band boundary; the smaller key wins), then
//      this band's components whose class starts elsewhere are linked: to the
//      other component's node in this band, or to a foreign slot (-2-slot)
//   C  roots + numbering scan of the band -> N_band; the band-local labels
//      of the band's boundary-slot roots (both need only the band itself)
//   X2 all-gather of the band records (N_band, then those 2W labels): the
//      foreign-label table and the counts in one collective (a foreign
//      root's label = its band-local label + the N of the bands before its
//      band; round 1 gathered N and the labels in two)
//   D  offset of this band = sum of N over earlier bands; N (K4's first
//      thread, from the gathered records)
//   E  labels of merged components + label write
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <numeric>
#include <unordered_map>
#include <vector>

#include "ccl.h"
#include "ccl_internal.cuh"

using namespace cclb;

namespace {

// ---------------------------------------------------------------- resolver
// Cross-band classes over the boundary-row keys.  rows[2k] / rows[2k+1] are
// band k's first / last row (per-pixel keys, -1 = background).  Pixels of two
// consecutive bands' facing rows that are 8-adjacent are joined; equal keys
// are the same node.  Returns, for every key, the minimum key of its class.
struct Resolver {
    std::vector<int64_t> keys;  // sorted distinct keys
    std::vector<int32_t> par;   // union-find over key indices (parent <= child)

    int idx(int64_t k) const {
        return (int)(std::lower_bound(keys.begin(), keys.end(), k) - keys.begin());
    }
    int find(int x) {
        while (par[x] != x) {
            par[x] = par[par[x]];
            x = par[x];
        }
        return x;
    }
    void unite(int a, int b) {
        a = find(a);
        b = find(b);
        if (a == b) return;
        if (a < b) std::swap(a, b);
        par[a] = b;  // the smaller key (earlier raster position) stays the root
    }
    void build(int nb, int W, const int64_t *const *rows) {
        keys.clear();
        for (int r = 0; r < 2 * nb; r++)
            for (int c = 0; c < W; c++)
                if (rows[r][c] >= 0) keys.push_back(rows[r][c]);
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        par.resize(keys.size());
        std::iota(par.begin(), par.end(), 0);
        for (int k = 0; k + 1 < nb; k++) {
            const int64_t *up = rows[2 * k + 1], *lo = rows[2 * (k + 1)];
            for (int c = 0; c < W; c++) {
                if (lo[c] < 0) continue;
                const int a = idx(lo[c]);
                for (int dc = -1; dc <= 1; dc++) {
                    const int cc = c + dc;
                    if (cc >= 0 && cc < W && up[cc] >= 0) unite(a, idx(up[cc]));
                }
            }
        }
    }
    int64_t class_min(int64_t k) { return keys[find(idx(k))]; }
};

// ---------------------------------------------------------------- one band
struct Band {
    Geometry g;
    Workspace ws;
    void *mem = nullptr;
    int32_t *d_nodes = nullptr;    // 2W band-local root node of each slot (-1 background)
    unsigned long long *d_noderep = nullptr;  // scratch: (epoch, first slot) of each node
    size_t noderep_count = 0;
    uint32_t epoch = 0;              // calls on this band (band_rep's epoch)
    int32_t *d_small = nullptr;    // [0] N_band, [1] band offset
    int32_t *hint = nullptr;       // mapped pinned host word: K1's last hand-over count (Workspace::k1hint_dev)
    int band_H = 0, row0 = 0;

    ~Band() { release(); }
    void release() {
        if (hint) cudaFreeHost(hint);
        hint = nullptr;
        if (mem) cudaFree(mem);
        if (d_nodes) cudaFree(d_nodes);
        if (d_noderep) cudaFree(d_noderep);
        if (d_small) cudaFree(d_small);
        mem = nullptr;
        d_nodes = nullptr;
        d_noderep = nullptr;
        d_small = nullptr;
    }
};

// Cross-band tables shared by the bands of one image (replicated per rank).
struct XBand {
    int nb = 0, W = 0;
    int64_t *keys = nullptr;  // nb*2W slot keys (-1 background)
    int32_t *reps = nullptr;  // nb*2W representative slot (band-local index)
    int32_t *spar = nullptr;  // nb*2W slot union-find
    int32_t *recs = nullptr;  // nb*(2W+1) band records: N_band, then its slots' band-local root labels
    ~XBand() { release(); }
    void release() {
        if (keys) cudaFree(keys);
        if (reps) cudaFree(reps);
        if (spar) cudaFree(spar);
        if (recs) cudaFree(recs);
        keys = nullptr;
        reps = nullptr;
        spar = nullptr;
        recs = nullptr;
    }
};

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess)                                                   \
            return e_ == cudaErrorMemoryAllocation ? CCL_OUT_OF_MEMORY : CCL_CUDA_ERROR; \
    } while (0)
#define CKN(x)                                              \
    do {                                                    \
        if ((x) != ncclSuccess) return CCL_NCCL_ERROR;      \
    } while (0)

ccl_status band_init(Band &b, int band_H, int W, int row0) {
    b.band_H = band_H;
    b.row0 = row0;
    b.g = make_geometry(band_H, W);
    b.g.row0 = row0;
    size_t offs[32], total;
    workspace_layout(b.g, offs, &total);
    CK(cudaMalloc(&b.mem, total));
    b.ws = workspace_bind(b.g, b.mem);
    CK(workspace_poison(b.mem, total, 0));
    CK(workspace_init(b.ws, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMalloc(&b.d_nodes, sizeof(int32_t) * 2 * W));
    b.noderep_count = (size_t)b.g.nT * b.g.capb;
    CK(cudaMalloc(&b.d_noderep, sizeof(unsigned long long) * b.noderep_count));
    CK(cudaMemset(b.d_noderep, 0xFF, sizeof(unsigned long long) * b.noderep_count));
    CK(cudaMalloc(&b.d_small, sizeof(int32_t) * 4));
    b.ws.boff = b.d_small + 1;
    // the hand-over hint (as a plan's): later band steps launch K1's idle
    // hand-over pass small
    int32_t *hint_dev = nullptr;
    if (cudaHostAlloc(&b.hint, sizeof(int32_t), cudaHostAllocMapped) == cudaSuccess) {
        *b.hint = -1;
        if (cudaHostGetDevicePointer(reinterpret_cast<void **>(&hint_dev), b.hint, 0) == cudaSuccess) {
            b.ws.k1hint_dev = hint_dev;
            b.ws.k1hint_host = b.hint;
        }
    }
    cudaGetLastError();  // (no hint: the full hand-over grid every step)
    return CCL_OK;
}

ccl_status xband_init(XBand &x, int nb, int W) {
    x.nb = nb;
    x.W = W;
    const size_t n = (size_t)nb * 2 * W;
    CK(cudaMalloc(&x.keys, sizeof(int64_t) * n));
    CK(cudaMalloc(&x.reps, sizeof(int32_t) * n));
    CK(cudaMalloc(&x.spar, sizeof(int32_t) * n));
    CK(cudaMalloc(&x.recs, sizeof(int32_t) * ((size_t)nb * (2 * W + 1))));
    return CCL_OK;
}

// A: local labeling; slot keys / nodes / representatives into (keys, reps)
// Profiling events of a band step (ShardPlan profiling), SHARD_EV per set:
// 0 K1, 1 K2, 2 cross-band exchange (row roots, representatives,
// all-gather, slot unions, links), 3 K3, 4 export + record all-gather +
// offsets, 5 K4, 6 K5, 7 end.
constexpr int SHARD_EV = 8;
const char *const kShardNames[SHARD_EV - 1] = {"k_tile_local", "k_border", "xband_exchange", "k_number",
                                                "xband_export", "k_fixup", "k_write"};

ccl_status band_phase_a(Band &b, const uint8_t *img, int64_t *keys, int32_t *reps, int32_t *spar, int spar_lo,
                        int spar_hi, cudaStream_t s, cudaEvent_t *ev = nullptr) {
    const int W = b.g.W;
    CK(run_stage_local(b.g, b.ws, img, s, ev));
    if (ev) CK(cudaEventRecord(ev[2], s));
    CK(band_row_roots(b.g, b.ws, keys, b.d_nodes, b.d_noderep, ++b.epoch, s));
    CK(band_rep(b.d_nodes, 2 * W, b.d_noderep, reps, spar, spar_lo, spar_hi, s));
    return CCL_OK;
}

// B (after the slot tables are complete): link this band's components whose
// class starts elsewhere.  C: roots + numbering scan -> N_band, then the
// band-local labels of its slots' roots: the band's record (N_band, 2W
// labels) of the gathered table, complete before the one all-gather X2.
ccl_status band_phase_bc(Band &b, const XBand &x, int self, cudaStream_t s, cudaEvent_t *ev = nullptr) {
    int32_t *rec = x.recs + (size_t)self * (2 * x.W + 1);
    CK(band_link(b.ws, x.W, self, x.keys, x.spar, b.d_nodes, s));
    CK(run_stage_count(b.g, b.ws, rec, s, ev ? ev + 3 : nullptr));  // ev[3]
    if (ev) CK(cudaEventRecord(ev[4], s));
    CK(band_export(b.g, b.ws, b.d_nodes, rec + 1, 2 * x.W, s));
    return CCL_OK;
}

// D + E (every record gathered): labels of merged components (foreign ones
// from the gathered records; K4's first thread also stores the band offset =
// N of the earlier bands, and N) + label write
ccl_status band_phase_e(Band &b, const XBand &x, int self, int32_t *n_total, int32_t *labels, cudaStream_t s,
                        cudaEvent_t *ev = nullptr) {
    b.ws.xlab = x.recs;
    b.ws.xself = self;
    b.ws.xnb = x.nb;
    b.ws.xntotal = n_total;
    CK(run_stage_final(b.g, b.ws, labels, s, ev ? ev + 5 : nullptr));  // ev[5], ev[6], ev[7]
    return CCL_OK;
}

}  // namespace

extern "C" {

int ccl_xband_resolve(int nb, int W, const int64_t *const *rows, int self, int64_t *out_min) {
    if (nb < 1 || W < 1 || !rows || !out_min || self < 0 || self >= nb) return CCL_INVALID_ARGUMENT;
    Resolver res;
    res.build(nb, W, rows);
    for (int r = 0; r < 2; r++)
        for (int c = 0; c < W; c++) {
            const int64_t k = rows[2 * self + r][c];
            out_min[(size_t)r * W + c] = k >= 0 ? res.class_min(k) : -1;
        }
    return CCL_OK;
}

ccl_status ccl_label_banded(const uint8_t *img, int H, int W, int nbands, int32_t *labels,
                            int32_t *n_components, ccl_stream_t stream) {
    if (H < 1 || W < 1 || nbands < 1 || nbands > H || !img || !labels || !n_components)
        return CCL_INVALID_ARGUMENT;
    if ((int64_t)H * W > INT32_MAX) return CCL_TOO_LARGE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    std::vector<int> bh(nbands), r0(nbands);
    for (int k = 0, acc = 0; k < nbands; k++) {
        bh[k] = H / nbands + (k >= nbands - H % nbands ? 1 : 0);
        r0[k] = acc;
        acc += bh[k];
    }
    std::vector<Band> bands(nbands);
    XBand x;
    ccl_status st = xband_init(x, nbands, W);
    if (st != CCL_OK) return st;
    for (int k = 0; k < nbands; k++)
        if ((st = band_init(bands[k], bh[k], W, r0[k])) != CCL_OK) return st;
    const size_t slots = 2 * (size_t)W;
    // A (+ X1: every band writes its slots straight into the shared tables)
    for (int k = 0; k < nbands; k++)
        if ((st = band_phase_a(bands[k], img + (size_t)r0[k] * W, x.keys + k * slots, x.reps + k * slots, x.spar,
                               (int)(k * slots), (int)((k + 1) * slots), s)) != CCL_OK)
            return st;
    CK(band_resolve(nbands, W, x.keys, x.reps, x.spar, s));
    // B + C (+ X2: every band writes its record straight into the shared table)
    for (int k = 0; k < nbands; k++)
        if ((st = band_phase_bc(bands[k], x, k, s)) != CCL_OK) return st;
    // D + E
    for (int k = 0; k < nbands; k++)
        if ((st = band_phase_e(bands[k], x, k, k == 0 ? n_components : nullptr, labels + (size_t)r0[k] * W, s)) !=
            CCL_OK)
            return st;
    CK(cudaStreamSynchronize(s));  // the band workspaces are freed on return
    return CCL_OK;
}

}  // extern "C"

struct ccl_shard_plan_st {
    Band b;
    XBand x;
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, W = 0;
    int prof_sets = 0;          // profiling ring size (0 = off)
    cudaEvent_t *ev = nullptr;  // prof_sets * SHARD_EV events
    long long prof_calls = 0;
    void free_events() {
        if (ev) {
            for (int i = 0; i < prof_sets * SHARD_EV; i++)
                if (ev[i]) cudaEventDestroy(ev[i]);
            delete[] ev;
        }
        ev = nullptr;
        prof_sets = 0;
        prof_calls = 0;
    }
    ~ccl_shard_plan_st() { free_events(); }
};

extern "C" {

// The argument check is collective: every rank's (band_H, row0, W, H_total,
// local verdict) is all-gathered BEFORE any rank returns, so a rank with bad
// arguments makes every rank return CCL_INVALID_ARGUMENT / CCL_TOO_LARGE
// instead of leaving the others blocked in the all-gather.  `extra` is the
// caller's own local verdict (e.g. the buffer checks of ccl_label_sharded).
static ccl_status shard_plan_create(int band_H, int W, int row0, int H_total, ccl_nccl_comm_t comm_,
                                    ccl_stream_t stream, ccl_status extra, ccl_shard_plan *plan_out) {
    if (!plan_out) return CCL_INVALID_ARGUMENT;  // (no communicator use is possible without a result slot)
    *plan_out = nullptr;
    if (!comm_) return CCL_INVALID_ARGUMENT;     // no collective without a communicator
    ccl_status local = extra;
    if (local == CCL_OK && (band_H < 1 || W < 1 || row0 < 0 || H_total < 1 || row0 + band_H > H_total))
        local = CCL_INVALID_ARGUMENT;
    if (local == CCL_OK && (int64_t)H_total * W > INT32_MAX) local = CCL_TOO_LARGE;
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(comm_);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int nranks = 0, rank = 0;
    CKN(ncclCommCount(comm, &nranks));
    CKN(ncclCommUserRank(comm, &rank));
    // collective argument check: every rank's (band_H, row0, W, H_total, status)
    constexpr int NM = 5;
    int32_t *d_meta = nullptr;
    CK(cudaMalloc(&d_meta, sizeof(int32_t) * NM * (nranks + 1)));
    int32_t mine[NM] = {band_H, row0, W, H_total, (int32_t)local};
    CK(cudaMemcpyAsync(d_meta, mine, sizeof(mine), cudaMemcpyHostToDevice, s));
    CKN(ncclAllGather(d_meta, d_meta + NM, NM, ncclInt32, comm, s));
    std::vector<int32_t> meta(NM * (size_t)nranks);
    CK(cudaMemcpyAsync(meta.data(), d_meta + NM, sizeof(int32_t) * NM * nranks, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(d_meta);
    int64_t acc = 0;
    bool ok = true;
    ccl_status worst = CCL_OK;
    for (int k = 0; k < nranks; k++) {
        const int32_t *m = &meta[(size_t)NM * k];
        if (m[4] != CCL_OK && worst == CCL_OK) worst = (ccl_status)m[4];
        ok = ok && m[1] == acc && m[2] == W && m[3] == H_total && m[0] >= 1;
        acc += m[0];
    }
    if (worst != CCL_OK) return worst;
    if (!ok || acc != H_total) return CCL_INVALID_ARGUMENT;
    ccl_shard_plan p = new (std::nothrow) ccl_shard_plan_st;
    if (!p) return CCL_OUT_OF_MEMORY;
    p->comm = comm;
    p->nranks = nranks;
    p->rank = rank;
    p->W = W;
    ccl_status st = band_init(p->b, band_H, W, row0);
    if (st == CCL_OK) st = xband_init(p->x, nranks, W);
    if (st != CCL_OK) {
        delete p;
        return st;
    }
    *plan_out = p;
    return CCL_OK;
}

ccl_status ccl_shard_plan_create(int band_H, int W, int row0, int H_total, ccl_nccl_comm_t comm_,
                                 ccl_stream_t stream, ccl_shard_plan *plan_out) {
    return shard_plan_create(band_H, W, row0, H_total, comm_, stream, CCL_OK, plan_out);
}

ccl_status ccl_shard_plan_destroy(ccl_shard_plan p) {
    if (!p) return CCL_INVALID_ARGUMENT;
    delete p;
    return CCL_OK;
}

ccl_status ccl_shard_plan_label(ccl_shard_plan p, const uint8_t *band_img, int32_t *band_labels,
                                int32_t *n_components, ccl_stream_t stream) {
    if (!p || !band_img || !band_labels || !n_components) return CCL_INVALID_ARGUMENT;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Band &b = p->b;
    XBand &x = p->x;
    const size_t slots = 2 * (size_t)p->W;
    const int self = p->rank;
    cudaEvent_t *ev = nullptr;
    if (p->prof_sets > 0) {
        ev = p->ev + (p->prof_calls % p->prof_sets) * SHARD_EV;
        p->prof_calls++;
    }
    // A + X1 (own slots written in place, then gathered)
    ccl_status st = band_phase_a(b, band_img, x.keys + self * slots, x.reps + self * slots, x.spar, 0,
                                 (int)(p->nranks * slots), s, ev);
    if (st != CCL_OK) return st;
    CKN(ncclGroupStart());
    CKN(ncclAllGather(x.keys + self * slots, x.keys, slots, ncclInt64, p->comm, s));
    CKN(ncclAllGather(x.reps + self * slots, x.reps, slots, ncclInt32, p->comm, s));
    CKN(ncclGroupEnd());
    // B + C + X2
    CK(band_resolve(p->nranks, p->W, x.keys, x.reps, x.spar, s));
    if ((st = band_phase_bc(b, x, self, s, ev)) != CCL_OK) return st;
    // X2: every band's record (N_band + its slots' band-local root labels)
    const size_t rec = slots + 1;
    CKN(ncclAllGather(x.recs + self * rec, x.recs, rec, ncclInt32, p->comm, s));
    // D + E
    return band_phase_e(b, x, self, n_components, band_labels, s, ev);
}

ccl_status ccl_shard_plan_set_profiling(ccl_shard_plan p, int nsets) {
    if (!p || nsets < 0) return CCL_INVALID_ARGUMENT;
    p->free_events();
    if (nsets == 0) return CCL_OK;
    p->ev = new (std::nothrow) cudaEvent_t[(size_t)nsets * SHARD_EV]();
    if (!p->ev) return CCL_OUT_OF_MEMORY;
    p->prof_sets = nsets;
    for (int i = 0; i < nsets * SHARD_EV; i++)
        if (cudaEventCreate(&p->ev[i]) != cudaSuccess) return CCL_CUDA_ERROR;
    return CCL_OK;
}

ccl_status ccl_shard_plan_kernel_times(ccl_shard_plan p, const char **names, float *ms, int cap, int *count) {
    if (!p || !count) return CCL_INVALID_ARGUMENT;
    *count = SHARD_EV - 1;
    if (p->prof_sets == 0 || p->prof_calls == 0) return CCL_INVALID_ARGUMENT;
    const int nset = (int)(p->prof_calls < p->prof_sets ? p->prof_calls : p->prof_sets);
    for (int i = 0; i < SHARD_EV - 1 && i < cap; i++) {
        if (names) names[i] = kShardNames[i];
        if (!ms) continue;
        double acc = 0;
        for (int k = 0; k < nset; k++) {
            cudaEvent_t *e = p->ev + (size_t)k * SHARD_EV;
            if (cudaEventSynchronize(e[i + 1]) != cudaSuccess) return CCL_CUDA_ERROR;
            float t = 0;
            if (cudaEventElapsedTime(&t, e[i], e[i + 1]) != cudaSuccess) return CCL_CUDA_ERROR;
            acc += t;
        }
        ms[i] = (float)(acc / nset);
    }
    return CCL_OK;
}

ccl_status ccl_label_sharded(const uint8_t *band_img, int band_H, int W, int row0, int H_total,
                             int32_t *band_labels, int32_t *n_components, ccl_nccl_comm_t comm,
                             ccl_stream_t stream) {
    const ccl_status local = (!band_img || !band_labels || !n_components) ? CCL_INVALID_ARGUMENT : CCL_OK;
    ccl_shard_plan p = nullptr;
    ccl_status st = shard_plan_create(band_H, W, row0, H_total, comm, stream, local, &p);
    if (st != CCL_OK) return st;
    st = ccl_shard_plan_label(p, band_img, band_labels, n_components, stream);
    // the plan's buffers are freed next: the enqueued work must be done with them
    if (cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess && st == CCL_OK)
        st = CCL_CUDA_ERROR;
    ccl_shard_plan_destroy(p);
    return st;
}

}  // extern "C"
