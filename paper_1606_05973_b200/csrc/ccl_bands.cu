// ccl_bands.cu -- one image as contiguous row bands (multi-GPU), the B200
// analogue of PARemSP's row chunks: every band is labelled
// locally with keys that carry its global row offset (PARemSP's per-thread
// label base, "count <- start x col"); the boundary rows of
// all bands are all-gathered and the small cross-band equivalence graph is
// resolved (PARemSP's boundary merge); per-band root counts
// are all-gathered so each band numbers its labels after the earlier bands.
//
// Protocol per band (the same code drives NCCL ranks and the single-GPU
// "virtual bands" mode, which only differs in how the three all-gathers move
// bytes):
//   A  pack + tile labeling + tile-edge merge of the band (device)
//      per-pixel root keys of the band's first and last row (device)
//   X1 all-gather of those keys
//   B  host: resolve the cross-band classes; a band root whose class minimum
//      is another key is re-linked -- to that root's node when it is in the
//      same band, else to a foreign-label slot (-2-f)
//   C  roots + numbering scan of the band -> N_band
//   X2 all-gather of N_band -> offset of this band = sum over earlier bands
//   D  labels of the band's boundary-row roots (device)
//   X3 all-gather of those labels; host fills the foreign-label table
//   E  component labels + label write (device)
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
    // device buffers: [0] first row, [1] last row
    int64_t *d_keys = nullptr;  // 2 * W
    int32_t *d_nodes = nullptr; // 2 * W
    int32_t *d_exp = nullptr;   // 2 * W
    int32_t *d_small = nullptr; // [0] N_band
    int32_t *d_xlab = nullptr;  // foreign labels
    int2 *d_act = nullptr;      // re-links
    size_t xlab_cap = 0, act_cap = 0;
    // host copies
    std::vector<int64_t> keys;   // 2 * W
    std::vector<int32_t> nodes;  // 2 * W
    std::vector<int64_t> fkeys;  // foreign class minima (index f -> key)
    int band_H = 0, row0 = 0;
    int32_t offset = 0;          // labels of earlier bands (phase D)

    ~Band() { release(); }
    void release() {
        if (mem) cudaFree(mem);
        if (d_keys) cudaFree(d_keys);
        if (d_nodes) cudaFree(d_nodes);
        if (d_exp) cudaFree(d_exp);
        if (d_small) cudaFree(d_small);
        if (d_xlab) cudaFree(d_xlab);
        if (d_act) cudaFree(d_act);
        mem = nullptr;
        d_keys = nullptr;
        d_nodes = nullptr;
        d_exp = nullptr;
        d_small = nullptr;
        d_xlab = nullptr;
        d_act = nullptr;
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
    CK(cudaMalloc(&b.d_keys, sizeof(int64_t) * 2 * W));
    CK(cudaMalloc(&b.d_nodes, sizeof(int32_t) * 2 * W));
    CK(cudaMalloc(&b.d_exp, sizeof(int32_t) * 2 * W));
    CK(cudaMalloc(&b.d_small, sizeof(int32_t) * 4));
    b.keys.resize(2 * (size_t)W);
    b.nodes.resize(2 * (size_t)W);
    return CCL_OK;
}

// A: local labeling + boundary-row root keys (device), then copy the keys and
// nodes to the host.
ccl_status band_phase_a(Band &b, const uint8_t *img, cudaStream_t s) {
    const int W = b.g.W;
    CK(run_stage_local(b.g, b.ws, img, s, nullptr));
    CK(band_row_roots(b.g, b.ws, 0, b.d_keys, b.d_nodes, s));
    CK(band_row_roots(b.g, b.ws, b.band_H - 1, b.d_keys + W, b.d_nodes + W, s));
    CK(cudaMemcpyAsync(b.nodes.data(), b.d_nodes, sizeof(int32_t) * 2 * W, cudaMemcpyDeviceToHost, s));
    return CCL_OK;
}

// B: re-link the band's roots whose cross-band class minimum is another key.
ccl_status band_phase_b(Band &b, Resolver &res, const std::vector<int> &row0s,
                        const std::vector<int> &bandHs, int self, cudaStream_t s) {
    const int W = b.g.W;
    const int64_t keys_per_row = (int64_t)b.g.nTx * MAXRUN;  // key = grow * keys_per_row + ...
    std::unordered_map<int64_t, int32_t> own_node;           // key -> node, this band
    for (int i = 0; i < 2 * W; i++)
        if (b.keys[i] >= 0) own_node[b.keys[i]] = b.nodes[i];
    std::unordered_map<int64_t, int32_t> fidx;
    std::unordered_map<int32_t, int32_t> act;  // node -> new parent
    b.fkeys.clear();
    for (const auto &kv : own_node) {
        const int64_t m = res.class_min(kv.first);
        if (m == kv.first) continue;
        const int grow = (int)(m / keys_per_row);
        int target;
        if (grow >= b.row0 && grow < b.row0 + b.band_H) {
            target = own_node.at(m);
        } else {
            auto it = fidx.find(m);
            int f;
            if (it == fidx.end()) {
                f = (int)b.fkeys.size();
                fidx[m] = f;
                b.fkeys.push_back(m);
            } else {
                f = it->second;
            }
            target = -2 - f;
        }
        act[kv.second] = target;
    }
    (void)row0s;
    (void)bandHs;
    (void)self;
    std::vector<int2> h(act.size());
    size_t i = 0;
    for (const auto &kv : act) h[i++] = make_int2(kv.first, kv.second);
    if (h.size() > b.act_cap) {
        if (b.d_act) cudaFree(b.d_act);
        b.act_cap = h.size();
        CK(cudaMalloc(&b.d_act, sizeof(int2) * b.act_cap));
    }
    if (!h.empty()) {
        CK(cudaMemcpyAsync(b.d_act, h.data(), sizeof(int2) * h.size(), cudaMemcpyHostToDevice, s));
        CK(band_apply(b.ws, b.d_act, (int)h.size(), s));
        CK(cudaStreamSynchronize(s));  // h is a host temporary
    }
    return CCL_OK;
}

// C: roots + numbering scan of the band; N_band -> d_small[0]
ccl_status band_phase_c(Band &b, cudaStream_t s) {
    CK(run_stage_count(b.g, b.ws, b.d_small, s, nullptr));
    return CCL_OK;
}

// D: with the band offset, the labels of the boundary-row roots
ccl_status band_phase_d(Band &b, int32_t offset, cudaStream_t s) {
    const int W = b.g.W;
    b.offset = offset;
    CK(band_export(b.g, b.ws, b.d_nodes, b.d_exp, offset, s));
    CK(band_export(b.g, b.ws, b.d_nodes + W, b.d_exp + W, offset, s));
    return CCL_OK;
}

// E: foreign labels from the gathered exports, then the final stage
ccl_status band_phase_e(Band &b, const int64_t *const *all_keys, const int32_t *const *all_exp,
                        int nb, int32_t *labels, cudaStream_t s) {
    const int W = b.g.W;
    std::vector<int32_t> xl(b.fkeys.size(), 0);
    if (!b.fkeys.empty()) {
        std::unordered_map<int64_t, int32_t> lab;
        for (int j = 0; j < nb; j++)
            for (int i = 0; i < 2 * W; i++)
                if (all_exp[j][i] >= 0) lab[all_keys[j][i]] = all_exp[j][i];
        for (size_t f = 0; f < b.fkeys.size(); f++) {
            auto it = lab.find(b.fkeys[f]);
            if (it == lab.end()) return CCL_CUDA_ERROR;  // protocol invariant broken
            xl[f] = it->second;
        }
        if (xl.size() > b.xlab_cap) {
            if (b.d_xlab) cudaFree(b.d_xlab);
            b.xlab_cap = xl.size();
            CK(cudaMalloc(&b.d_xlab, sizeof(int32_t) * b.xlab_cap));
        }
        CK(cudaMemcpyAsync(b.d_xlab, xl.data(), sizeof(int32_t) * xl.size(), cudaMemcpyHostToDevice, s));
    }
    b.ws.xlab = b.d_xlab;
    CK(run_stage_final(b.g, b.ws, labels, b.offset, s, nullptr));
    CK(cudaStreamSynchronize(s));  // xl is a host temporary
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
    for (int k = 0; k < nbands; k++) {
        ccl_status st = band_init(bands[k], bh[k], W, r0[k]);
        if (st != CCL_OK) return st;
    }
    // A + X1
    std::vector<const int64_t *> rows(2 * nbands);
    for (int k = 0; k < nbands; k++) {
        ccl_status st = band_phase_a(bands[k], img + (size_t)r0[k] * W, s);
        if (st != CCL_OK) return st;
        CK(cudaMemcpyAsync(bands[k].keys.data(), bands[k].d_keys, sizeof(int64_t) * 2 * W,
                           cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    for (int k = 0; k < nbands; k++) {
        rows[2 * k] = bands[k].keys.data();
        rows[2 * k + 1] = bands[k].keys.data() + W;
    }
    Resolver res;
    res.build(nbands, W, rows.data());
    // B + C + X2
    std::vector<int32_t> nband(nbands);
    for (int k = 0; k < nbands; k++) {
        ccl_status st = band_phase_b(bands[k], res, r0, bh, k, s);
        if (st == CCL_OK) st = band_phase_c(bands[k], s);
        if (st != CCL_OK) return st;
        CK(cudaMemcpyAsync(&nband[k], bands[k].d_small, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    // D + X3
    std::vector<std::vector<int32_t>> exps(nbands, std::vector<int32_t>(2 * (size_t)W));
    int32_t off = 0;
    for (int k = 0; k < nbands; k++) {
        ccl_status st = band_phase_d(bands[k], off, s);
        if (st != CCL_OK) return st;
        off += nband[k];
        CK(cudaMemcpyAsync(exps[k].data(), bands[k].d_exp, sizeof(int32_t) * 2 * W, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    std::vector<const int64_t *> akeys(nbands);
    std::vector<const int32_t *> aexp(nbands);
    for (int k = 0; k < nbands; k++) {
        akeys[k] = bands[k].keys.data();
        aexp[k] = exps[k].data();
    }
    // E
    for (int k = 0; k < nbands; k++) {
        ccl_status st = band_phase_e(bands[k], akeys.data(), aexp.data(), nbands,
                                     labels + (size_t)r0[k] * W, s);
        if (st != CCL_OK) return st;
    }
    CK(cudaMemcpyAsync(n_components, &off, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    return CCL_OK;
}

}  // extern "C"

struct ccl_shard_plan_st {
    Band b;
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, W = 0;
    int32_t total = 0;
    int64_t *d_allkeys = nullptr;
    int32_t *d_allexp = nullptr, *d_alln = nullptr;
    std::vector<int64_t> allkeys;
    std::vector<int32_t> allexp, nband;
    ~ccl_shard_plan_st() {
        if (d_allkeys) cudaFree(d_allkeys);
        if (d_allexp) cudaFree(d_allexp);
        if (d_alln) cudaFree(d_alln);
    }
};

extern "C" {

ccl_status ccl_shard_plan_create(int band_H, int W, int row0, int H_total, ccl_nccl_comm_t comm_,
                                 ccl_stream_t stream, ccl_shard_plan *plan_out) {
    if (!plan_out) return CCL_INVALID_ARGUMENT;
    *plan_out = nullptr;
    if (!comm_ || band_H < 1 || W < 1 || row0 < 0 || H_total < 1 || row0 + band_H > H_total)
        return CCL_INVALID_ARGUMENT;
    if ((int64_t)H_total * W > INT32_MAX) return CCL_TOO_LARGE;
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(comm_);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int nranks = 0, rank = 0;
    CKN(ncclCommCount(comm, &nranks));
    CKN(ncclCommUserRank(comm, &rank));
    // collective argument check: every rank's (band_H, row0, W, H_total)
    int32_t *d_meta = nullptr;
    CK(cudaMalloc(&d_meta, sizeof(int32_t) * 4 * (nranks + 1)));
    int32_t mine[4] = {band_H, row0, W, H_total};
    CK(cudaMemcpyAsync(d_meta, mine, sizeof(mine), cudaMemcpyHostToDevice, s));
    CKN(ncclAllGather(d_meta, d_meta + 4, 4, ncclInt32, comm, s));
    std::vector<int32_t> meta(4 * (size_t)nranks);
    CK(cudaMemcpyAsync(meta.data(), d_meta + 4, sizeof(int32_t) * 4 * nranks, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(d_meta);
    int acc = 0;
    bool ok = true;
    for (int k = 0; k < nranks; k++) {
        ok = ok && meta[4 * k + 1] == acc && meta[4 * k + 2] == W && meta[4 * k + 3] == H_total &&
             meta[4 * k] >= 1;
        acc += meta[4 * k];
    }
    if (!ok || acc != H_total) return CCL_INVALID_ARGUMENT;
    ccl_shard_plan p = new (std::nothrow) ccl_shard_plan_st;
    if (!p) return CCL_OUT_OF_MEMORY;
    p->comm = comm;
    p->nranks = nranks;
    p->rank = rank;
    p->W = W;
    ccl_status st = band_init(p->b, band_H, W, row0);
    if (st != CCL_OK) {
        delete p;
        return st;
    }
    if (cudaMalloc(&p->d_allkeys, sizeof(int64_t) * 2 * W * nranks) != cudaSuccess ||
        cudaMalloc(&p->d_allexp, sizeof(int32_t) * 2 * W * nranks) != cudaSuccess ||
        cudaMalloc(&p->d_alln, sizeof(int32_t) * nranks) != cudaSuccess) {
        delete p;
        return CCL_OUT_OF_MEMORY;
    }
    p->allkeys.resize(2 * (size_t)W * nranks);
    p->allexp.resize(2 * (size_t)W * nranks);
    p->nband.resize(nranks);
    *plan_out = p;
    return CCL_OK;
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
    const int W = p->W, nranks = p->nranks, rank = p->rank;
    // A + X1
    ccl_status st = band_phase_a(b, band_img, s);
    if (st != CCL_OK) return st;
    CKN(ncclAllGather(b.d_keys, p->d_allkeys, 2 * (size_t)W, ncclInt64, p->comm, s));
    CK(cudaMemcpyAsync(p->allkeys.data(), p->d_allkeys, sizeof(int64_t) * p->allkeys.size(),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    memcpy(b.keys.data(), p->allkeys.data() + 2 * (size_t)W * rank, sizeof(int64_t) * 2 * W);
    std::vector<const int64_t *> rows(2 * nranks);
    for (int k = 0; k < nranks; k++) {
        rows[2 * k] = p->allkeys.data() + 2 * (size_t)W * k;
        rows[2 * k + 1] = rows[2 * k] + W;
    }
    Resolver res;
    res.build(nranks, W, rows.data());
    // B + C + X2
    st = band_phase_b(b, res, {}, {}, rank, s);
    if (st == CCL_OK) st = band_phase_c(b, s);
    if (st != CCL_OK) return st;
    CKN(ncclAllGather(b.d_small, p->d_alln, 1, ncclInt32, p->comm, s));
    CK(cudaMemcpyAsync(p->nband.data(), p->d_alln, sizeof(int32_t) * nranks, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int32_t off = 0, total = 0;
    for (int k = 0; k < nranks; k++) {
        if (k < rank) off += p->nband[k];
        total += p->nband[k];
    }
    // D + X3
    st = band_phase_d(b, off, s);
    if (st != CCL_OK) return st;
    CKN(ncclAllGather(b.d_exp, p->d_allexp, 2 * (size_t)W, ncclInt32, p->comm, s));
    CK(cudaMemcpyAsync(p->allexp.data(), p->d_allexp, sizeof(int32_t) * p->allexp.size(),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<const int64_t *> akeys(nranks);
    std::vector<const int32_t *> aexp(nranks);
    for (int k = 0; k < nranks; k++) {
        akeys[k] = p->allkeys.data() + 2 * (size_t)W * k;
        aexp[k] = p->allexp.data() + 2 * (size_t)W * k;
    }
    // E
    st = band_phase_e(b, akeys.data(), aexp.data(), nranks, band_labels, s);
    if (st != CCL_OK) return st;
    p->total = total;
    CK(cudaMemcpyAsync(n_components, &p->total, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    return CCL_OK;
}

ccl_status ccl_label_sharded(const uint8_t *band_img, int band_H, int W, int row0, int H_total,
                             int32_t *band_labels, int32_t *n_components, ccl_nccl_comm_t comm,
                             ccl_stream_t stream) {
    if (!band_img || !band_labels || !n_components) return CCL_INVALID_ARGUMENT;
    ccl_shard_plan p = nullptr;
    ccl_status st = ccl_shard_plan_create(band_H, W, row0, H_total, comm, stream, &p);
    if (st != CCL_OK) return st;
    st = ccl_shard_plan_label(p, band_img, band_labels, n_components, stream);
    ccl_shard_plan_destroy(p);
    return st;
}

}  // extern "C"
