// ccl_kernels.cu -- B200 (sm_100a) kernels of the two-pass 8-connectivity CCL
// pipeline.  DESIGN.md explains the design; paper citations are PAPER.md lines.
//
//   K1 k_tile_local   one CTA per 32x1024 tile.  Loads the image tile (128-bit
//                     streaming loads), packs it into 32-bit row masks, and
//                     labels it with the paper's two-pass scheme in shared
//                     memory: 8 warps each scan a 4-row strip row by row
//                     (Scan_ARemSP's "copy the label of an upper neighbour,
//                     else a new label, merge the rest"),
//                     working on whole runs with ballots/popc instead of
//                     pixels; strips are then merged at their boundary rows
//                     (PARemSP's boundary loop) with a
//                     lock-free Rem's union with splicing (merge / merger,
//                     PAPER.md:669-698, 1001-1046); a tile-level flatten
//                      numbers the tile's components in
//                     raster order of their first pixel.
//   K2 k_border       lock-free atomicCAS union of the components that touch
//                     across tile edges (PARemSP's boundary merge, with CAS in
//                     place of omp locks).
//   K3 k_roots        per tile: which components are global roots, and their
//                     rank inside their (row, tile-column) segment.
//   K4 k_scan         hand-written decoupled-lookback exclusive scan of the
//                     per-segment root counts = flatten's consecutive numbering
//                     k++  in raster order; writes N.
//   K5 k_write        labeling phase: every pixel gets its
//                     component's canonical label; 16-byte streaming stores.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "ccl_internal.cuh"

namespace cclb {

#define FULL 0xFFFFFFFFu

const char *const kKernelNames[K_COUNT] = {"k_tile_local", "k_border", "k_roots", "k_scan",
                                           "k_write"};

// ===================================================================== helpers
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// bits 0..b set
__device__ __forceinline__ uint32_t upto(int b) { return FULL >> (31 - b); }

// Segmented inclusive OR-smear of t towards higher bits within runs of x
// (t is a subset of x): bit i = OR of t[j], j <= i, x[j..i] all ones.
__device__ __forceinline__ uint32_t smear_up(uint32_t t, uint32_t x) {
    uint32_t m = x & (x << 1);
    uint32_t s = t;
    s |= (s << 1) & m;  m &= m << 1;
    s |= (s << 2) & m;  m &= m << 2;
    s |= (s << 4) & m;  m &= m << 4;
    s |= (s << 8) & m;  m &= m << 8;
    s |= (s << 16) & m;
    return s;
}
// Same towards lower bits.
__device__ __forceinline__ uint32_t smear_down(uint32_t t, uint32_t x) {
    uint32_t m = x & (x >> 1);
    uint32_t s = t;
    s |= (s >> 1) & m;  m &= m >> 1;
    s |= (s >> 2) & m;  m &= m >> 2;
    s |= (s >> 4) & m;  m &= m >> 4;
    s |= (s >> 8) & m;  m &= m >> 8;
    s |= (s >> 16) & m;
    return s;
}

// Carry-lookahead across the 32 lanes of a warp: with per-lane generate g and
// propagate p, C_j = g_j | (p_j & C_{j-1}); returns C_{lane-1} (0 for lane 0).
// One integer addition on the ballots does the whole chain.
__device__ __forceinline__ uint32_t carry_in_fwd(bool g, bool p) {
    uint32_t G = __ballot_sync(FULL, g), P = __ballot_sync(FULL, p) | G;
    uint32_t c = (P + G) ^ P ^ G;  // carry into bit j
    return (c >> lane_id()) & 1u;
}
// Reverse direction: C_j = g_j | (p_j & C_{j+1}); returns C_{lane+1}.
__device__ __forceinline__ uint32_t carry_in_bwd(bool g, bool p) {
    uint32_t G = __brev(__ballot_sync(FULL, g)), P = __brev(__ballot_sync(FULL, p)) | G;
    uint32_t c = (P + G) ^ P ^ G;
    return (c >> (31 - lane_id())) & 1u;
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t &total) {
    uint32_t x = v;
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(FULL, x, 31);
    return x - v;
}

// Row structure of one 1024-px tile row held as one word per lane.
struct RowView {
    uint32_t x, xp, xn;  // this lane's word, left / right neighbour words
    uint32_t hx;         // run heads
    uint32_t base;       // runs whose head lies in lanes < this lane
    uint32_t nr;         // runs in the row
};

__device__ __forceinline__ RowView make_row(uint32_t x) {
    RowView r;
    const int lane = lane_id();
    r.x = x;
    uint32_t xp = __shfl_up_sync(FULL, x, 1);
    uint32_t xn = __shfl_down_sync(FULL, x, 1);
    r.xp = lane == 0 ? 0u : xp;
    r.xn = lane == 31 ? 0u : xn;
    r.hx = x & ~((x << 1) | (r.xp >> 31));
    r.base = warp_excl_scan(__popc(r.hx), r.nr);
    return r;
}

__device__ __forceinline__ uint32_t dilate(const RowView &r) {
    return r.x | (r.x << 1) | (r.xp >> 31) | (r.x >> 1) | (r.xn << 31);
}

// First set bit of t inside each run of x, across lanes (t subset of x).
__device__ __forceinline__ uint32_t first_in_run(uint32_t t, uint32_t x) {
    uint32_t s = smear_up(t, x);
    uint32_t cin = carry_in_fwd(((x >> 31) & (s >> 31)) != 0, x == FULL) & x & 1u;
    uint32_t lead = x & ~(x + 1);  // run segment that contains bit 0
    uint32_t earlier = ((s << 1) & x & (x << 1)) | (cin ? lead : 0u);
    return t & ~earlier;
}

// Heads of runs of x that contain no bit of t, across lanes.
__device__ __forceinline__ uint32_t untouched_heads(uint32_t t, const RowView &r) {
    uint32_t x = r.x;
    uint32_t s = smear_down(t, x);
    uint32_t cin = carry_in_bwd((x & s & 1u) != 0, x == FULL) & (x >> 31);
    int k = __clz(~x);  // leading ones = run segment that contains bit 31
    uint32_t trail = k == 0 ? 0u : (k == 32 ? FULL : (FULL << (32 - k)));
    return r.hx & ~(s | (cin ? trail : 0u));
}

// ordinal of the run containing pixel b of lane-word (heads h, base bs)
__device__ __forceinline__ int run_ord(uint32_t h, uint32_t bs, int b) {
    return (int)bs + __popc(h & upto(b)) - 1;
}

// bit (p-1), p, (p+1) of a row (own word w, neighbours wp, wn), b = p & 31:
// returns the offset (-1, 0, +1) of the leftmost set one (caller knows one is set).
__device__ __forceinline__ int leftmost3(uint32_t w, uint32_t wp, uint32_t wn, int b) {
    uint32_t lo = b == 0 ? (wp >> 31) : (w >> (b - 1)) & 1u;
    if (lo) return -1;
    if ((w >> b) & 1u) return 0;
    return 1;
}

// ---------------------------------------------------------------- union-find
// Lock-free Rem's union with splicing on a shared-memory parent array in
// which parent < child for every non-root (labels are created in raster
// order).  This is the paper's merge run concurrently the
// way its merger does: the root link is an atomicCAS
// (the role of merger's lock + "still a root?" re-check)
// and the splice is a plain store, unlocked as in merger (PAPER.md:1025,
// 1039).  Every value stored into p[x] is smaller than x, so no cycle forms.
__device__ void merge_smem(uint16_t *p, uint32_t x, uint32_t y) {
    volatile uint16_t *vp = p;
    while (true) {
        uint32_t px = vp[x], py = vp[y];
        if (px == py) return;
        if (px < py) {
            uint32_t t = x; x = y; y = t;
            t = px; px = py; py = t;
        }
        // now p[x] > p[y]
        if (px == x) {
            if (atomicCAS(reinterpret_cast<unsigned short *>(p + x), (unsigned short)x,
                          (unsigned short)py) == (unsigned short)x)
                return;
            continue;  // x stopped being a root meanwhile: retry from x
        }
        vp[x] = (uint16_t)py;  // splice: x's subtree becomes a sibling under py
        x = px;
    }
}

// Global union-find over border components, ordered by raster key.
__device__ __forceinline__ int gfind(int32_t *par, int x) {
    while (true) {
        int px = __ldcg(par + x);
        if (px == x) return x;
        int ppx = __ldcg(par + px);
        if (ppx != px) __stcg(par + x, ppx);  // path halving (stores only ancestors)
        x = ppx;
    }
}
__device__ __forceinline__ int gfind_ro(const int32_t *par, int x) {
    while (true) {
        int px = __ldcg(par + x);
        if (px == x) return x;
        x = px;
    }
}
// Links the root with the larger key under the root with the smaller key.
__device__ void gunion(int32_t *par, const int32_t *key, int a, int b) {
    while (true) {
        a = gfind(par, a);
        b = gfind(par, b);
        if (a == b) return;
        if (__ldg(key + a) < __ldg(key + b)) { int t = a; a = b; b = t; }
        if (atomicCAS(par + a, a, b) == a) return;
    }
}

// 16 bytes of pixels -> 16 bits (bit k = byte k != 0)
__device__ __forceinline__ uint32_t pack16(uint4 v) {
    auto nz4 = [](uint32_t w) -> uint32_t {
        uint32_t m = (((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u;
        return ((m >> 7) * 0x01020408u) >> 24;
    };
    return nz4(v.x) | (nz4(v.y) << 4) | (nz4(v.z) << 8) | (nz4(v.w) << 12);
}

// Load the 32 pixels of lane-word (row, word) as a bitmask.
__device__ __forceinline__ uint32_t load_word(const uint8_t *__restrict__ img, const Geometry &g,
                                              int row, int col0) {
    if (col0 >= g.W) return 0u;
    const uint8_t *src = img + (int64_t)row * g.W + col0;
    if (g.aligned) {
        uint32_t m = pack16(__ldcs(reinterpret_cast<const uint4 *>(src)));
        if (col0 + 16 < g.W) m |= pack16(__ldcs(reinterpret_cast<const uint4 *>(src + 16))) << 16;
        return m;
    }
    uint32_t m = 0;
    int n = min(32, g.W - col0);
    for (int i = 0; i < n; i++) m |= (uint32_t)(__ldcs(src + i) != 0) << i;
    return m;
}

// ========================================================================= K1
struct K1Smem {
    uint16_t p[CAP];               // parent of each provisional label (tile-local index)
    uint16_t lpos[CAP];            // position (row*1024 + col) of the pixel that created it;
                                   // after the flatten, a root's entry holds its component
    union {
        uint16_t lab[NW][3][MAXRUN];  // run labels: 2 ping-pong rows + the strip's first row
        uint16_t cnode[CAPC];         // Phase III: border flag, then border index + 1
    } u;
    uint32_t hd[NW][3][WPR];       // run heads per lane, same buffers
    uint32_t bs[NW][3][WPR];       // run base per lane, same buffers
    uint32_t bm[TH][WPR];          // the tile's masks
    uint16_t toplab[MAXRUN];       // run labels of the tile's first row
    uint16_t botlab[MAXRUN];       // run labels of the tile's last row
    int16_t left[TH], right[TH];   // label of the first / last column pixel of each row, -1 bg
    int32_t used[NW];              // labels created by each strip
    int32_t last[NW];              // buffer holding each strip's last row
    int32_t nrow[NW][2];           // runs in each strip's first / last row
    int32_t wscan[NW];             // scan scratch
};

// Block-wide exclusive scan of one int per thread (NW warps); returns prefix,
// sets total.
__device__ __forceinline__ int block_excl_scan(int v, int *scratch, int &total) {
    uint32_t tot;
    int pre = (int)warp_excl_scan((uint32_t)v, tot);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if (lane_id() == 0) scratch[w] = (int)tot;
    __syncthreads();
    int off = 0, all = 0;
#pragma unroll
    for (int i = 0; i < NW; i++) {
        int s = scratch[i];
        off += i < w ? s : 0;
        all += s;
    }
    total = all;
    return pre + off;
}

// Upper-side edges that the copy step does not already cover.  With the
// spanning edge set {(L, leftmost upper of L)} U {(U, leftmost lower of U)},
// the second family is redundant unless U's head h touches the lower run L
// through pixel h-1 AND L reaches an upper pixel at h-2 or further left (then
// L's leftmost upper neighbour is another run).  S is the segmented smear of
// the touch pixels t along the lower runs (incl. carries from left lanes).
__device__ __forceinline__ uint32_t upper_merge_heads(uint32_t hu, uint32_t u, uint32_t up,
                                                      uint32_t x, uint32_t xp, uint32_t S) {
    const uint32_t Sp = __shfl_up_sync(FULL, S, 1);
    const uint32_t sp = lane_id() == 0 ? 0u : Sp;
    const uint32_t x1 = (x << 1) | (xp >> 31);              // lower pixel at h-1
    const uint32_t s2 = (S << 2) | (sp >> 30);              // smear at h-2
    const uint32_t u2 = (u << 2) | (up >> 30);              // upper pixel at h-2
    return hu & x1 & (s2 | u2);
}

__global__ void __launch_bounds__(NW * 32, 3)
k_tile_local(const uint8_t *__restrict__ img, Geometry g, Workspace ws) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    K1Smem &sm = *reinterpret_cast<K1Smem *>(smem_raw);

    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int tx = blockIdx.x % g.nTx, ty = blockIdx.x / g.nTx;
    const int tile = blockIdx.x;
    const int R0 = ty * TH, C0 = tx * TW;
    const int rows = min(TH, g.H - R0);
    const int vcols = min(TW, g.W - C0);
    const int gword = tx * WPR + lane;  // this lane's word index in the image row
    const int col0 = C0 + 32 * lane;

    // ---- load this strip's rows (all loads in flight together)
    const int r0 = w * S;
    const int nrows = max(0, min(S, rows - r0));
    uint32_t xs[S];
#pragma unroll
    for (int i = 0; i < S; i++) xs[i] = i < nrows ? load_word(img, g, R0 + r0 + i, col0) : 0u;

    // ---- Phase I: strip scan, one row at a time (Scan_ARemSP)
    uint32_t next = w * CAPS;  // strip-local label counter (count <- start)
    uint32_t u = 0, up = 0, un = 0, hu = 0, bu = 0;
    int prev = 2, cur = 2;
#pragma unroll
    for (int i = 0; i < S; i++) {
        if (i >= nrows) break;
        const int rl = r0 + i;
        cur = (i == 0) ? 2 : (prev == 0 ? 1 : 0);
        uint16_t *labc = sm.u.lab[w][cur];
        const uint16_t *labp = sm.u.lab[w][prev];
        const uint32_t x = xs[i];
        const uint32_t xpr = __shfl_up_sync(FULL, x, 1), xnr = __shfl_down_sync(FULL, x, 1);
        const uint32_t xp = lane == 0 ? 0u : xpr, xn = lane == 31 ? 0u : xnr;
        const uint32_t hx = x & ~((x << 1) | (xp >> 31));

        // touch pixels: this-row pixels with a foreground pixel among the three above
        const uint32_t t = x & (u | (u << 1) | (up >> 31) | (u >> 1) | (un << 31));
        // first touch pixel of each run, and the run smear S (for the merge test)
        const uint32_t s = smear_up(t, x);
        const uint32_t cin = carry_in_fwd(((x >> 31) & (s >> 31)) != 0, x == FULL) & x & 1u;
        const uint32_t lead = x & ~(x + 1);
        const uint32_t S = s | (cin ? lead : 0u);
        const uint32_t ft = t & ~(((s << 1) & x & (x << 1)) | (cin ? lead : 0u));
        // heads of runs with no touch pixel -> new labels
        uint32_t nh;
        {
            const uint32_t sd = smear_down(t, x);
            const uint32_t cr = carry_in_bwd((x & sd & 1u) != 0, x == FULL) & (x >> 31);
            const int k = __clz(~x);
            const uint32_t trail = k == 0 ? 0u : (k == 32 ? FULL : (FULL << (32 - k)));
            nh = hx & ~(sd | (cr ? trail : 0u));
        }
        // one scan for both run ordinals and new-label numbers
        uint32_t tot;
        const uint32_t pre = warp_excl_scan(__popc(hx) | (__popc(nh) << 16), tot);
        const uint32_t base = pre & 0xFFFFu, nbase = pre >> 16;
        const uint32_t nr = tot & 0xFFFFu, nnew = tot >> 16;
        sm.hd[w][cur][lane] = hx;
        sm.bs[w][cur][lane] = base;
        sm.bm[rl][lane] = x;
        if (gword < g.WW) ws.bm[(int64_t)(R0 + rl) * g.WW + gword] = x;

        // new labels, numbered in column order = raster order
        {
            uint32_t m = nh, k = next + nbase;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                labc[run_ord(hx, base, b)] = (uint16_t)k;
                sm.p[k] = (uint16_t)k;
                sm.lpos[k] = (uint16_t)(rl * TW + 32 * lane + b);
                k++;
            }
        }
        next += nnew;
        // copy: a touched run takes the label of its leftmost upper neighbour
        // (the decision tree's copy(b)/copy(a)/copy(c))
        {
            uint32_t m = ft;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int q = 32 * lane + b + leftmost3(u, up, un, b);
                const int lq = q >> 5;
                const int ou = run_ord(sm.hd[w][prev][lq], sm.bs[w][prev][lq], q & 31);
                labc[run_ord(hx, base, b)] = labp[ou];
            }
        }
        __syncwarp();
        // merge: the few upper runs whose lower neighbour copied another
        // label (the decision tree's copy(c,a)/copy(c,d) merges)
        if (i > 0) {
            uint32_t m = upper_merge_heads(hu, u, up, x, xp, S);
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int q = 32 * lane + b - 1;  // lower pixel h-1 of the run below
                const int lq = q >> 5;
                const uint32_t lx = labc[run_ord(sm.hd[w][cur][lq], sm.bs[w][cur][lq], q & 31)];
                const uint32_t lu = labp[run_ord(hu, bu, b)];
                if (lx != lu) merge_smem(sm.p, lu, lx);
            }
        }
        // per-row outputs: run labels (for K5) and the border-column labels
        {
            uint32_t *dst = reinterpret_cast<uint32_t *>(ws.runlab + ((int64_t)(R0 + rl) * g.nTx + tx) * MAXRUN);
            const uint32_t *src = reinterpret_cast<const uint32_t *>(labc);
            for (int k = lane; 2 * k < (int)nr; k += 32) dst[k] = src[k];
            if (lane == 0) sm.left[rl] = (x & 1u) ? (int16_t)labc[0] : (int16_t)-1;
            const int lc = vcols - 1;
            if (lane == (lc >> 5)) sm.right[rl] = ((x >> (lc & 31)) & 1u) ? (int16_t)labc[nr - 1] : (int16_t)-1;
            if (lane == 0) {
                if (i == 0) sm.nrow[w][0] = (int)nr;
                sm.nrow[w][1] = (int)nr;
            }
        }
        __syncwarp();
        u = x;
        up = xp;
        un = xn;
        hu = hx;
        bu = base;
        prev = cur;
    }
    if (lane == 0) {
        sm.used[w] = (int)(next - w * CAPS);
        sm.last[w] = prev;
    }
    __syncthreads();

    // ---- Phase II: merge across strip boundaries (PARemSP boundary loop,
    // PAPER.md:971-988, lock-free merger)
    if (w > 0 && r0 < rows) {
        const int pw = w - 1, pb = sm.last[pw];
        const uint32_t uu = sm.bm[r0 - 1][lane], x = sm.bm[r0][lane];
        const uint16_t *labu = sm.u.lab[pw][pb];
        const uint16_t *labx = sm.u.lab[w][2];
        const uint32_t *hdu = sm.hd[pw][pb], *bsu = sm.bs[pw][pb];
        const uint32_t *hdx = sm.hd[w][2], *bsx = sm.bs[w][2];
        RowView X = make_row(x);
        RowView U = make_row(uu);
        const uint32_t t = x & dilate(U);
        const uint32_t s = smear_up(t, x);
        const uint32_t cin = carry_in_fwd(((x >> 31) & (s >> 31)) != 0, x == FULL) & x & 1u;
        const uint32_t lead = x & ~(x + 1);
        const uint32_t S = s | (cin ? lead : 0u);
        uint32_t m = t & ~(((s << 1) & x & (x << 1)) | (cin ? lead : 0u));
        while (m) {  // each lower run with its leftmost upper neighbour
            const int b = __ffs(m) - 1;
            m &= m - 1;
            const int q = 32 * lane + b + leftmost3(uu, U.xp, U.xn, b);
            const int lq = q >> 5;
            const uint32_t lu = labu[run_ord(hdu[lq], bsu[lq], q & 31)];
            const uint32_t lx = labx[run_ord(X.hx, X.base, b)];
            if (lx != lu) merge_smem(sm.p, lu, lx);
        }
        m = upper_merge_heads(U.hx, uu, U.xp, x, X.xp, S);
        while (m) {  // upper runs whose leftmost lower neighbour has another leftmost upper
            const int b = __ffs(m) - 1;
            m &= m - 1;
            const int q = 32 * lane + b - 1;
            const int lq = q >> 5;
            const uint32_t lx = labx[run_ord(hdx[lq], bsx[lq], q & 31)];
            const uint32_t lu = labu[run_ord(U.hx, U.base, b)];
            if (lx != lu) merge_smem(sm.p, lu, lx);
        }
    }
    // keep the tile's first and last row labels (the lab buffers are reused below)
    const int wl = (rows - 1) / S;  // strip holding the tile's last row
    if (w == 0) {
        const uint16_t *src = sm.u.lab[0][2];
        for (int k = lane; k < sm.nrow[0][0]; k += 32) sm.toplab[k] = src[k];
    }
    if (w == wl) {
        const uint16_t *src = sm.u.lab[wl][sm.last[wl]];
        for (int k = lane; k < sm.nrow[wl][1]; k += 32) sm.botlab[k] = src[k];
    }
    __syncthreads();

    // ---- Phase III: tile flatten: roots in label order
    // (= raster order of the creating pixel) get consecutive component
    // indices.  Warp w walks its own strip's labels in order.
    const int used_w = sm.used[w];
    const int lbase = w * CAPS;
    volatile uint16_t *vp = sm.p;
    // (a) full path compression
    for (int i = lane; i < used_w; i += 32) {
        const int l = lbase + i;
        uint32_t r = vp[l];
        while (vp[r] != r) r = vp[r];
        vp[l] = (uint16_t)r;
    }
    __syncthreads();
    // (b) count roots per strip, then number them in label order
    int nroot = 0;
    for (int i0 = 0; i0 < used_w; i0 += 32) {
        const int i = i0 + lane;
        nroot += __popc(__ballot_sync(FULL, i < used_w && sm.p[lbase + i] == (uint16_t)(lbase + i)));
    }
    if (lane == 0) sm.wscan[w] = nroot;
    __syncthreads();
    int coff = 0, ncomp = 0;
#pragma unroll
    for (int k = 0; k < NW; k++) {
        const int v = sm.wscan[k];
        coff += k < w ? v : 0;
        ncomp += v;
    }
    int32_t *compkey = ws.compkey + (int64_t)tile * CAPC;
    for (int i0 = 0; i0 < used_w; i0 += 32) {
        const int i = i0 + lane;
        const int l = lbase + i;
        const bool root = i < used_w && sm.p[l] == (uint16_t)l;
        const uint32_t bal = __ballot_sync(FULL, root);
        if (root) {
            const int c = coff + __popc(bal & ((1u << lane) - 1));
            const int pos = sm.lpos[l];
            compkey[c] = (R0 + (pos >> 10)) * g.W + C0 + (pos & (TW - 1));
            sm.lpos[l] = (uint16_t)c;  // a root's lpos now holds its component
        }
        coff += __popc(bal);
    }
    __syncthreads();
    // (c) provisional label -> component (for K5); clear the border flags
    uint16_t *lmap = ws.lmap + (int64_t)tile * CAP;
    for (int i = lane; i < used_w; i += 32) {
        const int l = lbase + i;
        lmap[l] = sm.lpos[sm.p[l]];
    }
    for (int c = threadIdx.x; c < ncomp; c += NW * 32) sm.u.cnode[c] = 0;
    __syncthreads();
    // (d) mark components that touch the tile border
    auto comp_of = [&](int l) -> int { return sm.lpos[sm.p[l]]; };
    const int ntop = sm.nrow[0][0], nbot = sm.nrow[wl][1];
    for (int k = threadIdx.x; k < ntop; k += NW * 32) sm.u.cnode[comp_of(sm.toplab[k])] = 1;
    for (int k = threadIdx.x; k < nbot; k += NW * 32) sm.u.cnode[comp_of(sm.botlab[k])] = 1;
    for (int r = threadIdx.x; r < rows; r += NW * 32) {
        if (sm.left[r] >= 0) sm.u.cnode[comp_of(sm.left[r])] = 1;
        if (sm.right[r] >= 0) sm.u.cnode[comp_of(sm.right[r])] = 1;
    }
    __syncthreads();
    // (e) border components -> global union-find nodes
    const int cper = (ncomp + NW * 32 - 1) / (NW * 32);
    const int c0 = threadIdx.x * cper, c1 = min(ncomp, c0 + cper);
    int bc = 0;
    for (int c = c0; c < c1; c++) bc += sm.u.cnode[c] != 0;
    int nborder;
    int bidx = block_excl_scan(bc, sm.wscan, nborder);
    int32_t *compnode = ws.compnode + (int64_t)tile * CAPC;
    const int nodebase = tile * CAPB;
    for (int c = c0; c < c1; c++) {
        if (sm.u.cnode[c]) {
            const int node = nodebase + bidx;
            compnode[c] = node;
            ws.gparent[node] = node;
            ws.gkey[node] = compkey[c];
            sm.u.cnode[c] = (uint16_t)(bidx + 1);
            bidx++;
        } else {
            compnode[c] = -1;
        }
    }
    __syncthreads();
    // (f) nodes of the border pixels, for K2
    auto node_of = [&](int l) -> int { return nodebase + (int)sm.u.cnode[comp_of(l)] - 1; };
    for (int k = threadIdx.x; k < ntop; k += NW * 32) ws.topnode[tile * MAXRUN + k] = node_of(sm.toplab[k]);
    for (int k = threadIdx.x; k < nbot; k += NW * 32) ws.botnode[tile * MAXRUN + k] = node_of(sm.botlab[k]);
    for (int r = threadIdx.x; r < rows; r += NW * 32) {
        const int64_t o = (int64_t)tx * g.H + R0 + r;
        ws.leftnode[o] = sm.left[r] >= 0 ? node_of(sm.left[r]) : -1;
        ws.rightnode[o] = sm.right[r] >= 0 ? node_of(sm.right[r]) : -1;
    }
    if (threadIdx.x == 0) {
        int32_t *meta = ws.meta + (int64_t)tile * META;
        meta[META_NCOMP] = ncomp;
        meta[META_NBORDER] = nborder;
        meta[META_ROWS] = rows;
    }
    if (lane == 0) ws.meta[(int64_t)tile * META + META_USED + w] = used_w;
}

// ========================================================================= K2
// Horizontal tile edges: one warp per (tile row boundary, tile column); the
// runs of the last row above and the first row below are united along the
// same two edge families as the strip merge.  Vertical tile edges (incl.
// corner pixels): one thread per (tile column boundary, row).
__global__ void __launch_bounds__(256)
k_border(Geometry g, Workspace ws, int nh_warps) {
    __shared__ uint32_t shd[8][2][WPR], sbs[8][2][WPR];
    const int lane = lane_id(), wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * 8 + wib;
    if (gw < nh_warps) {
        const int tx = gw % g.nTx, ty = 1 + gw / g.nTx;
        const int ru = ty * TH - 1, rx = ty * TH;
        const int gword = tx * WPR + lane;
        const uint32_t u = gword < g.WW ? ws.bm[(int64_t)ru * g.WW + gword] : 0u;
        const uint32_t x = gword < g.WW ? ws.bm[(int64_t)rx * g.WW + gword] : 0u;
        RowView U = make_row(u), X = make_row(x);
        shd[wib][0][lane] = U.hx; sbs[wib][0][lane] = U.base;
        shd[wib][1][lane] = X.hx; sbs[wib][1][lane] = X.base;
        __syncwarp();
        const int32_t *bot = ws.botnode + (int64_t)((ty - 1) * g.nTx + tx) * MAXRUN;
        const int32_t *top = ws.topnode + (int64_t)(ty * g.nTx + tx) * MAXRUN;
        uint32_t m = first_in_run(x & dilate(U), x);
        while (m) {
            int b = __ffs(m) - 1;
            m &= m - 1;
            int q = 32 * lane + b + leftmost3(u, U.xp, U.xn, b);
            int lq = q >> 5;
            int nu = bot[run_ord(shd[wib][0][lq], sbs[wib][0][lq], q & 31)];
            int nx = top[run_ord(X.hx, X.base, b)];
            gunion(ws.gparent, ws.gkey, nu, nx);
        }
        m = first_in_run(u & dilate(X), u);
        while (m) {
            int b = __ffs(m) - 1;
            m &= m - 1;
            int q = 32 * lane + b + leftmost3(x, X.xp, X.xn, b);
            int lq = q >> 5;
            int nx = top[run_ord(shd[wib][1][lq], sbs[wib][1][lq], q & 31)];
            int nu = bot[run_ord(U.hx, U.base, b)];
            gunion(ws.gparent, ws.gkey, nu, nx);
        }
        return;
    }
    // vertical edges
    const int64_t t = (int64_t)(gw - nh_warps) * 32 + lane;
    const int64_t nv = (int64_t)(g.nTx - 1) * g.H;
    if (t >= nv) return;
    const int tx = 1 + (int)(t / g.H), r = (int)(t % g.H);
    const int a = ws.rightnode[(int64_t)(tx - 1) * g.H + r];
    if (a < 0) return;
    const int32_t *L = ws.leftnode + (int64_t)tx * g.H;
    const int b = L[r];
    if (b >= 0) {
        gunion(ws.gparent, ws.gkey, a, b);  // (r-1) and (r+1) are then joined through b
        return;
    }
    if (r > 0 && L[r - 1] >= 0) gunion(ws.gparent, ws.gkey, a, L[r - 1]);
    if (r + 1 < g.H && L[r + 1] >= 0) gunion(ws.gparent, ws.gkey, a, L[r + 1]);
}

// ========================================================================= K3
// Per tile: component c is a global root iff it lies inside the tile or its
// node is a root of the global forest (its key is the component's minimum,
// i.e. its first pixel in raster order).  Counts roots per row and gives
// each root its rank inside its (row, tile-column) segment.
__global__ void __launch_bounds__(256)
k_roots(Geometry g, Workspace ws) {
    __shared__ int cntrow[TH], rowbase[TH], wscan[8];
    const int tile = blockIdx.x;
    const int tx = tile % g.nTx, ty = tile / g.nTx, R0 = ty * TH;
    if (tile == 0) {  // reset the scan's lookback state for K4
        for (int i = threadIdx.x; i < g.nscan; i += blockDim.x) ws.scanstate[i] = 0ull;
        if (threadIdx.x == 0) *ws.ticket = 0;
    }
    const int32_t *meta = ws.meta + (int64_t)tile * META;
    const int ncomp = meta[META_NCOMP], rows = meta[META_ROWS];
    if (threadIdx.x < TH) cntrow[threadIdx.x] = 0;
    const int32_t *compnode = ws.compnode + (int64_t)tile * CAPC;
    const int32_t *compkey = ws.compkey + (int64_t)tile * CAPC;
    uint32_t *comprank = ws.comprank + (int64_t)tile * CAPC;
    const int per = (ncomp + 255) / 256;
    const int c0 = threadIdx.x * per, c1 = min(ncomp, c0 + per);
    int cnt = 0;
    for (int c = c0; c < c1; c++) {
        int node = compnode[c];
        cnt += node < 0 || __ldcg(ws.gparent + node) == node;
    }
    __syncthreads();
    // block scan over 8 warps
    uint32_t tot;
    int pre = (int)warp_excl_scan((uint32_t)cnt, tot);
    if (lane_id() == 0) wscan[threadIdx.x >> 5] = (int)tot;
    __syncthreads();
    int off = 0;
    for (int i = 0; i < (int)(threadIdx.x >> 5); i++) off += wscan[i];
    int rank = pre + off;
    // per-row counts
    for (int c = c0; c < c1; c++) {
        int node = compnode[c];
        bool root = node < 0 || __ldcg(ws.gparent + node) == node;
        if (root) atomicAdd(&cntrow[compkey[c] / g.W - R0], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int r = 0; r < TH; r++) { rowbase[r] = s; s += cntrow[r]; }
    }
    __syncthreads();
    for (int c = c0; c < c1; c++) {
        int node = compnode[c];
        bool root = node < 0 || __ldcg(ws.gparent + node) == node;
        if (root) {
            int rl = compkey[c] / g.W - R0;
            int rk = rank - rowbase[rl];
            comprank[c] = ((uint32_t)rl << 16) | (uint32_t)rk;
            if (node >= 0) {
                ws.gnodeseg[node] = (R0 + rl) * g.nTx + tx;
                ws.gnoderank[node] = rk;
            }
            rank++;
        } else {
            comprank[c] = 0xFFFFFFFFu;
        }
    }
    if (threadIdx.x < rows) ws.segcnt[(int64_t)(R0 + threadIdx.x) * g.nTx + tx] = cntrow[threadIdx.x];
}

// ========================================================================= K4
// Single-pass decoupled-lookback exclusive scan of segcnt -> segoff, in the
// raster order of the segments; partitions are claimed through a ticket so
// a partition only ever waits on partitions that are already running.
// Descriptor: bits 62-63 status (1 aggregate, 2 inclusive prefix), low 32 bits value.
__global__ void __launch_bounds__(SCAN_THREADS)
k_scan(Geometry g, Workspace ws, int32_t *n_components) {
    __shared__ int s_part, s_excl;
    __shared__ int wsum[SCAN_THREADS / 32];
    if (threadIdx.x == 0) s_part = atomicAdd(ws.ticket, 1);
    __syncthreads();
    const int part = s_part;
    const int64_t base = (int64_t)part * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int v[SCAN_ITEMS];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
        int64_t k = base + i;
        v[i] = k < g.nseg ? ws.segcnt[k] : 0;
        sum += v[i];
    }
    uint32_t wt;
    int pre = (int)warp_excl_scan((uint32_t)sum, wt);
    const int wid = threadIdx.x >> 5;
    if (lane_id() == 0) wsum[wid] = (int)wt;
    __syncthreads();
    int off = 0, agg = 0;
    for (int i = 0; i < SCAN_THREADS / 32; i++) {
        off += i < wid ? wsum[i] : 0;
        agg += wsum[i];
    }
    if (threadIdx.x == 0) {
        volatile unsigned long long *st = ws.scanstate;
        if (part == 0) {
            atomicExch(ws.scanstate, (2ull << 62) | (uint32_t)agg);
            s_excl = 0;
        } else {
            atomicExch(ws.scanstate + part, (1ull << 62) | (uint32_t)agg);
            int excl = 0;
            int j = part - 1;
            while (true) {
                unsigned long long d = st[j];
                unsigned s = (unsigned)(d >> 62);
                if (s == 0) continue;  // predecessor not published yet: spin
                excl += (int)(uint32_t)d;
                if (s == 2) break;
                j--;
            }
            __threadfence();
            atomicExch(ws.scanstate + part, (2ull << 62) | (uint32_t)(excl + agg));
            s_excl = excl;
        }
        if (part == g.nscan - 1) *n_components = s_excl + agg;
    }
    __syncthreads();
    int run = s_excl + off + pre;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
        int64_t k = base + i;
        if (k < g.nseg) ws.segoff[k] = run;
        run += v[i];
    }
}

// ========================================================================= K5
struct K5Smem {
    int32_t flab[CAP];           // provisional label -> final label
    int32_t rowbuf[NW][TW];      // per-warp row staging (run labels, then the swizzled output row)
};

// Final label of a tile component (flatten's consecutive numbering,
// PAPER.md:714-715, in raster order): roots from their segment offset and
// rank; border components that are not roots from their global root's.
__device__ __forceinline__ int32_t comp_label(const Geometry &g, const Workspace &ws, int tile,
                                              int R0, int tx, int c) {
    const uint32_t cr = ws.comprank[(int64_t)tile * CAPC + c];
    if (cr != 0xFFFFFFFFu)
        return ws.segoff[(int64_t)(R0 + (int)(cr >> 16)) * g.nTx + tx] + (int)(cr & 0xFFFF) + 1;
    const int root = gfind_ro(ws.gparent, ws.compnode[(int64_t)tile * CAPC + c]);
    return ws.segoff[ws.gnodeseg[root]] + ws.gnoderank[root] + 1;
}

__global__ void __launch_bounds__(NW * 32, 3)
k_write(Geometry g, Workspace ws, int32_t *__restrict__ labels) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    K5Smem &sm = *reinterpret_cast<K5Smem *>(smem_raw);
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int tile = blockIdx.x;
    const int tx = tile % g.nTx, ty = tile / g.nTx;
    const int R0 = ty * TH, C0 = tx * TW;
    const int32_t *meta = ws.meta + (int64_t)tile * META;
    const int rows = meta[META_ROWS];
    const int vcols = min(TW, g.W - C0);
    const int gword = tx * WPR + lane;

    // this warp's rows are w, w+NW, ...; the next row's mask is always in flight
    auto load_mask = [&](int rl) -> uint32_t {
        return (rl < rows && gword < g.WW) ? __ldcs(ws.bm + (int64_t)(R0 + rl) * g.WW + gword) : 0u;
    };
    uint32_t xnext = load_mask(w);
    // provisional label -> final label (warp w: strip w's labels)
    {
        const int used = meta[META_USED + w];
        const uint16_t *lmap = ws.lmap + (int64_t)tile * CAP + w * CAPS;
        for (int i = lane; i < used; i += 32)
            sm.flab[w * CAPS + i] = comp_label(g, ws, tile, R0, tx, lmap[i]);
    }
    __syncthreads();

    int32_t *buf = sm.rowbuf[w];
    int32_t *rowlab = buf + MAXRUN;  // upper half: run labels of the current row
#pragma unroll 1
    for (int i = 0; i < TH / NW; i++) {
        const int rl = w + i * NW;
        if (rl >= rows) break;
        const int row = R0 + rl;
        const uint32_t x = xnext;
        xnext = load_mask(rl + NW);
        const uint32_t xl = __shfl_up_sync(FULL, x, 1);
        const uint32_t hx = x & ~((x << 1) | (lane == 0 ? 0u : (xl >> 31)));
        uint32_t nr;
        const uint32_t base = warp_excl_scan(__popc(hx), nr);
        const uint16_t *rlab = ws.runlab + ((int64_t)row * g.nTx + tx) * MAXRUN;
        for (int k = lane; k < (int)nr; k += 32) rowlab[k] = sm.flab[__ldcs(rlab + k)];
        __syncwarp();
        // walk this lane's 32 pixels: the label changes only at run heads
        int v[32];
        {
            int ord = (int)base;
            int cur = ((x & 1u) && !(hx & 1u)) ? rowlab[ord - 1] : 0;
#pragma unroll
            for (int b = 0; b < 32; b++) {
                if ((hx >> b) & 1u) cur = rowlab[ord++];
                v[b] = ((x >> b) & 1u) ? cur : 0;
            }
        }
        __syncwarp();
        // stage the row: lane's 32 labels = 8 16-byte chunks, XOR-swizzled so
        // both the row-wise writes and the coalesced reads are conflict-free
#pragma unroll
        for (int j = 0; j < 8; j++)
            *reinterpret_cast<int4 *>(buf + lane * 32 + ((j ^ (lane & 7)) << 2)) =
                make_int4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        __syncwarp();
        int32_t *out = labels + (int64_t)row * g.W + C0;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const int P = 128 * c + 4 * lane;          // first pixel of this lane's chunk
            const int jw = P >> 5, jj = (P >> 2) & 7;  // source lane-word and chunk
            const int4 o = *reinterpret_cast<const int4 *>(buf + jw * 32 + ((jj ^ (jw & 7)) << 2));
            if (g.aligned) {
                if (P < vcols) __stcs(reinterpret_cast<int4 *>(out + P), o);
            } else {
                if (P < vcols) __stcs(out + P, o.x);
                if (P + 1 < vcols) __stcs(out + P + 1, o.y);
                if (P + 2 < vcols) __stcs(out + P + 2, o.z);
                if (P + 3 < vcols) __stcs(out + P + 3, o.w);
            }
        }
        __syncwarp();
    }
}

// ==================================================================== host
static bool g_attr_done = false;

cudaError_t run_pipeline(const Geometry &g, const Workspace &ws, const uint8_t *img,
                         int32_t *labels, int32_t *n_components, cudaStream_t stream,
                         cudaEvent_t *ev) {
    cudaError_t e;
    const int k1smem = (int)sizeof(K1Smem), k5smem = (int)sizeof(K5Smem);
    if (!g_attr_done) {
        e = cudaFuncSetAttribute(k_tile_local, cudaFuncAttributeMaxDynamicSharedMemorySize, k1smem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(k_write, cudaFuncAttributeMaxDynamicSharedMemorySize, k5smem);
        if (e != cudaSuccess) return e;
        g_attr_done = true;
    }
    auto mark = [&](int i) {
        if (ev) cudaEventRecord(ev[i], stream);
    };
    mark(K_TILE);
    k_tile_local<<<g.nT, NW * 32, k1smem, stream>>>(img, g, ws);
    mark(K_BORDER);
    const int nh = (g.nTy - 1) * g.nTx;
    const int64_t nv = (int64_t)(g.nTx - 1) * g.H;
    const int64_t warps = nh + (nv + 31) / 32;
    if (warps > 0) k_border<<<(unsigned)((warps + 7) / 8), 256, 0, stream>>>(g, ws, nh);
    mark(K_ROOTS);
    k_roots<<<g.nT, 256, 0, stream>>>(g, ws);
    mark(K_SCAN);
    k_scan<<<g.nscan, SCAN_THREADS, 0, stream>>>(g, ws, n_components);
    mark(K_WRITE);
    k_write<<<g.nT, NW * 32, k5smem, stream>>>(g, ws, labels);
    mark(K_COUNT);
    return cudaGetLastError();
}

}  // namespace cclb
