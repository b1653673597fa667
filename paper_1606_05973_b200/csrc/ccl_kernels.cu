// ccl_kernels.cu -- B200 (sm_100a) kernels of the two-pass 8-connectivity CCL
// pipeline.  DESIGN.md explains the design; paper citations are PAPER.md lines.
//
//   K1 k_tile_local   one CTA per 32x1024 image tile: reads the pixels once
//                     (32-byte streaming loads; fg = byte != 0),
//                     packs them to row masks and fills bridged single-pixel
//                     holes; the runs of the tile are its provisional labels
//                     (index order = raster order).  Scan: every run copies its
//                     leftmost upper neighbour's label (Scan_ARemSP's copy,
//                     PAPER.md:871-892), 8 strips at once; a short find resolves
//                     the copies; the few remaining edges are
//                     merged with a lock-free Rem's union with splicing (merge /
//                     merger); roots numbered in
//                     raster order.
//   K2 k_border       lock-free atomicCAS union of the components that touch
//                     across tile edges (PARemSP's boundary merge, PAPER.md:971-988,
//                     with CAS in place of omp locks).
//   K3 k_number       one CTA per tile row: which components are global roots,
//                     root counts per (row, tile-column) segment, a hand-written
//                     decoupled-lookback scan over the tile rows = flatten's
//                     consecutive numbering k++  in raster
//                     order; labels of all roots; writes N.
//   K4 k_fixup        labels of the border components that are not global roots
//                     (their root's label).
//   K5 k_write        labeling phase: every pixel gets its
//                     component's label; coalesced 32-byte stores (evict_first).
#include <cuda_runtime.h>
#include <algorithm>
#include <stdint.h>
#include <stdio.h>

#include "ccl_internal.cuh"

namespace cclb {

#define FULL 0xFFFFFFFFu

const char *const kKernelNames[K_COUNT] = {"k_tile_local", "k_border", "k_number", "k_fixup", "k_write"};

// ===================================================================== helpers
// Programmatic dependent launch: a kernel waits for its predecessor's grid to
// complete (memory visible) before touching what it wrote, and lets its
// successor be scheduled once each of its CTAs has issued its last store, so
// the launch gaps between the pipeline's kernels overlap the tails.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Component labels (K3b/K4) are stored with the evict_last L2 priority: K5
// gathers them while 1.87 GB of evict_first label stores stream past (-4 us);
// the policy is made once per thread.
__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_keep(int32_t *p, int32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.s32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

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
// Lock-free union on a shared-memory parent array in which parent < child for
// every non-root (labels are created in raster order).  This replaces the
// paper's Rem's merge with splicing as its parallel merger
// runs it (lock the root, re-check it is still a root,
// link; the splice is unlocked).  On the GPU the splice is what breaks: it
// moves a subtree from one tree into another before the two trees are joined,
// so for a moment a set is split, and a concurrent merge that reads through
// the split can stop early (round 1 lost about 1 union in 150 C3 runs that
// way).  Here p changes only by
//   (link)     atomicCAS(p[r], r, s): a root r goes under s < r; the CAS
//              succeeds only while r is still a root (merger's re-check);
//   (halving)  p[x] <- p[p[x]] for a non-root x: an ancestor of x.
// Neither moves a node out of its tree, so trees (the sets) only ever merge,
// and p[x] <= x always holds (no cycles).  union(a, b) returns only when
// find(a) == find(b) was observed (trees only grow: they are joined from then
// on) or after its own successful link; a failed CAS means another link
// succeeded (lock-free).  The root of a set is its minimum index = its first
// run in raster order, as with Rem's min-linking (DESIGN.md "Tile-local
// union").
__device__ __forceinline__ uint32_t find_smem(volatile uint16_t *vp, uint32_t x) {
    while (true) {
        const uint32_t px = vp[x];
        if (px == x) return x;
        const uint32_t ppx = vp[px];
        if (ppx == px) return px;
        vp[x] = (uint16_t)ppx;  // path halving: x is not a root, ppx is its ancestor
        x = ppx;
    }
}
__device__ __forceinline__ void union_smem(uint16_t *p, uint32_t a, uint32_t b) {
    volatile uint16_t *vp = p;
    a = find_smem(vp, a);
    b = find_smem(vp, b);
    while (a != b) {
        if (a < b) { const uint32_t t = a; a = b; b = t; }
        // a > b: link the root a under b while a is still a root
        const uint32_t o = atomicCAS(reinterpret_cast<unsigned short *>(p + a), (unsigned short)a,
                                     (unsigned short)b);
        if (o == a) return;
        a = find_smem(vp, o);  // a was linked meanwhile: continue from its new root
        b = find_smem(vp, b);
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
// Read-only find; returns the root node, or a negative parent (-2-f) when the
// tree hangs under a root owned by another row band.
__device__ __forceinline__ int gfind_ro(const int32_t *par, int x) {
    while (true) {
        int px = __ldcg(par + x);
        if (px == x || px < 0) return px;
        x = px;
    }
}
// Find with path halving on a forest that may hang under foreign roots (row
// bands: a parent -2-f is a root owned by another band, terminal).  Used
// after the unions (K4): only non-roots are rewritten, each to an ancestor
// (possibly the foreign reference), so roots and the partition are unchanged;
// concurrent finds shorten each other's chains (C5b comb: chains of 512 tile
// rows).
__device__ __forceinline__ int gfind_halve(int32_t *par, int x) {
    while (true) {
        const int px = __ldcg(par + x);
        if (px == x || px < 0) return px;
        const int ppx = __ldcg(par + px);
        if (ppx == px) return px;
        __stcg(par + x, ppx);
        if (ppx < 0) return ppx;
        x = ppx;
    }
}
// Links the root with the larger key under the root with the smaller key.
// Links the root with the larger key under the root with the smaller key
// (merger's lock + "still a root?" re-check, as a CAS).
// (Rem's interleaved climb without the splice, linking a root under the
// other side's parent, was measured too: C4 K2 37 -> 91 us, C5b 0.7 -> 5.3
// ms -- two key loads per step and no compression on the long chains.)
__device__ void gunion(int32_t *par, const int64_t *key, int a, int b) {
    while (true) {
        a = gfind(par, a);
        // a's key is in flight during the second find (C5a serpentine K2
        // 109 -> 73 us; C4 unchanged)
        const int64_t ka = __ldg(key + a);
        b = gfind(par, b);
        if (a == b) return;
        if (ka < __ldg(key + b)) { int t = a; a = b; b = t; }
        if (atomicCAS(par + a, a, b) == a) return;
    }
}

// 8 bytes of pixels (words a, b) -> 8 bits, bit k = (byte k != 0).  Bit 7 of
// every byte of f is its "nonzero" flag; the flags of a go to bit 0 and those
// of b to bit 4 of each byte, and one multiply gathers bit 8j -> 24+j and
// 8j+4 -> 28+j (the partial products never overlap, so nothing carries).
__device__ __forceinline__ uint32_t pack8(uint32_t a, uint32_t b) {
    const uint32_t fa = ((a & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | a;
    const uint32_t fb = ((b & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | b;
    const uint32_t v = ((fa >> 7) & 0x01010101u) | ((fb >> 3) & 0x10101010u);
    return (v * 0x01020408u) >> 24;
}
// 16 bytes of pixels -> 16 bits (bit k = byte k != 0)
__device__ __forceinline__ uint32_t pack16(uint4 v) {
    return pack8(v.x, v.y) | (pack8(v.z, v.w) << 8);
}
// The same for bytes known to be 0 or 1 (binary images stored as 0/1): the
// bytes' low bits go straight into the gather multiply (bit 8j of a -> 24+j,
// bit 8j+4 of b<<4 -> 28+j).
__device__ __forceinline__ uint32_t pack8_01(uint32_t a, uint32_t b) {
    return ((a | (b << 4)) * 0x01020408u) >> 24;
}
__device__ __forceinline__ uint32_t pack16_01(uint4 v) {
    return pack8_01(v.x, v.y) | (pack8_01(v.z, v.w) << 8);
}

// Threshold on load (the paper's im2bw step,
// PAPER.md:1084-1089): foreground <=> byte > thr.  Bit 7 of every byte of the
// result is that flag: the carry out of the low 7 bits of a + ~t decides it
// (a majority of a7, ~t7 and that carry), no byte borrows from its neighbour.
__device__ __forceinline__ uint32_t gt_flags(uint32_t a, uint32_t t4) {
    const uint32_t s = (a & 0x7F7F7F7Fu) + (~t4 & 0x7F7F7F7Fu);
    return (a & ~t4) | ((a | ~t4) & s);
}
__device__ __forceinline__ uint32_t pack8_gt(uint32_t a, uint32_t b, uint32_t t4) {
    const uint32_t v = ((gt_flags(a, t4) >> 7) & 0x01010101u) | ((gt_flags(b, t4) >> 3) & 0x10101010u);
    return (v * 0x01020408u) >> 24;
}
__device__ __forceinline__ uint32_t pack16_gt(uint4 v, uint32_t t4) {
    return pack8_gt(v.x, v.y, t4) | (pack8_gt(v.z, v.w, t4) << 8);
}
// 16 bytes -> 16 foreground bits (THR: byte > thr, else byte != 0)
template <bool THR>
__device__ __forceinline__ uint32_t pack16_fg(uint4 v, uint32_t thr) {
    return THR ? pack16_gt(v, thr * 0x01010101u) : pack16(v);
}

// Rows whose length is not a multiple of 16 bytes: byte loads (kept out of line).
__device__ __noinline__ uint32_t load_word_bytes(const uint8_t *src, int n, uint32_t thr) {
    uint32_t m = 0;
#pragma unroll 1
    for (int i = 0; i < n; i++) m |= (uint32_t)(__ldcs(src + i) > thr) << i;
    return m;
}

// Load the 32 pixels of lane-word (row, word) as a bitmask.
template <bool THR>
__device__ __forceinline__ uint32_t load_word(const uint8_t *__restrict__ img, const Geometry &g,
                                              int row, int col0) {
    if (col0 >= g.W) return 0u;
    const uint8_t *src = img + (int64_t)row * g.W + col0;
    const uint32_t thr = THR ? (uint32_t)g.thr : 0u;
    if (g.aligned) {
        uint32_t m = pack16_fg<THR>(__ldcs(reinterpret_cast<const uint4 *>(src)), thr);
        if (col0 + 16 < g.W) m |= pack16_fg<THR>(__ldcs(reinterpret_cast<const uint4 *>(src + 16)), thr) << 16;
        return m;
    }
    return load_word_bytes(src, min(32, g.W - col0), thr);
}

// Run mask of image row `row`, word `gword` (lane = word within the tile
// column; whole warp): the foreground with the tile-local bridged single-pixel
// holes filled, exactly as K1 P0b fills them (holes whose left/right
// neighbours are in the tile, bridged by the pixel above or below inside the
// tile).  *fg receives the foreground word itself.
__device__ __forceinline__ uint32_t run_mask(const Geometry &g, const uint32_t *__restrict__ bm,
                                             int row, int gword, int rl, int rows, uint32_t *fg) {
    const int lane = lane_id();
    const bool ok = gword < g.WW;
    const int64_t i = (int64_t)row * g.WW + gword;
    const uint32_t x0 = ok ? __ldcg(bm + i) : 0u;
    const uint32_t u = (ok && rl > 0) ? __ldcg(bm + i - g.WW) : 0u;
    const uint32_t d = (ok && rl + 1 < rows) ? __ldcg(bm + i + g.WW) : 0u;
    const uint32_t xlr = __shfl_up_sync(FULL, x0, 1), xrr = __shfl_down_sync(FULL, x0, 1);
    const uint32_t xl = lane == 0 ? 0u : xlr, xr = lane == 31 ? 0u : xrr;
    const uint32_t holes = ~x0 & ((x0 << 1) | (xl >> 31)) & ((x0 >> 1) | (xr << 31));
    if (fg) *fg = x0;
    return x0 | (holes & (u | d));
}

// ========================================================================= K1
// Tile-local two-pass labeling with runs as the provisional labels.  The run
// with ordinal o in tile row r has index k = r*MAXRUN + o; indices grow in
// raster order of the runs' heads and play the role of ARemSP's provisional
// labels, so "link to the smaller index" keeps every root at its component's
// first pixel.  Every warp owns S consecutive rows (a strip); per-run work is
// done a row at a time with lane = run ordinal.
constexpr int MLCAP = 256;  // P2a -> P2b merge list entries in k_tile_big (4x in k_tile_local; the rest stay in mc)
// Runs per tile row the main K1 holds in shared memory (16 KB union-find
// array: 6 CTAs/SM).  A tile with a row of more runs (alternating pixels)
// is left to k_tile_big, which holds the full MAXRUN per row (5 CTAs/SM).
constexpr int K1_MR = 256;
template <int MR, int MLN = (MR == MAXRUN ? MLCAP : 4 * MLCAP)>
struct K1SmemT {
    static constexpr int ML = MLN;  // merge list entries
    uint16_t p[TH * MR];           // parent of each run (the union-find array p of Alg. merge)
    uint32_t bm[TH][WPR];          // run masks (foreground + filled holes)
    // P0: raw foreground; P2a/P2b: upper-side merge heads; P3 on: bitmap of
    // the roots of components that touch the tile border (run k = r*MAXRUN+o
    // -> word [r][o/32], so every warp clears exactly the words it read)
    uint32_t mc[TH][WPR];
    // P0b-P2b: runs whose head lies in earlier words of the row; P4 on: row
    // w holds warp w's copy of the border nodes before each tile row
    uint16_t hbase[TH][WPR];
    int32_t nrun[TH];              // runs per row
    int32_t rowcnt[TH];            // components whose root run lies in the row
    int32_t bcnt[TH];              // border components whose root run lies in the row
    uint32_t mlist[MLN];           // P2a -> P2b: merge pairs (upper | lower << 16)
    int32_t nmerge;
};
using K1Smem = K1SmemT<MAXRUN>;
constexpr int MLWIDE = 2048;  // merge list of the 32-warp K1 (small images: dense tiles, smem to spare)
using K1SmemWide = K1SmemT<MAXRUN, MLWIDE>;

// Upper-side edges that the copy step does not already cover.  The edge set
// {(L, leftmost upper run of L)} U {(U, leftmost lower run of U)} connects
// everything two adjacent rows connect; the second family is redundant unless
// U's head h touches the lower run L through pixel h-1 AND L reaches an upper
// pixel at h-2 or further left (then L's leftmost upper neighbour is another
// run).  S is the segmented smear of the touch pixels along the lower runs,
// including carries from the lanes to the left.
__device__ __forceinline__ uint32_t upper_merge_heads(uint32_t hu, uint32_t u, uint32_t up,
                                                      uint32_t x, uint32_t xp, uint32_t S) {
    const uint32_t Sp = __shfl_up_sync(FULL, S, 1);
    const uint32_t sp = lane_id() == 0 ? 0u : Sp;
    const uint32_t x1 = (x << 1) | (xp >> 31);              // lower pixel at h-1
    const uint32_t s2 = (S << 2) | (sp >> 30);              // smear at h-2
    const uint32_t u2 = (u << 2) | (up >> 30);              // upper pixel at h-2
    return hu & x1 & (s2 | u2);
}


// THR: foreground <=> byte > g.thr (threshold on load) instead of byte != 0;
// a separate instantiation so the plain path carries no threshold code.
// BATCH: a stack of images (tile rows are placed per image); the single-image
// instantiation keeps the plain row arithmetic.
// Development knob (scripts/k1_phases.py): K1 truncated after a phase.  Only
// in builds with -DCCL_PHASE_KNOB=1 -- the checks cost the product K1 ~3 us.
#if CCL_PHASE_KNOB
#define K1_STOP(cond) \
    if (cond) return
#else
#define K1_STOP(cond) (void)0
#endif
// MR: runs per row held in shared memory (K1_MR in k_tile_local, MAXRUN in
// k_tile_big).  Run (row r, ordinal o) has index k = r*MR + o.
template <bool THR, bool BATCH, bool BANDS, int MR, int SR = S>
__device__ __forceinline__ void k1_tile(const uint8_t *__restrict__ img, const Geometry &g, const Workspace &ws,
                                        const int tile, const int tx, const int ty, int pfd, int pfx, int pfy,
                                        int stop) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    using Sm = K1SmemT<MR, SR == 1 ? MLWIDE : (MR == MAXRUN ? MLCAP : 4 * MLCAP)>;
    Sm &sm = *reinterpret_cast<Sm *>(smem_raw);
    auto kidx = [](int r, int o) { return r * MR + o; };
    constexpr int NWK = TH / SR;  // warps of the CTA (SR rows each)

    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int R0 = BATCH ? tile_r0(g, ty) : ty * TH, C0 = tx * TW;
    const int rows = BATCH ? tile_rows(g, ty) : min(TH, g.H - R0);
    const int vcols = min(TW, g.W - C0);
    const int gword = tx * WPR + lane;  // this lane's word index in the image row
    const int r0 = w * SR;
    volatile uint16_t *vp = sm.p;
    uint32_t *bbits = &sm.mc[0][0];

    // Warm L2 with the pixels of the tile that will start about a quarter
    // wave of resident CTAs later (pfd = a quarter of the resident CTAs on
    // the device; measured against 3/8, 1/2, 5/8, 1, 1.5 and 2 waves): its
    // loads then hit L2 instead of waiting on HBM.
    {
        if (pfd > 0 && tile + pfd < g.nT) {
            // tile + pfd = (ty + pfy, tx + pfx) with a carry (no division)
            int ptx = tx + pfx, pty = ty + pfy;
            if (ptx >= g.nTx) {
                ptx -= g.nTx;
                pty++;
            }
            const int prow = (BATCH ? tile_r0(g, pty) : pty * TH) + (threadIdx.x >> 3);
            const int pcol = ptx * TW + (threadIdx.x & 7) * 128;
            if ((int)(threadIdx.x >> 3) < TH && (BATCH ? (int)(threadIdx.x >> 3) < tile_rows(g, pty) : prow < g.H) &&
                pcol < g.W) {
                const uint8_t *a = img + (int64_t)prow * g.W + pcol;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                if ((threadIdx.x & 7) == 7 && pcol + 127 < g.W)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a + 127));
            }
        }
    }
    // The tiles of the first quarter wave are nobody's look-ahead: they warm
    // their own lines.  (Prefetches may run before the grid dependency wait:
    // they only move lines into L2, the coherence point.)
    if (tile < pfd) {
        const int prow = R0 + (threadIdx.x >> 3), pcol = C0 + (threadIdx.x & 7) * 128;
        if ((int)(threadIdx.x >> 3) < rows && pcol < g.W)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(img + (int64_t)prow * g.W + pcol));
    }
    // Every run starts as its own label: the warp's rows
    // are one contiguous range of p, set to the identity with 16-byte stores
    // (8 entries each; entries past a row's runs are never read) before the
    // grid dependency wait -- shared memory only.
    {
        constexpr int NV = SR * MR / 8;  // uint4 per warp
        static_assert(NV % 32 == 0, "p init: whole uint4 per lane");
        uint4 *pv = reinterpret_cast<uint4 *>(sm.p + kidx(r0, 0));
        const uint32_t e0 = (uint32_t)kidx(r0, 0);
#pragma unroll
        for (int v = lane; v < NV; v += 32) {
            const uint32_t w0 = (e0 + 8u * v) * 0x10001u + 0x10000u;  // entries e, e+1
            pv[v] = make_uint4(w0, w0 + 0x20002u, w0 + 0x40004u, w0 + 0x60006u);
        }
    }
    // The image may be written by the kernel just before this one on the
    // stream (the caller's producer): no pixel is loaded before the wait.
    pdl_wait();
    // ---- P0: the pixels of the tile, read once with 16-byte streaming loads:
    // fg = byte != 0 (reading A10) -- or byte > thr when a
    // threshold is set -- one bit per pixel.  The warp's SR rows are all in
    // flight before the first is used.
    uint32_t xs[SR];
    if (g.aligned && C0 + TW <= g.W && rows == TH) {  // interior tile: all 2*SR loads in flight
        const uint8_t *src = img + (int64_t)(R0 + r0) * g.W + C0 + 32 * lane;
        uint4 v[2 * SR];
        if (((reinterpret_cast<uintptr_t>(img) | (uintptr_t)g.W) & 31u) == 0) {
            // rows 32-byte aligned: one 256-bit load per lane and row (K1
            // 279 -> 273 us on C4 against two 128-bit loads)
#pragma unroll
            for (int i = 0; i < SR; i++) {
                uint4 &a = v[2 * i], &b = v[2 * i + 1];
                asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                             : "l"(src + (int64_t)i * g.W));
            }
        } else
#pragma unroll
        for (int i = 0; i < SR; i++) {
            v[2 * i] = __ldcs(reinterpret_cast<const uint4 *>(src + (int64_t)i * g.W));
            v[2 * i + 1] = __ldcs(reinterpret_cast<const uint4 *>(src + (int64_t)i * g.W + 16));
        }
        if (!THR) {
            // warp-uniform fast path when every byte the warp loaded is 0 or 1
            uint32_t o = 0;
#pragma unroll
            for (int j = 0; j < 2 * SR; j++) o |= v[j].x | v[j].y | v[j].z | v[j].w;
            if (!__any_sync(FULL, (o & 0xFEFEFEFEu) != 0u)) {
#pragma unroll
                for (int i = 0; i < SR; i++) xs[i] = pack16_01(v[2 * i]) | (pack16_01(v[2 * i + 1]) << 16);
            } else {
#pragma unroll
                for (int i = 0; i < SR; i++) xs[i] = pack16(v[2 * i]) | (pack16(v[2 * i + 1]) << 16);
            }
        } else {
            const uint32_t t4 = (uint32_t)g.thr * 0x01010101u;
#pragma unroll
            for (int i = 0; i < SR; i++) xs[i] = pack16_gt(v[2 * i], t4) | (pack16_gt(v[2 * i + 1], t4) << 16);
        }
    } else {
#pragma unroll
        for (int i = 0; i < SR; i++)
            xs[i] = (r0 + i < rows && gword < g.WW) ? load_word<THR>(img, g, R0 + r0 + i, 32 * gword) : 0u;
    }
    // bm (1/8 B per pixel) is read again by K2 and K5 while ~5 B/px of image
    // and labels stream through L2: it is stored with the evict_last priority
    // (K5's label stores are evict_first), measured -10 us on C4
    uint64_t pol_last;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
    if ((MR < MAXRUN || SR != S) && tile == 0) {  // reset the numbering scan's lookback state (K3)
        for (int i = threadIdx.x; i < g.nTy; i += NWK * 32) ws.scanstate[i] = 0ull;
        if (threadIdx.x == 0) *ws.ticket = 0;
    }
#pragma unroll
    for (int i = 0; i < SR; i++) {
        sm.mc[r0 + i][lane] = xs[i];  // raw masks (mc is free until P2a)
        if (r0 + i < rows && gword < g.WW) {
            asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(ws.bm + (int64_t)(R0 + r0 + i) * g.WW + gword),
                         "r"(xs[i]), "l"(pol_last) : "memory");
        }
    }
    if (lane < SR) sm.bcnt[r0 + lane] = 0;
    if (threadIdx.x == 0) sm.nmerge = 0;
    __syncthreads();
    K1_STOP(stop < 0);
    // ---- P0b: run mask = foreground + bridged single-pixel holes (a background
    // pixel whose left and right neighbours and the pixel above or below are
    // foreground).  Only holes whose neighbours lie in
    // this tile are filled: any subset of bridged holes preserves the
    // partition of the foreground, and K2/K5 read the same run mask.
    // Then run heads and per-word run counts (p was set to the identity
    // above).
    bool over = false;  // a row of this warp has more runs than the p array holds
#pragma unroll
    for (int i = 0; i < SR; i++) {
        const int rl = r0 + i;
        const uint32_t x0 = xs[i];
        const uint32_t xlr = __shfl_up_sync(FULL, x0, 1), xrr = __shfl_down_sync(FULL, x0, 1);
        const uint32_t xl = lane == 0 ? 0u : xlr, xr = lane == 31 ? 0u : xrr;
        const uint32_t u = rl > 0 ? sm.mc[rl - 1][lane] : 0u;
        const uint32_t d = rl + 1 < rows ? sm.mc[rl + 1][lane] : 0u;
        const uint32_t holes = ~x0 & ((x0 << 1) | (xl >> 31)) & ((x0 >> 1) | (xr << 31));
        const uint32_t x = x0 | (holes & (u | d));
        const uint32_t xfl = __shfl_up_sync(FULL, x, 1);
        const uint32_t hx = x & ~((x << 1) | (lane == 0 ? 0u : (xfl >> 31)));
        uint32_t nr;
        const uint32_t base = warp_excl_scan(__popc(hx), nr);
        sm.bm[rl][lane] = x;
        sm.hbase[rl][lane] = (uint16_t)base;
        if (lane == 0) sm.nrun[rl] = (int)nr;
        over |= (int)nr > MR;
    }
    if (MR < MAXRUN) {
        if (__syncthreads_or(over)) {  // too many runs in a row: k_tile_big takes the tile
            if (threadIdx.x == 0) {
                ws.k1over[atomicAdd(ws.k1over_n, 1)] = tile;
                atomicAdd(ws.stats + STAT_K1_HANDOVER, 1ull);
            }
            return;
        }
    } else {
        __syncthreads();
    }
    K1_STOP(stop <= 0);

    // ---- P2a: scan.  A run with a foreground pixel among the three above any
    // of its pixels copies its leftmost upper neighbour's label (the decision
    // tree's copy(b)/copy(a)/copy(c)).  Each warp walks its
    // own rows in order, so inside a strip a run copies its upper neighbour's
    // parent (already final within the strip); a strip's first row copies the
    // upper run's index (a run of the strip above).
#pragma unroll 1
    for (int i = 0; i < SR; i++) {
        const int rl = r0 + i;
        if (rl >= rows || rl == 0) {
            sm.mc[rl][lane] = 0u;
            continue;
        }
        const uint32_t x = sm.bm[rl][lane], u = sm.bm[rl - 1][lane];
        const uint32_t xpr = __shfl_up_sync(FULL, x, 1);
        const uint32_t upr = __shfl_up_sync(FULL, u, 1), unr = __shfl_down_sync(FULL, u, 1);
        const uint32_t xp = lane == 0 ? 0u : xpr;
        const uint32_t up = lane == 0 ? 0u : upr, un = lane == 31 ? 0u : unr;
        const uint32_t hx = x & ~((x << 1) | (xp >> 31));
        // upper row: heads and run-index base of lanes lane-1, lane, lane+1
        const uint32_t hu = u & ~((u << 1) | (up >> 31));
        const int ub = kidx(rl - 1, sm.hbase[rl - 1][lane]);
        const uint32_t hun = __shfl_down_sync(FULL, hu, 1);
        const uint32_t uL = (u << 1) | (up >> 31);  // upper pixel at p-1
        const uint32_t t = x & (u | uL | (u >> 1) | (un << 31));
        // First touch of every run and S_ = the run pixels at or after it,
        // by one addition: q = untouched run pixels; adding the untouched run
        // heads (bit 0 counts as a head while the run from the left lanes has
        // no touch yet) carries through each head's untouched prefix P and
        // stops at the first touch.  Across lanes: a carry-lookahead on
        // "touched by bit 31" through all-ones words (tests/test_lemmas.py).
        const uint32_t hv0 = hx | (x & 1u);
        const uint32_t q = x & ~t;
        const uint32_t P0 = q & ~(q + (hv0 & ~t));
        const uint32_t cin = carry_in_fwd(((x & ~P0) >> 31) != 0u, x == FULL) & x & 1u;
        const uint32_t lead = x & ~(x + 1);
        const uint32_t P = cin ? (P0 & ~lead) : P0;
        const uint32_t S_ = x & ~P;
        uint32_t ft = t & ((P << 1) | (cin ? hx : hv0));
        uint32_t mc = upper_merge_heads(hu, u, up, x, xp, S_);
        // (K2 also drops the edges whose gap pixel is a hole bridged from the
        // row above -- redundant ones; here the merges are shared out over the
        // CTA and cost less than the filter: every listed edge is a real
        // 8-adjacency of the two runs)
        const int lbase = kidx(rl, sm.hbase[rl][lane]) - 1;
        // the row's merges go to a tile-wide list that all threads work
        // through in P2b (balanced); what does not fit stays in mc
        if (mc) {
            int idx = atomicAdd(&sm.nmerge, __popc(mc));
            while (mc && idx < Sm::ML) {
                const int b = __ffs(mc) - 1;
                const int a = ub + __popc(hu & upto(b)) - 1;         // the upper run with head h
                const int c = lbase + __popc(hx & ((1u << b) - 1u));  // the lower run containing h-1
                sm.mlist[idx++] = (uint32_t)a | ((uint32_t)c << 16);
                mc &= mc - 1;
            }
        }
        sm.mc[rl][lane] = mc;
        const bool instrip = i > 0;
        // The run of the leftmost upper foreground pixel q among b-1, b, b+1
        // is ub - 1 + (upper heads at <= q).  Heads at <= q = heads at <= b+1
        // less the head at b+1 when q = b-1 (q = b-1 rules out a head at b,
        // q = b one at b+1), so with hnext (bit b = upper head at b+1; bit 31
        // the next word's first pixel) and hb (q = b-1 and a head at b+1) the
        // count is (hu & 1) + popc(hnext & bits 0..b) - hb[b]: two popcounts
        // and three-input logic per touch, no 64-bit or variable shifts.
        const uint32_t hnext = (hu >> 1) | (lane == 31 ? 0u : hun << 31);  // no word right of the tile
        const uint32_t hb = uL & hnext;
        const int ubc = ub - 1 + (int)(hu & 1u);
        while (ft) {
            const uint32_t f1 = ft - 1u;
            const uint32_t m = ft ^ f1;              // bits 0..b, b = lowest touch
            const uint32_t xb = hb & ft & ~f1;       // bit b if q = b-1 skips a head at b+1
            ft &= f1;
            const int ui = ubc + __popc(hnext & (m ^ xb));
            vp[lbase + __popc(hx & m)] = instrip ? vp[ui] : (uint16_t)ui;
        }
        __syncwarp();
    }
    __syncthreads();
    K1_STOP(stop <= 1);
    // ---- P2b: the remaining edges, merged with lock-free Rem's splicing
    // (the decision tree's copy(c,a)/copy(c,d) merges).  The
    // parent chains may still cross strips (a strip's first row points into
    // the strip above): Rem's algorithm works on any forest with p[x] <= x.
    // The tile's merge list is shared out over all 256 threads (a strip with
    // many merges no longer holds the barrier); rows whose merges did not fit
    // in the list finish them per lane below.
    const int nmerge = sm.nmerge;
    constexpr int MLC = Sm::ML;
    if (threadIdx.x == 0 && nmerge > 0) {  // path counters (ccl_plan_counters)
        atomicAdd(ws.stats + STAT_K1_MERGES, (unsigned long long)nmerge);
        if (nmerge > MLC)
            atomicAdd(ws.stats + (MR == MAXRUN && SR == S ? STAT_K1BIG_LIST_OVERFLOW : STAT_K1_LIST_OVERFLOW), 1ull);
    }
    // All 256 threads work through the list at once (union_smem is safe
    // under concurrency, see above).
    for (int i = threadIdx.x; i < min(nmerge, MLC); i += NWK * 32) {
        const uint32_t e = sm.mlist[i], a = e & 0xFFFFu, c = e >> 16;
        if (vp[a] != vp[c]) union_smem(sm.p, a, c);
    }
    if (nmerge <= MLC) {  // nothing left per lane: clear the rows for bbits
#pragma unroll
        for (int i = 0; i < SR; i++) sm.mc[r0 + i][lane] = 0u;
    } else
#pragma unroll 1
    for (int i = 0; i < SR; i++) {
        const int rl = r0 + i;
        uint32_t m = (rl < rows) ? sm.mc[rl][lane] : 0u;
        sm.mc[rl][lane] = 0u;  // becomes this row's part of bbits
        if (__ballot_sync(FULL, m != 0u) == 0u) continue;  // warp-uniform
        const uint32_t u = sm.bm[rl - 1][lane], x = sm.bm[rl][lane];
        const uint32_t upr = __shfl_up_sync(FULL, u, 1), xpr = __shfl_up_sync(FULL, x, 1);
        const uint32_t hu = u & ~((u << 1) | (lane == 0 ? 0u : (upr >> 31)));
        const int ub = kidx(rl - 1, sm.hbase[rl - 1][lane]);
        const int xb = kidx(rl, sm.hbase[rl][lane]);
        const uint32_t hx = x & ~((x << 1) | (lane == 0 ? 0u : (xpr >> 31)));
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            const int a = ub + __popc(hu & upto(b)) - 1;  // the upper run with head h
            // the lower run containing pixel h-1
            const int c = xb - 1 + __popc(hx & ((1u << b) - 1u));
            if (vp[a] != vp[c]) union_smem(sm.p, (uint32_t)a, (uint32_t)c);
        }
    }
    __syncthreads();
    K1_STOP(stop <= 2);
    // ---- P3: flatten -- every run -> its root (Alg. flatten's p[i] <- p[p[i]],
    // PAPER.md:711-712), own rows, lane = run ordinal.  A root r's entry
    // becomes 0x8000 | (its rank among the roots of its row); finds treat a
    // flagged entry as a root.  A run on the tile border marks its root in
    // bbits, and the first mark of a root counts it in its row's border-root
    // count (row of run r = r / MAXRUN).
    const int lc = vcols - 1;
#pragma unroll 1
    for (int i = 0; i < SR; i++) {
        const int rl = r0 + i, n = sm.nrun[rl];
        const bool edge_row = rl == 0 || rl == rows - 1;
        const bool lfirst = sm.bm[rl][0] & 1u, llast = (sm.bm[rl][lc >> 5] >> (lc & 31)) & 1u;
        int cnt = 0;
#pragma unroll 1
        for (int o0 = 0; o0 < n; o0 += 32) {
            const int o = o0 + lane, k = kidx(rl, o);
            bool root = false;
            if (o < n) {
                // the first hop is usually shared: later rows of the strip
                // copied the same upper-strip run, so it is compressed too
                const uint32_t j = vp[k];
                uint32_t r = j;
                // (j is never flagged: only this warp ranks its own runs,
                // below; j == k: a root, no second load)
                // (a non-root's parent is below it; a root points to itself or
                // holds 0x8000 | rank > any index: one compare stops at both)
                if (j != (uint32_t)k)
                    while (true) {
                        const uint32_t v = vp[r];
                        if (v >= r) break;
                        r = v;
                    }
                root = r == (uint32_t)k;
                if (j != r) {  // more than one hop (a root has j == r == k)
                    vp[k] = (uint16_t)r;
                    vp[j] = (uint16_t)r;
                }
                if (edge_row || (o == 0 && lfirst) || (o == n - 1 && llast)) {
                    const uint32_t bit = 1u << (r & 31);
                    uint32_t *wd = bbits + (r / MR) * WPR + ((r % MR) >> 5);
                    if (!(atomicOr(wd, bit) & bit)) atomicAdd(&sm.bcnt[r / MR], 1);
                }
            }
            const uint32_t bal = __ballot_sync(FULL, root);
            if (root) vp[k] = (uint16_t)(0x8000u | (uint32_t)(cnt + __popc(bal & ((1u << lane) - 1u))));
            cnt += __popc(bal);
        }
        if (lane == 0) sm.rowcnt[rl] = cnt;
    }
    __syncthreads();
    K1_STOP(stop <= 3);
    // ---- P4: roots in index order = raster order of first pixels get the
    // consecutive component numbers (Alg. flatten's k++):
    // component = (roots in earlier rows) + (rank in its row).  Every run ->
    // its component (for K5); border roots become nodes of the global
    // union-find in index order; key = (image row, tile column, run ordinal):
    // raster order.
    uint32_t rtot, btot;
    const int rowfirst = (int)warp_excl_scan((uint32_t)sm.rowcnt[lane], rtot);  // lane = row
    const int bfirst = (int)warp_excl_scan((uint32_t)sm.bcnt[lane], btot);
    const int ncomp = (int)rtot, nborder = (int)btot;
    // this warp's copy of the border nodes before each row (lane = row), for
    // the node lookups below in lane-divergent code (hbase is free after P2b;
    // every warp has its own row of it, so no barrier follows P3's)
    static_assert(WPR == TH, "hbase rows hold one entry per tile row");
    uint16_t *bfrow = sm.hbase[w];
    bfrow[lane] = (uint16_t)bfirst;
    __syncwarp();
    int32_t *compnode = ws.compnode + (int64_t)tile * g.capc;
    const int nodebase = tile * g.capb;
    const int64_t dstride = (int64_t)g.nTx * g.maxrun;
    {
        // every run -> runcomp = (root row << 9) | rank of the root in its
        // row; the component is rowfirst[row] + rank (K5 needs the row).  A
        // per-lane loop (no ballot, no warp-uniform chunking): the row's only
        // loop-carried state is o.
        uint16_t *dst = ws.runcomp + ((int64_t)(R0 + r0) * g.nTx + tx) * g.maxrun;
#pragma unroll 1
        for (int i = 0; i < SR; i++, dst += dstride) {
            const int rl = r0 + i, n = sm.nrun[rl];
            const uint16_t *prow = sm.p + kidx(rl, 0);
#pragma unroll 1
            for (int o = lane; o < n; o += 32) {
                const uint32_t pk = prow[o];
                const uint32_t r = (pk & 0x8000u) ? (uint32_t)kidx(rl, o) : pk;
                const uint32_t pr = (pk & 0x8000u) ? pk : sm.p[r];
                dst[o] = (uint16_t)(((r / MR) << 9) | (pr & 0x1FFu));
            }
        }
    }
    // border roots (rows with any; most rows have none): nodes of the global
    // union-find in index order, key = (image row, tile column, run ordinal)
#pragma unroll 1
    for (int i = 0; i < SR; i++) {
        const int rl = r0 + i;
        if (sm.bcnt[rl] == 0) continue;  // warp-uniform
        const int n = sm.nrun[rl];
        int bi = __shfl_sync(FULL, bfirst, rl);
        const int rf = __shfl_sync(FULL, rowfirst, rl);
        const uint32_t *brow = bbits + rl * WPR;
#pragma unroll 1
        for (int o0 = 0; o0 < n; o0 += 32) {
            const int o = o0 + lane;
            const uint32_t pk = o < n ? sm.p[kidx(rl, o)] : 0u;
            const bool broot = o < n && (pk & 0x8000u) && ((brow[o >> 5] >> (o & 31)) & 1u);
            const uint32_t bbal = __ballot_sync(FULL, broot);
            if (broot) {  // a root of this row: component rowfirst[row] + rank
                const int c = rf + (int)(pk & 0x1FFu);
                const int node = nodebase + bi + __popc(bbal & ((1u << lane) - 1u));
                if (BANDS) compnode[c] = node;  // only the row-band path reads it
                ws.gparent[node] = node;
                ws.gnodecomp[node] = (rl << 16) | c;
                ws.gkey[node] = ((int64_t)(g.row0 + R0 + rl) * g.nTx + tx) * MAXRUN + o;
            }
            bi += __popc(bbal);
        }
    }
    K1_STOP(stop <= 4);
    // ---- P4c: nodes of the border pixels (for K2).  A border run's root r is
    // a border root; its node is the border roots of earlier rows (bfrow)
    // plus those before it in its row's bitmap words -- all in shared memory,
    // final since P3's barrier.  Top row, bottom row and the rows' end runs
    // as one list over the CTA.
    {
        auto node_of = [&](int k) -> int {
            const uint32_t pk = sm.p[k];
            const int r = (pk & 0x8000u) ? k : (int)pk;
            const int rr = r / MR, ro = r % MR;
            const uint32_t *bw = bbits + rr * WPR;
            int nd = nodebase + bfrow[rr] + __popc(bw[ro >> 5] & ((1u << (ro & 31)) - 1u));
            for (int j = 0; j < (ro >> 5); j++) nd += __popc(bw[j]);
            return nd;
        };
        const int ntop = sm.nrun[0], nbot = sm.nrun[rows - 1];
        for (int it = threadIdx.x; it < ntop + nbot + rows; it += NWK * 32) {
            if (it < ntop) {
                ws.topnode[(int64_t)tile * g.maxrun + it] = node_of(kidx(0, it));
            } else if (it < ntop + nbot) {
                const int o = it - ntop;
                ws.botnode[(int64_t)tile * g.maxrun + o] = node_of(kidx(rows - 1, o));
            } else {
                const int r = it - ntop - nbot;
                const int64_t off = (int64_t)tx * g.H + R0 + r;
                ws.leftnode[off] = (sm.bm[r][0] & 1u) ? node_of(kidx(r, 0)) : -1;
                ws.rightnode[off] = ((sm.bm[r][lc >> 5] >> (lc & 31)) & 1u) ? node_of(kidx(r, sm.nrun[r] - 1)) : -1;
            }
        }
    }
    // the first and last row's run masks for K2's horizontal edges
    if (w == NWK - 1) ws.edgerow[(int64_t)tile * 2 * WPR + lane] = sm.bm[0][lane];
    if (w == NWK - 2) ws.edgerow[((int64_t)tile * 2 + 1) * WPR + lane] = sm.bm[rows - 1][lane];
    int32_t *meta = ws.meta + (int64_t)tile * META;
    if (w == 0) {  // first component of every tile row (components are in key order)
        meta[META_ROWFIRST + lane] = rowfirst;
        if (lane == 0) {
            meta[META_ROWFIRST + TH] = ncomp;
            meta[META_NCOMP] = ncomp;
            meta[META_NBORDER] = nborder;
            meta[META_ROWS] = rows;
        }
    }
}

#ifndef K1_SR
#define K1_SR S  // rows per warp of the main K1 (TH / K1_SR warps per CTA)
#endif
constexpr int K1_THREADS = TH / K1_SR * 32;
template <bool THR, bool BATCH, bool BANDS = false>
#ifndef K1_MINB
#define K1_MINB 6  // CTAs per SM (40 registers; 7 forces 32 and spills)
#endif
__global__ void __launch_bounds__(K1_THREADS, K1_MINB)
k_tile_local(const uint8_t *__restrict__ img, Geometry g, Workspace ws, int pfd, int pfx, int pfy, int stop) {
    pdl_trigger();
    // a 2-D grid (tile columns x tile rows; CTAs still start in raster
    // order) spares the divisions, unless nTy exceeds the grid's y limit
    int tile, tx, ty;
    if (gridDim.y > 1 || g.nTy == 1) {
        tx = blockIdx.x;
        ty = blockIdx.y;
        tile = ty * g.nTx + tx;
    } else {
        tile = blockIdx.x;
        tx = tile % g.nTx;
        ty = tile / g.nTx;
    }
    k1_tile<THR, BATCH, BANDS, K1_MR, K1_SR>(img, g, ws, tile, tx, ty, pfd, pfx, pfy, stop);
}

// Images of few tiles (fewer than the SMs can hold twice over): one warp per
// tile row, 32 warps per CTA, so a tile's rows are worked on in parallel --
// the single-image latency of the <= 1 MB regime.  It
// holds the full MAXRUN runs per row (44 KB), so it never hands a tile over
// and the hand-over pass is not launched.
template <bool THR, bool BATCH, bool BANDS = false>
__global__ void __launch_bounds__(TH * 32, 1)
k_tile_local_wide(const uint8_t *__restrict__ img, Geometry g, Workspace ws, int stop) {
    pdl_trigger();
    const int tile = blockIdx.x;
    k1_tile<THR, BATCH, BANDS, MAXRUN, 1>(img, g, ws, tile, tile % g.nTx, tile / g.nTx, 0, 0, 0, stop);
}

// The tiles k_tile_local handed over (a row with more than K1_MR runs); the
// list is final once k_tile_local completed.  Usually empty.
template <bool THR, bool BATCH, bool BANDS = false>
__global__ void __launch_bounds__(NW * 32, 5)
k_tile_big(const uint8_t *__restrict__ img, Geometry g, Workspace ws, int stop) {
    pdl_trigger();
    pdl_wait();
    const int n = __ldcg(ws.k1over_n);
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const int tile = __ldcg(ws.k1over + i);
        k1_tile<THR, BATCH, BANDS, MAXRUN>(img, g, ws, tile, tile % g.nTx, tile / g.nTx, 0, 0, 0, stop);
        __syncthreads();  // shared memory is reused by the next tile
    }
}

// ========================================================================= K2
// Horizontal tile edges: one warp per (tile row boundary, tile column); the
// runs of the last row above and the first row below are united along the
// same two edge families as the strip merge.  Vertical tile edges (incl.
// corner pixels): one thread per (tile column boundary, row).
#ifndef CCL_K2_WARPS
#define CCL_K2_WARPS 4
#endif
constexpr int K2_WARPS = CCL_K2_WARPS;  // measured vs 2 and 8 warps per CTA
__global__ void __launch_bounds__(K2_WARPS * 32)
k_border(Geometry g, Workspace ws, int nh_warps, int hsplit) {
    pdl_trigger();
    pdl_wait();
    __shared__ uint32_t shd[K2_WARPS][2][WPR], sbs[K2_WARPS][2][WPR];
    constexpr int PCAP = 128;
    __shared__ uint32_t plist[K2_WARPS][PCAP];  // the edge's unions: (upper run, lower run) ordinals
    const int lane = lane_id(), wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * K2_WARPS + wib;
    if (gw < nh_warps) {
        // hsplit warps per horizontal edge (images of few tiles: more lanes
        // for the edge's unions); each lists them all and works on its share
        const int he = gw / hsplit, hs = gw - he * hsplit;
        const int tx = he % g.nTx, ty = 1 + he / g.nTx;
        if (ty % g.tpi == 0) return;  // first tile row of an image of a batch: no edge
        // the run masks of the two rows, as K1 left them
        const uint32_t u = __ldcg(ws.edgerow + ((int64_t)((ty - 1) * g.nTx + tx) * 2 + 1) * WPR + lane);
        const uint32_t x = __ldcg(ws.edgerow + (int64_t)(ty * g.nTx + tx) * 2 * WPR + lane);
        RowView U = make_row(u), X = make_row(x);
        shd[wib][0][lane] = U.hx; sbs[wib][0][lane] = U.base;
        shd[wib][1][lane] = X.hx; sbs[wib][1][lane] = X.base;
        __syncwarp();
        const int32_t *bot = ws.botnode + (int64_t)((ty - 1) * g.nTx + tx) * g.maxrun;
        const int32_t *top = ws.topnode + (int64_t)(ty * g.nTx + tx) * g.maxrun;
        // the edge's unions are listed first (run ordinals, shared memory
        // only) and then done one per lane: a lane with several edges no
        // longer runs their global union chains one after another.  Every
        // lane's edges get consecutive list positions (a warp scan of its
        // counts); a dense edge (more than PCAP unions) is worked through in
        // windows of PCAP, each fully lane-parallel.
        const uint32_t m1 = first_in_run(x & dilate(U), x);
        uint32_t m2;
        // upper runs whose leftmost lower neighbour has another leftmost upper
        // neighbour (see upper_merge_heads in K1)
        {
            const uint32_t t = x & dilate(U);
            const uint32_t s = smear_up(t, x);
            const uint32_t cin = carry_in_fwd(((x >> 31) & (s >> 31)) != 0, x == FULL) & x & 1u;
            const uint32_t S_ = s | (cin ? (x & ~(x + 1)) : 0u);
            // (no hole-bridged filter: it only drops redundant edges)
            m2 = upper_merge_heads(U.hx, u, U.xp, x, X.xp, S_);
        }
        uint32_t tot;
        const int base = (int)warp_excl_scan(__popc(m1) + __popc(m2), tot);
        for (int w0 = 0; w0 < (int)tot; w0 += PCAP) {
            int idx = base - w0;  // this lane's next entry, relative to the window
            for (uint32_t m = m1; m && idx < PCAP; m &= m - 1, idx++) {
                if (idx < 0) continue;
                const int b = __ffs(m) - 1;
                const int q = 32 * lane + b + leftmost3(u, U.xp, U.xn, b), lq = q >> 5;
                plist[wib][idx] = (uint32_t)run_ord(shd[wib][0][lq], sbs[wib][0][lq], q & 31) |
                                  ((uint32_t)run_ord(X.hx, X.base, b) << 16);
            }
            for (uint32_t m = m2; m && idx < PCAP; m &= m - 1, idx++) {
                if (idx < 0) continue;
                const int b = __ffs(m) - 1;
                const int q = 32 * lane + b - 1, lq = q >> 5;  // lower pixel h-1
                plist[wib][idx] = (uint32_t)run_ord(U.hx, U.base, b) |
                                  ((uint32_t)run_ord(shd[wib][1][lq], sbs[wib][1][lq], q & 31) << 16);
            }
            __syncwarp();
            const int np = min(PCAP, (int)tot - w0);
            if (hsplit == 1) {
                // consecutive entries often join the same two nodes (one region
                // crossing the edge in several runs): a union equal to the
                // previous lane's is skipped, as on the vertical edges (C4
                // step -2 us; K4 then walks a little more)
                for (int i0 = 0; i0 < np; i0 += 32) {
                    const int i = i0 + lane;
                    const uint32_t e = i < np ? plist[wib][i] : 0u;
                    const int a = i < np ? bot[e & 0xFFFFu] : -1, b = i < np ? top[e >> 16] : -1;
                    const int ap = __shfl_up_sync(FULL, a, 1), bp = __shfl_up_sync(FULL, b, 1);
                    if (i < np && !(lane > 0 && ap == a && bp == b)) gunion(ws.gparent, ws.gkey, a, b);
                }
            } else {
                for (int i = 32 * hs + lane; i < np; i += 32 * hsplit) {
                    const uint32_t e = plist[wib][i];
                    gunion(ws.gparent, ws.gkey, bot[e & 0xFFFFu], top[e >> 16]);
                }
            }
            __syncwarp();
        }
        return;
    }
    // vertical edges; lanes = consecutive rows of one edge, and a union that
    // the row above already made (same pair of nodes) is skipped -- a region
    // crossing the edge repeats its pair on every row it spans
    const int64_t t = (int64_t)(gw - nh_warps) * 32 + lane;
    const int64_t nv = (int64_t)(g.nTx - 1) * g.H;
    int tx = 0, r = 0, a = -1, b = -1, bu = -1, bd = -1;
    if (t < nv) {
        tx = 1 + (int)(t / g.H);
        r = (int)(t % g.H);
    }
    // rows r-1 / r+1 of the same image (a batch stacks images: no edges across)
    const bool has_up = r % g.IH != 0, has_dn = r + 1 < g.H && (r + 1) % g.IH != 0;
    if (t < nv) {  // the four node loads of the lane at once
        const int32_t *L = ws.leftnode + (int64_t)tx * g.H;
        a = ws.rightnode[(int64_t)(tx - 1) * g.H + r];
        const int bs = L[r];
        if (has_up) bu = L[r - 1];
        if (has_dn) bd = L[r + 1];
        b = a >= 0 ? bs : -1;
    }
    const int ap = __shfl_up_sync(FULL, a, 1), bp = __shfl_up_sync(FULL, b, 1);
    const int an = __shfl_down_sync(FULL, a, 1), bn = __shfl_down_sync(FULL, b, 1);
    const bool up_ok = lane > 0 && has_up;   // lane-1 is row r-1 of this edge
    const bool dn_ok = lane < 31 && has_dn;  // lane+1 is row r+1 of this edge
    if (a < 0) return;
    if (b >= 0) {
        // (r-1) and (r+1) are then joined through b
        if (!(up_ok && ap == a && bp == b)) gunion(ws.gparent, ws.gkey, a, b);
        return;
    }
    // diagonal neighbours; skipped when the adjacent row makes the same union
    if (bu >= 0 && !(up_ok && ap == a && bp == bu)) gunion(ws.gparent, ws.gkey, a, bu);
    if (bd >= 0 && !(dn_ok && an == a && bn == bd)) gunion(ws.gparent, ws.gkey, a, bd);
}

// ========================================================================= K4
// A border component that is not a global root takes its root's label (a
// root of this image's forest, or -- row bands -- a root owned by another
// band, whose global label arrived in xlab; labels stored here are band-local,
// K5 adds the band offset).  One warp per tile, over its border nodes.
#ifndef CCL_K4_WARPS
#define CCL_K4_WARPS 4  // measured vs 2, 8, 16: -0.5 us
#endif
constexpr int K4_WARPS = CCL_K4_WARPS;
// K4's work for one tile (one warp).  (Folded into K3 -- one warp per
// tile-row CTA works through 2-3 tiles' finds one after another, with flags
// for the earlier rows' root labels -- it took C4 K3 + K4 from 39 to 56 us.)
__device__ __forceinline__ void fixup_tile(const Geometry &g, const Workspace &ws, const int tile, const int lane) {
    const int nborder = __ldcg(ws.meta + (int64_t)tile * META + META_NBORDER);
    const int nodebase = tile * g.capb;
    int32_t *nrlab = ws.nrlab + (int64_t)tile * g.capc;
    const uint32_t *tbits = ws.tbits + (int64_t)tile * g.capw;
    const int32_t *twpre = ws.twpre + (int64_t)tile * g.capw;
    const uint64_t keep = pol_evict_last();  // the labels stay in L2 for K5
    auto root_label = [&](int r) -> int32_t {
        if (r < 0) {  // a root owned by another band: its band-local label + that band's
                      // offset, less this band's (the label stored here is band-local)
            const int f = -2 - r, k = f / (2 * g.W), stride = 2 * g.W + 1;
            int off = 0;
            for (int j = 0; j < max(k, ws.xself); j++) {
                const int c = __ldcg(ws.xlab + (size_t)j * stride);
                off += (j < k ? c : 0) - (j < ws.xself ? c : 0);
            }
            return __ldcg(ws.xlab + (size_t)k * stride + 1 + (f - k * 2 * g.W)) + off;
        }
        return __ldcg(ws.gnodelab + r);
    };
    // the non-root's position among the tile's non-root border components
    // (K3b's bitmap): its slot in nrlab
    auto slot = [&](int c) -> int {
        return __ldcg(twpre + (c >> 5)) + __popc(__ldcg(tbits + (c >> 5)) & ((1u << (c & 31)) - 1u));
    };
    // the parents and components of 4 nodes per lane are loaded at once
    int par[4], gcv[4];
#pragma unroll
    for (int t = 0; t < 4; t++) {
        const int j = lane + 32 * t;
        par[t] = j < nborder ? __ldcg(ws.gparent + nodebase + j) : nodebase + j;
        gcv[t] = j < nborder ? __ldcg(ws.gnodecomp + nodebase + j) : 0;
    }
#pragma unroll
    for (int t = 0; t < 4; t++) {
        if (par[t] == nodebase + lane + 32 * t) continue;  // a root (or past nborder)
        const int sl = slot(gcv[t] & 0xFFFF);
        const int r = par[t] < 0 ? par[t] : gfind_halve(ws.gparent, par[t]);
        const int32_t lab = root_label(r);
        st_keep(nrlab + sl, lab, keep);
    }
    for (int j = lane + 128; j < nborder; j += 32) {
        const int node = nodebase + j;
        if (__ldcg(ws.gparent + node) == node) continue;
        const int sl = slot(__ldcg(ws.gnodecomp + node) & 0xFFFF);
        const int r = gfind_halve(ws.gparent, node);
        const int32_t lab = root_label(r);
        st_keep(nrlab + sl, lab, keep);
    }
}

__global__ void __launch_bounds__(K4_WARPS * 32)
k_fixup(Geometry g, Workspace ws) {
    pdl_trigger();
    pdl_wait();
    if (ws.xlab && blockIdx.x == 0 && threadIdx.x == 0) {
        // row bands: this band's offset (N of the earlier bands, for K5) and
        // N from the gathered records (N_band first in each)
        int off = 0, tot = 0;
        for (int k = 0; k < ws.xnb; k++) {
            const int c = __ldcg(ws.xlab + (size_t)k * (2 * g.W + 1));
            off += k < ws.xself ? c : 0;
            tot += c;
        }
        *const_cast<int32_t *>(ws.boff) = off;
        if (ws.xntotal) *ws.xntotal = tot;
    }
    const int tile = blockIdx.x * K4_WARPS + (threadIdx.x >> 5);
    if (tile >= g.nT) return;
    fixup_tile(g, ws, tile, lane_id());
}

// ========================================================================= K3
// One CTA per tile row (32 image rows x all tile columns), claimed in raster
// order through a ticket so that a CTA only ever waits on CTAs already running.
// A component is a global root iff it lies inside its tile or its node is a
// root of the global forest after K2 (its key is the component's minimum, i.e.
// its first pixel in raster order).  Components of a tile are numbered in key
// order (K1), so the roots of tile row r are the index range
// [rowfirst[r], rowfirst[r+1]) minus the few border components that are not
// roots.  The root counts of the tile row's segments (row, tile column) are
// scanned in raster order, chained across tile rows with a decoupled
// lookback: flatten's consecutive numbering k++  made
// canonical.  Per tile (one warp) the kernel leaves what K4 and K5 need to
// label any component c = rowfirst[row] + rank of the tile:
//   tbits / twpre  bitmap of the non-root border components + its popcount
//                  prefix (nonroots_before(c) = twpre[c/32] + popc(...));
//   tlb[row]       excl(tile row) + segoff(row, tile) + non-roots in earlier
//                  rows + 1, so a root's label = tlb[row] + rank -
//                  nonroots_before(c);
//   gnodelab       the labels of the tile's root border nodes (K4 reads them
//                  for the components merged into them).
#if CCL_K3_TRACE
// development trace (build knob; scripts/k3_trace.py): per tile row,
// globaltimer at the kernel's entry, after pdl_wait, after phase 1, after
// phase 2, after the lookback barrier and at the end
__device__ unsigned long long g_k3trace[4096][6];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define K3T(ty, i) \
    if (threadIdx.x == 0 && (ty) < 4096) g_k3trace[ty][i] = gtimer()
#else
#define K3T(ty, i) (void)0
#endif
template <int NWN>
struct KNSmem {
    int32_t nrrow[NWN][TH];           // non-root border components per row
    uint32_t bits[NWN][CAPC / 32];    // the warp's tile's non-root bitmap
    int32_t wsum[NWN];
    int32_t part, excl;
};

// NWN warps per tile-row CTA (8; fewer for images of 1-4 tile columns, so
// the idle warps do not hold SM slots: C2 batches of 1024-px-wide images).
template <int NWN>
__global__ void __launch_bounds__(NWN * 32, NWN >= 16 ? 64 / NWN : NWN == 8 ? 6 : 16)
k_number(Geometry g, Workspace ws, int32_t *n_components) {
#if CCL_K3_TRACE
    const unsigned long long t_in = gtimer();
#endif
    pdl_trigger();
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (ws.k1hint_dev) *reinterpret_cast<volatile int32_t *>(ws.k1hint_dev) = __ldcg(ws.k1over_n);
        *ws.k1over_n = 0;  // K1's hand-over list, for the next call
    }
    __shared__ KNSmem<NWN> sm;
    const int lane = lane_id(), w = threadIdx.x >> 5;
    if (threadIdx.x == 0) sm.part = atomicAdd(ws.ticket, 1);
    __syncthreads();
    const int ty = sm.part;
#if CCL_K3_TRACE
    if (threadIdx.x == 0 && ty < 4096) g_k3trace[ty][0] = t_in;
#endif
    K3T(ty, 1);
    const int R0 = tile_r0(g, ty), rows = tile_rows(g, ty);
    const bool first = ty % g.tpi == 0;  // first tile row of its image: numbering starts at 1
    // ---- phase 1: non-root border components of every tile (bitmap, prefix,
    // counts per row) and the root counts of the segments (R0 + r, tx)
    for (int tx = w; tx < g.nTx; tx += NWN) {
        const int tile = ty * g.nTx + tx;
        const int32_t *meta = ws.meta + (int64_t)tile * META;
        const int nodebase = tile * g.capb;
        // every load of the tile at once: the node entries of the first 4*32
        // node slots do not wait for the node count (they lie inside the
        // tile's capb slots either way)
        const int ncomp = __ldcg(meta + META_NCOMP), nborder = __ldcg(meta + META_NBORDER);
        const int rf = __ldcg(meta + META_ROWFIRST + lane);
        const int rfx = __ldcg(meta + META_ROWFIRST + (lane + 1 < TH ? lane + 1 : TH));
        int par[4], gcv[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const int j = lane + 32 * t;
            par[t] = j < g.capb ? __ldcg(ws.gparent + nodebase + j) : nodebase + j;
            gcv[t] = j < g.capb ? __ldcg(ws.gnodecomp + nodebase + j) : 0;
        }
        const int nbw = (ncomp + 31) >> 5;
        int32_t *nrrow = sm.nrrow[w];
        uint32_t *bits = sm.bits[w];
        nrrow[lane] = 0;
        for (int j = lane; j < nbw; j += 32) bits[j] = 0u;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 4; t++)
            if (lane + 32 * t < nborder && par[t] != nodebase + lane + 32 * t) {
                const int c = gcv[t] & 0xFFFF;
                atomicOr(bits + (c >> 5), 1u << (c & 31));
                atomicAdd(nrrow + (gcv[t] >> 16), 1);
            }
        for (int j = lane + 128; j < nborder; j += 32) {
            const int node = nodebase + j;
            if (__ldcg(ws.gparent + node) != node) {
                const int gc = __ldcg(ws.gnodecomp + node), c = gc & 0xFFFF;
                atomicOr(bits + (c >> 5), 1u << (c & 31));
                atomicAdd(nrrow + (gc >> 16), 1);
            }
        }
        __syncwarp();
        const int rfn = lane + 1 < rows ? rfx : ncomp;
        if (lane < rows) ws.segcnt[(int64_t)(R0 + lane) * g.nTx + tx] = rfn - rf - nrrow[lane];
        // the bitmap and its popcount prefix (K4, K5); the non-roots of the
        // earlier rows (lane = row) wait in tlb for phase 3
        uint32_t *tbits = ws.tbits + (int64_t)tile * g.capw;
        int32_t *twpre = ws.twpre + (int64_t)tile * g.capw;
        for (int j0 = 0, acc = 0; j0 < nbw; j0 += 32) {
            const int j = j0 + lane;
            const uint32_t b = j < nbw ? bits[j] : 0u;
            uint32_t tot;
            const int pre = (int)warp_excl_scan(__popc(b), tot);
            if (j < nbw) {
                tbits[j] = b;
                twpre[j] = acc + pre;
            }
            acc += (int)tot;
        }
        uint32_t tot;
        ws.tlb[(int64_t)tile * TH + lane] = (int)warp_excl_scan((uint32_t)nrrow[lane], tot);
        __syncwarp();
    }
    __syncthreads();
    K3T(ty, 2);
    // ---- phase 2: exclusive scan of the tile row's rows*nTx segment counts
    // (raster order), then the lookback over earlier tile rows
    const int64_t sbase = (int64_t)R0 * g.nTx;
    const int nS = rows * g.nTx;
    int carry = 0;
    for (int c0 = 0; c0 < nS; c0 += NWN * 32 * KN_ITEMS) {
        const int i0 = c0 + threadIdx.x * KN_ITEMS;
        int v[KN_ITEMS], sum = 0;
#pragma unroll
        for (int i = 0; i < KN_ITEMS; i++) {
            v[i] = i0 + i < nS ? __ldcg(ws.segcnt + sbase + i0 + i) : 0;
            sum += v[i];
        }
        uint32_t wt;
        const int pre = (int)warp_excl_scan((uint32_t)sum, wt);
        if (lane == 0) sm.wsum[w] = (int)wt;
        __syncthreads();
        int off = 0, all = 0;
#pragma unroll
        for (int i = 0; i < NWN; i++) {
            off += i < w ? sm.wsum[i] : 0;
            all += sm.wsum[i];
        }
        int run = carry + off + pre;
#pragma unroll
        for (int i = 0; i < KN_ITEMS; i++) {
            if (i0 + i < nS) ws.segoff[sbase + i0 + i] = run;
            run += v[i];
        }
        carry += all;
        __syncthreads();  // wsum reuse
    }
    K3T(ty, 3);
    // descriptor: bits 62-63 status (1 aggregate, 2 inclusive prefix), low 32
    // bits value.  Warp 0 looks back over 32 predecessors at a time.
    if (w == 0) {
        if (lane == 0)
            atomicExch(ws.scanstate + ty, ((first ? 2ull : 1ull) << 62) | (uint32_t)carry);
        int excl = 0;
        if (!first) {
            const volatile unsigned long long *st = ws.scanstate;
            int j = ty - 1;
            while (true) {
                const int idx = j - lane;
                const unsigned long long d = idx >= 0 ? st[idx] : (2ull << 62);
                const unsigned s2 = (unsigned)(d >> 62);
                const uint32_t incl = __ballot_sync(FULL, s2 == 2), zero = __ballot_sync(FULL, s2 == 0);
                const int first = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive prefix
                const uint32_t need = (2u << first) - 1u;         // lanes 0..first
                if (zero & need) {                                // not all published yet: spin
#if CCL_K3_BACKOFF
                    __nanosleep(CCL_K3_BACKOFF);
#endif
                    continue;
                }
                int v = lane <= first ? (int)(uint32_t)d : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
                excl += v;
                if (incl) break;
                j -= 32;
            }
            if (lane == 0) {
                __threadfence();
                atomicExch(ws.scanstate + ty, (2ull << 62) | (uint32_t)(excl + carry));
            }
        }
        if (lane == 0) {
            sm.excl = excl;
            if (ty % g.tpi == g.tpi - 1) n_components[ty / g.tpi] = excl + carry;
        }
    }
    __syncthreads();
    // ---- phase 3: label bases of every tile row segment and the labels of
    // the root border nodes (offset(segment) + rank in segment + 1)
    K3T(ty, 4);
    const int excl = sm.excl;
    for (int tx = w; tx < g.nTx; tx += NWN) {
        const int tile = ty * g.nTx + tx;
        const int32_t *meta = ws.meta + (int64_t)tile * META;
        const int nodebase = tile * g.capb;
        const int nborder = __ldcg(meta + META_NBORDER);
        const int rf = __ldcg(meta + META_ROWFIRST + lane);
        // (segoff, tlb, tbits and twpre were stored by this CTA in phases 1-2:
        // plain loads after the barrier, not L1-bypassing ones)
        const int so = lane < rows ? ws.segoff[(int64_t)(R0 + lane) * g.nTx + tx] : 0;
        int32_t *tlb = ws.tlb + (int64_t)tile * TH;
        const int lb = excl + so + tlb[lane] + 1;
        tlb[lane] = lb;
        const uint32_t *tbits = ws.tbits + (int64_t)tile * g.capw;
        const int32_t *twpre = ws.twpre + (int64_t)tile * g.capw;
        for (int j0 = 0; j0 < nborder; j0 += 32) {  // warp-uniform: the shuffles need every lane
            const int node = nodebase + j0 + lane;
            const bool valid = j0 + lane < nborder;
            const bool root = valid && __ldcg(ws.gparent + node) == node;
            const int gc = valid ? __ldcg(ws.gnodecomp + node) : 0, c = gc & 0xFFFF, row = gc >> 16;
            const int rfr = __shfl_sync(FULL, rf, row), lbr = __shfl_sync(FULL, lb, row);
            if (root) {
                const int nrb =
                    twpre[c >> 5] + __popc(tbits[c >> 5] & ((1u << (c & 31)) - 1u));
                ws.gnodelab[node] = lbr + (c - rfr) - nrb;
            }
        }
    }
    if (threadIdx.x == 0) ws.rowexcl[ty] = excl;
#if CCL_K3_TRACE
    __syncthreads();
    K3T(ty, 5);
#endif
}
#if CCL_K3_TRACE
extern "C" int ccl_debug_k3trace(unsigned long long *host, int rows) {
    return (int)cudaMemcpyFromSymbol(host, g_k3trace, (size_t)rows * 6 * sizeof(unsigned long long));
}
#endif

// ============================================================ small images
// K2 + K3 + K4 in ONE CTA for images of one tile column and at most 32 tile
// rows (W <= 1024, H <= 1024: the paper's <= 1 MB regime, PAPER.md:1172-
// 1177).  Every border node's parent lives in shared memory, so the tile-edge
// unions, the flatten, the numbering (one block scan over the image rows; no
// lookback) and the non-root labels cost shared-memory latency instead of a
// chain of five global-memory kernels.  With one tile column the node index
// order IS the raster key order (tiles stacked vertically, nodes of a tile in
// raster order), so the union links by index.  Outputs are those of K2-K4:
// tbits / twpre / tlb / gnodelab / nrlab and N.
constexpr int SMALL_MAX_TILES = 32;  // one warp per tile
constexpr int SMALL_MAX_ROWS = 1024; // one thread per image row in the scan
constexpr int SMALL_THREADS = 1024;
__device__ __forceinline__ int sfind(volatile int32_t *par, int x) {
    while (true) {
        const int px = par[x];
        if (px == x) return x;
        const int ppx = par[px];
        if (ppx == px) return px;
        par[x] = ppx;  // path halving: an ancestor
        x = ppx;
    }
}
__device__ __forceinline__ void sunion(int32_t *par, int a, int b) {
    volatile int32_t *vp = par;
    a = sfind(vp, a);
    b = sfind(vp, b);
    while (a != b) {
        if (a < b) { const int t = a; a = b; b = t; }
        const int o = atomicCAS(par + a, a, b);  // link the larger root under the smaller (see union_smem)
        if (o == a) return;
        a = sfind(vp, o);
        b = sfind(vp, b);
    }
}
__global__ void __launch_bounds__(SMALL_THREADS, 1)
k_small_middle(Geometry g, Workspace ws, int32_t *n_components) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ int32_t s_seg[SMALL_MAX_ROWS];       // root count per image row, then its exclusive prefix
    __shared__ int32_t s_nrp[SMALL_MAX_TILES][TH];  // non-roots in earlier rows of the tile
    __shared__ int32_t s_wsum[SMALL_THREADS / 32];
    __shared__ uint32_t s_hx[SMALL_MAX_TILES][2][WPR], s_hb[SMALL_MAX_TILES][2][WPR];
    int32_t *par = reinterpret_cast<int32_t *>(smem_raw);  // nT * capb node parents
    // per warp CAPC / 32 words after them: an edge's unions (upper | lower run
    // ordinal << 16), later the tile's non-root bitmap
    uint32_t(*s_pl)[CAPC / 32] = reinterpret_cast<uint32_t(*)[CAPC / 32]>(smem_raw + (size_t)g.nT * g.capb * 4);
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int nT = g.nT, capb = g.capb;
    if (threadIdx.x == 0) *ws.k1over_n = 0;  // K1's hand-over list, for the next call
    // per tile (warp w = tile w): its counts and row offsets, the first
    // SMALL_NODES_REG border nodes' (row, component) in registers (lane + 32 t),
    // and the parents of its border nodes (only those are ever read) in
    // shared memory -- all loads of the warp in flight together
    constexpr int NR = 8;  // 256 nodes in registers
    const int tile = w, nodebase = w * capb;
    const int32_t *meta = ws.meta + (int64_t)tile * META;
    const int nborder = w < nT ? __ldcg(meta + META_NBORDER) : 0;
    const int ncomp = w < nT ? __ldcg(meta + META_NCOMP) : 0;
    const int rf = w < nT ? __ldcg(meta + META_ROWFIRST + lane) : 0;
    const int rfx = w < nT ? __ldcg(meta + META_ROWFIRST + (lane + 1 < TH ? lane + 1 : TH)) : 0;
    int gcv[NR];
#pragma unroll
    for (int t = 0; t < NR; t++) {
        const int j = 32 * t + lane;
        gcv[t] = j < min(nborder, capb) && w < nT ? __ldcg(ws.gnodecomp + nodebase + j) : 0;
    }
    if (w < nT) {
        for (int j0 = 0; j0 < nborder; j0 += 128) {
            int v[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int j = j0 + 32 * t + lane;
                v[t] = j < nborder ? __ldcg(ws.gparent + nodebase + j) : 0;
            }
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int j = j0 + 32 * t + lane;
                if (j < nborder) par[nodebase + j] = v[t];
            }
        }
    }
    __syncthreads();
    // ---- K2: the horizontal tile edges (one tile column: no vertical ones),
    // the same two edge families as k_border; unions straight in shared memory
    if (w >= 1 && w < nT) {
        const int ty = w;
        const uint32_t u = __ldcg(ws.edgerow + ((int64_t)(ty - 1) * 2 + 1) * WPR + lane);
        const uint32_t x = __ldcg(ws.edgerow + (int64_t)ty * 2 * WPR + lane);
        RowView U = make_row(u), X = make_row(x);
        s_hx[w][0][lane] = U.hx; s_hb[w][0][lane] = U.base;
        s_hx[w][1][lane] = X.hx; s_hb[w][1][lane] = X.base;
        __syncwarp();
        const int32_t *bot = ws.botnode + (int64_t)(ty - 1) * g.maxrun;
        const int32_t *top = ws.topnode + (int64_t)ty * g.maxrun;
        // listed first (consecutive positions per lane by a warp scan), then
        // in windows of 128: all node loads of a window in flight, then the
        // shared-memory unions
        const uint32_t m1 = first_in_run(x & dilate(U), x);
        uint32_t m2;
        {
            const uint32_t t = x & dilate(U);
            const uint32_t sm_ = smear_up(t, x);
            const uint32_t cin = carry_in_fwd(((x >> 31) & (sm_ >> 31)) != 0, x == FULL) & x & 1u;
            m2 = upper_merge_heads(U.hx, u, U.xp, x, X.xp, sm_ | (cin ? (x & ~(x + 1)) : 0u));
        }
        uint32_t tot;
        const int base = (int)warp_excl_scan(__popc(m1) + __popc(m2), tot);
        uint32_t *pl = s_pl[w];
        for (int w0 = 0; w0 < (int)tot; w0 += 128) {
            int idx = base - w0;
            for (uint32_t m = m1; m && idx < 128; m &= m - 1, idx++) {
                if (idx < 0) continue;
                const int b = __ffs(m) - 1;
                const int q = 32 * lane + b + leftmost3(u, U.xp, U.xn, b), lq = q >> 5;
                pl[idx] = (uint32_t)run_ord(s_hx[w][0][lq], s_hb[w][0][lq], q & 31) |
                          ((uint32_t)run_ord(X.hx, X.base, b) << 16);
            }
            for (uint32_t m = m2; m && idx < 128; m &= m - 1, idx++) {
                if (idx < 0) continue;
                const int b = __ffs(m) - 1;
                const int q = 32 * lane + b - 1, lq = q >> 5;  // lower pixel h-1
                pl[idx] = (uint32_t)run_ord(U.hx, U.base, b) |
                          ((uint32_t)run_ord(s_hx[w][1][lq], s_hb[w][1][lq], q & 31) << 16);
            }
            __syncwarp();
            const int np = min(128, (int)tot - w0);
            int na[4], nbn[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int i = 32 * t + lane;
                const uint32_t e = i < np ? pl[i] : 0u;
                na[t] = i < np ? __ldcg(bot + (e & 0xFFFFu)) : 0;
                nbn[t] = i < np ? __ldcg(top + (e >> 16)) : 0;
            }
#pragma unroll
            for (int t = 0; t < 4; t++)
                if (32 * t + lane < np) sunion(par, na[t], nbn[t]);
            __syncwarp();
        }
    }
    __syncthreads();
    // (no flatten: the root test needs no more than par[x] == x, and K4
    // below walks each non-root up to its root, read-only)
    // ---- K3 phase 1, one warp per tile: the non-root bitmap + prefix, the
    // non-roots per row and the root count of every row.  The first
    // SMALL_NODES_REG border nodes of the tile are held in registers (lane +
    // 32 t), and so are the first 32 bitmap words and their prefix (lane =
    // word): the phases below run on shuffles, with a handful of batched
    // global round trips (larger tiles take the global fallback).
    const int rows_t = w < nT ? tile_rows(g, w) : 0;
    bool nonr[NR];
#pragma unroll
    for (int t = 0; t < NR; t++) {
        const int j = 32 * t + lane;
        nonr[t] = j < nborder && par[nodebase + j] != nodebase + j;
    }
    const int nbw = (ncomp + 31) >> 5;
    uint32_t *tbits = ws.tbits + (int64_t)tile * g.capw;
    int32_t *twpre = ws.twpre + (int64_t)tile * g.capw;
    uint32_t *bits = s_pl[w];  // (the edge list is done): the tile's non-root bitmap
    int32_t *nrow = s_nrp[w];
    uint32_t bw = 0u;  // bitmap word `lane`
    int wp = 0;        // its exclusive popcount prefix
    if (w < nT) {
        for (int j = lane; j < nbw; j += 32) bits[j] = 0u;
        nrow[lane] = 0;
        __syncwarp();
        auto mark = [&](int gc) {
            const int c = gc & 0xFFFF;
            atomicOr(bits + (c >> 5), 1u << (c & 31));
            atomicAdd(nrow + (gc >> 16), 1);
        };
#pragma unroll
        for (int t = 0; t < NR; t++)
            if (nonr[t]) mark(gcv[t]);
        for (int j = 32 * NR + lane; j < nborder; j += 32)
            if (par[nodebase + j] != nodebase + j) mark(__ldcg(ws.gnodecomp + nodebase + j));
        __syncwarp();
        for (int j0 = 0, acc = 0; j0 < nbw; j0 += 32) {
            const int j = j0 + lane;
            const uint32_t bb = j < nbw ? bits[j] : 0u;
            uint32_t tot;
            const int pre = (int)warp_excl_scan(__popc(bb), tot);
            if (j < nbw) {
                tbits[j] = bb;
                twpre[j] = acc + pre;
            }
            if (j0 == 0) {
                bw = bb;
                wp = pre;
            }
            acc += (int)tot;
        }
        const int nr = nrow[lane];
        uint32_t tot;
        nrow[lane] = (int)warp_excl_scan((uint32_t)nr, tot);  // non-roots in earlier rows
        const int rfn = lane + 1 < rows_t ? rfx : ncomp;
        if (lane < rows_t) s_seg[tile * TH + lane] = rfn - rf - nr;
    }
    __syncthreads();
    // ---- K3 phase 2: exclusive scan of the row counts over the whole image
    {
        const int v = (int)threadIdx.x < g.H ? s_seg[threadIdx.x] : 0;
        uint32_t wt;
        const int pre = (int)warp_excl_scan((uint32_t)v, wt);
        if (lane == 0) s_wsum[w] = (int)wt;
        __syncthreads();
        int off = 0, all = 0;
        for (int i = 0; i < SMALL_THREADS / 32; i++) {
            off += i < w ? s_wsum[i] : 0;
            all += s_wsum[i];
        }
        __syncthreads();
        if ((int)threadIdx.x < g.H) s_seg[threadIdx.x] = off + pre;
        if (threadIdx.x == 0) n_components[0] = all;
    }
    __syncthreads();
    // non-roots before component c of this warp's tile (bitmap word + prefix;
    // past the 32 lane-held words, from the shared bitmap)
    const int pre32 = __shfl_sync(FULL, wp + __popc(bw), 31);  // non-roots in words 0..31
    auto nonroots_before = [&](int c) -> int {  // every lane calls it (shuffles)
        const int wd = c >> 5;
        uint32_t x = __shfl_sync(FULL, bw, wd & 31);
        int pre = __shfl_sync(FULL, wp, wd & 31);
        if (wd >= 32) {  // more than 1024 components in the tile (rare)
            x = bits[wd];
            pre = pre32;
            for (int k = 32; k < wd; k++) pre += __popc(bits[k]);
        }
        return pre + __popc(x & ((1u << (c & 31)) - 1u));
    };
    // ---- K3 phase 3: label bases of the tile rows and the root nodes' labels
    const int lb = (lane < rows_t ? s_seg[tile * TH + lane] : 0) + (w < nT ? nrow[lane] : 0) + 1;
    if (w < nT) {
        ws.tlb[(int64_t)tile * TH + lane] = lb;
#pragma unroll
        for (int t = 0; t < NR; t++) {
            if (32 * t >= nborder) break;  // warp-uniform
            const int c = gcv[t] & 0xFFFF, row = gcv[t] >> 16;
            const int rfr = __shfl_sync(FULL, rf, row), lbr = __shfl_sync(FULL, lb, row);
            const int nb = nonroots_before(c);
            const int j = 32 * t + lane;
            if (j < nborder && !nonr[t]) par[nodebase + j] = ~(lbr + (c - rfr) - nb);  // a root: ~label
        }
        for (int j0 = 32 * NR; j0 < nborder; j0 += 32) {
            const int j = j0 + lane;
            const bool root = j < nborder && par[nodebase + j] == nodebase + j;
            const int gc = j < nborder ? __ldcg(ws.gnodecomp + nodebase + j) : 0, c = gc & 0xFFFF;
            const int rfr = __shfl_sync(FULL, rf, gc >> 16), lbr = __shfl_sync(FULL, lb, gc >> 16);
            const int nb = nonroots_before(c);
            if (root) par[nodebase + j] = ~(lbr + (c - rfr) - nb);
        }
    }
    __syncthreads();
    // ---- K4: every non-root border component takes its root's label, at its
    // slot among the tile's non-roots
    if (w < nT) {
        int32_t *nrlab = ws.nrlab + (int64_t)tile * g.capc;
        // a root holds ~label (< 0) since phase 3, every other node a parent
        // (>= 0): walk read-only up to the root (no store may leave a node
        // pointing below its root -- see DESIGN.md "Small images")
        auto root_label = [&](int y) -> int {
            while (true) {
                const int v = reinterpret_cast<volatile int32_t *>(par)[y];
                if (v < 0) return ~v;
                y = v;
            }
        };
        int lab[NR];
#pragma unroll
        for (int t = 0; t < NR; t++) lab[t] = nonr[t] ? root_label(par[nodebase + 32 * t + lane]) : 0;
#pragma unroll
        for (int t = 0; t < NR; t++) {
            if (32 * t >= nborder) break;  // warp-uniform
            const int sl = nonroots_before(gcv[t] & 0xFFFF);
            if (nonr[t]) nrlab[sl] = lab[t];
        }
        for (int j0 = 32 * NR; j0 < nborder; j0 += 32) {
            const int j = j0 + lane;
            const int pj = j < nborder ? par[nodebase + j] : 0;
            const bool nonroot = j < nborder && pj >= 0;  // (roots hold ~label < 0)
            const int c = j < nborder ? __ldcg(ws.gnodecomp + nodebase + j) & 0xFFFF : 0;
            const int sl = nonroots_before(c);
            if (nonroot) nrlab[sl] = root_label(pj);
        }
    }
}

// The small-image path (k_small_middle): one image (no batch, no row band),
// one tile column, at most 32 tile rows, every border node in shared memory.
constexpr size_t SMALL_SMEM_MAX = 190 * 1024;  // dynamic; + ≈ 25 KB static < 227 KB
static size_t small_smem(const Geometry &g) {
    return (size_t)g.nT * g.capb * sizeof(int32_t) + (size_t)SMALL_MAX_TILES * (CAPC / 32) * sizeof(uint32_t);
}
extern int g_no_small;
static bool small_mode(const Geometry &g) {
    return !g_no_small && g.tpi == g.nTy && g.nTx == 1 && g.nT <= SMALL_MAX_TILES && g.H <= SMALL_MAX_ROWS &&
           small_smem(g) <= SMALL_SMEM_MAX;
}

// ========================================================================= K5
// Labeling phase: one warp per 1024-px row segment.  Lane
// j writes pixels 256c + 8j .. +7 (c = 0..3), so every 32-byte store of the
// warp is one contiguous 1 KB stretch of the output row (rows not 32-byte
// aligned: pixels 128c + 4j .. +3 with 16-byte stores).
#ifndef CCL_K5_WARPS
#define CCL_K5_WARPS 8
#endif
constexpr int K5_WARPS = CCL_K5_WARPS;  // 8 CTAs/SM; measured vs 4 and 16 (C4 step -6 us vs 16 since the 256-bit stores)
// (x & bit) ? v : 0
__device__ __forceinline__ int sel_bit(uint32_t x, uint32_t bit, int v) {
    int r;
    asm("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %1, 0;\n\tselp.b32 %0, %2, 0, p;\n\t}"
        : "=r"(r) : "r"(x & bit), "r"(v));
    return r;
}
__global__ void __launch_bounds__(K5_WARPS * 32, 64 / K5_WARPS)
k_write(Geometry g, Workspace ws, int32_t *__restrict__ labels, uint32_t magic, int mshift) {
    pdl_trigger();
    pdl_wait();
    // s_lab[w][1 + k] = final label of run k of warp w's row (entry 0 and the
    // two after the last run are read for pixels they do not label)
    __shared__ int32_t s_lab[K5_WARPS][MAXRUN + 4];
    __shared__ uint4 s_word[K5_WARPS][32];  // (foreground, run heads, runs before) of each lane-word
    const int lane = lane_id(), wi = threadIdx.x >> 5;
    // warp = one row segment; consecutive warps and CTAs take consecutive
    // segments in raster order, so the stores in flight cover one contiguous
    // stretch of the label image
    const uint32_t seg = blockIdx.x * K5_WARPS + wi;  // (row, tile column); nseg < 2^31
    if (seg >= (uint32_t)g.nseg) return;
    // seg / nTx by the host's magic multiplier (exact for seg < 2^31; m = 0: nTx = 1)
    const int row = magic ? (int)(__umulhi(seg, magic) >> mshift) : (int)seg;
    const int tx = (int)(seg - (uint32_t)row * (uint32_t)g.nTx);
    const int ty = row_tile(g, row);
    const int C0 = tx * TW, tile = ty * g.nTx + tx;
    const int vcols = min(TW, g.W - C0);
    const int gword = tx * WPR + lane;
    const uint16_t *rc = ws.runcomp + (int64_t)seg * g.maxrun;
    const int32_t off = ws.boff ? __ldcg(ws.boff) : 0;  // labels of earlier row bands
    // the first 32 run entries are loaded beside the masks (most rows have
    // fewer runs), and so are the tile's tables, one entry per lane: row
    // offsets and label bases (lane = tile row), the non-root bitmap and its
    // prefix (lane = word), the first 64 non-root labels (lane = slot).  All
    // independent: the labels below are computed with shuffles, no
    // dependent gather.
    const uint32_t rc0 = lane < g.maxrun ? (uint32_t)__ldcs(rc + lane) : 0u;
    const int rfv = __ldcg(ws.meta + (int64_t)tile * META + META_ROWFIRST + lane);
    const int lbv = __ldcg(ws.tlb + (int64_t)tile * TH + lane);
    const uint32_t *tbits = ws.tbits + (int64_t)tile * g.capw;
    const int32_t *twpre = ws.twpre + (int64_t)tile * g.capw;
    const int32_t *nrlab = ws.nrlab + (int64_t)tile * g.capc;
    const uint32_t bwv = lane < g.capw ? __ldcg(tbits + lane) : 0u;
    const int wpv = lane < g.capw ? __ldcg(twpre + lane) : 0;
    const int nlv = lane < g.capc ? __ldcg(nrlab + lane) : 0;
    const int nlv2 = lane + 32 < g.capc ? __ldcg(nrlab + 32 + lane) : 0;
    uint32_t x;                                          // foreground
    const uint32_t f = run_mask(g, ws.bm, row, gword, row - tile_r0(g, ty), tile_rows(g, ty), &x);  // runs
    const uint32_t fl = __shfl_up_sync(FULL, f, 1);
    const uint32_t hx = f & ~((f << 1) | (lane == 0 ? 0u : (fl >> 31)));
    uint32_t nr;
    const uint32_t base = warp_excl_scan(__popc(hx), nr);
    int32_t *rowlab = s_lab[wi] + 1;
    {
        // label of run entry v = (root row, rank): component c = rowfirst[row]
        // + rank; a non-root border component takes its slot's label (K4),
        // any other component tlb[row] + rank - (non-roots before c) (K3b).
        // Every lane runs the shuffles (entries past the row are harmless).
        auto run_label = [&](uint32_t v) -> int {
            const int row = (int)(v >> 9) & 31, rank = (int)(v & 0x1FFu);
            // (clamped: an entry past the row's runs is stale workspace and
            // decodes to anything; its label is never stored, but its loads
            // must stay inside the tile's tables)
            const int c = min(__shfl_sync(FULL, rfv, row) + rank, g.capc - 1), wd = c >> 5;
            uint32_t w = __shfl_sync(FULL, bwv, wd & 31);
            int pre = __shfl_sync(FULL, wpv, wd & 31);
            if (__any_sync(FULL, wd >= 32)) {  // warp-uniform: more than 1024 components in the tile
                if (wd >= 32) {
                    w = __ldcg(tbits + wd);
                    pre = __ldcg(twpre + wd);
                }
            }
            const int nb = pre + __popc(w & ((1u << (c & 31)) - 1u));
            const int lb = __shfl_sync(FULL, lbv, row);
            const bool nonroot = (w >> (c & 31)) & 1u;
            int lab = lb + rank - nb;
            if (__any_sync(FULL, nonroot)) {  // warp-uniform: most chunks have no merged border component
                const int nla = __shfl_sync(FULL, nlv, nb & 31), nlb = __shfl_sync(FULL, nlv2, nb & 31);
                if (nonroot) lab = nb < 32 ? nla : nlb;
                if (__any_sync(FULL, nonroot && nb >= 64))  // warp-uniform: more than 64 non-roots
                    if (nonroot && nb >= 64) lab = __ldcg(nrlab + min((uint32_t)nb, (uint32_t)g.capc - 1u));
            }
            return lab + off;
        };
        // (entries past the row's runs are decoded too -- clamped, see
        // run_label -- so the shuffles do not wait for the run count)
        const int l0 = run_label(rc0);
        if (lane < (int)nr) rowlab[lane] = l0;
#pragma unroll 1
        for (int k0 = 32; k0 < (int)nr; k0 += 32) {  // warp-uniform: the shuffles need every lane
            const int k = k0 + lane;
            const int l = run_label(k < (int)nr ? (uint32_t)__ldcs(rc + k) : 0u);
            if (k < (int)nr) rowlab[k] = l;
        }
    }
    s_word[wi][lane] = make_uint4(x, hx, base, 0u);
    __syncwarp();
    int32_t *out = labels + (int64_t)row * g.W + C0;
    uint64_t pol_first;  // labels are not read again: evict first (bm, runcomp stay in L2)
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    // labels of 4 pixels b..b+3 of lane-word t.  Heads of the run mask are
    // never adjacent, so pixels b+1..b+3 lie in the run of pixel b or one of
    // the next two: three independent shared loads and selects
    auto quad_at = [&](const uint4 &t, int b, uint32_t mb, int &v0, int &v1, int &v2, int &v3) {
        const uint32_t nib = t.x >> b, hn = t.y >> b;
        const int32_t *rp = rowlab + ((int)t.z + __popc(t.y & mb) - 1);  // run containing (or before) pixel b
        const int l0 = rp[0], l1 = rp[1], l2 = rp[2];
        const int a1 = (hn & 2u) ? l1 : l0;
        const int a2 = (hn & 6u) ? l1 : l0;
        const int a3 = (hn & 8u) ? ((hn & 2u) ? l2 : l1) : a2;
        // (a predicate test + select per pixel: two instructions; the plain
        // `? l : 0` compiles to a three-instruction sign mask)
        v0 = sel_bit(nib, 1u, l0);
        v1 = sel_bit(nib, 2u, a1);
        v2 = sel_bit(nib, 4u, a2);
        v3 = sel_bit(nib, 8u, a3);
    };
    if (g.aligned && vcols == TW && ((reinterpret_cast<uintptr_t>(out) & 31u) == 0)) {
        // interior segment: four full 1024-byte warp stores (256-bit per
        // lane: pixels 256c + 8*lane .. +7, two quads of lane-word 8c + lane/4)
        const int b8 = 8 * (lane & 3);
        const uint32_t mA = upto(b8), mB = upto(b8 + 4);
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const uint4 t = s_word[wi][8 * c + (lane >> 2)];
            int v0, v1, v2, v3, v4, v5, v6, v7;
            quad_at(t, b8, mA, v0, v1, v2, v3);
            quad_at(t, b8 + 4, mB, v4, v5, v6, v7);
            asm volatile("st.global.L2::cache_hint.v8.s32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;"
                         ::"l"(out + 256 * c + 8 * lane), "r"(v0), "r"(v1), "r"(v2), "r"(v3),
                         "r"(v4), "r"(v5), "r"(v6), "r"(v7), "l"(pol_first) : "memory");
        }
        return;
    }
    const int b0 = 4 * (lane & 7);  // lane's 4 pixels inside lane-word 4c + lane/8
    const uint32_t m0 = upto(b0);
    auto quad = [&](int c, int &v0, int &v1, int &v2, int &v3) {
        quad_at(s_word[wi][4 * c + (lane >> 3)], b0, m0, v0, v1, v2, v3);
    };
#pragma unroll 1
    for (int c = 0; c < 8; c++) {
        const int P = 128 * c + 4 * lane;
        if (128 * c >= vcols) break;
        int v0, v1, v2, v3;
        quad(c, v0, v1, v2, v3);
        if (g.aligned) {
            if (P < vcols) *reinterpret_cast<int4 *>(out + P) = make_int4(v0, v1, v2, v3);
        } else {
            if (P < vcols) __stcs(out + P, v0);
            if (P + 1 < vcols) __stcs(out + P + 1, v1);
            if (P + 2 < vcols) __stcs(out + P + 2, v2);
            if (P + 3 < vcols) __stcs(out + P + 3, v3);
        }
    }
}

// ================================================================ row bands
// Per pixel of a local row: the key and node of its component's root in the
// band's forest (after k_border).  One warp per 1024-px row segment.
__global__ void __launch_bounds__(256)
k_band_rows(Geometry g, Workspace ws, int64_t *keys, int32_t *nodes, unsigned long long *noderep, uint32_t epoch) {
    pdl_trigger();
    pdl_wait();
    __shared__ int32_t s_node[4][MAXRUN];
    __shared__ int64_t s_key[4][MAXRUN];
    const int lane = lane_id(), wi = threadIdx.x >> 5;
    const int seg = blockIdx.x * 4 + wi;  // the band's first row, then its last
    if (seg >= 2 * g.nTx) return;
    const int side = seg / g.nTx, tx = seg % g.nTx;
    const int row = side ? g.H - 1 : 0;
    keys += side * g.W;
    nodes += side * g.W;
    const int ty = row_tile(g, row);
    const int C0 = tx * TW, tile = ty * g.nTx + tx;
    const int gword = tx * WPR + lane;
    uint32_t x;
    const uint32_t f = run_mask(g, ws.bm, row, gword, row - tile_r0(g, ty), tile_rows(g, ty), &x);
    const uint32_t fl = __shfl_up_sync(FULL, f, 1);
    const uint32_t hx = f & ~((f << 1) | (lane == 0 ? 0u : (fl >> 31)));
    uint32_t nr;
    const uint32_t base = warp_excl_scan(__popc(hx), nr);
    const uint16_t *rc = ws.runcomp + ((int64_t)row * g.nTx + tx) * g.maxrun;
    const int32_t *compnode = ws.compnode + (int64_t)tile * g.capc;
    const int32_t *rowfirst = ws.meta + (int64_t)tile * META + META_ROWFIRST;
    // root node and key once per run, two runs per lane in flight together
    // (the chain rc -> rowfirst -> compnode -> parents -> key is all latency)
    for (int k = lane; k < (int)nr; k += 64) {
        const int k2 = k + 32;
        const bool two = k2 < (int)nr;
        const uint32_t v = rc[k], v2 = two ? rc[k2] : 0u;  // (root row << 9) | rank
        const int f = rowfirst[v >> 9], f2 = two ? rowfirst[v2 >> 9] : 0;
        int x = compnode[f + (int)(v & 0x1FFu)], x2 = two ? compnode[f2 + (int)(v2 & 0x1FFu)] : -1;
        // read-only finds in lockstep (a negative parent: a foreign root, terminal)
        bool a1 = x >= 0, a2 = two && x2 >= 0;
        while (a1 || a2) {
            const int p1 = a1 ? __ldcg(ws.gparent + x) : 0, p2 = a2 ? __ldcg(ws.gparent + x2) : 0;
            if (a1) {
                if (p1 == x || p1 < 0) { a1 = false; x = p1 == x ? x : p1; } else x = p1;
            }
            if (a2) {
                if (p2 == x2 || p2 < 0) { a2 = false; x2 = p2 == x2 ? x2 : p2; } else x2 = p2;
            }
        }
        const int64_t key = ws.gkey[x], key2 = two ? ws.gkey[x2] : 0;
        s_node[wi][k] = x;
        s_key[wi][k] = key;
        if (two) {
            s_node[wi][k2] = x2;
            s_key[wi][k2] = key2;
        }
    }
    __syncwarp();
    // ... then per pixel, lane = pixel within each 32-pixel word (coalesced)
    for (int c = 0; c < WPR; c++) {
        const uint32_t xw = __shfl_sync(FULL, x, c), hw = __shfl_sync(FULL, hx, c), bw = __shfl_sync(FULL, base, c);
        const int col = C0 + 32 * c + lane;
        if (col >= g.W) continue;
        const bool fg = (xw >> lane) & 1u;
        const int ord = (int)bw + __popc(hw & upto(lane)) - 1;
        keys[col] = fg ? s_key[wi][ord] : -1;
        nodes[col] = fg ? s_node[wi][ord] : -1;
        // the representative slot of every band-local root node (its first
        // slot: the minimum over the heads of its runs), see k_xb_rep2
        if (fg && ((hw >> lane) & 1u))
            atomicMin(noderep + s_node[wi][ord],
                      ((unsigned long long)(0xFFFFFFFFu - epoch) << 32) | (uint32_t)(side * g.W + col));
    }
}

// ------------------------------------------------------------ cross-band step
// Boundary slots: band k's first row then its last row, W slots each, at
// k*2W.  Every rank holds the keys of all bands' slots (all-gathered) and
// resolves the cross-band classes itself, identically: a union-find over the
// slots, joining the slots of one band-local component (via a representative
// slot) and 8-adjacent pixels across each band boundary, linking the root
// with the larger key under the smaller, so a class's root is its first pixel
// in raster order (PARemSP's boundary merge).

// Representative slot of every boundary slot of this band: the first slot
// whose pixel has the same band-local root node (k_band_rows takes the
// atomicMin over the run heads).  noderep entries carry the call's epoch in
// their high word (stored complemented, so a newer call's entries are
// smaller and win atomicMin): the scratch never needs clearing.
// (also starts the slot union-find: every slot in [lo, hi) its own root)
__global__ void k_xb_rep2(const int32_t *nodes, int n, const unsigned long long *noderep, int32_t *rep,
                          int32_t *spar, int lo, int hi) {
    pdl_trigger();
    pdl_wait();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n) rep[s] = nodes[s] >= 0 ? (int32_t)(uint32_t)__ldcg(noderep + nodes[s]) : -1;
    if (lo + s < hi) spar[lo + s] = lo + s;
}
__global__ void k_xb_union(int nb, int W, const int64_t *keys, const int32_t *reps, int32_t *spar) {
    pdl_trigger();
    pdl_wait();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nb * 2 * W || keys[t] < 0) return;
    const int k = t / (2 * W), s = t % (2 * W);
    const int r = reps[t];
    if (r >= 0 && r != s) gunion(spar, keys, t, k * 2 * W + r);
    if (s >= W && k + 1 < nb) {  // last row of band k against the first row of band k+1
        const int c = s - W;
        for (int dc = -1; dc <= 1; dc++) {
            const int cc = c + dc, t2 = (k + 1) * 2 * W + cc;
            if (cc >= 0 && cc < W && keys[t2] >= 0) gunion(spar, keys, t, t2);
        }
    }
}
// This band's components whose class starts elsewhere are linked to it: to
// the other component's node in this band, or to a foreign slot (-2-slot)
// whose label arrives with the exported labels.
__global__ void k_xb_apply(int W, int self, const int64_t *keys, const int32_t *spar, const int32_t *nodes,
                           int32_t *gparent) {
    pdl_trigger();
    pdl_wait();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = self * 2 * W + s;
    if (s >= 2 * W || keys[t] < 0) return;
    int r = t;
    while (spar[r] != r) r = spar[r];
    if (keys[r] == keys[t]) return;  // the class starts with this component
    gparent[nodes[s]] = r / (2 * W) == self ? nodes[r - self * 2 * W] : -2 - r;
}
// Band-local label of the root of every boundary slot of this band (-1: not
// a root after the cross-band links), written into the band's record of the
// gathered table (N_band is its entry 0, K3's output): one all-gather then
// carries both, and every rank adds the band offsets itself.
__global__ void k_band_export(Geometry g, Workspace ws, const int32_t *nodes, int32_t *out, int n) {
    pdl_trigger();
    pdl_wait();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int v = nodes[s];
    out[s] = (v >= 0 && __ldcg(ws.gparent + v) == v) ? __ldcg(ws.gnodelab + v) : -1;
}

// ==================================================================== host
static bool g_attr_done = false;
int g_k1_stop = 99, g_k1_exper = 0;
int g_no_small = 0, g_no_wide = 0;  // development knobs: force the general middle / the 8-warp K1  // development knob: truncate K1 after a phase (timing only)


// Launch with programmatic stream serialization (see pdl_wait / pdl_trigger).
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// The same with a 2-D grid.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl2(void (*kern)(KArgs...), dim3 grid, unsigned block, size_t smem, cudaStream_t stream,
                               Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

static int g_k1_resident = 0;
static int g_sms = 148;  // K1 CTAs resident on the device at once (L2 prefetch distance)
static int g_k1big_resident = 0;
static cudaError_t set_attrs() {
    if (g_attr_done) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    for (auto k : {k_tile_local<false, false>, k_tile_local<true, false>, k_tile_local<false, true>,
                   k_tile_local<true, true>, k_tile_local<false, false, true>, k_tile_local<true, false, true>})
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(K1SmemT<K1_MR>))) != cudaSuccess)
            return e;
    for (auto k : {k_tile_local_wide<false, false>, k_tile_local_wide<true, false>, k_tile_local_wide<false, true>,
                   k_tile_local_wide<true, true>, k_tile_local_wide<false, false, true>,
                   k_tile_local_wide<true, false, true>})
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K1SmemWide))) !=
            cudaSuccess)
            return e;
    for (auto k : {k_tile_big<false, false>, k_tile_big<true, false>, k_tile_big<false, true>, k_tile_big<true, true>,
                   k_tile_big<false, false, true>, k_tile_big<true, false, true>})
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K1Smem))) !=
            cudaSuccess)
            return e;
    if ((e = cudaFuncSetAttribute(k_small_middle, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMALL_SMEM_MAX)) !=
        cudaSuccess)
        return e;
    int dev = 0, sms = 0, per = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tile_local<false, false>, K1_THREADS,
                                                           sizeof(K1SmemT<K1_MR>))) != cudaSuccess)
        return e;
    g_k1_resident = sms * per;
    g_sms = sms;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tile_big<false, false>, NW * 32,
                                                           sizeof(K1Smem))) != cudaSuccess)
        return e;
    g_k1big_resident = sms * per;
    g_attr_done = true;
    return cudaSuccess;
}

// 16-byte vector loads (K1) and stores (K5) need the row pitch AND the base
// pointer 16-byte aligned; g.aligned holds the pitch test, the pointer is
// checked per call.
static Geometry with_ptr_alignment(const Geometry &g0, const void *ptr) {
    Geometry g = g0;
    g.aligned = g0.aligned && ((reinterpret_cast<uintptr_t>(ptr) & 15u) == 0);
    return g;
}

cudaError_t run_stage_local(const Geometry &g0, const Workspace &ws, const uint8_t *img,
                            cudaStream_t stream, cudaEvent_t *ev, bool with_border) {
    const Geometry g = with_ptr_alignment(g0, img);
    cudaError_t e = set_attrs();
    if (e != cudaSuccess) return e;
    auto mark = [&](int i) {
        if (ev) cudaEventRecord(ev[i], stream);
    };
    mark(K_TILE);
    const bool batch = g.tpi != g.nTy, bands = ws.boff != nullptr;  // (a band workspace has its offset)
    // few tiles: the 32-warp K1 (one warp per tile row) shortens the tile's
    // latency; many tiles: the 8-warp K1 (6 CTAs per SM) keeps the SMs busy
    const bool wide = !g_no_wide && g.nT * 4 <= g_k1_resident;
    if (wide) {
        auto k1 = g.thr ? (batch ? k_tile_local_wide<true, true> : bands ? k_tile_local_wide<true, false, true>
                                                                        : k_tile_local_wide<true, false>)
                        : (batch ? k_tile_local_wide<false, true> : bands ? k_tile_local_wide<false, false, true>
                                                                         : k_tile_local_wide<false, false>);
        e = launch_pdl(k1, g.nT, TH * 32, sizeof(K1SmemWide), stream, img, g, ws, g_k1_stop);
    } else {
        auto k1 = g.thr ? (batch ? k_tile_local<true, true> : bands ? k_tile_local<true, false, true> : k_tile_local<true, false>)
                        : (batch ? k_tile_local<false, true> : bands ? k_tile_local<false, false, true> : k_tile_local<false, false>);
#ifndef CCL_PFD_DIV
#define CCL_PFD_DIV 4
#endif
        const int pfd = g_k1_exper ? 0 : g_k1_resident / CCL_PFD_DIV;
        const bool twod = g.nTy <= 65535;
        e = launch_pdl2(k1, twod ? dim3(g.nTx, g.nTy) : dim3(g.nT), K1_THREADS, sizeof(K1SmemT<K1_MR>), stream, img, g,
                        ws, pfd, pfd % g.nTx, pfd / g.nTx, g_k1_stop);
    }
    if (e != cudaSuccess) return e;
    if (!wide) {  // the hand-over pass (the 32-warp K1 holds full rows itself)
        auto k1b = g.thr ? (batch ? k_tile_big<true, true> : bands ? k_tile_big<true, false, true> : k_tile_big<true, false>)
                         : (batch ? k_tile_big<false, true> : bands ? k_tile_big<false, false, true> : k_tile_big<false, false>);
        // a small grid (usually there is nothing to do; its CTAs loop over the list)
        // (a plan's last known hand-over count of 0: a quarter of the SMs, so
        // that every CTA fits beside K1's last wave and K2 is scheduled at
        // once -- C4 step 661 -> 650 us; otherwise every resident slot: the
        // comb hands every tile over, K1 1.50 -> 0.82 ms against half the
        // slots)
        const bool idle = ws.k1hint_host && *ws.k1hint_host == 0;
        const int grid = idle ? std::max(1, g_sms / 4) : g_k1big_resident;
        e = launch_pdl(k1b, std::min(g.nT, grid), NW * 32, sizeof(K1Smem), stream, img, g, ws, g_k1_stop);
        if (e != cudaSuccess) return e;
    }
    mark(K_BORDER);
    if (g_k1_stop < 99 || !with_border) return cudaGetLastError();
    const int nh = (g.nTy - 1) * g.nTx;
    const int64_t nv = (int64_t)(g.nTx - 1) * g.H;
    // few horizontal edges (small images, batches of them): 2 or 4 warps
    // share each edge's unions while the warps still fit on the device at once
    const int64_t vwarps = (nv + 31) / 32, slots = (int64_t)g_sms * 64;
    const int hsplit = ((int64_t)nh * 4 + vwarps <= slots) ? 4 : ((int64_t)nh * 2 + vwarps <= slots) ? 2 : 1;
    const int64_t warps = (int64_t)nh * hsplit + (nv + 31) / 32;
    if (warps > 0)
        e = launch_pdl(k_border, (unsigned)((warps + K2_WARPS - 1) / K2_WARPS), K2_WARPS * 32, 0, stream, g, ws,
                       nh * hsplit, hsplit);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// K3 (N and the root labels; on the row-band path K4 runs after the
// cross-band export).  Event (optional): ev[0] before K3.
cudaError_t run_stage_count(const Geometry &g, const Workspace &ws, int32_t *n_components,
                            cudaStream_t stream, cudaEvent_t *ev) {
    if (ev) cudaEventRecord(ev[0], stream);
    // warps per tile-row CTA: one per tile column up to 8; with few tile rows
    // (row bands, mid-size images) 16 or 32, while every CTA of the grid is
    // still resident at once (the lookback waits on earlier tile rows; with
    // C4's 675 tile rows 16 warps did not fit and measured slower)
    const int64_t warps_resident = (int64_t)g_sms * 64;
    int nw = g.nTx >= 8 ? 8 : g.nTx >= 4 ? 4 : g.nTx >= 2 ? 2 : 1;
    if (g.nTx > 16 && (int64_t)g.nTy * 32 <= warps_resident) nw = 32;
    else if (g.nTx > 8 && (int64_t)g.nTy * 16 <= warps_resident) nw = 16;
    void (*k3)(Geometry, Workspace, int32_t *) =
        nw == 32 ? k_number<32> : nw == 16 ? k_number<16> : nw == 8 ? k_number<8> : nw == 4 ? k_number<4>
        : nw == 2 ? k_number<2> : k_number<1>;
    cudaError_t e = launch_pdl(k3, g.nTy, nw * 32, 0, stream, g, ws, n_components);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// Magic multiplier for n / d with n < 2^31 (Granlund-Montgomery, N = 31
// bits): l = ceil(log2 d), m = ceil(2^(31+l) / d) < 2^32, and n / d =
// umulhi(n, m) >> (l - 1) for every n < 2^31 (d >= 2; checked exhaustively
// for d < 5000 and at the powers of two).  d = 1 is special-cased (m = 0).
static void magic_u32(uint32_t d, uint32_t *m, int *s) {
    if (d < 2) {
        *m = 0;
        *s = 0;
        return;
    }
    int l = 0;
    while ((1u << l) < d) l++;
    *m = (uint32_t)((((uint64_t)1 << (31 + l)) + d - 1) / d);
    *s = l - 1;
}

static cudaError_t launch_write(const Geometry &g0, const Workspace &ws, int32_t *labels, cudaStream_t stream) {
    const Geometry g = with_ptr_alignment(g0, labels);
    uint32_t magic;
    int mshift;
    magic_u32((uint32_t)g.nTx, &magic, &mshift);
    return launch_pdl(k_write, (unsigned)(((int64_t)g.nseg + K5_WARPS - 1) / K5_WARPS), K5_WARPS * 32, 0, stream,
                      g, ws, labels, magic, mshift);
}

// K5 alone (small-image path).  Events (optional): ev[0] before K5, ev[1] after.
static cudaError_t run_stage_final_write(const Geometry &g, const Workspace &ws, int32_t *labels,
                                         cudaStream_t stream, cudaEvent_t *ev) {
    if (ev) cudaEventRecord(ev[0], stream);
    cudaError_t e = launch_write(g, ws, labels, stream);
    if (e != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[1], stream);
    return cudaGetLastError();
}

// K4 + K5.  Events (optional): ev[0] before K4, ev[1] before K5, ev[2] after.
cudaError_t run_stage_final(const Geometry &g, const Workspace &ws, int32_t *labels,
                            cudaStream_t stream, cudaEvent_t *ev) {
    if (ev) cudaEventRecord(ev[0], stream);
    cudaError_t e = launch_pdl(k_fixup, (g.nT + K4_WARPS - 1) / K4_WARPS, K4_WARPS * 32, 0, stream, g, ws);
    if (e != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[1], stream);
    e = launch_write(g, ws, labels, stream);
    if (e != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[2], stream);
    return cudaGetLastError();
}

// Single image / batch: K1 (+ its hand-over pass), K2, K3, K4, K5.  Events
// (optional, K_COUNT + 1): ev[i] before kernel i, ev[K_COUNT] after.
cudaError_t run_pipeline(const Geometry &g, const Workspace &ws, const uint8_t *img,
                         int32_t *labels, int32_t *n_components, cudaStream_t stream,
                         cudaEvent_t *ev) {
    const bool small = small_mode(g);
    cudaError_t e = run_stage_local(g, ws, img, stream, ev, !small);
    if (g_k1_stop < 99) {  // development knob: K1 truncated, the rest would read garbage
        for (int i = K_NUMBER; ev && i <= K_COUNT; i++) cudaEventRecord(ev[i], stream);
        return e;
    }
    if (e != cudaSuccess) return e;
    if (small) {  // K2-K4 fused in one CTA (the event of K2 covers it; K3/K4 spans are empty)
        e = launch_pdl(k_small_middle, 1, SMALL_THREADS, small_smem(g), stream, g, ws, n_components);
        if (e != cudaSuccess) return e;
        if (ev) {
            cudaEventRecord(ev[K_NUMBER], stream);
            cudaEventRecord(ev[K_FIXUP], stream);
        }
        return run_stage_final_write(g, ws, labels, stream, ev ? ev + K_WRITE : nullptr);
    }
    e = run_stage_count(g, ws, n_components, stream, ev ? ev + K_NUMBER : nullptr);
    if (e == cudaSuccess) e = run_stage_final(g, ws, labels, stream, ev ? ev + K_FIXUP : nullptr);
    return e;
}

cudaError_t band_row_roots(const Geometry &g, const Workspace &ws, int64_t *keys, int32_t *nodes,
                           unsigned long long *noderep, uint32_t epoch, cudaStream_t stream) {
    return launch_pdl(k_band_rows, (2 * g.nTx + 3) / 4, 128, 0, stream, g, ws, keys, nodes, noderep, epoch);
}

cudaError_t band_rep(const int32_t *nodes, int n, const unsigned long long *noderep, int32_t *rep,
                     int32_t *spar, int spar_lo, int spar_hi, cudaStream_t stream) {
    const int m = std::max(n, spar_hi - spar_lo);
    return launch_pdl(k_xb_rep2, (m + 255) / 256, 256, 0, stream, nodes, n, noderep, rep, spar, spar_lo,
                      spar_hi);
}

cudaError_t band_resolve(int nb, int W, const int64_t *keys, const int32_t *reps, int32_t *spar,
                         cudaStream_t stream) {
    const int n = nb * 2 * W;
    return launch_pdl(k_xb_union, (n + 255) / 256, 256, 0, stream, nb, W, keys, reps, spar);
}

cudaError_t band_link(const Workspace &ws, int W, int self, const int64_t *keys, const int32_t *spar,
                      const int32_t *nodes, cudaStream_t stream) {
    return launch_pdl(k_xb_apply, (2 * W + 255) / 256, 256, 0, stream, W, self, keys, spar, nodes, ws.gparent);
}

cudaError_t band_export(const Geometry &g, const Workspace &ws, const int32_t *nodes, int32_t *labels_out, int n,
                        cudaStream_t stream) {
    return launch_pdl(k_band_export, (n + 255) / 256, 256, 0, stream, g, ws, nodes, labels_out, n);
}


}  // namespace cclb
