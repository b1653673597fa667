// ccl_internal.cuh -- shared definitions of the B200 CCL pipeline (product
// path).  No code here is shared with oracle/ (DESIGN.md "Independence").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cclb {

// ---- tiling ------------------------------------
constexpr int TW = 1024;               // tile width in pixels: one warp-row, 32 lanes x 32 bits
constexpr int WPR = TW / 32;           // 32-bit words per tile row
constexpr int NW = 8;                  // warps per K1 CTA
constexpr int S = 4;                   // rows per warp in K1
constexpr int TH = NW * S;             // tile height (32)
constexpr int MAXRUN = TW / 2;         // max runs in one tile row (smem bound)
constexpr int RCAP = TH * MAXRUN;      // max runs in one tile (16384 < 2^15)
// Components of a tile are at most its largest set of pairwise non-adjacent
// pixels (king's graph): ceil(TH/2) * ceil(TW/2).  Geometry::capc is the same
// bound for the actual tile width (narrow images get small workspaces).
constexpr int CAPC = (TH / 2) * (TW / 2);
constexpr int META = 40;               // ints of per-tile metadata
constexpr int META_NCOMP = 0, META_NBORDER = 1, META_ROWS = 2;
constexpr int META_ROWFIRST = 4;       // [TH+1] first component index of each tile row

constexpr int KN_WARPS = 8;            // k_number: warps per tile-row CTA (fewer for narrow images)
constexpr int KN_ITEMS = 4;            // k_number: segments per thread per scan chunk

struct Geometry {
    int H, W;
    int WW;        // 32-bit words per image row = ceil(W/32)
    int nTx, nTy;  // tile grid
    int nT;        // nTx * nTy
    int nseg;      // H * nTx: (row, tile-column) segments in raster order
    int maxrun;    // runs per tile row bound: ceil(min(W,TW)/2)
    int capc;      // components per tile bound: ceil(min(H,TH)/2) * maxrun
    int capb;      // border components per tile bound: 2*maxrun + min(H,TH)
    int capw;      // words of a tile's component bitmap: ceil(capc/32)
    int aligned;   // W % 16 == 0: 16-byte vector loads / stores are legal
    int IH;        // rows per image: a batch is B images of IH x W stacked in memory (H = B*IH)
    int tpi;       // tile rows per image = ceil(IH/TH); tile rows never straddle two images
    int row0;      // global row of this image's row 0 (row bands of a sharded image; else 0)
    int thr;       // foreground <=> byte > thr (0: byte != 0)
};

// Device workspace (all arrays carved from one allocation; see ccl_api.cu).
struct Workspace {
    uint32_t *bm;         // [H][WW]           foreground bitmask, bit i of word k = column 32k+i
    uint16_t *runcomp;    // [H][nTx][maxrun]  (root row << 9) | root rank in its row, of each run
                          //                   (tile component = rowfirst[root row] + rank)
    int32_t *compnode;    // [nT][capc]        border-node id of a border component (others unset)
    int32_t *nrlab;       // [nT][capc]        band-local label of the j-th non-root border component
                          //                   of the tile (j = non-roots before it, K4)
    int32_t *tlb;         // [nT][TH]          label base of each tile row r: label of a root
                          //                   component = tlb[r] + rank - (non-roots before it)
    uint32_t *tbits;      // [nT][capw]        bitmap of the tile's non-root border components
    int32_t *twpre;       // [nT][capw]        exclusive popcount prefix of tbits
    int32_t *gparent;     // [nT][capb]        global union-find over border components
    int64_t *gkey;        // [nT][capb]        (image row, tile column, run ordinal) key: raster order
    int32_t *gnodecomp;   // [nT][capb]        (root row in tile << 16) | tile component of the node
    int32_t *gnodelab;    // [nT][capb]        band-local label of a root node
    uint32_t *edgerow;    // [nT][2][WPR]      run masks of the tile's first and last row (for K2)
    int32_t *topnode;     // [nT][maxrun]      node of each run of the tile's first row
    int32_t *botnode;     // [nT][maxrun]      node of each run of the tile's last row
    int32_t *leftnode;    // [nTx][H]          node of the pixel in the tile's first column
    int32_t *rightnode;   // [nTx][H]          node of the pixel in the tile's last column
    int32_t *meta;        // [nT][META]        ncomp, nborder, rows, rowfirst[TH+1]
    int32_t *segcnt;      // [nseg]            global roots whose first pixel lies in the segment
    int32_t *segoff;      // [nseg]            exclusive prefix of segcnt inside its tile row
    unsigned long long *scanstate;  // [nTy]   decoupled-lookback descriptors (one per tile row)
    int32_t *ticket;      // [1]               dynamic partition counter
    int32_t *rowexcl;     // [nTy]             labels of earlier tile rows
    int32_t *k1over;      // [nT]              tiles K1 handed to its full-size pass
    int32_t *k1over_n;    // [1]               their count (0 between calls; K3 resets it)
    unsigned long long *stats;  // [STAT_COUNT]  cumulative path counters (ccl_plan_counters)
    // plans only (null otherwise): K3 stores the number of tiles K1 handed
    // over into a mapped pinned host word; the host sizes the next call's
    // hand-over pass from the last value it sees (a grid of 370 idle CTAs
    // held K2's launch back by ~10 us on C4; the comb needs the full grid)
    int32_t *k1hint_dev = nullptr;                  // device address of the word
    const volatile int32_t *k1hint_host = nullptr;  // host address (-1: nothing seen yet)
    // row bands only (null for a whole image):
    const int32_t *xlab;  // [nb][2W+1]        gathered band records (N_band, then the band-local
                          //                   labels of its boundary slots); a node whose parent
                          //                   is -2-f (f = k*2W + s) takes record k's label s
                          //                   plus the N of bands before k
    const int32_t *boff;  // [1]               labels of earlier bands (added to every label by K5;
                          //                   written by K4's first thread from the records)
    int xself = 0, xnb = 0;         // this band's index, the number of bands
    int32_t *xntotal = nullptr;     // [1] N of all bands (K4 writes it; null: not wanted)
};

Geometry make_geometry(int H, int W);
// B images of IH x W, contiguous (image b = rows b*IH .. b*IH+IH-1 of a B*IH x W image)
Geometry make_geometry_batch(int B, int IH, int W);

// Tile row ty: first memory row, rows; tile row of a memory row.
// (a single image -- tpi == nTy -- takes the division-free branch)
__host__ __device__ __forceinline__ int tile_r0(const Geometry &g, int ty) {
    if (g.tpi == g.nTy) return ty * TH;
    return (ty / g.tpi) * g.IH + (ty % g.tpi) * TH;
}
__host__ __device__ __forceinline__ int tile_rows(const Geometry &g, int ty) {
    const int r = g.tpi == g.nTy ? g.H - ty * TH : g.IH - (ty % g.tpi) * TH;
    return r < TH ? r : TH;
}
__host__ __device__ __forceinline__ int row_tile(const Geometry &g, int row) {
    if (g.tpi == g.nTy) return row / TH;
    return (row / g.IH) * g.tpi + (row % g.IH) / TH;
}
// Offsets of every Workspace array inside one allocation of *total bytes.
void workspace_layout(const Geometry &g, size_t offs[], size_t *total);
Workspace workspace_bind(const Geometry &g, void *base);
// Zeroes the counters a new workspace must start with (before its first call).
cudaError_t workspace_init(const Workspace &ws, cudaStream_t stream);
// test hook ccl_debug_set(5, seed): fill a fresh workspace with pseudo-random words
cudaError_t workspace_poison(void *mem, size_t bytes, cudaStream_t stream);


// Path counters (cumulative over a plan's calls; zeroed by workspace_init):
// which K1 code paths the tiles took, so tests can prove the dense paths ran.
enum {
    STAT_K1_LIST_OVERFLOW = 0,  // k_tile_local(_wide) tiles whose strip-merge list overflowed (per-row leftover pass)
    STAT_K1_HANDOVER,           // tiles k_tile_local handed to k_tile_big (a row of > 256 runs)
    STAT_K1BIG_LIST_OVERFLOW,   // k_tile_big tiles whose merge list overflowed
    STAT_K1_MERGES,             // strip merges listed (all tiles, both passes)
    STAT_COUNT
};

// kernels of the single-image pipeline (run_pipeline), for per-kernel events
enum { K_TILE = 0, K_BORDER, K_NUMBER, K_FIXUP, K_WRITE, K_COUNT };
extern const char *const kKernelNames[K_COUNT];

// Enqueues the whole single-GPU pipeline on `stream`.  If `ev` is non-null it
// must hold K_COUNT+1 events; event i is recorded before kernel i.
cudaError_t run_pipeline(const Geometry &g, const Workspace &ws, const uint8_t *img,
                         int32_t *labels, int32_t *n_components, cudaStream_t stream,
                         cudaEvent_t *ev);
// The same pipeline in three stages (row bands insert the cross-band step
// between them): local = tile labeling (incl. the foreground predicate) +
// tile-edge merge; count = roots, numbering scan and labels of the roots (N of
// this image/band -> *n_components); final = labels of merged components +
// label write.
cudaError_t run_stage_local(const Geometry &g, const Workspace &ws, const uint8_t *img,
                            cudaStream_t stream, cudaEvent_t *ev, bool with_border = true);
cudaError_t run_stage_count(const Geometry &g, const Workspace &ws, int32_t *n_components,
                            cudaStream_t stream, cudaEvent_t *ev);
cudaError_t run_stage_final(const Geometry &g, const Workspace &ws, int32_t *labels,
                            cudaStream_t stream, cudaEvent_t *ev);
// Row bands: per-pixel root key / root node of the band's first row (keys[0,W),
// nodes[0,W)) and last row ([W,2W)); -1 for background.  Also the
// representative slot of every band-local root node: atomicMin of
// ((~epoch) << 32 | slot) into noderep[node] over the run heads.
cudaError_t band_row_roots(const Geometry &g, const Workspace &ws, int64_t *keys, int32_t *nodes,
                           unsigned long long *noderep, uint32_t epoch, cudaStream_t stream);
// Cross-band step (row bands).  Slots: band k's first
// row then last row, W each, at k*2W.
// rep[s] = first slot (of this band's 2W) with the same band-local root node,
// read from noderep (one entry per node of the band, all-ones initially;
// epoch: a number that grows with every call on the same scratch, from 1).
// Also starts the slot union-find: spar[t] = t for t in [spar_lo, spar_hi).
cudaError_t band_rep(const int32_t *nodes, int n, const unsigned long long *noderep, int32_t *rep,
                     int32_t *spar, int spar_lo, int spar_hi, cudaStream_t stream);
// The unions over all nb*2W slots (keys / reps of every band gathered).
cudaError_t band_resolve(int nb, int W, const int64_t *keys, const int32_t *reps, int32_t *spar,
                         cudaStream_t stream);
// Link this band's components whose class starts in another component.
cudaError_t band_link(const Workspace &ws, int W, int self, const int64_t *keys, const int32_t *spar,
                      const int32_t *nodes, cudaStream_t stream);
// Band-local label of the root of each of n boundary slots (-1: not a root),
// into the band's record of the gathered table (record = N_band, then 2W
// labels; labels_out = record + 1).
cudaError_t band_export(const Geometry &g, const Workspace &ws, const int32_t *nodes, int32_t *labels_out, int n,
                        cudaStream_t stream);


}  // namespace cclb
