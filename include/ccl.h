/*
 * include/ccl.h -- C ABI of the B200-native two-pass 8-connectivity connected
 * component labeling library (libccl_b200.so), after arxiv 1606.05973
 * ("A New Parallel Algorithm for Two-Pass Connected Component Labeling",
 * ARemSP / PARemSP).
 *
 * Problem (Sec. "Proposed Algorithm"): the input is a 2-D
 * binary image; "the connected component labeling problem is to assign a
 * label to each object pixel so that connected object pixels have the same
 * label", under 8-connectedness only.  The output is a 2-D array "label
 * containing the final labels" (Alg. ARemSP / PARemSP, PAPER.md:819-820,
 * 959-960).
 *
 * Output contract (bit-exact; tested against oracle/):
 *   - pixel (r,c) is foreground  <=>  img[r*W + c] != 0          (reading A10)
 *   - labels[r*W + c] = 0 for background, else a label in 1..N
 *   - labels are numbered 1..N in raster (row-major) order of each component's
 *     first pixel (BASELINE.json configs; reading A9/A13), so the
 *     output is unique for every image
 *   - N (flatten's k-1) is written to *n_components.
 *
 * Layout: row-major, pitch == W (bytes for img, int32 elements for labels).
 * Sizes: 1 <= H, 1 <= W, (int64)H*W <= INT32_MAX.
 * Alignment: none required.  16-byte vector loads/stores are used only when
 * W % 16 == 0 AND the img (loads) / labels (stores) base pointer is 16-byte
 * aligned, 32-byte ones only when the rows are 32-byte aligned as well (img:
 * W % 32 == 0 and a 32-byte aligned base; labels: a 32-byte aligned base);
 * otherwise the kernels fall back to narrower accesses.
 *
 * Ordering: the first kernel of a call waits for the previous work on
 * `stream` (e.g. the caller's kernel that produced img) to complete before it
 * reads any pixel.
 *
 * Ownership: the caller owns img, labels and n_components; the library never
 * frees or reallocates them.  labels must not alias img.  All workspace is
 * owned by a ccl_plan (explicit) or allocated stream-ordered from the device's
 * default memory pool (ccl_label).
 *
 * Asynchrony: the device-pointer calls only enqueue work on `stream` and
 * return; the caller synchronizes the stream before reading *n_components or
 * labels.  Device-side faults surface at the caller's next synchronization as
 * a CUDA error (documented, not detectable at enqueue time).
 *
 * Errors: arguments are validated on the host BEFORE any CUDA call, so a bad
 * argument never launches work (and is safe to test without a GPU).
 */
#ifndef CCL_B200_H
#define CCL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CCL_OK = 0,
    CCL_INVALID_ARGUMENT = 1, /* H<1, W<1, a NULL pointer, aliasing, bad plan  */
    CCL_TOO_LARGE = 2,        /* (int64)H*W > INT32_MAX                         */
    CCL_CUDA_ERROR = 3,       /* a CUDA runtime call or launch failed           */
    CCL_NCCL_ERROR = 4,       /* an NCCL call failed (sharded entry point)      */
    CCL_OUT_OF_MEMORY = 5     /* workspace allocation failed                    */
} ccl_status;

/* Opaque stream type so this header needs no CUDA include (== cudaStream_t). */
typedef struct CUstream_st *ccl_stream_t;
/* Opaque NCCL communicator (== ncclComm_t). */
typedef struct ncclComm *ccl_nccl_comm_t;

/* Human-readable name of a status code; never NULL. */
const char *ccl_status_string(ccl_status s);

/* Library version as "major.minor.patch". */
const char *ccl_version(void);

/* ------------------------------------------------------------------------
 * ccl_label -- one image on one GPU (ARemSP's contract, Alg. ARemSP
 * PAPER.md:814-834, computed by the B200 pipeline described in DESIGN.md).
 *   img           DEVICE pointer, H*W bytes, read only
 *   labels        DEVICE pointer, H*W int32, written (every pixel)
 *   n_components  DEVICE pointer to one int32, written
 *   stream        CUDA stream (NULL = legacy default stream)
 * Workspace is allocated and freed stream-ordered (cudaMallocAsync).
 * ---------------------------------------------------------------------- */
ccl_status ccl_label(const uint8_t *img, int H, int W, int32_t *labels,
                     int32_t *n_components, ccl_stream_t stream);

/* ------------------------------------------------------------------------
 * ccl_label_threshold -- ccl_label on a grayscale image thresholded on load:
 * pixel (r,c) is foreground <=> img[r*W + c] > threshold (0..255; 0 gives
 * ccl_label's byte != 0).  This is the paper's im2bw preprocessing fused into
 * the pixel read ("converted to binary ... level 0.5";
 * for 8-bit images level 0.5 is threshold 127: gray >= 128).
 * section 8(f) row f1.  threshold outside 0..255 -> CCL_INVALID_ARGUMENT.
 * ---------------------------------------------------------------------- */
ccl_status ccl_label_threshold(const uint8_t *img, int H, int W, int threshold, int32_t *labels,
                               int32_t *n_components, ccl_stream_t stream);

/* ------------------------------------------------------------------------
 * ccl_label_batch -- B independent images of H x W in one call (SURVEY.md
 * section 8(f) row f3: the paper's images of 1 MB or less, PAPER.md:1172-1177,
 * where one image is too small to fill a GPU and launches dominate).
 *   imgs          DEVICE pointer, B*H*W bytes: image b is rows b*H..b*H+H-1
 *   labels        DEVICE pointer, B*H*W int32, written; image b's labels are
 *                 1..N_b in raster order of its own components (as ccl_label)
 *   n_components  DEVICE pointer to B int32, written: N_b
 * No component crosses from one image to the next.  B >= 1; (int64)B*H*W
 * <= INT32_MAX else CCL_TOO_LARGE.  Same ownership/asynchrony as ccl_label.
 * ---------------------------------------------------------------------- */
ccl_status ccl_label_batch(const uint8_t *imgs, int B, int H, int W, int32_t *labels,
                           int32_t *n_components, ccl_stream_t stream);

/* ------------------------------------------------------------------------
 * Plans: preallocate the workspace for one image shape once, then label many
 * images of that shape with no allocation.  A plan may be used by one stream
 * at a time.
 * ---------------------------------------------------------------------- */
typedef struct ccl_plan_st *ccl_plan;

/* Allocates device workspace for H x W images on the current device (and
 * one mapped pinned host word: the plan sizes each call's hand-over pass for
 * tiles with rows of > 256 runs from the count its earlier calls left there;
 * outputs never depend on it). */
ccl_status ccl_plan_create(int H, int W, ccl_plan *plan_out);
/* Workspace for batches of B images of H x W (ccl_label_batch's layout): the
 * plan's label calls then take B*H*W pixels and write B component counts. */
ccl_status ccl_plan_create_batch(int B, int H, int W, ccl_plan *plan_out);
ccl_status ccl_plan_destroy(ccl_plan plan);
/* Foreground <=> byte > threshold for the plan's later calls (0..255; the
 * default 0 is byte != 0).  See ccl_label_threshold. */
ccl_status ccl_plan_set_threshold(ccl_plan plan, int threshold);
/* Bytes of device workspace the plan holds. */
ccl_status ccl_plan_workspace_bytes(ccl_plan plan, uint64_t *bytes);

/* Same contract as ccl_label, using the plan's workspace (DEVICE pointers). */
ccl_status ccl_plan_label(ccl_plan plan, const uint8_t *img, int32_t *labels,
                          int32_t *n_components, ccl_stream_t stream);

/* End-to-end variant with HOST buffers: copies h_img (H*W bytes) to the
 * device, labels it, copies labels (H*W int32) and N back, and synchronizes
 * `stream` before returning.  Host buffers should be pinned
 * (cudaHostAlloc / torch pin_memory) for full copy bandwidth.  The device
 * staging buffers belong to the plan.  = ccl_plan_label_host_async + a
 * synchronization of `stream`. */
ccl_status ccl_plan_label_host(ccl_plan plan, const uint8_t *h_img, int32_t *h_labels,
                               int32_t *h_n_components, ccl_stream_t stream);

/* Pipelined end-to-end variant: enqueues the H2D copy, the labeling and the
 * D2H copy on the plan's own streams (two staging slots), makes `stream`
 * wait for the D2H, and returns.  The caller synchronizes `stream` (or calls
 * again) before reading h_labels / *h_n_components, and keeps h_img
 * unchanged and h_labels / h_n_components untouched until then.  Back-to-back
 * calls overlap: call i+1's H2D and kernels run while call i's labels are
 * copied back, so a stream of frames runs at the slower copy direction's
 * bandwidth.  Ordering: a plan's calls (this one, ccl_plan_label on any
 * stream) run in call order on its single workspace; the H2D of h_img is not
 * ordered after earlier work on `stream` (the host buffer must be ready when
 * the call is made). */
ccl_status ccl_plan_label_host_async(ccl_plan plan, const uint8_t *h_img, int32_t *h_labels,
                                     int32_t *h_n_components, ccl_stream_t stream);

/* Per-kernel timing.  ccl_plan_set_profiling(plan, n) arms a ring of n sets
 * of CUDA events (n = 0 disarms): every later ccl_plan_label call records one
 * event before each pipeline kernel and one after the last, on the launch
 * stream (no synchronization).  ccl_plan_kernel_times fills up to `cap`
 * entries of names/ms with each kernel's duration averaged over the last
 * min(calls, n) calls; *count receives the number of kernels.  It
 * synchronizes on those events. */
ccl_status ccl_plan_set_profiling(ccl_plan plan, int nsets);
ccl_status ccl_plan_kernel_times(ccl_plan plan, const char **names, float *ms, int cap,
                                 int *count);

/* ccl_plan_counters -- cumulative path counters of a plan (zeroed at
 * ccl_plan_create), so a caller can tell which code paths of the tile-local
 * scan (PAPER.md:865-930 Scan_ARemSP on a chunk) its
 * images took:
 *   out[0]  tiles whose strip-merge list overflowed (the per-row leftover
 *           unions ran beside the list; > 1024 merges in a 32x1024 tile)
 *   out[1]  tiles handed to the full-size pass (a tile row of > 256 runs)
 *   out[2]  handed-over tiles whose merge list overflowed (> 256 merges)
 *   out[3]  strip merges listed, all tiles
 * Fills min(cap, *count) entries of `out` (HOST array; may be NULL with
 * cap 0 to query *count).  Synchronizes the device (cudaMemcpy).
 * Errors: CCL_INVALID_ARGUMENT for a NULL plan/count, CCL_CUDA_ERROR. */
ccl_status ccl_plan_counters(ccl_plan plan, uint64_t *out, int cap, int *count);

/* ------------------------------------------------------------------------
 * ccl_label_sharded -- one image split into contiguous row bands, one band
 * per rank of an NCCL communicator (the B200 analogue of PARemSP's row
 * chunks with per-thread label offsets).
 * Collective: every rank of `comm` calls it with the same W and H_total.
 *   band_img       DEVICE pointer, band_H*W bytes = global rows row0..row0+band_H-1
 *   band_labels    DEVICE pointer, band_H*W int32: the SAME values the
 *                  single-GPU ccl_label writes for those rows of the full image
 *   n_components   DEVICE pointer, receives the GLOBAL N on every rank
 * Bands are contiguous in rank order: row0 of rank k = sum of band_H of ranks
 * < k, and sum(band_H) = H_total (checked collectively; mismatch ->
 * CCL_INVALID_ARGUMENT on every rank).  band_H >= 1.  Synchronizes `stream`
 * (the cross-band step needs host-visible sizes).
 * ---------------------------------------------------------------------- */
ccl_status ccl_label_sharded(const uint8_t *band_img, int band_H, int W, int row0,
                             int H_total, int32_t *band_labels, int32_t *n_components,
                             ccl_nccl_comm_t comm, ccl_stream_t stream);

/* Sharded plans: the workspace and exchange buffers of one rank's band,
 * created once (collective: every rank calls it; checks the band layout as
 * ccl_label_sharded does) and reused by ccl_shard_plan_label, which has the
 * contract of ccl_label_sharded.  ccl_label_sharded = create + label + destroy. */
typedef struct ccl_shard_plan_st *ccl_shard_plan;
ccl_status ccl_shard_plan_create(int band_H, int W, int row0, int H_total, ccl_nccl_comm_t comm,
                                 ccl_stream_t stream, ccl_shard_plan *plan_out);
ccl_status ccl_shard_plan_label(ccl_shard_plan plan, const uint8_t *band_img, int32_t *band_labels,
                                int32_t *n_components, ccl_stream_t stream);
ccl_status ccl_shard_plan_destroy(ccl_shard_plan plan);
/* Per-stage CUDA-event profiling of a sharded plan (as ccl_plan_set_profiling /
 * ccl_plan_kernel_times; events between the stages serialise the chained
 * launches, so time profiled calls apart from throughput runs).  Stages:
 * k_tile_local, k_border, xband_exchange (boundary-row roots, representatives,
 * the key all-gather, slot unions, links), k_number, k_label, xband_export
 * (count all-gather, band offset, boundary labels, label all-gather),
 * k_fixup, k_write.  Local calls, not collective. */
ccl_status ccl_shard_plan_set_profiling(ccl_shard_plan plan, int nsets);
ccl_status ccl_shard_plan_kernel_times(ccl_shard_plan plan, const char **names, float *ms, int cap,
                                       int *count);

/* ------------------------------------------------------------------------
 * ccl_label_banded -- the row-band protocol of ccl_label_sharded run on ONE
 * GPU: the image (DEVICE pointers, as in ccl_label) is split into `nbands`
 * contiguous row bands of near-equal height (remainder to the last bands),
 * every band is labelled as its own image and the bands are joined by the
 * same cross-band resolution, with the all-gathers done by local copies.
 * Output identical to ccl_label.  1 <= nbands <= H.  Synchronizes `stream`.
 * Exists to test the multi-GPU protocol where only one GPU is available.
 * ---------------------------------------------------------------------- */
ccl_status ccl_label_banded(const uint8_t *img, int H, int W, int nbands, int32_t *labels,
                            int32_t *n_components, ccl_stream_t stream);

/* ------------------------------------------------------------------------
 * ccl_xband_resolve -- the host-side cross-band step of the row-band protocol
 * (PARemSP's boundary merge), exposed for host tests.
 *   rows[2k], rows[2k+1]: HOST arrays of W keys for band k's first and last
 *     row: a per-pixel key of the pixel's band-local component (-1 =
 *     background); keys are unique per component and increase with the
 *     raster position of the component's first pixel.
 *   Pixels of band k's last row and band k+1's first row that are 8-adjacent
 *   join their components; equal keys are the same component.
 *   out_min: HOST array of 2*W; for band `self`'s first and last row, the
 *     smallest key of each pixel's joined class (-1 for background).
 * Returns CCL_OK or CCL_INVALID_ARGUMENT.  Pure host code, no GPU needed.
 * ---------------------------------------------------------------------- */
int ccl_xband_resolve(int nb, int W, const int64_t *const *rows, int self, int64_t *out_min);

/* NCCL bootstrap helpers (torch.distributed does not expose its ncclComm_t):
 * rank 0 creates the 128-byte unique id, the harness broadcasts it (e.g. via
 * torch.distributed over gloo), then every rank creates its communicator on
 * the current device. */
ccl_status ccl_nccl_get_unique_id(uint8_t id_out[128]);
ccl_status ccl_nccl_comm_create(const uint8_t id[128], int nranks, int rank,
                                ccl_nccl_comm_t *comm_out);
ccl_status ccl_nccl_comm_destroy(ccl_nccl_comm_t comm);

/* Development hook (timing experiments; not part of the labeling contract):
 *   ccl_debug_set(1, stop): truncate K1 after phase `stop` (99 = off); the
 *     rest of the pipeline is skipped.  K1 honours it only in builds with
 *     -DCCL_PHASE_KNOB=1 (the checks cost the product kernel ~3 us).  ccl_debug_set(2, x): K1 experiment
 *     bits (1 = no L2 prefetch).  ccl_debug_set(3, 1): no small-image path
 *     (the general K2-K4 for every image); ccl_debug_set(4, 1): no 32-warp K1.
 *     ccl_debug_set(5, seed): workspaces created from now on (plans,
 *     one-shot calls) are filled with pseudo-random words (0 = off), so tests
 *     can check that no kernel reads workspace this call has not written.
 *     Returns 0, or 1 for an unknown key. */
int ccl_debug_set(int key, int value);

#ifdef __cplusplus
}
#endif
#endif /* CCL_B200_H */
