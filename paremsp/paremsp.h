/*
 * paremsp/paremsp.h -- multi-core host baseline PARemSP (arxiv 1606.05973,
 * Alg. PARemSP, merger PAPER.md:1001-1046).
 * BASELINE / TEST INFRASTRUCTURE ONLY (bench.py cpu_baseline leg, tests/).
 */
#ifndef CCL_PAREMSP_H
#define CCL_PAREMSP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Labels img (H x W bytes, fg <=> != 0, 8-connectivity) with `nthreads`
 * OpenMP threads (<= 0: omp_get_max_threads(); capped at ceil(H/2)).
 * labels: H*W int32 HOST array, written with the canonical labels (1..N in
 * raster order of each component's first pixel, 0 background) -- the
 * oracle's output.  *threads_used (may be NULL) = the thread count used.
 * Returns 0, 1 invalid argument, 2 too large, 5 out of memory. */
int paremsp_label(const uint8_t *img, int H, int W, int nthreads,
                  int32_t *labels, int32_t *n_components, int *threads_used);

#ifdef __cplusplus
}
#endif
#endif
