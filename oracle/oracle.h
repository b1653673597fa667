/*
 * oracle/oracle.h -- CPU ORACLE for ARemSP (arxiv 1606.05973).
 * TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it; the product path may not.
 * Shares nothing with include/ccl.h or paper_1606_05973_b200/.
 */
#ifndef CCL_ORACLE_H
#define CCL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Alg. merge, PAPER.md:669-698 (returns the paper's p[root_x]). */
int32_t oracle_merge(int32_t *p, int32_t x, int32_t y);
/* Alg. flatten; iterates i = 1..count; returns N = k-1. */
int32_t oracle_flatten(int32_t *p, int32_t count);
/* Alg. ARemSP Scan Phase; returns next unused label. */
int32_t oracle_scan_aremsp(const uint8_t *img, int H, int W, int32_t *label, int32_t *p);
/* Labeling phase. */
void oracle_relabel(int32_t *label, int64_t n, const int32_t *p);
/* Raster-order first-occurrence renumbering. */
int oracle_canonicalize(int32_t *label, int64_t n, int32_t nlabels);
int64_t oracle_p_capacity(int H, int W);
/* CCLRemSP's one-line decision-tree scan, PAPER.md:509-554 + Fig. 3. */
int32_t oracle_scan_cclremsp(const uint8_t *img, int H, int W, int32_t *label, int32_t *p);
int64_t oracle_p_capacity_cclremsp(int H, int W);
int ccl_oracle_label_cclremsp(const uint8_t *img, int H, int W, int32_t *labels, int32_t *n_components);
/* Whole pipeline: scan -> flatten -> relabel -> canonicalize. */
int ccl_oracle_label(const uint8_t *img, int H, int W, int32_t *labels, int32_t *n_components);

#ifdef __cplusplus
}
#endif
#endif
