/*
 * oracle/aremsp.c -- the CPU ORACLE for two-pass 8-connectivity CCL (ARemSP).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1606_05973_b200/) never links, imports or calls it;
 * the two share no code, header, table or helper.
 *
 * Plain, slow, sequential C that follows the paper step by step, in the
 * paper's order and notation.  Citations are PAPER.md line numbers
 * (/root/reference/PAPER.md, the full-document copy) plus the algorithm name.
 *
 *   O1  storage: p[] zero-filled, p[0]=0, count=1           (reading A6)
 *   O2  Scan_ARemSP   Alg. "ARemSP Scan Phase" PAPER.md:855-933
 *   O2' merge         Alg. "merge"
 *   O3  flatten       Alg. "flatten"
 *   O4  relabel       Alg. "ARemSP" labeling phase PAPER.md:826-830
 *   O5  canonicalize  raster-order renumbering (readings A9, A13; BASELINE.json
 *                     "canonical labels (1..N in raster order of first pixel)")
 *   O6  Scan_CCLRemSP one-line decision-tree scan, PAPER.md:509-554 + Fig. 3
 *                     (a second, independent sequential variant: SURVEY f4)
 *
 * Readings of the paper (all listed in DESIGN.md "Readings"):
 *   A1  PAPER.md:879 "merge(p,label(a))" has one argument -> merge(p,label(e),label(a))
 *   A2  PAPER.md:920 branch e=0,g=1,d=0,f=0 writes label(e) -> label(g)
 *   A3  the scan walks row pairs (0,1),(2,3),... ("two lines at a time")
 *   A4  neighbours outside the image read as background
 *   A5  odd H: the last row pairs with a virtual all-background g row
 *   A6  count starts at 1; background label 0; p[0]=0
 *   A7  flatten runs i = 1 .. (count-1) = the max label assigned
 *   A8  merge's return value p[root_x] is not relied upon by ARemSP (CCLRemSP: A18)
 *   A10 a pixel is foreground iff its byte is non-zero
 *   A12 labels are int32; H*W <= INT32_MAX
 *   A17 CCLRemSP's own listing is missing (an ARemSP listing stands where it
 *       belongs): its scan is rebuilt from Fig. 3 and the
 *       copy / new-label definitions
 *   A18 copy(c,x) stores merge's return value p[root]: a
 *       member of the merged set, which is all a provisional label needs
 *
 * Parity status: pinned (see tests/test_oracle_pins.py) -- brute-force BFS on
 * every image with h*w <= 20, random images, closed forms, union-find traces
 * and the oracle-free property validator.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ------------------------------------------------------------------ */
/* O2'  merge -- Rem's union with splicing, Alg. merge */
/* ------------------------------------------------------------------ */
int32_t oracle_merge(int32_t *p, int32_t x, int32_t y)
{
    int32_t root_x = x, root_y = y;
    while (p[root_x] != p[root_y]) {
        if (p[root_x] > p[root_y]) {
            if (root_x == p[root_x]) {
                p[root_x] = p[root_y];
                return p[root_x];
            }
            int32_t z = p[root_x];
            p[root_x] = p[root_y];
            root_x = z;
        } else {
            if (root_y == p[root_y]) {
                p[root_y] = p[root_x];
                return p[root_x];
            }
            int32_t z = p[root_y];
            p[root_y] = p[root_x];
            root_y = z;
        }
    }
    return p[root_x];
}

/* ------------------------------------------------------------------ */
/* O3  flatten, Alg. flatten PAPER.md:708-718.  Returns k-1 = N.       */
/* ------------------------------------------------------------------ */
int32_t oracle_flatten(int32_t *p, int32_t count)
{
    int32_t k = 1;
    for (int32_t i = 1; i <= count; i++) {
        if (p[i] < i)
            p[i] = p[p[i]];
        else {
            p[i] = k;
            k++;
        }
    }
    return k - 1;
}

/* image(x) with reading A4 (outside -> 0) and A10 (non-zero -> 1) */
static inline int img_at(const uint8_t *img, int H, int W, int r, int c)
{
    if (r < 0 || r >= H || c < 0 || c >= W) return 0;
    return img[(int64_t)r * W + c] != 0;
}

#define LBL(r, c) label[(int64_t)(r) * W + (c)]

/* ------------------------------------------------------------------ */
/* O2  Scan_ARemSP, Alg. "ARemSP Scan Phase" PAPER.md:855-933.         */
/* Mask (Fig. 2b):  a b c / d e / f g, with          */
/* e=(r,c), g=(r+1,c), a=(r-1,c-1), b=(r-1,c), c'=(r-1,c+1),           */
/* d=(r,c-1), f=(r+1,c-1).  Returns count (next unused label).         */
/* p must hold ceil(H/2)*W + 2 zero-filled entries; label H*W zeros.   */
/* ------------------------------------------------------------------ */
int32_t oracle_scan_aremsp(const uint8_t *img, int H, int W,
                           int32_t *label, int32_t *p)
{
    int32_t count = 1;                              /* A6 */
    p[0] = 0;
    for (int r = 0; r < H; r += 2) {                /* A3: row pairs */
        for (int c = 0; c < W; c++) {
            int e  = img_at(img, H, W, r,     c);
            int g  = img_at(img, H, W, r + 1, c);   /* A5: 0 past the last row */
            int a  = img_at(img, H, W, r - 1, c - 1);
            int b  = img_at(img, H, W, r - 1, c);
            int cc = img_at(img, H, W, r - 1, c + 1);
            int d  = img_at(img, H, W, r,     c - 1);
            int f  = img_at(img, H, W, r + 1, c - 1);
            if (e) {
                if (!d) {
                    if (b) {
                        LBL(r, c) = LBL(r - 1, c);
                        if (f)
                            oracle_merge(p, LBL(r, c), LBL(r + 1, c - 1));
                    } else {
                        if (f) {
                            LBL(r, c) = LBL(r + 1, c - 1);
                            if (a)                              /* PAPER.md:878; A1 */
                                oracle_merge(p, LBL(r, c), LBL(r - 1, c - 1));
                            if (cc)
                                oracle_merge(p, LBL(r, c), LBL(r - 1, c + 1));
                        } else {
                            if (a) {
                                LBL(r, c) = LBL(r - 1, c - 1);
                                if (cc)
                                    oracle_merge(p, LBL(r, c), LBL(r - 1, c + 1));
                            } else {
                                if (cc) {
                                    LBL(r, c) = LBL(r - 1, c + 1);
                                } else {
                                    LBL(r, c) = count;
                                    p[count] = count;
                                    count++;
                                }
                            }
                        }
                    }
                } else {
                    LBL(r, c) = LBL(r, c - 1);
                    if (!b) {
                        if (cc)
                            oracle_merge(p, LBL(r, c), LBL(r - 1, c + 1));
                    }
                }
                if (g)
                    LBL(r + 1, c) = LBL(r, c);
            } else {
                if (g) {
                    if (d) {
                        LBL(r + 1, c) = LBL(r, c - 1);
                    } else {
                        if (f) {
                            LBL(r + 1, c) = LBL(r + 1, c - 1);
                        } else {                                /* PAPER.md:920-922; A2 */
                            LBL(r + 1, c) = count;
                            p[count] = count;
                            count++;
                        }
                    }
                }
            }
        }
    }
    return count;
}

/* ------------------------------------------------------------------ */
/* O6  Scan_CCLRemSP: the paper's second    */
/* sequential variant, "CCLRemSP", PAPER.md:509-554 + Fig. 3 (decision  */
/* tree of CCLLRPC).  Its pseudo-code (Alg. RemSP-I)  */
/* is missing from PAPER.md (reading A17), so the scan is rebuilt from  */
/* the prose: one image line at a time, forward mask a b c / d e        */
/* (Fig. 2a), and for every object pixel e the tree   */
/*   b ? copy(b)                                                         */
/*     : c ? (a ? copy(c,a) : d ? copy(c,d) : copy(c))                   */
/*         : (a ? copy(a) : d ? copy(d) : new label)                     */
/* with                                               */
/*   copy(x)   : label(e) = p[label(x)]                                  */
/*   copy(c,x) : label(e) = merge(p, label(c), label(x))  (Rem's merge   */
/*               with splicing, O2'; its return value p[root] is a       */
/*               member of the merged set, reading A18)                  */
/*   new label : label(e) = count, p[count] = count, count++.            */
/* p must hold ceil(H/2)*ceil(W/2) + 2 zero-filled entries (new labels   */
/* go to pairwise non-adjacent pixels); returns count.                   */
/* ------------------------------------------------------------------ */
int32_t oracle_scan_cclremsp(const uint8_t *img, int H, int W,
                             int32_t *label, int32_t *p)
{
    int32_t count = 1;                              /* A6 */
    p[0] = 0;
    for (int r = 0; r < H; r++) {
        for (int c = 0; c < W; c++) {
            if (!img_at(img, H, W, r, c)) continue;             /* background: label 0 */
            int a = img_at(img, H, W, r - 1, c - 1);     /* Fig. 2a mask */
            int b = img_at(img, H, W, r - 1, c);
            int cc = img_at(img, H, W, r - 1, c + 1);
            int d = img_at(img, H, W, r, c - 1);
            if (b) {
                LBL(r, c) = p[LBL(r - 1, c)];                   /* copy(b) */
            } else if (cc) {
                if (a)                                          /* copy(c,a) */
                    LBL(r, c) = oracle_merge(p, LBL(r - 1, c + 1), LBL(r - 1, c - 1));
                else if (d)                                     /* copy(c,d) */
                    LBL(r, c) = oracle_merge(p, LBL(r - 1, c + 1), LBL(r, c - 1));
                else                                            /* copy(c) */
                    LBL(r, c) = p[LBL(r - 1, c + 1)];
            } else if (a) {
                LBL(r, c) = p[LBL(r - 1, c - 1)];               /* copy(a) */
            } else if (d) {
                LBL(r, c) = p[LBL(r, c - 1)];                   /* copy(d) */
            } else {                                            /* new label */
                LBL(r, c) = count;
                p[count] = count;
                count++;
            }
        }
    }
    return count;
}

int64_t oracle_p_capacity_cclremsp(int H, int W)
{
    return (int64_t)((H + 1) / 2) * ((W + 1) / 2) + 2;
}

/* CCLRemSP (scan O6, flatten O3, labeling phase O4) followed by O5. */
int ccl_oracle_label_cclremsp(const uint8_t *img, int H, int W,
                              int32_t *labels, int32_t *n_components)
{
    if (!img || !labels || !n_components || H < 1 || W < 1) return 1;
    if ((int64_t)H * W > INT32_MAX) return 2;
    int64_t n = (int64_t)H * W;
    int32_t *p = (int32_t *)calloc((size_t)oracle_p_capacity_cclremsp(H, W), sizeof(int32_t));
    if (!p) return 5;
    memset(labels, 0, (size_t)n * sizeof(int32_t));
    int32_t count = oracle_scan_cclremsp(img, H, W, labels, p);     /* O6 */
    int32_t N = oracle_flatten(p, count - 1);                          /* O3 */
    oracle_relabel(labels, n, p);                                      /* O4 */
    free(p);
    if (oracle_canonicalize(labels, n, N) != 0) return 5;              /* O5 */
    *n_components = N;
    return 0;
}

/* O4  labeling phase: label(e) <- p[label(e)] */
void oracle_relabel(int32_t *label, int64_t n, const int32_t *p)
{
    for (int64_t i = 0; i < n; i++)
        label[i] = p[label[i]];                     /* p[0] = 0 keeps background */
}

/* O5  canonicalize: renumber 1..N by first occurrence in raster order */
int oracle_canonicalize(int32_t *label, int64_t n, int32_t nlabels)
{
    int32_t *map = (int32_t *)calloc((size_t)nlabels + 1, sizeof(int32_t));
    if (!map) return -1;
    int32_t next = 1;
    for (int64_t i = 0; i < n; i++) {
        int32_t L = label[i];
        if (L == 0) continue;
        if (map[L] == 0) map[L] = next++;
        label[i] = map[L];
    }
    free(map);
    return 0;
}

/* Capacity of p for an H x W image: one new label at most per (row pair,
 * column) because g copies e's label, plus p[0] and the
 * one-past-the-end slot flatten's literal bound may touch. */
int64_t oracle_p_capacity(int H, int W)
{
    return (int64_t)((H + 1) / 2) * W + 2;
}

/* ARemSP (Alg. ARemSP) followed by O5.
 * img: H*W bytes, labels: H*W int32 (output), *n_components: N.
 * Returns 0 on success, 1 invalid argument, 2 too large, 5 out of memory. */
int ccl_oracle_label(const uint8_t *img, int H, int W,
                     int32_t *labels, int32_t *n_components)
{
    if (!img || !labels || !n_components || H < 1 || W < 1) return 1;
    if ((int64_t)H * W > INT32_MAX) return 2;
    int64_t n = (int64_t)H * W;
    int64_t cap = oracle_p_capacity(H, W);
    int32_t *p = (int32_t *)calloc((size_t)cap, sizeof(int32_t));   /* O1 */
    if (!p) return 5;
    memset(labels, 0, (size_t)n * sizeof(int32_t));
    int32_t count = oracle_scan_aremsp(img, H, W, labels, p);        /* O2 */
    int32_t N = oracle_flatten(p, count - 1);                        /* O3, A7 */
    oracle_relabel(labels, n, p);                                    /* O4 */
    int rc = oracle_canonicalize(labels, n, N);                      /* O5 */
    free(p);
    if (rc) return 5;
    *n_components = N;
    return 0;
}
