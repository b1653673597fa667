/*
 * paremsp/paremsp.c -- multi-core HOST baseline: PARemSP (arxiv 1606.05973,
 * Sec. "Parallelizing ARemSP", Alg. PARemSP PAPER.md:954-998 and Alg. merger
 * PAPER.md:1001-1046), OpenMP, for SURVEY.md section 8(f) row f2.
 *
 * BASELINE / TEST INFRASTRUCTURE ONLY.  bench.py's cpu_baseline leg and
 * tests/ load it; the product path (paper_1606_05973_b200/) never does, and
 * it shares no code with the product or with oracle/ (its scan is the
 * paper's Scan_ARemSP restated for a row chunk).
 *
 * What it computes (the output is canonical, identical to the oracle's):
 *   P1 chunking   numiter = ceil(H/2) row pairs (reading A5:
 *                 an odd last row pairs with a background row); T threads
 *                 get chunk = numiter/T row pairs each, the remainder to the
 *                 last thread (reading A17).
 *   P2 local scan every thread runs Scan_ARemSP (readings
 *                 A1-A4) on its chunk alone -- rows above the chunk read as
 *                 background (reading A14) -- with provisional labels
 *                 count <- start*col + 1 where start is the thread's first
 *                 row-pair index (reading A15: "+1" keeps
 *                 0 for background; a row pair creates at most col labels,
 *                 so the chunks' label ranges are disjoint).  Inside a chunk
 *                 merge is the sequential Rem's merge with splicing
 *                 (PAPER.md:677-695): no other thread touches those labels.
 *   P3 boundary   for every chunk's first row i: object
 *                 pixel e=(i,col) is merged with b=(i-1,col), else with a
 *                 and c (the diagonals), through merger
 *                 -- lock, re-check that the node is still a root, link.
 *                 Reading B2: merger's unlocked splice is left out (the
 *                 climb moves to the parent instead): a splice moves a
 *                 subtree into another tree before the two are joined, and
 *                 a concurrent merger reading through that moment can stop
 *                 early (on the GPU this lost unions, DESIGN.md "Tile-local
 *                 union").  Locks are striped (PM_NLOCKS mutexes indexed by
 *                 the root's label): the same mutual exclusion, bounded
 *                 memory.
 *   P4 flatten    PAPER.md:700-721 (sequential in the paper, PAPER.md:989;
 *                 reading A18: the order does not change the output): in
 *                 parallel, every label -> its root; roots numbered in label
 *                 order by a per-thread count + exclusive prefix.
 *   P5 labeling   label(e) <- p[label(e)], parallel.
 *   P6 canonical  raster-order renumbering (readings A9/A13), parallel: the
 *                 first pixel of every label (min index), a prefix count of
 *                 first pixels in raster order, relabel.
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "paremsp.h"

#define PM_NLOCKS 4096

/* relaxed atomic access to the shared parent array (no torn or cached reads
 * between threads; the paper's memory model) */
static inline int32_t ld(const int32_t *p, int64_t i) { return __atomic_load_n(p + i, __ATOMIC_RELAXED); }
static inline void st(int32_t *p, int64_t i, int32_t v) { __atomic_store_n(p + i, v, __ATOMIC_RELAXED); }

/* ---------------------------------------------------------------- merge */
/* Alg. merge, PAPER.md:677-695 -- sequential Rem's union with splicing,  */
/* used inside one thread's chunk (its labels are its own).               */
static void merge_seq(int32_t *p, int32_t x, int32_t y)
{
    int32_t rx = x, ry = y;
    while (p[rx] != p[ry]) {
        if (p[rx] > p[ry]) {
            if (rx == p[rx]) { p[rx] = p[ry]; return; }
            int32_t z = p[rx]; p[rx] = p[ry]; rx = z;
        } else {
            if (ry == p[ry]) { p[ry] = p[rx]; return; }
            int32_t z = p[ry]; p[ry] = p[rx]; ry = z;
        }
    }
}

/* --------------------------------------------------------------- merger */
/* Alg. merger, without the splice (reading B2).      */
static void merger(int32_t *p, omp_lock_t *locks, int32_t x, int32_t y)
{
    int32_t rx = x, ry = y;
    for (;;) {
        int32_t px = ld(p, rx), py = ld(p, ry);
        if (px == py) return;
        if (px > py) {
            if (rx == px) {
                int ok = 0;
                omp_set_lock(&locks[rx % PM_NLOCKS]);
                if (ld(p, rx) == rx) { st(p, rx, py); ok = 1; }
                omp_unset_lock(&locks[rx % PM_NLOCKS]);
                if (ok) return;
                continue;
            }
            rx = px;                                        /* (splice dropped: B2) */
        } else {
            if (ry == py) {
                int ok = 0;
                omp_set_lock(&locks[ry % PM_NLOCKS]);
                if (ld(p, ry) == ry) { st(p, ry, px); ok = 1; }  /* PAPER.md:1030-1032, A16 */
                omp_unset_lock(&locks[ry % PM_NLOCKS]);
                if (ok) return;
                continue;
            }
            ry = py;
        }
    }
}

/* ------------------------------------------------------ Scan on a chunk */
/* Scan_ARemSP over rows [r0, r1): rows outside read as */
/* background (A14; A4 at the image edge).  Returns the next unused label. */
static int32_t scan_chunk(const uint8_t *img, int W, int r0, int r1,
                          int32_t *label, int32_t *p, int32_t count)
{
#define PX(r, c) ((r) >= r0 && (r) < r1 && (c) >= 0 && (c) < W && img[(int64_t)(r) * W + (c)] != 0)
#define L(r, c) label[(int64_t)(r) * W + (c)]
    for (int r = r0; r < r1; r += 2) {                       /* two rows at a time (A3) */
        for (int c = 0; c < W; c++) {
            const int e = PX(r, c), g = PX(r + 1, c);
            const int a = PX(r - 1, c - 1), b = PX(r - 1, c), cc = PX(r - 1, c + 1);
            const int d = PX(r, c - 1), f = PX(r + 1, c - 1);
            if (e) {
                if (!d) {
                    if (b) {
                        L(r, c) = L(r - 1, c);
                        if (f) merge_seq(p, L(r, c), L(r + 1, c - 1));
                    } else if (f) {
                        L(r, c) = L(r + 1, c - 1);
                        if (a) merge_seq(p, L(r, c), L(r - 1, c - 1));     /* A1 */
                        if (cc) merge_seq(p, L(r, c), L(r - 1, c + 1));
                    } else if (a) {
                        L(r, c) = L(r - 1, c - 1);
                        if (cc) merge_seq(p, L(r, c), L(r - 1, c + 1));
                    } else if (cc) {
                        L(r, c) = L(r - 1, c + 1);
                    } else {
                        L(r, c) = count; p[count] = count; count++;
                    }
                } else {
                    L(r, c) = L(r, c - 1);
                    if (!b && cc) merge_seq(p, L(r, c), L(r - 1, c + 1));
                }
                if (g) L(r + 1, c) = L(r, c);
            } else if (g) {
                if (d) L(r + 1, c) = L(r, c - 1);
                else if (f) L(r + 1, c) = L(r + 1, c - 1);
                else { L(r + 1, c) = count; p[count] = count; count++; }  /* A2 */
            }
        }
    }
#undef PX
#undef L
    return count;
}

int paremsp_label(const uint8_t *img, int H, int W, int nthreads,
                  int32_t *label, int32_t *n_components, int *threads_used)
{
    if (!img || !label || !n_components || H < 1 || W < 1) return 1;
    if ((int64_t)H * W > INT32_MAX) return 2;
    const int64_t n = (int64_t)H * W;
    const int numiter = (H + 1) / 2;                          /* PAPER.md:962, A5 */
    int T = nthreads > 0 ? nthreads : omp_get_max_threads();
    if (T > numiter) T = numiter;
    const int chunk = numiter / T;
    const int64_t cap = (int64_t)numiter * W + 2;
    int32_t *p = (int32_t *)calloc((size_t)cap, sizeof(int32_t));
    int64_t *tcnt = (int64_t *)calloc((size_t)T + 1, sizeof(int64_t));
    omp_lock_t *locks = (omp_lock_t *)malloc(sizeof(omp_lock_t) * PM_NLOCKS);
    if (!p || !tcnt || !locks) { free(p); free(tcnt); free(locks); return 5; }
    for (int i = 0; i < PM_NLOCKS; i++) omp_init_lock(&locks[i]);
    int rc = 0;
    int32_t N = 0;
    int32_t *map = NULL, *first = NULL;

#pragma omp parallel num_threads(T)
    {
        const int t = omp_get_thread_num();
        const int it0 = t * chunk, it1 = t == T - 1 ? numiter : it0 + chunk;   /* A17 */
        const int r0 = 2 * it0, r1 = 2 * it1 < H ? 2 * it1 : H;
        /* P2 local scan; labels from start*col + 1 (A15) */
        memset(label + (int64_t)r0 * W, 0, sizeof(int32_t) * (size_t)((int64_t)(r1 - r0) * W));
        const int32_t base = (int32_t)((int64_t)it0 * W) + 1;
        const int32_t end = scan_chunk(img, W, r0, r1, label, p, base);
        (void)end;
#pragma omp barrier
        /* P3 boundary merge: the first row of every chunk but the first */
#pragma omp for schedule(static)
        for (int k = 1; k < T; k++) {
            const int i = 2 * k * chunk;
            for (int c = 0; c < W; c++) {
                const int32_t le = label[(int64_t)i * W + c];
                if (!le) continue;
                const int32_t lb = label[(int64_t)(i - 1) * W + c];
                if (lb) {
                    merger(p, locks, le, lb);
                } else {
                    const int32_t la = c > 0 ? label[(int64_t)(i - 1) * W + c - 1] : 0;
                    const int32_t lc = c + 1 < W ? label[(int64_t)(i - 1) * W + c + 1] : 0;
                    if (la) merger(p, locks, le, la);
                    if (lc) merger(p, locks, le, lc);
                }
            }
        }
        /* (implicit barrier) P4 flatten: every label -> its root, in parallel
         * (labels of thread t's range are [it0*W+1, it1*W]); roots counted */
        const int64_t l0 = (int64_t)it0 * W + 1, l1 = (int64_t)it1 * W + 1;
        int64_t roots = 0;
        for (int64_t i = l0; i < l1; i++) {
            int32_t r = ld(p, i);
            if (r == 0) continue;                 /* an unused label (A7) */
            if (r == i) { roots++; continue; }
            while (ld(p, r) != r) r = ld(p, r);
            st(p, i, r);                          /* an ancestor: safe to publish */
        }
        tcnt[t + 1] = roots;
#pragma omp barrier
#pragma omp single
        {
            for (int k = 0; k < T; k++) tcnt[k + 1] += tcnt[k];
            N = (int32_t)tcnt[T];
            map = (int32_t *)calloc((size_t)N + 1, sizeof(int32_t));
            first = (int32_t *)malloc(sizeof(int32_t) * ((size_t)N + 1));
            if (!map || !first) rc = 5;
        }
        if (!rc) {
            /* roots numbered k = 1.. in label order (flatten's k++):
             * stored negated so a root's new number is not mistaken for a label */
            int64_t k = tcnt[t];
            for (int64_t i = l0; i < l1; i++)
                if (ld(p, i) == i) st(p, i, (int32_t)-(++k));
#pragma omp barrier
            for (int64_t i = l0; i < l1; i++) {
                const int32_t r = ld(p, i);
                if (r > 0) st(p, i, -ld(p, r));   /* a non-root: its root's number */
            }
#pragma omp barrier
            for (int64_t i = l0; i < l1; i++) {
                const int32_t r = ld(p, i);
                if (r < 0) st(p, i, -r);
            }
#pragma omp barrier
            /* P5 labeling phase and the first pixel of
             * every label (P6); pixels split evenly over the threads */
            const int64_t q0 = n * t / T, q1 = n * (t + 1) / T;
            for (int64_t i = q0; i < q1; i++) label[i] = label[i] ? p[label[i]] : 0;
#pragma omp for schedule(static)
            for (int64_t L = 0; L <= N; L++) first[L] = INT32_MAX;
            for (int64_t i = q0; i < q1; i++) {
                const int32_t L = label[i];
                if (!L) continue;
                int32_t cur = __atomic_load_n(first + L, __ATOMIC_RELAXED);
                while ((int32_t)i < cur &&
                       !__atomic_compare_exchange_n(first + L, &cur, (int32_t)i, 0, __ATOMIC_RELAXED,
                                                    __ATOMIC_RELAXED)) {
                }
            }
#pragma omp barrier
            int64_t nf = 0;
            for (int64_t i = q0; i < q1; i++) nf += label[i] && first[label[i]] == (int32_t)i;
            tcnt[t + 1] = nf;
#pragma omp barrier
#pragma omp single
            for (int k = 0; k < T; k++) tcnt[k + 1] += tcnt[k];
            int32_t next = (int32_t)tcnt[t] + 1;
            for (int64_t i = q0; i < q1; i++)
                if (label[i] && first[label[i]] == (int32_t)i) map[label[i]] = next++;
#pragma omp barrier
            for (int64_t i = q0; i < q1; i++) label[i] = map[label[i]];
        }
    }
    for (int i = 0; i < PM_NLOCKS; i++) omp_destroy_lock(&locks[i]);
    free(locks);
    free(p);
    free(tcnt);
    free(map);
    free(first);
    if (rc) return rc;
    *n_components = N;
    if (threads_used) *threads_used = T;
    return 0;
}
