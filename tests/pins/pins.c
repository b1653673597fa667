/*
 * tests/pins/pins.c -- independent checkers that PIN the oracle (and, on the
 * GPU box, the CUDA path) to the mathematics, not to itself.  Test code only;
 * shares no code with oracle/ or paper_1606_05973_b200/.
 *
 *  P1 pins_bfs_label   breadth-first flood fill under 8-connectivity
 *                      (PAPER.md:500-505), labels handed out in raster order
 *                      of discovery -> already canonical.
 *  P2 pins_dsu_label   naive union-find over every 8-adjacent foreground pixel
 *                      pair (transitive closure), then raster renumbering.
 *  P3 pins_validate    oracle-free property check: (i) 8-adjacent fg pairs
 *                      share a label, (ii) each label's pixels are 8-connected,
 *                      (iii) bg <=> 0, (iv) canonical raster numbering,
 *                      (v) N = max label.  (i)+(ii)+(iv) determine the output.
 *  exhaustive driver   runs two labelers on every h x w binary image.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static const int DR[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
static const int DC[8] = {-1, 0, 1, -1, 1, -1, 0, 1};

int pins_bfs_label(const uint8_t *img, int H, int W, int32_t *lab, int32_t *n_out)
{
    int64_t n = (int64_t)H * W;
    int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
    if (!queue) return 5;
    memset(lab, 0, sizeof(int32_t) * n);
    int32_t next = 0;
    for (int64_t s = 0; s < n; s++) {
        if (!img[s] || lab[s]) continue;
        next++;
        int64_t qh = 0, qt = 0;
        queue[qt++] = (int32_t)s;
        lab[s] = next;
        while (qh < qt) {
            int32_t v = queue[qh++];
            int r = v / W, c = v % W;
            for (int k = 0; k < 8; k++) {
                int rr = r + DR[k], cc = c + DC[k];
                if (rr < 0 || rr >= H || cc < 0 || cc >= W) continue;
                int64_t u = (int64_t)rr * W + cc;
                if (img[u] && !lab[u]) { lab[u] = next; queue[qt++] = (int32_t)u; }
            }
        }
    }
    free(queue);
    *n_out = next;
    return 0;
}

static int32_t dsu_find(int32_t *par, int32_t x)
{
    while (par[x] != x) x = par[x];
    return x;
}

int pins_dsu_label(const uint8_t *img, int H, int W, int32_t *lab, int32_t *n_out)
{
    int64_t n = (int64_t)H * W;
    int32_t *par = (int32_t *)malloc(sizeof(int32_t) * n);
    int32_t *map = (int32_t *)malloc(sizeof(int32_t) * n);
    if (!par || !map) { free(par); free(map); return 5; }
    for (int64_t i = 0; i < n; i++) { par[i] = (int32_t)i; map[i] = 0; }
    for (int r = 0; r < H; r++)
        for (int c = 0; c < W; c++) {
            int64_t v = (int64_t)r * W + c;
            if (!img[v]) continue;
            for (int k = 0; k < 8; k++) {
                int rr = r + DR[k], cc = c + DC[k];
                if (rr < 0 || rr >= H || cc < 0 || cc >= W) continue;
                int64_t u = (int64_t)rr * W + cc;
                if (!img[u]) continue;
                int32_t a = dsu_find(par, (int32_t)v), b = dsu_find(par, (int32_t)u);
                if (a != b) par[a > b ? a : b] = a < b ? a : b;
            }
        }
    int32_t next = 0;
    for (int64_t i = 0; i < n; i++) {
        if (!img[i]) { lab[i] = 0; continue; }
        int32_t root = dsu_find(par, (int32_t)i);
        if (!map[root]) map[root] = ++next;
        lab[i] = map[root];
    }
    free(par); free(map);
    *n_out = next;
    return 0;
}

/* Returns 0 if valid, else a code naming the first violated property:
 * 1 bg/fg mismatch (iii), 2 adjacent fg pair with different labels (i),
 * 3 non-canonical numbering (iv), 4 a label's pixels not 8-connected (ii),
 * 5 N != max label (v), 6 out of memory. */
int pins_validate(const uint8_t *img, int H, int W, const int32_t *lab, int32_t N)
{
    int64_t n = (int64_t)H * W;
    int32_t maxseen = 0;
    for (int64_t i = 0; i < n; i++) {
        if ((img[i] != 0) != (lab[i] != 0)) return 1;
        if (lab[i] < 0) return 3;
        if (lab[i] > maxseen) {
            if (lab[i] != maxseen + 1) return 3;
            maxseen = lab[i];
        }
    }
    if (maxseen != N) return 5;
    for (int r = 0; r < H; r++)
        for (int c = 0; c < W; c++) {
            int64_t v = (int64_t)r * W + c;
            if (!lab[v]) continue;
            for (int k = 4; k < 8; k++) { /* forward half of the neighbourhood */
                int rr = r + DR[k], cc = c + DC[k];
                if (rr >= H || cc < 0 || cc >= W) continue;
                int64_t u = (int64_t)rr * W + cc;
                if (lab[u] && lab[u] != lab[v]) return 2;
            }
        }
    /* (ii): flood from each label's first pixel through same-label pixels,
     * and require that every pixel of that label is reached. */
    uint8_t *seen = (uint8_t *)calloc((size_t)n, 1);
    int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
    if (!seen || !queue) { free(seen); free(queue); return 6; }
    int32_t nextlab = 1;
    for (int64_t s = 0; s < n; s++) {
        if (!lab[s] || seen[s]) continue;
        if (lab[s] != nextlab) { free(seen); free(queue); return 4; } /* label split */
        nextlab++;
        int64_t qh = 0, qt = 0;
        queue[qt++] = (int32_t)s;
        seen[s] = 1;
        while (qh < qt) {
            int32_t v = queue[qh++];
            int r = v / W, c = v % W;
            for (int k = 0; k < 8; k++) {
                int rr = r + DR[k], cc = c + DC[k];
                if (rr < 0 || rr >= H || cc < 0 || cc >= W) continue;
                int64_t u = (int64_t)rr * W + cc;
                if (!seen[u] && lab[u] == lab[s]) { seen[u] = 1; queue[qt++] = (int32_t)u; }
            }
        }
    }
    free(seen); free(queue);
    return 0;
}

typedef int (*labeler_fn)(const uint8_t *, int, int, int32_t *, int32_t *);

/* Runs labelers A and B on every h x w image whose index lies in
 * [first, last); returns the number of images where labels or N differ and
 * stores the first failing image index in *first_bad (or -1). */
int64_t pins_exhaustive(labeler_fn A, labeler_fn B, int h, int w,
                        int64_t first, int64_t last, int64_t *first_bad)
{
    int n = h * w;
    uint8_t img[64];
    int32_t la[64], lb[64];
    int64_t bad = 0;
    *first_bad = -1;
    for (int64_t m = first; m < last; m++) {
        for (int i = 0; i < n; i++) img[i] = (uint8_t)((m >> i) & 1);
        int32_t na = -1, nb = -2;
        int ra = A(img, h, w, la, &na), rb = B(img, h, w, lb, &nb);
        if (ra || rb || na != nb || memcmp(la, lb, sizeof(int32_t) * n) != 0) {
            if (*first_bad < 0) *first_bad = m;
            bad++;
        }
    }
    return bad;
}
