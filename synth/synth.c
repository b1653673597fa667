/*
 * synth/synth.c -- seeded synthetic binary images shaped like the paper's
 * workloads.  Shared by the
 * oracle tests, the GPU parity tests and bench.py.  Holds NONE of the CCL
 * method's arithmetic: it only draws pixels.
 *
 * PRNG: counter-based h(seed,stream,i) = mix64(mix64(seed ^ stream*C1) + i*C2),
 * mix64 = the SplitMix64 finaliser.  Bernoulli(p): fg <=> (h>>32) < floor(p*2^32).
 * Every generator is a pure function of its arguments (no global state), and
 * multi-threaded generators give the same bytes for any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t synth_hash(uint64_t seed, uint64_t stream, uint64_t i)
{
    return mix64(mix64(seed ^ (stream * 0xD1B54A32D192ED03ULL)) + i * 0x9E3779B97F4A7C15ULL);
}

static inline uint32_t bern_threshold(double p)
{
    if (p <= 0.0) return 0;
    if (p >= 1.0) return 0xFFFFFFFFu;
    return (uint32_t)floor(p * 4294967296.0);
}

/* iid Bernoulli(p); p >= 1 gives all-ones exactly. */
void synth_bernoulli(uint8_t *out, int H, int W, double p, uint64_t seed)
{
    int64_t n = (int64_t)H * W;
    uint32_t thr = bern_threshold(p);
    int all = p >= 1.0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        uint32_t v = (uint32_t)(synth_hash(seed, 0, (uint64_t)i) >> 32);
        out[i] = all ? 1 : (v < thr);
    }
}

/* U[0,1) noise -> separable Gaussian (sigma, radius = 4 sigma, mirror
 * boundary "d c b a | a b c d | d c b a", float64) -> fg <=> v > lower median
 * (the element of rank (n-1)/2), giving exactly floor(n/2) foreground pixels
 * when the filtered values are distinct. */
static int cmp_double(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

static inline int mirror(int i, int n)
{
    /* reflect about the edge, repeating the edge sample (scipy "reflect") */
    while (i < 0 || i >= n) {
        if (i < 0) i = -i - 1;
        if (i >= n) i = 2 * n - i - 1;
    }
    return i;
}

int synth_blobs(uint8_t *out, int H, int W, double sigma, uint64_t seed)
{
    int64_t n = (int64_t)H * W;
    int R = (int)ceil(4.0 * sigma);
    double *a = (double *)malloc(sizeof(double) * n);
    double *b = (double *)malloc(sizeof(double) * n);
    double *k = (double *)malloc(sizeof(double) * (2 * R + 1));
    if (!a || !b || !k) { free(a); free(b); free(k); return 5; }
    double ks = 0;
    for (int t = -R; t <= R; t++) { k[t + R] = exp(-0.5 * t * t / (sigma * sigma)); ks += k[t + R]; }
    for (int t = 0; t <= 2 * R; t++) k[t] /= ks;
    for (int64_t i = 0; i < n; i++)
        a[i] = (double)(synth_hash(seed, 0, (uint64_t)i) >> 11) * (1.0 / 9007199254740992.0);
    /* horizontal pass a -> b */
#pragma omp parallel for schedule(static)
    for (int r = 0; r < H; r++)
        for (int c = 0; c < W; c++) {
            double s = 0;
            for (int t = -R; t <= R; t++) s += k[t + R] * a[(int64_t)r * W + mirror(c + t, W)];
            b[(int64_t)r * W + c] = s;
        }
    /* vertical pass b -> a */
#pragma omp parallel for schedule(static)
    for (int r = 0; r < H; r++)
        for (int c = 0; c < W; c++) {
            double s = 0;
            for (int t = -R; t <= R; t++) s += k[t + R] * b[(int64_t)mirror(r + t, H) * W + c];
            a[(int64_t)r * W + c] = s;
        }
    memcpy(b, a, sizeof(double) * n);
    qsort(b, (size_t)n, sizeof(double), cmp_double);
    double med = b[(n - 1) / 2];
    for (int64_t i = 0; i < n; i++) out[i] = a[i] > med;
    free(a); free(b); free(k);
    return 0;
}

/* Voronoi class map: ncells seeds at integer coordinates (stream 1), pixel ->
 * nearest seed by int64 squared distance, ties -> lowest seed index; each cell
 * is foreground with probability pcell (stream 2); then every pixel is flipped
 * with probability pflip (stream 3, indexed by raster index). */
int synth_voronoi(uint8_t *out, int H, int W, int ncells, double pcell, double pflip,
                  uint64_t seed)
{
    if (ncells < 1) return 1;
    int32_t *sx = (int32_t *)malloc(sizeof(int32_t) * ncells);
    int32_t *sy = (int32_t *)malloc(sizeof(int32_t) * ncells);
    uint8_t *cf = (uint8_t *)malloc(ncells);
    if (!sx || !sy || !cf) { free(sx); free(sy); free(cf); return 5; }
    uint32_t thc = bern_threshold(pcell), thf = bern_threshold(pflip);
    for (int k = 0; k < ncells; k++) {
        sx[k] = (int32_t)(synth_hash(seed, 1, 2 * (uint64_t)k) % (uint64_t)W);
        sy[k] = (int32_t)(synth_hash(seed, 1, 2 * (uint64_t)k + 1) % (uint64_t)H);
        cf[k] = (uint32_t)(synth_hash(seed, 2, (uint64_t)k) >> 32) < thc;
    }
    /* bucket grid with cell size G ~ mean seed spacing */
    int G = (int)ceil(sqrt((double)H * W / ncells));
    if (G < 1) G = 1;
    int BX = (W + G - 1) / G, BY = (H + G - 1) / G;
    int32_t *bstart = (int32_t *)calloc((size_t)BX * BY + 1, sizeof(int32_t));
    int32_t *blist = (int32_t *)malloc(sizeof(int32_t) * ncells);
    if (!bstart || !blist) { free(sx); free(sy); free(cf); free(bstart); free(blist); return 5; }
    for (int k = 0; k < ncells; k++) bstart[(sy[k] / G) * BX + sx[k] / G + 1]++;
    for (int i = 0; i < BX * BY; i++) bstart[i + 1] += bstart[i];
    {
        int32_t *fill = (int32_t *)malloc(sizeof(int32_t) * BX * BY);
        memcpy(fill, bstart, sizeof(int32_t) * BX * BY);
        for (int k = 0; k < ncells; k++) blist[fill[(sy[k] / G) * BX + sx[k] / G]++] = k;
        free(fill);
    }
    int maxring = BX > BY ? BX : BY;
#pragma omp parallel for schedule(dynamic, 16)
    for (int r = 0; r < H; r++) {
        int by = r / G;
        for (int c = 0; c < W; c++) {
            int bx = c / G;
            int64_t best = INT64_MAX;
            int bestk = -1;
            for (int ring = 0; ring <= maxring; ring++) {
                for (int yy = by - ring; yy <= by + ring; yy++) {
                    if (yy < 0 || yy >= BY) continue;
                    for (int xx = bx - ring; xx <= bx + ring; xx++) {
                        if (xx < 0 || xx >= BX) continue;
                        if (yy != by - ring && yy != by + ring && xx != bx - ring && xx != bx + ring)
                            continue; /* interior buckets were scanned at smaller rings */
                        int b = yy * BX + xx;
                        for (int q = bstart[b]; q < bstart[b + 1]; q++) {
                            int k = blist[q];
                            int64_t dx = sx[k] - c, dy = sy[k] - r;
                            int64_t d = dx * dx + dy * dy;
                            if (d < best || (d == best && k < bestk)) { best = d; bestk = k; }
                        }
                    }
                }
                /* any seed outside rings 0..ring is at distance > ring*G */
                int64_t lim = (int64_t)ring * G;
                if (bestk >= 0 && best <= lim * lim) break;
            }
            int64_t i = (int64_t)r * W + c;
            uint8_t v = cf[bestk];
            if ((uint32_t)(synth_hash(seed, 3, (uint64_t)i) >> 32) < thf) v ^= 1;
            out[i] = v;
        }
    }
    free(sx); free(sy); free(cf); free(bstart); free(blist);
    return 0;
}

/* C5a serpentine: even rows fully fg; odd row r has one connector pixel at
 * column W-1 if (r-1)/2 is even, else at column 0. */
void synth_serpentine(uint8_t *out, int H, int W)
{
#pragma omp parallel for schedule(static)
    for (int r = 0; r < H; r++) {
        uint8_t *row = out + (int64_t)r * W;
        if (r % 2 == 0) { memset(row, 1, W); continue; }
        memset(row, 0, W);
        row[(((r - 1) / 2) % 2 == 0) ? W - 1 : 0] = 1;
    }
}

/* C5b comb: fg at even columns for rows 0..H-2, plus row H-1 fully fg. */
void synth_comb(uint8_t *out, int H, int W)
{
#pragma omp parallel for schedule(static)
    for (int r = 0; r < H; r++) {
        uint8_t *row = out + (int64_t)r * W;
        if (r == H - 1) { memset(row, 1, W); continue; }
        for (int c = 0; c < W; c++) row[c] = (c % 2 == 0);
    }
}

void synth_fill(uint8_t *out, int H, int W, int value)
{
    memset(out, value, (size_t)H * W);
}

int synth_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
