/*
 * synth/gen.c — seeded synthetic input generators (test/bench infrastructure).
 *
 * This module holds NONE of the method's arithmetic: no comparison, merge or
 * sort.  It only draws the inputs that both the oracle (oracle/) and the CUDA
 * path (paper_2402_01816_b200/) are run on, so the two sides see identical
 * bits.  Every generator is a pure function of (n, seed).
 *
 * PRNG: SplitMix64 (Steele, Lea, Flood 2014), one stream per (config, sub).
 *
 * Workload shapes follow the paper's measurement patterns
 * (§Methods and measurement) and BASELINE.json `configs`;
 * the concrete recipes are the readings listed in DESIGN.md §3 (SURVEY A10,
 * A11, A13, A14).
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t s; } sm64;

static inline uint64_t sm64_next(sm64 *g)
{
    uint64_t z = (g->s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* floor(x * m / 2^64): an unbiased-enough bounded draw in [0, m). */
static inline uint64_t bounded(uint64_t x, uint64_t m)
{
    return (uint64_t)(((unsigned __int128)x * m) >> 64);
}

/* Raw 64-bit stream (exported so tests can pin the PRNG to its published
 * first outputs). */
void gen_u64(uint64_t *out, size_t n, uint64_t seed)
{
    sm64 g = { seed };
    for (size_t i = 0; i < n; ++i) out[i] = sm64_next(&g);
}

/* U(0,1): u = (x >> 11) * 2^-53, exact on the 2^53 grid, never NaN (A13). */
void gen_uniform(double *out, size_t n, uint64_t seed)
{
    sm64 g = { seed };
    for (size_t i = 0; i < n; ++i)
        out[i] = (double)(sm64_next(&g) >> 11) * 0x1.0p-53;
}

/* Uniform random permutation of 0..n-1 as doubles (Fisher-Yates,
 * j = floor(x*(i+1)/2^64) for i = n-1 .. 1).  `permut`. */
void gen_permutation(double *out, size_t n, uint64_t seed)
{
    sm64 g = { seed };
    for (size_t i = 0; i < n; ++i) out[i] = (double)i;
    for (size_t i = n; i-- > 1;) {
        size_t j = (size_t)bounded(sm64_next(&g), (uint64_t)i + 1);
        double t = out[i]; out[i] = out[j]; out[j] = t;
    }
}

/* Heavy ties: integer uniform in [0, m) as double (A14); m = 24 at 2^24 is
 * `tielog2`. */
void gen_ties(double *out, size_t n, uint64_t seed, uint64_t m)
{
    sm64 g = { seed };
    for (size_t i = 0; i < n; ++i) out[i] = (double)bounded(sm64_next(&g), m);
}

/* `ascall` and `descall` on 0..n-1. */
void gen_ascending(double *out, size_t n)
{
    for (size_t i = 0; i < n; ++i) out[i] = (double)i;
}

void gen_descending(double *out, size_t n)
{
    for (size_t i = 0; i < n; ++i) out[i] = (double)(n - 1 - i);
}

/* Ascending 0..n-1 with 2*floor(n*permille/2000) distinct positions chosen by
 * a partial Fisher-Yates and swapped pairwise (A10: permille = 10 gives 1%). */
int gen_swapped(double *out, size_t n, uint64_t seed, unsigned permille)
{
    sm64 g = { seed };
    size_t npos = 2 * ((n * (size_t)permille) / 2000);
    for (size_t i = 0; i < n; ++i) out[i] = (double)i;
    if (npos < 2) return 0;
    size_t *idx = (size_t *)malloc(n * sizeof(size_t));
    if (!idx) return -1;
    for (size_t i = 0; i < n; ++i) idx[i] = i;
    for (size_t i = 0; i < npos; ++i) {             /* partial Fisher-Yates */
        size_t j = i + (size_t)bounded(sm64_next(&g), (uint64_t)(n - i));
        size_t t = idx[i]; idx[i] = idx[j]; idx[j] = t;
    }
    for (size_t i = 0; i + 1 < npos; i += 2) {
        double t = out[idx[i]]; out[idx[i]] = out[idx[i + 1]]; out[idx[i + 1]] = t;
    }
    free(idx);
    return 0;
}

/* `runs` ascending runs of consecutive integers with seeded random lengths,
 * concatenated in random order (A11).  runs-1 distinct cut points uniform in
 * [1, n-1] (rejection), runs shuffled by Fisher-Yates. */
int gen_runs(double *out, size_t n, uint64_t seed, unsigned runs)
{
    sm64 g = { seed };
    if (runs < 1 || (size_t)runs > n) runs = n ? (unsigned)(n < 16 ? n : 16) : 1;
    if (n == 0) return 0;
    size_t *cut = (size_t *)malloc((runs + 1) * sizeof(size_t));
    unsigned *ord = (unsigned *)malloc(runs * sizeof(unsigned));
    if (!cut || !ord) { free(cut); free(ord); return -1; }
    cut[0] = 0; cut[runs] = n;
    for (unsigned c = 1; c < runs; ++c) {
        for (;;) {
            size_t x = 1 + (size_t)bounded(sm64_next(&g), (uint64_t)(n - 1));
            int dup = 0;
            for (unsigned d = 1; d < c; ++d) dup |= (cut[d] == x);
            if (!dup) { cut[c] = x; break; }
        }
    }
    /* order the cut points (insertion; runs <= a few dozen) */
    for (unsigned a = 2; a < runs; ++a)
        for (unsigned b = a; b > 1 && cut[b - 1] > cut[b]; --b) {
            size_t t = cut[b]; cut[b] = cut[b - 1]; cut[b - 1] = t;
        }
    for (unsigned r = 0; r < runs; ++r) ord[r] = r;
    for (unsigned r = runs; r-- > 1;) {
        unsigned j = (unsigned)bounded(sm64_next(&g), (uint64_t)r + 1);
        unsigned t = ord[r]; ord[r] = ord[j]; ord[j] = t;
    }
    size_t o = 0;
    for (unsigned r = 0; r < runs; ++r)
        for (size_t v = cut[ord[r]]; v < cut[ord[r] + 1]; ++v) out[o++] = (double)v;
    free(cut); free(ord);
    return 0;
}

/* Paper patterns on the sqrt(n) block structure (
 * block length ceil(sqrt(n)) as SPEC.md:133 reads it).
 *  asclocal : values 0..n-1 shuffled, cut into blocks, each block ascending
 *  ascglobal: values 0..n-1 in ascending quantile blocks, each block permuted
 *  desc*    : mirrored. */
static size_t isqrt_ceil(size_t n)
{
    size_t r = 0;
    while (r * r < n) ++r;
    return r;
}

static void shuffle_range(double *a, size_t n, sm64 *g)
{
    for (size_t i = n; i-- > 1;) {
        size_t j = (size_t)bounded(sm64_next(g), (uint64_t)i + 1);
        double t = a[i]; a[i] = a[j]; a[j] = t;
    }
}

/* asclocal/desclocal: a uniformly random assignment of the values 0..n-1 to
 * the blocks (a shuffled multiset of block labels), then each block receives
 * its values in ascending (descending: reversed) order.  Same distribution as
 * "shuffle globally, then order each block", but needs no comparisons. */
int gen_pattern_local(double *out, size_t n, uint64_t seed, int descending)
{
    sm64 g = { seed };
    if (n == 0) return 0;
    size_t b = isqrt_ceil(n);
    size_t nblk = (n + b - 1) / b;
    uint32_t *label = (uint32_t *)malloc(n * sizeof(uint32_t));
    size_t *fill = (size_t *)calloc(nblk, sizeof(size_t));
    if (!label || !fill) { free(label); free(fill); return -1; }
    for (size_t i = 0; i < n; ++i) label[i] = (uint32_t)(i / b);
    for (size_t i = n; i-- > 1;) {
        size_t j = (size_t)bounded(sm64_next(&g), (uint64_t)i + 1);
        uint32_t t = label[i]; label[i] = label[j]; label[j] = t;
    }
    for (size_t v = 0; v < n; ++v) {
        size_t q = label[v], s = q * b, len = (s + b <= n) ? b : n - s;
        size_t o = fill[q]++;
        out[s + (descending ? len - 1 - o : o)] = (double)v;
    }
    free(label); free(fill);
    return 0;
}

int gen_pattern_global(double *out, size_t n, uint64_t seed, int descending)
{
    sm64 g = { seed };
    if (n == 0) return 0;
    size_t b = isqrt_ceil(n);
    for (size_t i = 0; i < n; ++i) out[i] = (double)i;
    if (descending) {
        /* quantile blocks in descending order: block q holds the q-th highest quantile */
        size_t o = 0;
        size_t nblk = (n + b - 1) / b;
        double *tmp = (double *)malloc(n * sizeof(double));
        if (!tmp) return -1;
        for (size_t q = nblk; q-- > 0;) {
            size_t s = q * b, e = (s + b <= n) ? s + b : n;
            for (size_t v = s; v < e; ++v) tmp[o++] = (double)v;
        }
        memcpy(out, tmp, n * sizeof(double));
        free(tmp);
    }
    for (size_t s = 0; s < n;) {
        /* block lengths follow the value quantiles, so recompute per block */
        size_t len = b;
        if (descending) {
            size_t nblk = (n + b - 1) / b;
            size_t last = n - (nblk - 1) * b;      /* the top quantile may be short */
            len = (s == 0) ? last : b;
        } else if (s + b > n) {
            len = n - s;
        }
        shuffle_range(out + s, len, &g);
        s += len;
    }
    return 0;
}

void gen_iota_u32(uint32_t *out, size_t n)
{
    for (size_t i = 0; i < n; ++i) out[i] = (uint32_t)i;
}
