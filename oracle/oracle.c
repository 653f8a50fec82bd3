/*
 * oracle/oracle.c — the CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this.  The product path
 * (paper_2402_01816_b200/) never calls, links or includes it, and this file
 * shares no code, header or constant with it.
 *
 * What it computes (§Definition of sorting, lines 121-142): the
 * *stable ascending* sort ("AscLeft": ties keep their input order left to
 * right) of contiguous binary64 keys, optionally moving a u32 payload with each
 * key.  Keys are ordered by IEEE `<`, so -0.0 == +0.0 and their relative order
 * is fixed by stability (reading R2).  NaN is rejected (reading R1,
 * SPEC.md:93 "NaN-like unordered keys rejected at ingestion").
 *
 * How (plain, slow, single-threaded, no tuning):
 *   - top-down binary divide&conquer mergesort with a 100% distant buffer
 *     allocated once before recursing (§Forgotten art);
 *   - split mid = lo + (hi-lo)/2 (reading R4);
 *   - Knuth's merge: the right run's head is taken only if it is strictly
 *     smaller than the left run's head, so the left run wins ties
 *     ("Knuthsort"; "left element wins ties");
 *   - the merged run is copied back from the buffer (no nocopy alternation,
 *     no insertion-sort cutoff: the plainest correct form).
 *   %RAM of this oracle is 2.0 (PAPER.md:26 formula, buffer = n elements).
 *
 * oracle_sort_target(): the four stable API targets of PAPER.md:137-142
 * (AscLeft, AscRight, DescLeft, DescRight), each written out as the same plain
 * mergesort with its own merge rule: the right run's head is taken iff it must
 * precede the left run's head in the target order, ties included for the
 * *Right targets (ties in reverse input order).  (NEXT f3.)
 *
 * oracle_sort_keys(): the same plain mergesort and per-target merge rule over
 * 8-byte keys of one of three types, given as bit patterns: binary64 under
 * IEEE < (kt 0; NaN rejected), two's-complement int64 (kt 1), uint64 (kt 2).
 * (NEXT f3, key types.)
 *
 * oracle_merge_runs(): one merge *level* of the same mergesort over runs of
 * length L ("per recursion-level one read-scan with comparisons ... and one
 * write-scan") — the definition a single GPU merge pass must
 * reproduce.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Knuth merge of a[lo:mid) and a[mid:hi) into t[lo:hi); left wins ties. */
static void merge_into(const double *k, const uint32_t *v, double *tk, uint32_t *tv,
                       size_t lo, size_t mid, size_t hi)
{
    size_t i = lo, j = mid, o = lo;
    while (i < mid && j < hi) {
        if (k[j] < k[i]) {               /* take right only if strictly smaller */
            tk[o] = k[j];
            if (v) tv[o] = v[j];
            ++j;
        } else {
            tk[o] = k[i];
            if (v) tv[o] = v[i];
            ++i;
        }
        ++o;
    }
    while (i < mid) { tk[o] = k[i]; if (v) tv[o] = v[i]; ++i; ++o; }
    while (j < hi) { tk[o] = k[j]; if (v) tv[o] = v[j]; ++j; ++o; }
}

static void msort(double *k, uint32_t *v, double *tk, uint32_t *tv, size_t lo, size_t hi)
{
    if (hi - lo <= 1) return;
    size_t mid = lo + (hi - lo) / 2;
    msort(k, v, tk, tv, lo, mid);
    msort(k, v, tk, tv, mid, hi);
    merge_into(k, v, tk, tv, lo, mid, hi);
    memcpy(k + lo, tk + lo, (hi - lo) * sizeof(double));
    if (v) memcpy(v + lo, tv + lo, (hi - lo) * sizeof(uint32_t));
}

/* target: 0 AscLeft, 1 AscRight, 2 DescLeft, 3 DescRight.  take_right(l, r):
 * the right head goes first.  AscLeft: r < l.  AscRight: r <= l.
 * DescLeft: r > l.  DescRight: r >= l. */
static int take_right(int target, double l, double r)
{
    switch (target) {
    case 1: return r <= l;
    case 2: return r > l;
    case 3: return r >= l;
    default: return r < l;
    }
}

static void merge_into_t(const double *k, const uint32_t *v, double *tk, uint32_t *tv,
                         size_t lo, size_t mid, size_t hi, int target)
{
    size_t i = lo, j = mid, o = lo;
    while (i < mid && j < hi) {
        if (take_right(target, k[i], k[j])) {
            tk[o] = k[j];
            if (v) tv[o] = v[j];
            ++j;
        } else {
            tk[o] = k[i];
            if (v) tv[o] = v[i];
            ++i;
        }
        ++o;
    }
    while (i < mid) { tk[o] = k[i]; if (v) tv[o] = v[i]; ++i; ++o; }
    while (j < hi) { tk[o] = k[j]; if (v) tv[o] = v[j]; ++j; ++o; }
}

static void msort_t(double *k, uint32_t *v, double *tk, uint32_t *tv, size_t lo, size_t hi, int target)
{
    if (hi - lo <= 1) return;
    size_t mid = lo + (hi - lo) / 2;
    msort_t(k, v, tk, tv, lo, mid, target);
    msort_t(k, v, tk, tv, mid, hi, target);
    merge_into_t(k, v, tk, tv, lo, mid, hi, target);
    memcpy(k + lo, tk + lo, (hi - lo) * sizeof(double));
    if (v) memcpy(v + lo, tv + lo, (hi - lo) * sizeof(uint32_t));
}

int oracle_sort_target(double *keys, uint32_t *vals, size_t n, int target)
{
    for (size_t i = 0; i < n; ++i)
        if (keys[i] != keys[i]) return 1;
    if (target < 0 || target > 3) return 3;
    if (n < 2) return 0;
    double *tk = (double *)malloc(n * sizeof(double));
    uint32_t *tv = vals ? (uint32_t *)malloc(n * sizeof(uint32_t)) : NULL;
    if (!tk || (vals && !tv)) { free(tk); free(tv); return 2; }
    msort_t(keys, vals, tk, tv, 0, n, target);
    free(tk);
    free(tv);
    return 0;
}

/* ---- 8-byte key types (bit patterns) ------------------------------------ */
/* -1 / 0 / +1 as a <, ==, > b in key type kt (0 f64, 1 i64, 2 u64). */
static int key_cmp(int kt, uint64_t a, uint64_t b)
{
    if (kt == 1) {
        int64_t x = (int64_t)a, y = (int64_t)b;
        return x < y ? -1 : (x > y ? 1 : 0);
    }
    if (kt == 2) return a < b ? -1 : (a > b ? 1 : 0);
    double x, y;
    memcpy(&x, &a, 8);
    memcpy(&y, &b, 8);
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* the right head r goes before the left head l in the target order */
static int take_right_k(int kt, int target, uint64_t l, uint64_t r)
{
    int c = key_cmp(kt, r, l);
    switch (target) {
    case 1: return c <= 0;
    case 2: return c > 0;
    case 3: return c >= 0;
    default: return c < 0;
    }
}

static void msort_k(uint64_t *k, uint32_t *v, uint64_t *tk, uint32_t *tv, size_t lo, size_t hi, int kt, int target)
{
    if (hi - lo <= 1) return;
    size_t mid = lo + (hi - lo) / 2;
    msort_k(k, v, tk, tv, lo, mid, kt, target);
    msort_k(k, v, tk, tv, mid, hi, kt, target);
    size_t i = lo, j = mid, o = lo;
    while (i < mid && j < hi) {
        if (take_right_k(kt, target, k[i], k[j])) {
            tk[o] = k[j];
            if (v) tv[o] = v[j];
            ++j;
        } else {
            tk[o] = k[i];
            if (v) tv[o] = v[i];
            ++i;
        }
        ++o;
    }
    while (i < mid) { tk[o] = k[i]; if (v) tv[o] = v[i]; ++i; ++o; }
    while (j < hi) { tk[o] = k[j]; if (v) tv[o] = v[j]; ++j; ++o; }
    memcpy(k + lo, tk + lo, (hi - lo) * sizeof(uint64_t));
    if (v) memcpy(v + lo, tv + lo, (hi - lo) * sizeof(uint32_t));
}

/* Returns 0, 1 on a NaN f64 key, 2 on OOM, 3 on a bad kt/target. */
int oracle_sort_keys(uint64_t *keys, uint32_t *vals, size_t n, int kt, int target)
{
    if (kt < 0 || kt > 2 || target < 0 || target > 3) return 3;
    if (kt == 0)
        for (size_t i = 0; i < n; ++i) {
            double x;
            memcpy(&x, &keys[i], 8);
            if (x != x) return 1;
        }
    if (n < 2) return 0;
    uint64_t *tk = (uint64_t *)malloc(n * sizeof(uint64_t));
    uint32_t *tv = vals ? (uint32_t *)malloc(n * sizeof(uint32_t)) : NULL;
    if (!tk || (vals && !tv)) { free(tk); free(tv); return 2; }
    msort_k(keys, vals, tk, tv, 0, n, kt, target);
    free(tk);
    free(tv);
    return 0;
}

/* Sorts keys[0:n) (and vals, if non-NULL) in place.
 * Returns 0 on success, 1 if a key is NaN (input untouched), 2 on OOM. */
int oracle_sort_f64_u32(double *keys, uint32_t *vals, size_t n)
{
    for (size_t i = 0; i < n; ++i)
        if (keys[i] != keys[i]) return 1;
    if (n < 2) return 0;
    double *tk = (double *)malloc(n * sizeof(double));
    uint32_t *tv = vals ? (uint32_t *)malloc(n * sizeof(uint32_t)) : NULL;
    if (!tk || (vals && !tv)) { free(tk); free(tv); return 2; }
    msort(keys, vals, tk, tv, 0, n);
    free(tk);
    free(tv);
    return 0;
}

/* One merge level: for q = 0,1,..: merges the sorted runs
 * in[2qL : 2qL+L) and in[2qL+L : 2qL+2L) (clipped to n) into out[2qL : ...).
 * Returns 0, or 1 on NaN. */
int oracle_merge_runs(const double *keys, const uint32_t *vals, size_t n, size_t L,
                      double *out_keys, uint32_t *out_vals)
{
    for (size_t i = 0; i < n; ++i)
        if (keys[i] != keys[i]) return 1;
    if (L == 0) return 1;
    for (size_t lo = 0; lo < n; lo += 2 * L) {
        size_t mid = lo + L < n ? lo + L : n;
        size_t hi = lo + 2 * L < n ? lo + 2 * L : n;
        merge_into(keys, vals, out_keys, out_vals, lo, mid, hi);
    }
    return 0;
}
