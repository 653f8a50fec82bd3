// gns_kernels.cuh — sm_100a device code of the stable f64 mergesort hot path.
//
// Kernels (PAPER.md line cites in each):
//   K1    tile_sort2_kernel    (row a2) stable sort of one 8192-key tile per CTA,
//                              per-tile omission / reversal of ordered tiles (f2)
//   K2+K3 merge_tstore_kernel  (rows a3+a4) one merge level, src -> dst ping-pong,
//                              warp-specialised: sample-guided co-rank search
//                              warps, TMA producer, merge warps; also the
//                              two-run merge of the distributed sort (f4)
//   K2    partition_kernel     (row a3) stable co-rank split per output tile (for K4)
//   K4    merge_inplace_kernel (row a6) ordered in-place top merge of the limited-
//                              buffer modes (0.5 and p < 0.5, f1)
//         inplace_deps_kernel  (row a6) which earlier tiles each K4 tile must wait for
//         reverse_kernel       (f3) the Right targets
//         split_cuts_kernel    (f4) splitter cuts of the distributed sort
//         omit_plan_kernel, omit_prep_kernel, omit_final_kernel and the
//         list-driven merge_tstore_kernel<.., OL = true>
//                              (f2) the Omitsort / Octosort schedule
//         nan_count_kernel     GNS_DEBUG=1 pre-scan (R1)
// Keys of every type (f64, int64, uint64; f3) travel as 8-byte patterns; the
// template parameter ORD = direction | key type << 1 selects the order.
//
// No code here is shared with oracle/ (the CPU oracle); the two are compared
// only through their outputs.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

namespace gns {

// Debug build (make debug -> libgns_debug.so, GNS_LIB=libgns_debug.so): bounds
// assertions on every shared-memory slot, slice and bulk-copy range.
// compute-sanitizer is closed on this GPU pool, so these are the memory checks.
#ifdef GNS_DEBUG_BOUNDS
#define GNS_DASSERT(c)                                                                          \
    do {                                                                                        \
        if (!(c)) {                                                                             \
            printf("GNS_DASSERT failed %s:%d block %d thread %d\n", __FILE__, __LINE__,          \
                   (int)blockIdx.x, (int)threadIdx.x);                                          \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define GNS_DASSERT(c) \
    do {               \
    } while (0)
#endif

// Profiling build (make prof -> libgns_prof.so): thread 0 of each merge CTA
// accumulates clock64 phase times into g_prof (tools/prof_merge.py).
#ifdef GNS_PROF
__device__ unsigned long long g_prof[16];
// timeline: [launch slot][0] = min start, [1] = max end (globaltimer ns); slot 0 =
// tile sort, slot 1 + log2(L / TILE) = merge pass of run length L
__device__ unsigned long long g_tl[32][2];
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define GNS_TL_START(slot) do { if (threadIdx.x == 0) atomicMin(&g_tl[slot][0], gtimer()); } while (0)
#define GNS_TL_END(slot) do { if (threadIdx.x == 0) atomicMax(&g_tl[slot][1], gtimer()); } while (0)
#define GNS_PT(var) const long long var = clock64()
#define GNS_PADD(slot, v) acc[slot] += (unsigned long long)(v)
#else
#define GNS_PT(var) do {} while (0)
#define GNS_PADD(slot, v) do {} while (0)
#define GNS_TL_START(slot) do {} while (0)
#define GNS_TL_END(slot) do {} while (0)
#endif

constexpr int NT = 256;            // merge threads per CTA
constexpr int VT = 16;             // outputs per merge thread
constexpr int MTILE = NT * VT;     // K3/K4 output tile = 4096 elements
constexpr int MTILE_LOG2 = 12;
static_assert((1 << MTILE_LOG2) == MTILE, "MTILE_LOG2");
// tile-sort merge rounds inside one warp synchronise that warp only (K1 with
// payload here, key-only in gns_tile64.cuh); 0 = CTA barriers in every round
// merge passes wait for the previous launch (PDL) after their shared-memory
// prologue instead of at entry
#ifndef GNS_TMAP_PREFETCH
#define GNS_TMAP_PREFETCH 1
#endif
#ifndef GNS_LATE_PDL_WAIT
#define GNS_LATE_PDL_WAIT 1
#endif
#ifndef GNS_K1_WSYNC
#define GNS_K1_WSYNC 1
#endif
#ifndef GNS_NT1
#define GNS_NT1 256
#endif
constexpr int NT1 = GNS_NT1;       // K1 threads per CTA (three CTAs per SM key-only, two with payload)
#ifndef GNS_VT1
#define GNS_VT1 32
#endif
// K1 CTAs per SM: key-only 3 (80 registers, 3 x 67.5 KB shared: 2^24 keys
// tile sort 272 -> 249 us), with payload 2 (its 100 KB of shared memory)
#ifndef GNS_T1_MINB
#define GNS_T1_MINB (512 / GNS_NT1)
#endif
#ifndef GNS_T1_MINB_KEYS
#define GNS_T1_MINB_KEYS (768 / GNS_NT1)
#endif
constexpr int VT1 = GNS_VT1;       // K1 keys per thread
constexpr int TILE = NT1 * VT1;    // K1 tile = 8192 elements (runs entering the merge passes)
constexpr int TILE_LOG2 = TILE == 16384 ? 14 : TILE == 8192 ? 13 : 12;
static_assert((1 << TILE_LOG2) == TILE, "TILE must be 4096, 8192 or 16384");
static_assert(TILE % MTILE == 0, "pair boundaries must fall on merge-tile boundaries");

// ---------------------------------------------------------------- global I/O
// 256-bit vector accesses (LDG/STG.E.ENL2.256 on sm_100a).
__device__ __forceinline__ void st_v8(uint32_t *p, const uint32_t *u)
{
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]),
                    "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// ---- programmatic dependent launch (PDL): every kernel of a sort waits for
// its predecessor's completion before touching memory, and lets its successor
// be scheduled early, hiding the launch latency between the ~25 launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- mbarrier + TMA bulk copy (cp.async.bulk, SASS UBLKCP) helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n"
                 "GNS_WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra GNS_WAIT_%=;\n}"
                 :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
// TMA tensor store (2-D map over the key array viewed as [n/16][16] doubles,
// 128-byte swizzle) from shared memory, and its bulk-group completion.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, const void *src, int c0, int c1)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 :: "l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
// Shared-memory f64 load at a 32-bit shared address (volatile: two such loads
// under complementary predicates stay two predicated LDS instead of one LDS
// followed by four 32-bit selects).
__device__ __forceinline__ double lds_f64(uint32_t a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
// the same with an L2 cache-policy hint (evict-first for data read once)
__device__ __forceinline__ void tma_load_2d_hint(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar,
                                                 uint64_t policy)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                 " [%0], [%1, {%2, %3}], [%4], %5;"
                 :: "r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
__device__ __forceinline__ void lds128(const void *p, double &a, double &b)
{
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void lds128u(const void *p, uint32_t *u)
{
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void sts128u(void *p, const uint32_t *u)
{
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" :: "r"(smem_u32(p)), "r"(u[0]), "r"(u[1]), "r"(u[2]),
                 "r"(u[3]) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void sts128(void *p, double a, double b)
{
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" :: "r"(smem_u32(p)), "d"(a), "d"(b) : "memory");
}

// 1-D bulk copy global -> shared, completion counted on `bar` (16-byte aligned
// addresses, size a multiple of 16).  L2 evict-first: every byte is read once.
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                            uint64_t policy)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                 " [%0], [%1], %2, [%3], %4;"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
#ifndef GNS_LOAD_POLICY
#define GNS_LOAD_POLICY 0
#endif
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
#if GNS_LOAD_POLICY == 1
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#elif GNS_LOAD_POLICY == 2
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
    return p;
}

// ------------------------------------------------------------ merge device code
// Key order of the sort target: ascending (AscLeft) or
// descending (DescLeft); ties always keep input order (the left run wins).
// The *Right targets are the reversal of the opposite-direction Left target
// (gns.cu).  before<ORD>(x, y): x must be output strictly before y.
// ORD = DESC | (key type << 1): key types (NEXT f3) share the 8-byte layout;
// keys travel as double bit patterns and are compared as binary64 (GNS_KEY_F64,
// IEEE <: -0.0 == +0.0), two's-complement int64 (GNS_KEY_I64) or uint64
// (GNS_KEY_U64).
constexpr int KT_F64 = 0, KT_I64 = 1, KT_U64 = 2;
constexpr int ord_of(bool desc, int kt) { return (desc ? 1 : 0) | (kt << 1); }
template <int ORD>
__device__ __forceinline__ bool before(double x, double y)
{
    constexpr bool DESC = ORD & 1;
    constexpr int KT = ORD >> 1;
    if (KT == KT_I64) {
        const long long a = __double_as_longlong(x), b = __double_as_longlong(y);
        return DESC ? (a > b) : (a < b);
    } else if (KT == KT_U64) {
        const unsigned long long a = (unsigned long long)__double_as_longlong(x);
        const unsigned long long b = (unsigned long long)__double_as_longlong(y);
        return DESC ? (a > b) : (a < b);
    }
    return DESC ? (x > y) : (x < y);
}
// A key no real key sorts after (ties with it keep real keys first because
// pads are placed after every real key): +inf / -inf, INT64_MAX / MIN,
// UINT64_MAX / 0.
template <int ORD>
__device__ __forceinline__ double pad_key()
{
    constexpr bool DESC = ORD & 1;
    constexpr int KT = ORD >> 1;
    if (KT == KT_I64) return __longlong_as_double(DESC ? (long long)0x8000000000000000ULL : 0x7FFFFFFFFFFFFFFFLL);
    if (KT == KT_U64) return __longlong_as_double(DESC ? 0LL : (long long)0xFFFFFFFFFFFFFFFFULL);
    return __longlong_as_double(DESC ? (long long)0xFFF0000000000000ULL : 0x7FF0000000000000LL);
}

// ----------------------------------------------------------- merge geometry
// Pair q merges A_q = ak[q*2L : q*2L + na_q) with B_q = bk[q*2L : q*2L + nb_q)
// into out[q*2L : ...), na_q = min(L, n - 2qL), nb_q = clamp(n - 2qL - L, 0, L).
//   uniform pass : ak = src, bk = src + L, out = dst
//   in-place top merge (single = 1): ak = buffer, bk = data + nl, L = nl,
//                  out = data, one pair with na = nl, nb = n - nl
constexpr int SMP_LOG2_DEF = 9;   // = SMP_LOG2 (below): split-search sample spacing 512
struct MergeGeo {
    const double *ak;
    const uint32_t *av;
    const double *bk;
    const uint32_t *bv;
    double *ok;
    uint32_t *ov;
    long long n;
    long long L;
    int single;     // 1: one pair, A = ak[0:L), B = bk[0:n-L) (any lengths; the in-place top merge)
    int tpp;        // uniform pass: output tiles per pair, 2L / MTILE
    int tpp_log2;   // log2(tpp) if tpp is a power of two, else -1
    const double *sa;   // samples of the source region (key at every SMP_G-th position), or nullptr
    double *so;         // samples of the output region written by this pass, or nullptr
    const double *sb;   // single (two-run) geometry: samples of B (every SMP_G-th key of bk), or nullptr
    long long off = 0;  // single geometry: outputs [off, n) only; ok = the output of merge position off
    int so_log2 = SMP_LOG2_DEF;   // spacing of the output samples `so` (6 before a 4-way pass, gns_merge4.cuh)
};

struct TileSpan {
    long long g0, pbase;
    int na, nb, k0, k1;
};

__device__ __forceinline__ TileSpan tile_span(const MergeGeo &g, int t)
{
    TileSpan s;
    s.g0 = (long long)t * MTILE;
    if (g.single) {
        s.pbase = 0;
        s.na = (int)g.L;
        s.nb = (int)(g.n - g.L);
    } else {
        const long long span = 2 * g.L;
        const unsigned q = g.tpp_log2 >= 0 ? ((unsigned)t >> g.tpp_log2) : (unsigned)t / (unsigned)g.tpp;
        s.pbase = (long long)q * span;
        const long long rem = g.n - s.pbase;
        s.na = (int)min(g.L, rem);
        s.nb = (int)max(0LL, min(g.L, rem - g.L));
    }
    s.k0 = (int)(s.g0 - s.pbase + (g.single ? g.off : 0));
    // (64-bit: the last tile of a 2^31 - 1 element pair starts at 2^31 - 4096)
    s.k1 = (int)min((long long)s.k0 + MTILE, (long long)s.na + s.nb);
    return s;
}

// gns_merge_two into a destination that is not 32-byte aligned: the first
// `off` (<= 7) outputs of the stable merge (A first, left wins ties,
// PAPER.md:221), one thread; the pipelined merge writes the rest from dst + off.
template <bool HV, int ORD>
__global__ void merge_head_kernel(const double *A, const uint32_t *AV, long long la, const double *B,
                                  const uint32_t *BV, long long lb, double *dst, uint32_t *dv, int off)
{
    pdl_wait();
    if (threadIdx.x == 0) {
        long long i = 0, j = 0;
        for (int x = 0; x < off; ++x) {
            const bool tb = j < lb && (i >= la || before<ORD>(B[j], A[i]));
            dst[x] = tb ? B[j] : A[i];
            if (HV) dv[x] = tb ? BV[j] : AV[i];
            if (tb) ++j;
            else ++i;
        }
    }
    pdl_trigger();
}

// ---------------------------------------------------------- K2 partition
// One warp per output tile: the stable co-rank of the tile's first diagonal,
// found by a 32-ary search (each round probes 32 split points in parallel and
// keeps the interval between the last true and first false predicate), about
// 5 dependent rounds at L = 2^23 instead of 23 for a binary search.
// "parallelize over an arbitrary number of processes".
// Warp-cooperative stable co-rank of tile t's first diagonal (all 32 lanes
// return the result).
template <int ORD>
__device__ __forceinline__ int warp_corank(const MergeGeo &g, int t, int lane)
{
    const TileSpan s = tile_span(g, t);
    const double *A = g.ak + s.pbase;
    const double *B = g.bk + s.pbase;
    const int d = s.k0;
    int lo = max(0, d - s.nb), hi = min(d, s.na);
    while (lo < hi) {
        const int span = hi - lo;
        int m, nprobe;
        if (span <= 32) {
            m = lo + lane;
            nprobe = span;
        } else {
            m = lo + (int)(((long long)span * (lane + 1)) / 33);
            nprobe = 32;
        }
        bool p = false;
        if (lane < nprobe) p = !before<ORD>(B[d - 1 - m], A[m]);
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, p);
        const int c = __popc(bal);
        const int m_prev = __shfl_sync(0xFFFFFFFFu, m, (c > 0 ? c - 1 : 0));
        const int m_next = __shfl_sync(0xFFFFFFFFu, m, (c < nprobe ? c : 0));
        const int nlo = (c == 0) ? lo : m_prev + 1;
        const int nhi = (c == nprobe) ? hi : m_next;
        lo = nlo;
        hi = max(nlo, nhi);
    }
    return lo;
}

// ------------------------------------------- sample-guided co-rank search
// Every pass (and the tile sort) also writes the key at every SMP_G-th output
// position into a small sample array (n / 512 keys, L2-resident).  The next
// pass finds a split first on the samples -- Q(x) = A[x] <= B[y_lo(x)] with
// x a multiple of G and y_lo(x) = G * floor((d-1-x) / G), monotone in x --
// which brackets the co-rank c of diagonal d (d a multiple of G) in a window
// of 2G: Q(x) true  => A[x] <= B[d-1-x]          => c >= x + 1;
//        Q(x) false => B[d-1-x-G] <= B[y_lo(x)] < A[x] <= A[x+G] => c <= x + G.
// Then the exact search runs in that window (2 rounds of 33-ary probes),
// instead of ~5 rounds spread over the whole run.
constexpr int SMP_LOG2 = SMP_LOG2_DEF;
constexpr int SMP_G = 1 << SMP_LOG2;   // 512

// (W+1)-ary search of the last true of a monotone predicate over [lo, hi]
// (indices), by a group of W lanes; returns the number of trues in [lo, hi].
template <int W, class P>
__device__ __forceinline__ int group_count_true(int lo, int hi, int gl, unsigned mask, int gbase, P pred)
{
    // invariant: pred true on [lo0, lo), false on [hi, hi0]; answer in [lo, hi+1)
    const int lo0 = lo;
    hi += 1;
    while (lo < hi) {
        const int span = hi - lo;
        int m, nprobe;
        if (span <= W) {
            m = lo + gl;
            nprobe = span;
        } else {
            m = lo + (int)(((long long)span * (gl + 1)) / (W + 1));
            nprobe = W;
        }
        bool p = false;
        if (gl < nprobe) p = pred(m);
        const unsigned bal = (__ballot_sync(mask, p) & mask) >> gbase;
        const int c = __popc(bal);
        const int m_prev = __shfl_sync(mask, m, gbase + (c > 0 ? c - 1 : 0));
        const int m_next = __shfl_sync(mask, m, gbase + (c < nprobe ? c : 0));
        const int nlo = (c == 0) ? lo : m_prev + 1;
        const int nhi = (c == nprobe) ? hi : m_next;
        lo = nlo;
        hi = max(nlo, nhi);
    }
    return lo - lo0;
}

// Stable co-rank of tile t's first diagonal by a group of W lanes, sample-guided
// when the pass has samples (uniform passes), else over the whole range.
template <int W, int ORD>
__device__ __forceinline__ int tile_corank(const MergeGeo &g, int t, int gl, unsigned mask, int gbase)
{
    const TileSpan s = tile_span(g, t);
    const double *A = g.ak + s.pbase;
    const double *B = g.bk + s.pbase;
    const int d = s.k0;
    int lo = max(0, d - s.nb), hi = min(d, s.na);
    if (lo >= hi) return lo;
    if (g.sa != nullptr && (!g.single || g.sb != nullptr)) {
        const int s_lo = (lo + SMP_G - 1) >> SMP_LOG2;
        const int s_hi = (hi - 1) >> SMP_LOG2;
        if (s_lo <= s_hi) {
            const double *SA = g.sa + (s.pbase >> SMP_LOG2);
            const double *SB = g.single ? g.sb : g.sa + ((s.pbase + g.L) >> SMP_LOG2);
            const int cnt = group_count_true<W>(s_lo, s_hi, gl, mask, gbase, [&](int sx) {
                const int yb = (d - 1 - (sx << SMP_LOG2)) >> SMP_LOG2;
                return !before<ORD>(SB[yb], SA[sx]);
            });
            if (cnt > 0) lo = max(lo, ((s_lo + cnt - 1) << SMP_LOG2) + 1);
            if (s_lo + cnt <= s_hi) hi = min(hi, ((s_lo + cnt) << SMP_LOG2) + SMP_G);
        }
    }
    // exact: number of m in [lo, hi) with A[m] <= B[d-1-m]
    return lo + group_count_true<W>(lo, hi - 1, gl, mask, gbase,
                                    [&](int m) { return !before<ORD>(B[d - 1 - m], A[m]); });
}

// One group of PW lanes per tile (PW = 32: one warp; 16 / 8: two / four tiles
// per warp, fewer waves of latency-bound searches).
template <int ORD, int PW = 32>
__global__ void __launch_bounds__(256)
partition_kernel(MergeGeo g, int ntiles, int *__restrict__ corank)
{
    pdl_wait();
    pdl_trigger();
    const int t = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) / PW);
    const int lane = threadIdx.x & 31;
    const int gl = lane % PW, gbase = lane - gl;
    const unsigned mask = PW == 32 ? 0xFFFFFFFFu : ((1u << PW) - 1u) << gbase;
    if (t >= ntiles) return;
    const int c = tile_corank<PW, ORD>(g, t, gl, mask, gbase);   // sample-guided if g has samples
    if (gl == 0) corank[t] = c;
}

// Samples of the two runs of an in-place top merge (every SMP_G-th key of
// each), so its partition can run the sample-guided split search.
__global__ void __launch_bounds__(256)
gather_samples_kernel(const double *a, long long na, double *sa, const double *b, long long nb, double *sb)
{
    pdl_wait();
    pdl_trigger();
    const long long ca = (na + SMP_G - 1) >> SMP_LOG2, cb = (nb + SMP_G - 1) >> SMP_LOG2;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ca + cb; i += (long long)gridDim.x * blockDim.x) {
        if (i < ca) sa[i] = a[i << SMP_LOG2];
        else sb[i - ca] = b[(i - ca) << SMP_LOG2];
    }
}

// ---------------------------------------------- K4 dependency ranges (row a6)
// In the in-place top merge, output tile t writes data[k0:k1); tile u reads
// B = data[L + j0(u) : L + j1(u)).  Tile t may only write once every earlier
// tile u < t whose read range intersects its write range has loaded its
// inputs (later tiles never intersect: k1(t) <= L + j1(t) <= L + j0(u)).
// deps[t] = {u_lo, u_hi} (empty if u_lo > u_hi).
__device__ __forceinline__ long long j_start(const int *corank, int u)
{
    return (long long)u * MTILE - corank[u];
}

__global__ void __launch_bounds__(256)
inplace_deps_kernel(const int *__restrict__ corank, int ntiles, long long L, long long n, int2 *deps,
                    unsigned *flags)
{
    pdl_wait();
    pdl_trigger();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    flags[t] = 0u;           // flags[0:ntiles) = "loaded", flags[ntiles] = ticket counter
    if (t == ntiles) return;
    const long long k0 = (long long)t * MTILE;
    const long long k1 = min(k0 + MTILE, n);
    // u_lo: first u in [0,t) with L + j1(u) > k0, where j1(u) = j_start(u+1)
    int lo = 0, hi = t;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (L + j_start(corank, m + 1) > k0) hi = m;
        else lo = m + 1;
    }
    const int u_lo = lo;
    // u_hi: last u in [0,t) with L + j0(u) < k1
    lo = 0;
    hi = t;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (L + j_start(corank, m) < k1) lo = m + 1;
        else hi = m;
    }
    deps[t] = make_int2(u_lo, lo - 1);
}

// ------------------------------------------------ K3 pipelined (persistent)
// The production merge pass.  A persistent grid (2 CTAs per SM) walks the
// output tiles t = blockIdx.x, +gridDim.x, ...; each CTA double-buffers its
// tiles in shared memory: while all 256 threads merge tile i from one stage,
// the TMA engine (cp.async.bulk, issued by one thread) streams the inputs of
// tile i+1 -- exactly A[i0:i1) and B[j0:j1), from the co-ranks -- into the
// other stage, so HBM reads run continuously under the merge arithmetic.
// Keys arrive by TMA tensor loads of whole 128-byte rows (16 keys) in boxes of
// KROWS rows, with the 128-byte swizzle (16-byte chunk c of stage row r at
// chunk c ^ (r & 7)), so stride-16 reads (threads at neighbouring 16-output
// segments of a copy-like tile: ties, presorted data) spread over the banks
// instead of hitting one.  A's rows fill stage rows [0, RA), B's rows start at
// row RA (a multiple of KROWS); key slot s = 16 * stage row + column.  Rows past
// an array's last full row are out of the map (zero filled); their few real
// keys are patched by the merge warps from global memory.  Vals keep 1-D bulk
// copies into their own region (slot = base + (g mod 4) + ..., so every copy
// is 16-byte aligned; at most three vals at an unaligned array end are read
// with plain loads).
// rows per key box: 32 (4 KB) key-only, 16 (2 KB) with payload (shared
// memory for two CTAs per SM); fewer, larger boxes measured faster
constexpr int krows(bool hv) { return hv ? 16 : 32; }
// stage key rows: >= 4096/16 + 4 + 2 * (krows - 1), rounded up to a multiple of krows
constexpr int stage_key_rows(bool hv) { return ((MTILE / 16 + 4 + 2 * (krows(hv) - 1)) + krows(hv) - 1) / krows(hv) * krows(hv); }
constexpr int PIPE_VSLOTS = MTILE + 128;

// key slot s of a stage whose 1 KiB-aligned base is `base` (shared address)
__device__ __forceinline__ uint32_t stage_addr(uint32_t base, int s)
{
    const uint32_t b = 8u * (uint32_t)s;
    return base + (b ^ ((b >> 3) & 0x70u));
}

struct PipeGeo {
    MergeGeo g;
    const double *a_lim;   // end of the array holding the A runs (keys)
    const double *b_lim;   // end of the array holding the B runs (keys)
    long long a_idx0;      // element index of g.ak[0] in the A key map's array
    long long b_idx0;      // element index of g.bk[0] in the B key map's array
    long long a_rows;      // full 16-key rows of the A map (row a_rows is patched by hand)
    long long b_rows;
    int coop = 0;          // merge_tstore_kernel: 1 = the whole producer warp issues a tile's TMA boxes
                           // (one box per lane), 0 = one lane issues them all
};

struct PipeMeta {
    int t, ca, cb;
    int offa, bslot;       // key slots of A[0], B[0]
    int voffa, vbslot;     // val slots of A[0], B[0]
    int pa_slot, pa_cnt;   // A keys at slots [pa_slot, +pa_cnt) to patch from pa_src
    int pb_slot, pb_cnt;
    const double *pa_src;
    const double *pb_src;
};

// Thread-0 side: computes tile t's input slices and issues their copies into
// the stage (keys at sk, vals at sv), completing on `bar`.
template <bool HV>
__device__ __forceinline__ void pipe_issue(const PipeGeo &pg, const CUtensorMap &amap, const CUtensorMap &bmap,
                                           int t, int i0, int i1next, double *sk, uint32_t *sv, uint64_t *bar,
                                           PipeMeta *meta, uint64_t policy, int ln = -1)
{
    // ln >= 0: called by all 32 lanes of a warp (lane ln); lane 0 posts the
    // byte count, writes the meta and arrives, lane b issues key box b.
    const bool coop = ln >= 0;
    const bool lead = !coop || ln == 0;
    const MergeGeo &g = pg.g;
    const TileSpan s = tile_span(g, t);
    const int cnt = s.k1 - s.k0;
    int i1 = (s.k1 == s.na + s.nb) ? s.na : i1next;
    i1 = min(min(max(max(i1, i0), s.k1 - s.nb), i0 + cnt), s.na);
    const int j0 = s.k0 - i0;
    const int ca = i1 - i0, cb = cnt - ca;
    const double *Ak = g.ak + s.pbase + i0;
    const double *Bk = g.bk + s.pbase + j0;
    const uint32_t *Av = HV ? g.av + s.pbase + i0 : nullptr;
    const uint32_t *Bv = HV ? g.bv + s.pbase + j0 : nullptr;
    GNS_DASSERT(i0 >= 0 && ca >= 0 && cb >= 0 && i0 + ca <= s.na && j0 >= 0 && j0 + cb <= s.nb);
    // ---- keys: rows [r0, r1] of the slice, boxes of KROWS rows
    const long long ga = pg.a_idx0 + s.pbase + i0, gb = pg.b_idx0 + s.pbase + j0;
    constexpr int KROWS = krows(HV);
    const int nba = ca > 0 ? (int)((((ga + ca - 1) >> 4) - (ga >> 4)) / KROWS) + 1 : 0;
    const int nbb = cb > 0 ? (int)((((gb + cb - 1) >> 4) - (gb >> 4)) / KROWS) + 1 : 0;
    const int rb0 = nba * KROWS;                                   // B's first stage row
    GNS_DASSERT(rb0 + nbb * KROWS <= stage_key_rows(HV));
    // ---- vals: 1-D bulk copies (16-byte chunks of 4) + plain loads at an unaligned end
    const int voffa = HV ? (int)(((uintptr_t)Av >> 2) & 3) : 0;
    const int voffb = HV ? (int)(((uintptr_t)Bv >> 2) & 3) : 0;
    const int vbbase = (voffa + ca + 3) & ~3;
    auto vrange = [&](const double *K, int c, int off, const double *lim, int &vs, int &ve) {
        const long long avail = lim - K;           // elements readable
        vs = -off;
        ve = vs + ((c - vs + 3) & ~3);
        if (ve > avail) ve = vs + (int)((avail - vs) & ~3LL);
    };
    uint32_t total = (uint32_t)(nba + nbb) * (KROWS * 128u);
    int vsa = 0, vea = 0, vsb = 0, veb = 0;
    if (HV) {
        if (ca > 0) vrange(Ak, ca, voffa, pg.a_lim, vsa, vea);
        if (cb > 0) vrange(Bk, cb, voffb, pg.b_lim, vsb, veb);
        if (vea > vsa) total += (uint32_t)(vea - vsa) * 4u;
        if (veb > vsb) total += (uint32_t)(veb - vsb) * 4u;
    }
    // Post the expected byte count first (no arrival yet), then issue.
    if (lead) mbar_expect_tx(bar, total);
    if (coop) {
        GNS_DASSERT(nba + nbb <= 32);
        __syncwarp();
        if (ln < nba)
            tma_load_2d_hint(sk + ln * KROWS * 16, &amap, 0, (int)((ga >> 4) + ln * KROWS), bar, policy);
        else if (ln - nba < nbb)
            tma_load_2d_hint(sk + (rb0 + (ln - nba) * KROWS) * 16, &bmap, 0, (int)((gb >> 4) + (ln - nba) * KROWS),
                             bar, policy);
        if (!lead) return;
    } else {
        for (int b = 0; b < nba; ++b)
            tma_load_2d_hint(sk + b * KROWS * 16, &amap, 0, (int)((ga >> 4) + b * KROWS), bar, policy);
        for (int b = 0; b < nbb; ++b)
            tma_load_2d_hint(sk + (rb0 + b * KROWS) * 16, &bmap, 0, (int)((gb >> 4) + b * KROWS), bar, policy);
    }
    if (HV) {
        if (vea > vsa) tma_load_1d(sv + voffa + vsa, Av + vsa, (uint32_t)(vea - vsa) * 4u, bar, policy);
        for (int e = max(vea, 0); e < ca; ++e) sv[voffa + e] = Av[e];
        if (veb > vsb) tma_load_1d(sv + vbbase + voffb + vsb, Bv + vsb, (uint32_t)(veb - vsb) * 4u, bar, policy);
        for (int e = max(veb, 0); e < cb; ++e) sv[vbbase + voffb + e] = Bv[e];
    }
    PipeMeta mt;
    mt.t = t;
    mt.ca = ca;
    mt.cb = cb;
    mt.offa = (int)(ga & 15);
    mt.bslot = rb0 * 16 + (int)(gb & 15);
    mt.voffa = voffa;
    mt.vbslot = vbbase + voffb;
    // keys past the last full row of a map (out of the box, zero filled)
    auto patch = [&](long long gi, int c, int slot0, long long rows, const double *src, int &pslot, int &pcnt,
                     const double *&psrc) {
        const long long lim = rows * 16;
        pcnt = 0;
        pslot = 0;
        psrc = src;
        if (c > 0 && gi + c > lim) {
            const int e0 = (int)max(0LL, lim - gi);
            pcnt = c - e0;
            pslot = slot0 + e0;
            psrc = src + e0;
        }
    };
    patch(ga, ca, mt.offa, pg.a_rows, Ak, mt.pa_slot, mt.pa_cnt, mt.pa_src);
    patch(gb, cb, mt.bslot, pg.b_rows, Bk, mt.pb_slot, mt.pb_cnt, mt.pb_src);
    *meta = mt;
    // The stage's phase completes only after this arrive (the barrier expects
    // one arrival) and the copies' bytes: everything written above by this
    // thread (meta, unaligned tail vals) is released to the waiters.
    mbar_arrive(bar);
}

// Merge-warp side, after the stage's full barrier: copy the keys the TMA box
// could not deliver (past a map's last full row; at most 15 per run, only at
// an array end) into their swizzled slots, then sync the merge warps.
__device__ __forceinline__ void stage_patch(uint32_t kbase, const PipeMeta &mt, int tid)
{
    if ((mt.pa_cnt | mt.pb_cnt) == 0) return;
    if (tid < mt.pa_cnt)
        asm volatile("st.shared.f64 [%0], %1;" :: "r"(stage_addr(kbase, mt.pa_slot + tid)), "d"(mt.pa_src[tid])
                     : "memory");
    if (tid < mt.pb_cnt)
        asm volatile("st.shared.f64 [%0], %1;" :: "r"(stage_addr(kbase, mt.pb_slot + tid)), "d"(mt.pb_src[tid])
                     : "memory");
    asm volatile("bar.sync 1, %0;" :: "n"(NT) : "memory");
}

// Stable co-rank (merge path) of diagonal d for the stage's runs (key slots
// A: a0.., B: b0..): the number of A keys among the first d outputs, A wins
// ties.  Predicate: A[m] <= B[d-1-m].
template <int ORD>
__device__ __forceinline__ int merge_path_stage(uint32_t kbase, int a0, int na, int b0, int nb, int d)
{
    int lo = max(0, d - nb), hi = min(d, na);
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        const double bk = lds_f64(stage_addr(kbase, b0 + d - 1 - m));
        const double ak = lds_f64(stage_addr(kbase, a0 + m));
        if (!before<ORD>(bk, ak)) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// Serial merge of VT outputs from the stage, starting at key slots ai (A) and
// bi (B), run ends aend / bend (exclusive).  B's head is taken only if
// strictly before A's (left wins ties).  The consumed side's next key is
// loaded straight into its head register (predicated loads); reads at most
// one slot past a run end (the value is never used).
template <bool HV, int ORD>
__device__ __forceinline__ void serial_merge_stage(uint32_t kbase, const uint32_t *sv, const PipeMeta &mt, int ai,
                                                   int aend, int bi, int bend, double (&k)[VT], uint32_t (&v)[VT])
{
    // (A's slots precede B's when A is non-empty; an empty A may sit anywhere)
    GNS_DASSERT(ai >= 0 && bi >= 0 && (ai >= aend || aend <= bend) && bend <= stage_key_rows(HV) * 16 &&
                aend <= stage_key_rows(HV) * 16);
    double ka = lds_f64(stage_addr(kbase, ai)), kb = lds_f64(stage_addr(kbase, bi));
#pragma unroll
    for (int x = 0; x < VT; ++x) {
        const bool p = (bi < bend) && ((ai >= aend) || before<ORD>(kb, ka));
        k[x] = p ? kb : ka;
        const int src = p ? bi : ai;
        if (HV) v[x] = sv[src < mt.bslot ? src - mt.offa + mt.voffa : src - mt.bslot + mt.vbslot];
        const int nxt = src + 1;
        GNS_DASSERT(nxt < stage_key_rows(HV) * 16);
        const uint32_t a = stage_addr(kbase, nxt);
        if (p) {
            bi = nxt;
            kb = lds_f64(a);
        } else {
            ai = nxt;
            ka = lds_f64(a);
        }
    }
}


// ------------------------------- shared pieces of the fused merge kernels
#ifndef GNS_SEARCH_WARPS
#define GNS_SEARCH_WARPS 2
#endif
constexpr int SEARCH_WARPS = GNS_SEARCH_WARPS;
constexpr int SPL_RING = 64;

__device__ __forceinline__ void bar_merge_warps() { asm volatile("bar.sync 1, %0;" :: "n"(NT) : "memory"); }

// ---------------------------- K2+K3 fused: the production merge pass (row a3+a4)
// A persistent grid (2 CTAs per SM); CTA c owns the contiguous output tiles
// [first, last) of 4096 keys, so it needs the co-rank splits at first..last
// only (tile t ends where t+1 starts).  Warp roles (warp-specialised, no
// CTA-wide barrier inside the tile loop):
//   warps 0-7  merge: each thread merges 16 outputs of the tile in stage
//              i % NS (merge path + serial merge, left wins ties), then writes
//              them into the same stage as the output staging box;
//   warp 8     producer (one lane): issues the TMA bulk copies (cp.async.bulk,
//              UBLKCP) of exactly A[i0:i1) and B[j0:j1) into a free stage,
//              and the TMA tensor store (UTMASTG) of each staged tile;
//   warps 9-10 search: run ahead computing the splits (two concurrent 16-lane
//              17-ary searches per warp, predicate A[m] <= B[d-1-m]) into a
//              shared ring; at kernel start warps 0-7 compute the first splits.
// Keys and vals of global element g share one shared slot (offset g mod 4) so
// every copy is 16-byte aligned.  Stage hand-off: full[st] (producer -> merge
// warps, tx-count of the bulk copies) and staged[st] (8 merge-warp arrivals ->
// producer, after the swizzled output box is in shared memory).  The producer
// reuses a stage for tile i+NS once the store of tile i has read it out.
// Staging: thread t writes its 16 outputs (= row t of a [256][16] double box)
// with conflict-free st.shared.v2 into the 128-byte-swizzled layout; one
// cp.async.bulk.tensor stores the 32 KB tile.  Vals (if any) are stored by the
// merge threads with 256-bit stores.
constexpr size_t ts_key_bytes(bool hv) { return (size_t)stage_key_rows(hv) * 128; }   // 43,008 / 38,912 B
constexpr size_t TS_VAL_BYTES = ((size_t)PIPE_VSLOTS * 4 + 1023) / 1024 * 1024;
constexpr size_t ts_stage_bytes(bool hv) { return ts_key_bytes(hv) + (hv ? TS_VAL_BYTES : 0); }
constexpr size_t ts_smem(bool hv, int ns = 2) { return ns * ts_stage_bytes(hv) + 1024; }
constexpr int MERGE_WARPS = NT / 32;                 // 8
constexpr int PRODUCER_WARP = MERGE_WARPS;           // 8
// NEXT f2 adaptivity of the full-buffer sort, decided on the device from the
// tile sort's flag word (bit 0: some descent, bit 1: some adjacent pair not
// strictly reversed).  The host schedules, per merge pass, what an ordered or
// strictly reversed input needs instead of the merge: a copy of the tile
// sort's output into this pass's destination (pre_*) and, for a reversed
// input, a tile-order reversal (gather) or a copy (rev_*).
struct Adapt {
    const unsigned *flag;         // nullptr: no adaptivity
    const double *pre_k;          // ordered input: copy source, or nullptr
    const uint32_t *pre_v;
    const double *rev_k;          // strictly reversed input: source, or nullptr
    const uint32_t *rev_v;
    int rev_gather;               // 1: out[j] = tile-sorted src at 2tT + c_t - n + j; 0: plain copy
    int run_log2 = TILE_LOG2;     // log2 T: the tile sort's run length (TILE, or a K1 cluster's C x TILE)
};

// The CTA's share of the output [lo, hi).  gather: the stable sort of a
// strictly reversed input is its reversal; tile t of src holds input tile t
// sorted (= reversed), so out[j] = src[2tT + c_t - n + j] with
// t = (n-1-j) / T and c_t = min(T, n - tT) (contiguous within each tile).
template <bool HV>
__device__ void adapt_move(const MergeGeo &g, int per_cta, const double *sk, const uint32_t *sv, bool gather,
                           int rl)
{
    const long long n = g.n;
    const long long lo = (long long)blockIdx.x * per_cta * MTILE;
    const long long hi = min(n, lo + (long long)per_cta * MTILE);
    for (long long j = lo + threadIdx.x; j < hi; j += blockDim.x) {
        long long s = j;
        if (gather) {
            const long long t = (n - 1 - j) >> rl;
            const long long c = min(1LL << rl, n - (t << rl));
            s = 2 * (t << rl) + c - n + j;
        }
        g.ok[j] = sk[s];
        if (HV) g.ov[j] = sv[s];
    }
}

constexpr int WS_THREADS = NT + 32 + 32 * SEARCH_WARPS;   // 352

// NEXT f2 Omitsort (OL = true): the pass merges only the tiles listed in
// ol.tiles[0:*ol.count) (ascending; every tile of a listed pair), split
// evenly over the grid on the device.  Bit 31 (OMIT_DIR) of an entry selects the
// direction: 0 = pg (data -> buffer) with omap/amap/bmap, 1 = ol.pg1 (buffer
// -> data) with omap1/amap1/bmap1.
constexpr unsigned OMIT_DIR = 1u << 31;        // list-entry bit: buffer -> data
struct OmitList {
    const int *tiles;
    const int *count;
    PipeGeo pg1;
};

// Chained uniform passes of a full-buffer sort (no griddepcontrol.wait): the
// pass triggers its dependent launch at start, its CTAs start as the previous
// pass's CTAs exit, and every tile waits -- before its co-rank search reads
// anything -- until the previous pass has stored its pair region
// [q 2L, (q+1) 2L) (dep[q] counts the stored previous-pass tiles there; it
// also covers the write-after-read hazard on this pass's output, which the
// previous pass read within the same region).  At exit the producer adds
// the CTA's tiles to this pass's counters, per next-pass region of 4L
// (sig), after its last store completed.  Deadlock-free: a pass launches
// only once every CTA of the previous one has started (PDL trigger at start),
// so every region it waits on belongs to resident CTAs.
struct Chain {
    const unsigned *dep;     // previous pass's region counters, or nullptr (griddepcontrol.wait)
    unsigned *sig;           // this pass's region counters, or nullptr (last pass)
};
__device__ __forceinline__ void red_release_add(unsigned *p, unsigned v)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void chain_wait(const Chain &ch, const MergeGeo &g, int t)
{
    const long long span = 2 * g.L;
    const long long q = ((long long)t * MTILE) / span;
    const long long lo = q * span, hi = min(g.n, lo + span);
    const unsigned want = (unsigned)((hi - lo + MTILE - 1) / MTILE);
    while (ld_acquire(ch.dep + q) < want) __nanosleep(64);
}

template <bool HV, int ORD, int NS = 2, bool OL = false>
__global__ void __launch_bounds__(WS_THREADS, 2)
merge_tstore_kernel(PipeGeo pg, int ntiles, int per_cta, const __grid_constant__ CUtensorMap omap,
                    const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, Adapt ad,
                    const OmitList ol, const __grid_constant__ CUtensorMap omap1,
                    const __grid_constant__ CUtensorMap amap1, const __grid_constant__ CUtensorMap bmap1, Chain ch)
{
#ifdef GNS_PROF
    unsigned long long acc[16] = {};
    const long long t_entry = clock64();
    const int tl_slot = min(31, 1 + (63 - __clzll(pg.g.L)) - TILE_LOG2);
#endif
    const bool chained = !OL && ch.dep != nullptr;
    // The previous launch's results are first read below the shared-memory
    // set-up (the list-driven variant reads its list before): waiting for it
    // there lets a CTA that starts early do its prologue meanwhile.
    constexpr bool LATE_WAIT = GNS_LATE_PDL_WAIT && !OL;
    if (chained) pdl_trigger();          // (the next pass may launch once every CTA of this one started)
    else if (!LATE_WAIT) pdl_wait();
    GNS_TL_START(tl_slot);
    extern __shared__ __align__(16) unsigned char smem_raw0[];
    // 1 KiB alignment for the swizzled TMA boxes; pointer arithmetic (not an
    // integer round trip) keeps the shared address space visible to ptxas.
    unsigned char *smem_raw = smem_raw0 + ((1024u - (smem_u32(smem_raw0) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t full[NS];
    __shared__ __align__(8) uint64_t staged[NS];
    __shared__ PipeMeta meta[NS];
    __shared__ int spl[SPL_RING];
    __shared__ volatile int spl_tag[SPL_RING];
    __shared__ volatile int spl_used;
    auto skb = [&](int st) { return reinterpret_cast<double *>(smem_raw + st * ts_stage_bytes(HV)); };
    auto svb = [&](int st) {
        return reinterpret_cast<uint32_t *>(smem_raw + st * ts_stage_bytes(HV) + ts_key_bytes(HV));
    };
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    int nlist = ntiles;
    if (OL) {
        nlist = *ol.count;
        per_cta = (nlist + (int)gridDim.x - 1) / (int)gridDim.x;
    }
    const int first = blockIdx.x * per_cta;
    const int last = min(first + per_cta, nlist);
    const int m = last - first;
    if (m <= 0) return;
    // the CTA's j-th tile; j = m: the tile after its last one (its split ends the last tile)
    auto entry = [&](int j) -> int { return ol.tiles[first + min(j, m - 1)]; };
    auto tile_of = [&](int j) -> int {
        if (!OL) return first + j;
        const int e = (int)((unsigned)entry(j) & ~OMIT_DIR);
        return j < m ? e : e + 1;
    };
    // direction of the CTA's j-th tile (j = m: the last tile's)
    auto rev = [&](int j) -> bool { return OL && ((unsigned)entry(j) & OMIT_DIR) != 0u; };
    auto geo = [&](int j) -> const PipeGeo & { return rev(j) ? ol.pg1 : pg; };
    const int nspl = (tile_of(m - 1) + 1 < ntiles) ? m + 1 : m;
    for (int j = tid; j < SPL_RING; j += WS_THREADS) spl_tag[j] = -1;
    if (GNS_TMAP_PREFETCH && tid == 32) {
        // the tensor maps are launch parameters: their descriptors can be
        // fetched before the previous launch has finished
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&omap)) : "memory");
    }
    if (tid == 0) {
#pragma unroll
        for (int b = 0; b < NS; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&staged[b], MERGE_WARPS);
        }
        fence_mbar_init();
        spl_used = 0;
    }
    __syncthreads();
    if (LATE_WAIT && !chained) pdl_wait();
    // NEXT f2 flag word: loaded now, tested after the first split searches
    // (which only read), so its latency hides behind them
    const unsigned f_adapt = ad.flag ? *(volatile const unsigned *)ad.flag : 3u;
#ifdef GNS_PROF
    const long long t_flag = clock64();
#endif
    auto publish = [&](int j, int c) {
        spl[j % SPL_RING] = c;
        __threadfence_block();
        spl_tag[j % SPL_RING] = j;
    };
    // the first splits: every warp computes one (32-lane sample-guided search)
    const int init = min(nspl, WS_THREADS / 32);
    const bool adapt = (f_adapt & 1u) == 0u || (f_adapt & 2u) == 0u;
    if (warp < init && !(chained && adapt)) {
        if (chained) {
            if (lane == 0) chain_wait(ch, geo(warp).g, tile_of(warp));
            __syncwarp();
        }
        const int c = tile_corank<32, ORD>(geo(warp).g, tile_of(warp), lane, 0xFFFFFFFFu, 0);
        if (lane == 0) publish(warp, c);
    }
#ifdef GNS_PROF
    const long long t_split0 = clock64();
    long long t_full0 = 0;
#endif
    if ((f_adapt & 1u) == 0u || (f_adapt & 2u) == 0u) {
        // NEXT f2: the whole input was already in order (no descent: every
        // merge is an omission, "Omitsort"), or strictly
        // reversed (its stable sort is the reversal).
        // Only the steps the host scheduled for this pass move data.
        const bool pre = (f_adapt & 1u) == 0u;
        const double *ck = pre ? ad.pre_k : ad.rev_k;
        const uint32_t *cv = pre ? ad.pre_v : ad.rev_v;
        if (chained) pdl_wait();          // (the moves read the previous pass's moves: full completion)
        if (ck) adapt_move<HV>(pg.g, per_cta, ck, cv, !pre && ad.rev_gather, ad.run_log2);
        pdl_trigger();
        return;
    }
    __syncthreads();      // the first splits are published

    if (warp > PRODUCER_WARP) {
        // ------------------------------------------------ search warps
        const int sw = warp - PRODUCER_WARP - 1;
        const int h = lane >> 4, gl = lane & 15;
        const unsigned mask = 0xFFFFu << (16 * h);
        for (int j0 = init + 2 * sw; j0 < nspl; j0 += 2 * SEARCH_WARPS) {
            const int j = j0 + h;
            while (j0 + 1 - spl_used >= SPL_RING) { __nanosleep(64); }
            if (j < nspl) {
                if (chained) {
                    if (gl == 0) chain_wait(ch, geo(j).g, tile_of(j));
                    __syncwarp(mask);
                }
                const int c = tile_corank<16, ORD>(geo(j).g, tile_of(j), gl, mask, 16 * h);
                if (gl == 0) publish(j, c);
            }
            __syncwarp();
        }
        return;
    }

    if (warp == PRODUCER_WARP) {
        // ------------------------------------------------ producer (one lane, or the
        // whole warp issuing the loads with pg.coop; stores and their waits stay on lane 0)
        if (!pg.coop && lane != 0) return;
        const int pln = pg.coop ? lane : -1;
        const uint64_t policy = policy_evict_first();
        auto get_split = [&](int j) -> int {
#ifdef GNS_PROF
            const long long a = clock64();
            while (spl_tag[j % SPL_RING] != j) { }
            acc[8] += clock64() - a;
#else
            while (spl_tag[j % SPL_RING] != j) { }
#endif
            return spl[j % SPL_RING];
        };
        auto issue = [&](int i) {
            const int st = i % NS;
            const bool r = rev(i);
            const int s0 = get_split(i);
            const int s1 = (i + 1 < nspl) ? get_split(i + 1) : 0;
            if (chained) fence_proxy_async_global();   // the region's stores (acquired by a search lane) before our loads
            pipe_issue<HV>(geo(i), r ? amap1 : amap, r ? bmap1 : bmap, tile_of(i), s0, s1, skb(st), svb(st),
                           &full[st], &meta[st], policy, pln);
            if (lane == 0) spl_used = i;
        };
        for (int i = 0; i < NS && i < m; ++i) issue(i);
#ifdef GNS_PROF
        GNS_PADD(0, clock64() - t_entry);
#endif
        for (int i = 0; i < m; ++i) {
            const int st = i % NS;
            GNS_PT(p0);
            mbar_wait(&staged[st], (uint32_t)((i / NS) & 1));     // tile i staged by the 8 merge warps
            GNS_PT(p1);
            GNS_PADD(1, p1 - p0);
            if (pg.g.n - pg.g.off >= 16 && lane == 0) {   // (< 16 outputs: no full row; the merge warps stored the partial row)
                tma_store_2d(rev(i) ? &omap1 : &omap, skb(st), 0, (int)((long long)tile_of(i) * (MTILE / 16)));
                bulk_commit();
            }
            if (i + NS < m) {
                if (lane == 0) bulk_wait_read0();                  // stage st read out -> reusable
                if (pg.coop) __syncwarp();
                GNS_PT(p2);
                GNS_PADD(5, p2 - p1);
                issue(i + NS);
                GNS_PT(p3);
                GNS_PADD(6, p3 - p2);
            }
        }
        if (lane == 0) bulk_wait0();
        if (!OL && ch.sig != nullptr && lane == 0) {
            // this CTA's stored tiles, per next-pass region of 4L
            __threadfence();
            const long long span = 4 * pg.g.L;
            long long t = first;
            while (t < last) {
                const long long r = (t * MTILE) / span;
                const long long tend = min((long long)last, ((r + 1) * span + MTILE - 1) / MTILE);
                red_release_add(ch.sig + r, (unsigned)(tend - t));
                t = tend;
            }
        }
#ifdef GNS_PROF
        atomicMax(&g_tl[tl_slot][1], gtimer());
        acc[7] = clock64() - t_entry;
        acc[9] = m;
        acc[10] = 1;
        if (lane == 0)
            for (int q = 0; q < 11; ++q) atomicAdd(&g_prof[q], acc[q]);
#endif
        pdl_trigger();
        return;
    }

    // ---------------------------------------------------- merge warps 0-7
    const long long n = pg.g.n - pg.g.off;           // outputs of this launch (from ok)
    const long long full_rows = n >> 4;              // rows stored by TMA; a partial last row is stored by hand
    for (int i = 0; i < m; ++i) {
        const int st = i % NS;
        mbar_wait(&full[st], (uint32_t)((i / NS) & 1));
#ifdef GNS_PROF
        if (i == 0) t_full0 = clock64();
#endif
        const PipeMeta mt = meta[st];
        const int cnt = mt.ca + mt.cb;
        const int d = min(tid * VT, cnt);
        double *sk = skb(st);
        const uint32_t *sv = svb(st);
        const uint32_t kbase = smem_u32(sk);
        stage_patch(kbase, mt, tid);
        double k[VT];
        uint32_t v[VT];
        const int ii = merge_path_stage<ORD>(kbase, mt.offa, mt.ca, mt.bslot, mt.cb, d);
        serial_merge_stage<HV, ORD>(kbase, sv, mt, mt.offa + ii, mt.offa + mt.ca, mt.bslot + d - ii, mt.bslot + mt.cb, k,
                                    v);
        const long long t = tile_of(i);
        const MergeGeo &G = geo(i).g;
        const long long row = t * (MTILE / 16) + tid;    // global row of this thread's 16 outputs
        if (G.so != nullptr && (tid & ((1 << (G.so_log2 - 4)) - 1)) == 0 && d < cnt)
            G.so[(row * 16) >> G.so_log2] = k[0];     // sample of output position row*16
        bar_merge_warps();                               // stage st fully read
        unsigned char *rowp = reinterpret_cast<unsigned char *>(sk) + tid * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) sts128(rowp + ((c ^ (tid & 7)) << 4), k[2 * c], k[2 * c + 1]);
        fence_proxy_async();
        if (HV) {
            const int mv = cnt - d;
            if (mv >= VT) {
#pragma unroll
                for (int x = 0; x < VT; x += 8) st_v8(G.ov + row * 16 + x, &v[x]);
            } else {
#pragma unroll
                for (int x = 0; x < VT; ++x)
                    if (x < mv) G.ov[row * 16 + x] = v[x];
            }
        }
        if (row == full_rows && d < cnt) {                  // the partial last row (n % 16 != 0)
#pragma unroll
            for (int x = 0; x < VT; ++x)
                if (x < cnt - d) G.ok[row * 16 + x] = k[x];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&staged[st]);
    }
#ifdef GNS_PROF
    if (tid == 0) {
        atomicAdd(&g_prof[11], (unsigned long long)(t_flag - t_entry));
        atomicAdd(&g_prof[12], (unsigned long long)(t_split0 - t_entry));
        atomicAdd(&g_prof[13], (unsigned long long)(t_full0 - t_entry));
        atomicAdd(&g_prof[14], (unsigned long long)(clock64() - t_entry));
    }
#endif
    pdl_trigger();
}


// ------------------------------------------------- K1 v2: TMA-fed tile sort
// 256 threads x 32 keys (TILE = 8192).  The tile arrives by TMA tensor
// load (2-D maps: keys [n/16][16] f64, vals [n/32][32] u32, 128-byte swizzle)
// and leaves by one TMA tensor store; the blocked register<->smem transfers
// use 16-byte accesses in the swizzled layout.  In registers: one stable
// odd-even transposition sort of the thread's 32 keys; then log2(8192/32) = 8
// shared-memory merge rounds (merge path + serial merge, left wins ties).
// With 32 outputs per thread the merge-path searches per key are halved vs 16.
constexpr size_t T1_KEY_BYTES = TILE * 8 + 1024;
constexpr size_t T1_VAL_BYTES = TILE * 4 + 1024;
constexpr size_t t1_smem(bool hv) { return T1_KEY_BYTES + (hv ? T1_VAL_BYTES : 0) + 1024; }

// merge-round layouts (blocked spill e = 32t + x and merge reads conflict-light)
__device__ __forceinline__ int swm(int e) { return e ^ ((e >> 5) & 15); }
// Tile-sort key layout on absolute shared byte addresses (the key array is
// 1 KiB aligned): the 8-byte slot within each 128-byte line is XORed with bits
// 8-11 of the address (the 32-key row), so the blocked spill (thread t writes
// row t) and stride-16 merge reads spread over the banks.  Working on byte
// addresses saves the index->address shift in the merge steps.
__device__ __forceinline__ uint32_t swa(uint32_t a) { return a ^ ((a >> 5) & 0x78u); }
struct SwM { __device__ __forceinline__ int operator()(int e) const { return swm(e); } };
// Stable co-rank over the tile-sort layout (keys at swa(base + 8e)); A wins ties.
template <int ORD>
__device__ __forceinline__ int merge_path_tile(uint32_t base, int a0, int na, int b0, int nb, int d)
{
    int lo = max(0, d - nb), hi = min(d, na);
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        const double b = lds_f64(swa(base + 8u * (b0 + d - 1 - m)));
        const double a = lds_f64(swa(base + 8u * (a0 + m)));
        if (!before<ORD>(b, a)) lo = m + 1;
        else hi = m;
    }
    return lo;
}
// TMA 128-byte swizzle layouts (16-byte chunk c of row r stored at chunk c ^ (r & 7))
__device__ __forceinline__ int tk_slot(int e)     // doubles, 16 per row
{
    const int r = e >> 4;
    return (r << 4) | ((((e >> 1) & 7) ^ (r & 7)) << 1) | (e & 1);
}
__device__ __forceinline__ int tv_slot(int e)     // u32, 32 per row
{
    const int r = e >> 5;
    return (r << 5) | ((((e >> 2) & 7) ^ (r & 7)) << 2) | (e & 3);
}

// Stable odd-even transposition sort of k[O:O+N) (adjacent compare-exchange,
// swap only if the right key is strictly before the left one).
template <int O, int N, bool HV, int ORD>
__device__ __forceinline__ void transpose_sort(double (&k)[VT1], uint32_t (&v)[VT1])
{
#pragma unroll
    for (int r = 0; r < N; ++r) {
#pragma unroll
        for (int i = r & 1; i + 1 < N; i += 2) {
            const bool p = before<ORD>(k[O + i + 1], k[O + i]);
            const double lo = p ? k[O + i + 1] : k[O + i];
            const double hi = p ? k[O + i] : k[O + i + 1];
            k[O + i] = lo;
            k[O + i + 1] = hi;
            if (HV) {
                const uint32_t vl = p ? v[O + i + 1] : v[O + i];
                const uint32_t vh = p ? v[O + i] : v[O + i + 1];
                v[O + i] = vl;
                v[O + i + 1] = vh;
            }
        }
    }
}


// Serial merge of VT1 outputs for the tile sort's merge rounds.  Heads ka/kb,
// indices ai/bi; B's head is taken only if strictly before A's (left wins
// ties).  The next key of the consumed side is loaded straight into that
// side's head register (predicated loads), so a step costs one compare, two
// selects for the output, the index update and the swizzled address.
template <bool HV, int ORD>
__device__ __forceinline__ void serial_merge32(const double *sk, const uint32_t *sv, int ai, int aend, int bi, int bend,
                                               double (&k)[VT1], uint32_t (&v)[VT1])
{
    GNS_DASSERT(ai >= 0 && bi >= ai && bend <= TILE);
    const uint32_t base = smem_u32(sk);
    // heads as (unswizzled) byte addresses; guards compare addresses
    uint32_t pa = base + 8u * ai, pb = base + 8u * bi;
    const uint32_t pae = base + 8u * aend, pbe = base + 8u * bend;
    double ka = lds_f64(swa(pa)), kb = lds_f64(swa(pb));
#pragma unroll
    for (int x = 0; x < VT1; ++x) {
        const bool p = (pb < pbe) && ((pa >= pae) || before<ORD>(kb, ka));
        k[x] = p ? kb : ka;
        const uint32_t src = p ? pb : pa;
        // vals sit at the keys' swizzled slot positions (4 bytes per slot):
        // byte offset = (swizzled key byte offset) / 2
        if (HV) v[x] = sv[(swa(src) - base) >> 3];
        const uint32_t nxt = src + 8u;
        GNS_DASSERT(nxt >= base && nxt <= base + 8u * TILE);
        const uint32_t a = swa(nxt);
        if (p) {
            pb = nxt;
            kb = lds_f64(a);
        } else {
            pa = nxt;
            ka = lds_f64(a);
        }
    }
}

template <bool HV, int ORD>
__global__ void __launch_bounds__(NT1, HV ? GNS_T1_MINB : GNS_T1_MINB_KEYS)
tile_sort2_kernel(const double *src_k, const uint32_t *src_v, double *dst_k, uint32_t *dst_v, long long n,
                  const __grid_constant__ CUtensorMap ksrc, const __grid_constant__ CUtensorMap vsrc,
                  const __grid_constant__ CUtensorMap kdst, const __grid_constant__ CUtensorMap vdst,
                  unsigned *unsorted, double *smp, unsigned char *tdesc, double *smp_src)
{
    pdl_wait();
    GNS_TL_START(0);
    extern __shared__ __align__(16) unsigned char smem_raw0[];
    unsigned char *smem = smem_raw0 + ((1024u - (smem_u32(smem_raw0) & 1023u)) & 1023u);
    double *sk = reinterpret_cast<double *>(smem);
    uint32_t *sv = reinterpret_cast<uint32_t *>(smem + T1_KEY_BYTES);
    __shared__ __align__(8) uint64_t bar;
    __shared__ unsigned s_flags;
    const int tid = threadIdx.x;
    const long long tile = blockIdx.x;
    if (tid == 0) s_flags = 0;
    const long long base = tile * TILE;
    const int cnt = (int)min((long long)TILE, n - base);
    const bool full = cnt == TILE;
    double k[VT1];
    uint32_t v[VT1];
    if (full) {
        if (tid == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
            mbar_expect_tx(&bar, (uint32_t)(TILE * 8 + (HV ? TILE * 4 : 0)));
#pragma unroll
            for (int b = 0; b < TILE / 4096; ++b) {          // boxes of 256 rows
                tma_load_2d(sk + b * 4096, &ksrc, 0, (int)(tile * (TILE / 16) + b * 256), &bar);
                if (HV && (b & 1) == 0)
                    tma_load_2d(sv + b * 4096, &vsrc, 0, (int)(tile * (TILE / 32) + (b / 2) * 256), &bar);
            }
            mbar_arrive(&bar);
        }
        __syncthreads();
        mbar_wait(&bar, 0);
#pragma unroll
        for (int c = 0; c < VT1 / 2; ++c) lds128(sk + tk_slot(tid * VT1 + 2 * c), k[2 * c], k[2 * c + 1]);
        if (HV) {
#pragma unroll
            for (int c = 0; c < VT1 / 4; ++c) lds128u(sv + tv_slot(tid * VT1 + 4 * c), &v[4 * c]);
        }
    } else {
        __syncthreads();                   // s_flags initialised (the full path has its own barrier)
#pragma unroll
        for (int x = 0; x < VT1; ++x) {
            const int e = tid * VT1 + x;
            const bool ok = e < cnt;
            // pads sort after every real key (+inf ascending, -inf descending;
            // real infinities come first among ties because pads are last)
            k[x] = ok ? src_k[base + e] : pad_key<ORD>();
            if (HV) v[x] = ok ? src_v[base + e] : 0u;
        }
    }
    const int e0 = tid * VT1;
    // NEXT f2 (Omitsort's omitted merges; Octosort's reversal of
    // descending runs), per tile: is the tile already in
    // order (no key must move before its predecessor), or strictly reversed
    // (every key strictly before its predecessor; its stable sort is its
    // reversal)?  Each thread checks its real keys and the key after them.
    // The same tests across tile boundaries feed the whole-input flag word
    // (bit 0: some descent, bit 1: some pair not strictly reversed).
    int mode = 0;          // 0 sort, 1 tile in order (omit), 2 tile strictly reversed (reverse)
    {
        // one compare per adjacent pair: "descent" = next strictly before
        // current; in order <=> no descent, strictly reversed <=> all descents
        int pairs = 0, desc = 0;
#pragma unroll
        for (int x = 0; x + 1 < VT1; ++x) {
            if (e0 + x + 1 < cnt) {
                ++pairs;
                desc += before<ORD>(k[x + 1], k[x]) ? 1 : 0;
            }
        }
        unsigned fl = 0;       // bit 0/1: in-tile some descent / some non-descent; bit 2/3: across the tile end
        const long long nx = base + e0 + VT1;
        if (nx < n) {
            const double kn = (full && e0 + VT1 < TILE) ? sk[tk_slot(e0 + VT1)] : src_k[nx];
            const bool d = before<ORD>(kn, k[VT1 - 1]);
            fl |= (e0 + VT1 < cnt) ? (d ? 1u : 2u) : (d ? 4u : 8u);
        }
        fl |= (desc > 0 ? 1u : 0u) | (desc < pairs ? 2u : 0u);
        fl = __reduce_or_sync(0xFFFFFFFFu, fl);
        if (lane_id() == 0 && fl) atomicOr(&s_flags, fl);
        __syncthreads();
        fl = s_flags;
        mode = !(fl & 1u) ? 1 : (!(fl & 2u) && full) ? 2 : 0;
        if (unsorted && tid == 0) {
            const unsigned g = ((fl | (fl >> 2)) & 3u);   // whole-input flag word (see merge_tstore_kernel)
            if (g) atomicOr(unsorted, g);
        }
    }
    if (mode == 0) {
    // the thread's 32 keys: one stable odd-even transposition sort in
    // registers (trades ALU, which has headroom, for the shared-memory round
    // that merged two sorted halves: measured -1.6 %)
    transpose_sort<0, VT1, HV, ORD>(k, v);
    __syncthreads();                       // the TMA-layout reads are done before the first spill
#pragma unroll 1
    for (int coop = 2; coop <= NT1; coop <<= 1) {
#pragma unroll
        for (int x = 0; x < VT1; ++x) {
            *reinterpret_cast<double *>(reinterpret_cast<unsigned char *>(sk) +
                                        (swa(smem_u32(sk) + 8u * (e0 + x)) - smem_u32(sk))) = k[x];
            if (HV) sv[(swa(smem_u32(sk) + 8u * (e0 + x)) - smem_u32(sk)) >> 3] = v[x];
        }
        // a pair of <= 32 threads lies inside one warp (its spills, its reads
        // and the swizzle, which stays inside a 128-byte line): the first
        // five rounds synchronise the warp only
        const bool wsync = GNS_K1_WSYNC && coop <= 32;
        if (wsync) __syncwarp();
        else __syncthreads();
        {
            const int local = tid & (coop - 1);
            const int a0 = (tid - local) * VT1;
            const int run = (coop >> 1) * VT1;
            const int b0 = a0 + run;
            const int d = local * VT1;
            const int i = merge_path_tile<ORD>(smem_u32(sk), a0, run, b0, run, d);
            serial_merge32<HV, ORD>(sk, sv, a0 + i, b0, b0 + d - i, b0 + run, k, v);
        }
        if (wsync) __syncwarp();
        else __syncthreads();
    }
    } else {
        __syncthreads();                   // the TMA-layout reads are done before the staging writes
    }
    // Omitsort schedule (tdesc != nullptr): per tile bit 0 = kept as a
    // descending run, bit 1 = written to dst (not in src's region)
    if (tdesc != nullptr && tid == 0)
        tdesc[tile] = (unsigned char)((mode == 2 ? 1 : 0) | ((mode == 0 && dst_k != src_k) ? 2 : 0));
    if (tdesc != nullptr && mode != 0) {
        // Omitsort / Octosort (NEXT f2): a tile in order,
        // or strictly reversed (a descending run: its reversal is its stable
        // sort), stays where it is; only its samples are written
        if (smp_src != nullptr && e0 < cnt && (tid & (SMP_G / VT1 - 1)) == 0)
            smp_src[(base + e0) >> SMP_LOG2] = k[0];
        GNS_TL_END(0);
        pdl_trigger();
        return;
    }
    if (mode == 2) {
        // full tile, strictly reversed: output position TILE-1-e gets input e
#pragma unroll
        for (int c = 0; c < VT1 / 2; ++c) sts128(sk + tk_slot(TILE - 2 - e0 - 2 * c), k[2 * c + 1], k[2 * c]);
        if (HV) {
#pragma unroll
            for (int c = 0; c < VT1 / 4; ++c) {
                const uint32_t r[4] = {v[4 * c + 3], v[4 * c + 2], v[4 * c + 1], v[4 * c]};
                sts128u(sv + tv_slot(TILE - 4 - e0 - 4 * c), r);
            }
        }
        fence_proxy_async();
        __syncthreads();
        if (smp != nullptr && (tid & (SMP_G / VT1 - 1)) == 0)
            smp[(base + e0) >> SMP_LOG2] = sk[tk_slot(e0)];
        if (tid == 0) {
#pragma unroll
            for (int b = 0; b < TILE / 4096; ++b) {
                tma_store_2d(&kdst, sk + b * 4096, 0, (int)(tile * (TILE / 16) + b * 256));
                if (HV && (b & 1) == 0) tma_store_2d(&vdst, sv + b * 4096, 0, (int)(tile * (TILE / 32) + (b / 2) * 256));
            }
            bulk_commit();
            bulk_wait_read0();
        }
        GNS_TL_END(0);
        pdl_trigger();
        return;
    }
    if (smp != nullptr && e0 < cnt && (tid & (SMP_G / VT1 - 1)) == 0)
        smp[(base + e0) >> SMP_LOG2] = k[0];          // sample of output position base + e0
    if (mode == 1 && dst_k == src_k) {                // in place and in order: nothing moves (Omitsort)
        GNS_TL_END(0);
        pdl_trigger();
        return;
    }
    if (full) {
#pragma unroll
        for (int c = 0; c < VT1 / 2; ++c) sts128(sk + tk_slot(e0 + 2 * c), k[2 * c], k[2 * c + 1]);
        if (HV) {
#pragma unroll
            for (int c = 0; c < VT1 / 4; ++c) sts128u(sv + tv_slot(e0 + 4 * c), &v[4 * c]);
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int b = 0; b < TILE / 4096; ++b) {
                tma_store_2d(&kdst, sk + b * 4096, 0, (int)(tile * (TILE / 16) + b * 256));
                if (HV && (b & 1) == 0) tma_store_2d(&vdst, sv + b * 4096, 0, (int)(tile * (TILE / 32) + (b / 2) * 256));
            }
            bulk_commit();
            bulk_wait_read0();
        }
    } else {
#pragma unroll
        for (int x = 0; x < VT1; ++x) {
            const int e = e0 + x;
            if (e < cnt) {
                dst_k[base + e] = k[x];
                if (HV) dst_v[base + e] = v[x];
            }
        }
    }
    GNS_TL_END(0);
    pdl_trigger();
}


// ------------------------- K4 v2: pipelined ordered in-place top merge (row a6)
// The 0.5 mode's last merge: A = the buffer (left half, sorted), B = data[nl:n)
// (right half, sorted), output = data[0:n).  Persistent CTAs claim output
// tiles in atomic-ticket order (so every claimed tile belongs to a running
// CTA), load each tile's inputs by TMA bulk copies (co-ranks precomputed by
// partition_kernel) into a double-buffered stage and publish flags[t]
// (st.release.gpu) as soon as that load has landed.  Before a tile's outputs
// are stored (TMA tensor store of the keys, 256-bit stores of the vals), the
// tile waits (ld.acquire.gpu) on the flags of the earlier tiles whose B read
// range intersects its write range (deps[], inplace_deps_kernel).  Later tiles
// never intersect: k1(t) <= nl + j1(t) <= nl + j0(u) for u > t.  Deadlock-free:
// the smallest tile in flight only depends on tiles whose loads have landed.
template <bool HV, int ORD>
__global__ void __launch_bounds__(NT + 32, 2)
merge_inplace_kernel(PipeGeo pg, int ntiles, const int *__restrict__ corank, const int2 *__restrict__ deps,
                     unsigned *flags, unsigned *ticket, const __grid_constant__ CUtensorMap omap,
                     const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, Adapt ad)
{
    pdl_wait();
    if (ad.flag) {
        // NEXT f2 (as in merge_tstore_kernel): ordered or strictly reversed input
        const unsigned f = *(volatile const unsigned *)ad.flag;
        if ((f & 1u) == 0u || (f & 2u) == 0u) {
            const bool pre = (f & 1u) == 0u;
            const double *ck = pre ? ad.pre_k : ad.rev_k;
            const uint32_t *cv = pre ? ad.pre_v : ad.rev_v;
            const int per = (ntiles + gridDim.x - 1) / gridDim.x;
            if (ck) adapt_move<HV>(pg.g, per, ck, cv, !pre && ad.rev_gather, ad.run_log2);
            pdl_trigger();
            return;
        }
    }
    extern __shared__ __align__(16) unsigned char smem_raw0[];
    unsigned char *smem_raw = smem_raw0 + ((1024u - (smem_u32(smem_raw0) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t full[2];
    __shared__ __align__(8) uint64_t staged[2];
    __shared__ PipeMeta meta[2];
    auto skb = [&](int st) { return reinterpret_cast<double *>(smem_raw + st * ts_stage_bytes(HV)); };
    auto svb = [&](int st) {
        return reinterpret_cast<uint32_t *>(smem_raw + st * ts_stage_bytes(HV) + ts_key_bytes(HV));
    };
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&staged[b], MERGE_WARPS);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == PRODUCER_WARP) {
        // ---------------------------------------- producer (lane 0): tickets, loads, stores
        if (lane != 0) return;
        const uint64_t policy = policy_evict_first();
        // claim a tile in ticket order and load it into stage st, or tell the
        // merge warps there is none left (meta.t = ntiles, arrival without bytes)
        // the next ticket and its co-ranks are fetched one tile ahead, so the
        // atomic and the two loads are off the stage-refill path (claiming a
        // ticket before loading it keeps ticket order: every tile still only
        // waits on smaller tickets, and the smallest unfinished tile has its
        // dependencies' loads landed)
        int pf = (int)atomicAdd(ticket, 1u);
        int pf_i0 = pf < ntiles ? corank[pf] : 0;
        int pf_i1 = pf + 1 < ntiles ? corank[pf + 1] : 0;
        auto claim = [&](int st) -> bool {
            const int c = pf;
            if (c < ntiles) {
                pipe_issue<HV>(pg, amap, bmap, c, pf_i0, pf_i1, skb(st), svb(st), &full[st], &meta[st], policy);
                pf = (int)atomicAdd(ticket, 1u);
                if (pf < ntiles) {
                    pf_i0 = corank[pf];
                    pf_i1 = pf + 1 < ntiles ? corank[pf + 1] : 0;
                }
                return true;
            }
            meta[st].t = ntiles;
            mbar_arrive(&full[st]);
            return false;
        };
        bool more = claim(0) && claim(1);
        for (int i = 0;; ++i) {
            const int st = i & 1;
            mbar_wait(&staged[st], (uint32_t)((i >> 1) & 1));    // merged, deps waited, staged
            const int t = meta[st].t;
            if (t >= ntiles) break;
            fence_proxy_async_global();
            tma_store_2d(&omap, skb(st), 0, t * (MTILE / 16));
            bulk_commit();
            bulk_wait_read0();                                    // stage st read out -> reusable
            if (more) more = claim(st);
            else {                                                // no tile for this stage: end marker
                meta[st].t = ntiles;
                mbar_arrive(&full[st]);
            }
        }
        bulk_wait0();
        pdl_trigger();
        return;
    }

    // -------------------------------------------------------- merge warps 0-7
    const long long n = pg.g.n;
    const long long full_rows = n >> 4;
    for (int i = 0;; ++i) {
        const int st = i & 1;
        mbar_wait(&full[st], (uint32_t)((i >> 1) & 1));
        const PipeMeta mt = meta[st];
        const int t = mt.t;
        if (t >= ntiles) {                                      // end: let the producer see it too
            __syncwarp();
            if (lane == 0) mbar_arrive(&staged[st]);
            break;
        }
        if (tid == 0 && flags) st_release(flags + t, 1u);      // inputs of tile t are in shared memory
        const int cnt = mt.ca + mt.cb;
        const int d = min(tid * VT, cnt);
        double *sk = skb(st);
        const uint32_t *sv = svb(st);
        const uint32_t kbase = smem_u32(sk);
        stage_patch(kbase, mt, tid);
        double k[VT];
        uint32_t v[VT];
        const int ii = merge_path_stage<ORD>(kbase, mt.offa, mt.ca, mt.bslot, mt.cb, d);
        serial_merge_stage<HV, ORD>(kbase, sv, mt, mt.offa + ii, mt.offa + mt.ca, mt.bslot + d - ii, mt.bslot + mt.cb, k,
                                    v);
        const long long row = (long long)t * (MTILE / 16) + tid;
        if (pg.g.so != nullptr && (tid & ((1 << (pg.g.so_log2 - 4)) - 1)) == 0 && d < cnt)
            pg.g.so[(row * 16) >> pg.g.so_log2] = k[0];         // sample of output position row*16
        bar_merge_warps();                                     // stage st fully read
        unsigned char *rowp = reinterpret_cast<unsigned char *>(sk) + tid * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) sts128(rowp + ((c ^ (tid & 7)) << 4), k[2 * c], k[2 * c + 1]);
        fence_proxy_async();
        if (deps) {
            // wait until every earlier tile that reads B slots we overwrite has loaded
            const int2 dp = deps[t];
            GNS_DASSERT(dp.x >= 0 && dp.y < t);
            for (int u = dp.x + tid; u <= dp.y; u += NT)
                while (ld_acquire(flags + u) == 0u) { __nanosleep(32); }
            bar_merge_warps();                                 // every dependency seen by some merge thread
            fence_proxy_async_global();
        }
        if (HV) {
            const int mv = cnt - d;
            if (mv >= VT) {
#pragma unroll
                for (int x = 0; x < VT; x += 8) st_v8(pg.g.ov + row * 16 + x, &v[x]);
            } else {
#pragma unroll
                for (int x = 0; x < VT; ++x)
                    if (x < mv) pg.g.ov[row * 16 + x] = v[x];
            }
        }
        if (row == full_rows && d < cnt) {
#pragma unroll
            for (int x = 0; x < VT; ++x)
                if (x < cnt - d) pg.g.ok[row * 16 + x] = k[x];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&staged[st]);
    }
    pdl_trigger();
}


// ------------------------------ NEXT f2: Omitsort with run-location tracking
// PAPER.md:228 (§Full adaptivity): "the merge function simply returns the
// location of the data and the sort function checks whether after its two
// merges the data are in the same memory region, if not, it copies one to the
// data region ... diagnosing presortedness as non-overlap of the two input
// sequences".  Level-p runs (L = TILE << p keys, the last one shorter) each
// live in the data (0) or the buffer (1) region.  Pair q = runs 2q, 2q+1:
//   * no B run: the run is carried, location kept (no move);
//   * locations differ: the buffer-resident run is copied to the data region;
//   * B[0] not before A[L-1] (non-overlap): the merge is omitted, location
//     kept; else both runs are merged into the other region.
// Every decision depends only on the run boundaries: a merged run's smallest
// and largest key are the smaller / larger of its runs' (only comparisons are
// made, so which of two equal keys is irrelevant).  So one CTA plans all
// levels right after the tile sort (omit_plan_kernel).  Run state: region
// (data / buffer), direction (ascending, or strictly descending = Octosort's
// lazily kept reversed run: its reversal is its stable sort),
// smallest and largest key.  Pair (A, B):
//   * no B run: carried unchanged;
//   * both descending and every key of B strictly before every key of A:
//     A ++ B is strictly descending -- omitted as a descending run (after
//     copying the buffer-resident one to the data region if they differ);
//   * else each descending run is reversed (in place, or while it is copied),
//     the buffer-resident run is copied to the data region if the regions
//     differ, then the pair is omitted if B's smallest key is not
//     before A's largest, else merged into the other region.
// Per level p and pair q: an action byte act[p][q] and the exclusive prefix
// pre[p][q] of merge tiles over the level's pairs; per level the merge-tile
// count; at the end the sorted run's state.  Per level, omit_prep_kernel (all
// SMs) writes the merge-tile list (ascending, OMIT_DIR = buffer -> data),
// reverses and copies runs; one list-driven merge launch follows.
constexpr int OMIT_THREADS = 1024;
constexpr int OMIT_SMEM_RUNS = 2048;            // run state in shared memory up to 2048 level-0 runs (2^24 keys)
constexpr size_t OMIT_SMEM = 34 * OMIT_SMEM_RUNS;
// action byte: copy A / B from the buffer to the data region, merge (buffer ->
// data if OMIT_REV), reverse A / B, A / B currently in the buffer
constexpr unsigned OMIT_COPY_A = 1u, OMIT_COPY_B = 2u, OMIT_MERGE = 4u, OMIT_REV = 8u, OMIT_FLIP_A = 16u,
                   OMIT_FLIP_B = 32u, OMIT_BUF_A = 64u, OMIT_BUF_B = 128u;
constexpr unsigned OMIT_ST_BUF = 1u, OMIT_ST_DESC = 2u;   // run state bits
struct OmitState {                  // per-run state of two levels (ping-pong), scratch
    unsigned char *st[2];           // OMIT_ST_BUF | OMIT_ST_DESC
    double *lo[2];                  // smallest key (target order)
    double *hi[2];                  // largest key
};
template <int ORD>
__global__ void __launch_bounds__(OMIT_THREADS)
omit_plan_kernel(const double *dk, const double *bk, const unsigned char *tdesc, long long n, int levels, OmitState S,
                 unsigned char *act, int *pre, int *counts)
{
    pdl_wait();
    __shared__ int wsum[OMIT_THREADS / 32];
    __shared__ int carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned un = (unsigned)n;            // n < 2^31: positions fit 32 bits (unsigned: a0 + 2L < 2^32)
    // level 0: the tile-sorted runs, all in the data region
    const int nr0 = (int)((n + TILE - 1) / TILE);
    extern __shared__ __align__(16) unsigned char omit_smem[];
    if (nr0 <= OMIT_SMEM_RUNS) {            // small sorts: the run state in shared memory
        double *f = reinterpret_cast<double *>(omit_smem);
        S.lo[0] = f;
        S.lo[1] = f + OMIT_SMEM_RUNS;
        S.hi[0] = f + 2 * OMIT_SMEM_RUNS;
        S.hi[1] = f + 3 * OMIT_SMEM_RUNS;
        S.st[0] = omit_smem + 32 * OMIT_SMEM_RUNS;
        S.st[1] = S.st[0] + OMIT_SMEM_RUNS;
    }
    for (int r = tid; r < nr0; r += OMIT_THREADS) {
        const unsigned d = (tdesc[r] & 1) ? OMIT_ST_DESC : 0u;
        const unsigned b = (tdesc[r] & 2) ? OMIT_ST_BUF : 0u;
        const double *R = b ? bk : dk;
        const double f = R[(long long)r * TILE], l = R[min(n, (long long)(r + 1) * TILE) - 1];
        S.st[0][r] = (unsigned char)(d | b);
        S.lo[0][r] = d ? l : f;
        S.hi[0][r] = d ? f : l;
    }
    __syncthreads();
    int off = 0, cur = 0;
    for (int p = 0; p < levels; ++p) {
        const unsigned L = (unsigned)TILE << p;
        const int npairs = (int)((n + 2 * (long long)L - 1) / (2 * (long long)L));
        const unsigned tpp = 2 * L / MTILE;     // merge tiles per full pair
        if (tid == 0) carry = 0;
        __syncthreads();
        for (int c0 = 0; c0 < npairs; c0 += OMIT_THREADS) {
            const int q = c0 + tid;
            int nt = 0;
            unsigned a = 0;
            if (q < npairs) {
                const unsigned a0 = 2u * (unsigned)q * L, b0 = a0 + L;
                unsigned sa = S.st[cur][2 * q];
                double lo = S.lo[cur][2 * q], hi = S.hi[cur][2 * q];
                unsigned so = sa;
                if (b0 < un) {
                    const unsigned sb = S.st[cur][2 * q + 1];
                    const double blo = S.lo[cur][2 * q + 1], bhi = S.hi[cur][2 * q + 1];
                    a = ((sa & OMIT_ST_BUF) ? OMIT_BUF_A : 0u) | ((sb & OMIT_ST_BUF) ? OMIT_BUF_B : 0u);
                    unsigned ra = sa & OMIT_ST_BUF, rb = sb & OMIT_ST_BUF;
                    const bool desc_omit = (sa & sb & OMIT_ST_DESC) && before<ORD>(bhi, lo);
                    if (!desc_omit) {
                        if (sa & OMIT_ST_DESC) a |= OMIT_FLIP_A;
                        if (sb & OMIT_ST_DESC) a |= OMIT_FLIP_B;
                    }
                    if (ra != rb) {      // copy the buffer-resident run to the data region
                        a |= ra ? OMIT_COPY_A : OMIT_COPY_B;
                        ra = 0;
                    }
                    if (desc_omit) {
                        so = ra | OMIT_ST_DESC;                 // omitted, still descending
                    } else if (before<ORD>(blo, hi)) {          // overlap: merge into the other region
                        so = ra ^ 1u;
                        a |= OMIT_MERGE | (ra ? OMIT_REV : 0u);
                        nt = (int)min(tpp, (un - a0 + MTILE - 1) / MTILE);
                    } else {
                        so = ra;                                // omitted (0 moves)
                    }
                    if (before<ORD>(blo, lo)) lo = blo;
                    if (!before<ORD>(bhi, hi)) hi = bhi;
                }
                S.st[cur ^ 1][q] = (unsigned char)so;
                S.lo[cur ^ 1][q] = lo;
                S.hi[cur ^ 1][q] = hi;
                act[off + q] = (unsigned char)a;
            }
            int x = nt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            if (warp == 0) {
                int w = wsum[lane];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xFFFFFFFFu, w, o);
                    if (lane >= o) w += y;
                }
                wsum[lane] = w;
            }
            __syncthreads();
            if (q < npairs) pre[off + q] = carry + x - nt + (warp ? wsum[warp - 1] : 0);
            __syncthreads();
            if (tid == 0) carry += wsum[OMIT_THREADS / 32 - 1];
            __syncthreads();
        }
        if (tid == 0) counts[p] = carry;
        off += npairs;
        cur ^= 1;
        __syncthreads();                        // the level's state is complete
    }
    if (tid == 0) counts[levels] = S.st[cur][0];   // the sorted run's state (region, direction)
    pdl_trigger();
}

// Per level (run length L = 1 << lg), one pass over the merge tiles on all
// SMs: tile t of a merging pair q goes to list[pre[q] + t - first tile of q]
// (with OMIT_DIR for buffer -> data); a tile of a run to be moved and / or
// reversed is processed by one CTA: plain copy buffer -> data, reversed copy
// buffer -> data, or (first half of the run only) in-place swaps with the
// mirrored positions in the run's region -- keys, vals and the split-search
// samples of the touched positions.
template <bool HV>
__global__ void __launch_bounds__(256)
omit_prep_kernel(double *dk, uint32_t *dv, double *bk, uint32_t *bv, double *smp_d, double *smp_b, long long n, int lg,
                 const unsigned char *act, const int *pre, int *list)
{
    pdl_trigger();          // (the merge launch may become resident early; it waits for this grid to finish)
    pdl_wait();
    const int ntiles = (int)((n + MTILE - 1) / MTILE);
    const int tq_log2 = lg + 1 - MTILE_LOG2;                       // tiles per pair = 1 << tq_log2
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
        const int q = t >> tq_log2;
        const unsigned a = act[q];
        if (a & OMIT_MERGE)
            list[pre[q] + (t & ((1 << tq_log2) - 1))] = (int)((unsigned)t | ((a & OMIT_REV) ? OMIT_DIR : 0u));
    }
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const long long s0 = (long long)t * MTILE;
        const unsigned a = act[t >> tq_log2];
        const bool in_a = ((s0 >> lg) & 1) == 0;
        const bool copy = (a & (in_a ? OMIT_COPY_A : OMIT_COPY_B)) != 0;
        const bool flip = (a & (in_a ? OMIT_FLIP_A : OMIT_FLIP_B)) != 0;
        if (!copy && !flip) continue;
        const long long e = min(n, s0 + MTILE);
        const long long rs = (s0 >> lg) << lg;                     // the run [rs, rs + len)
        const long long len = min((long long)1 << lg, n - rs);
        const long long mir = 2 * rs + len - 1;                     // position i <-> mir - i
        if (copy && !flip) {
            if (e - s0 == MTILE) {         // full tile: 16-byte vectors (regions are 32-byte aligned)
                const double2 *src = reinterpret_cast<const double2 *>(bk + s0);
                double2 *dst = reinterpret_cast<double2 *>(dk + s0);
                for (int i = threadIdx.x; i < MTILE / 2; i += blockDim.x) dst[i] = src[i];
                if (HV) {
                    const uint4 *vs = reinterpret_cast<const uint4 *>(bv + s0);
                    uint4 *vd = reinterpret_cast<uint4 *>(dv + s0);
                    for (int i = threadIdx.x; i < MTILE / 4; i += blockDim.x) vd[i] = vs[i];
                }
            } else {
                for (long long i = s0 + threadIdx.x; i < e; i += blockDim.x) {
                    dk[i] = bk[i];
                    if (HV) dv[i] = bv[i];
                }
            }
            for (long long i = ((s0 + SMP_G - 1) >> SMP_LOG2) + threadIdx.x; (i << SMP_LOG2) < e; i += blockDim.x)
                smp_d[i] = smp_b[i];
        } else if (copy) {                 // reversed copy, buffer -> data
            for (long long i = s0 + threadIdx.x; i < e; i += blockDim.x) {
                const double x = bk[mir - i];
                dk[i] = x;
                if (HV) dv[i] = bv[mir - i];
                if ((i & (SMP_G - 1)) == 0) smp_d[i >> SMP_LOG2] = x;
            }
        } else {                           // in place, in the run's region; the first half swaps
            const bool buf = (a & (in_a ? OMIT_BUF_A : OMIT_BUF_B)) != 0;
            double *K = buf ? bk : dk;
            uint32_t *V = buf ? bv : dv;
            double *Sm = buf ? smp_b : smp_d;
            const long long half = rs + len / 2;
            for (long long i = s0 + threadIdx.x; i < min(e, half); i += blockDim.x) {
                const long long j = mir - i;
                const double x = K[i], y = K[j];
                K[i] = y;
                K[j] = x;
                if (HV) {
                    const uint32_t u = V[i], w = V[j];
                    V[i] = w;
                    V[j] = u;
                }
                if ((i & (SMP_G - 1)) == 0) Sm[i >> SMP_LOG2] = y;
                if ((j & (SMP_G - 1)) == 0) Sm[j >> SMP_LOG2] = x;
            }
        }
    }
}

// The sorted run's state `st` (OMIT_ST_BUF, OMIT_ST_DESC): copy it back to the
// data region, reverse it in place, or both (reversed copy); nothing if it is
// an ascending run in the data region.
template <bool HV>
__global__ void __launch_bounds__(256)
omit_final_kernel(double *dk, uint32_t *dv, const double *bk, const uint32_t *bv, long long n, const int *st)
{
    pdl_wait();
    const unsigned s = (unsigned)*st;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s == OMIT_ST_BUF) {
        const double2 *src = reinterpret_cast<const double2 *>(bk);
        double2 *dst = reinterpret_cast<double2 *>(dk);
        for (long long i = i0; i < (n >> 1); i += stride) dst[i] = src[i];
        if ((n & 1) && i0 == 0) dk[n - 1] = bk[n - 1];
        if (HV) for (long long i = i0; i < n; i += stride) dv[i] = bv[i];
    } else if (s == (OMIT_ST_BUF | OMIT_ST_DESC)) {
        for (long long i = i0; i < n; i += stride) {
            dk[i] = bk[n - 1 - i];
            if (HV) dv[i] = bv[n - 1 - i];
        }
    } else if (s == OMIT_ST_DESC) {
        for (long long i = i0; i < (n >> 1); i += stride) {
            const long long j = n - 1 - i;
            const double x = dk[i], y = dk[j];
            dk[i] = y;
            dk[j] = x;
            if (HV) {
                const uint32_t u = dv[i], w = dv[j];
                dv[i] = w;
                dv[j] = u;
            }
        }
    }
    pdl_trigger();
}

// NEXT f3: 64-bit payloads (gns_sort_keys_u64) ride as a u32 index through
// the pairs sort, then are gathered: idx[i] = i before, tmp[i] = vals[idx[i]]
// after (random 8-byte reads, coalesced writes).
__global__ void __launch_bounds__(256) iota_u32_kernel(uint32_t *idx, long long n)
{
    pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        idx[i] = (uint32_t)i;
    pdl_trigger();
}
__global__ void __launch_bounds__(256) gather_u64_kernel(uint64_t *out, const uint64_t *vals, const uint32_t *idx,
                                                          long long n)
{
    pdl_wait();
    // 8 outputs per thread and step: 8 independent random loads in flight
    // (the gather is latency-bound), 16-byte index loads and stores
    const long long n8 = n >> 3;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n8; g += stride) {
        const uint4 a = reinterpret_cast<const uint4 *>(idx)[2 * g];
        const uint4 b = reinterpret_cast<const uint4 *>(idx)[2 * g + 1];
        const uint64_t v0 = __ldg(vals + a.x), v1 = __ldg(vals + a.y), v2 = __ldg(vals + a.z), v3 = __ldg(vals + a.w);
        const uint64_t v4 = __ldg(vals + b.x), v5 = __ldg(vals + b.y), v6 = __ldg(vals + b.z), v7 = __ldg(vals + b.w);
        ulonglong2 *o = reinterpret_cast<ulonglong2 *>(out + 8 * g);
        o[0] = make_ulonglong2(v0, v1);
        o[1] = make_ulonglong2(v2, v3);
        o[2] = make_ulonglong2(v4, v5);
        o[3] = make_ulonglong2(v6, v7);
    }
    for (long long i = 8 * n8 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = vals[idx[i]];
    pdl_trigger();
}

// GNS_DEBUG=1 pre-scan (R1): number of NaN keys (f64 only).
__global__ void __launch_bounds__(256) nan_count_kernel(const double *k, long long n, unsigned *cnt)
{
    unsigned c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        c += (k[i] != k[i]) ? 1u : 0u;
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// ------------------------------------- target reversal (NEXT f3, AscRight/DescRight)
// AscRight = reverse(DescLeft), DescRight = reverse(AscLeft) (PAPER.md:137-142:
// the Right targets are the Left targets read from the other end of memory).
// In place: thread pairs element i with n-1-i; both ranges are read coalesced.
template <bool HV>
__global__ void __launch_bounds__(256)
reverse_kernel(double *k, uint32_t *v, long long n)
{
    pdl_wait();
    const long long half = n >> 1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < half;
         i += (long long)gridDim.x * blockDim.x) {
        const long long j = n - 1 - i;
        const double a = k[i], b = k[j];
        k[i] = b;
        k[j] = a;
        if (HV) {
            const uint32_t x = v[i], y = v[j];
            v[i] = y;
            v[j] = x;
        }
    }
    pdl_trigger();
}

// ----------------------------------- NEXT f4: distributed sort, splitter cuts
// For splitter i = (key, owner rank r_i, position p_i in r_i's sorted shard),
// the number of this rank's sorted keys that precede it in the global stable
// order (key, rank, position): ranks below r_i keep their ties first
// (count of keys <= key), ranks above put theirs after (count of keys < key),
// the owner cuts at p_i.  One thread per splitter, binary search.
template <int ORD>
__global__ void __launch_bounds__(128)
split_cuts_kernel(const double *keys, long long n, const double *spl_key, const int *spl_rank,
                  const long long *spl_pos, int nsplit, int my_rank, long long *cuts)
{
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nsplit) {
        long long c;
        if (spl_rank[i] == my_rank) {
            c = min(max(spl_pos[i], 0LL), n);
        } else {
            const bool upper = my_rank < spl_rank[i];
            const double x = spl_key[i];
            long long lo = 0, hi = n;      // first position whose key does not precede x
            while (lo < hi) {
                const long long m = (lo + hi) >> 1;
                const bool pre = upper ? !before<ORD>(x, keys[m]) : before<ORD>(keys[m], x);
                if (pre) lo = m + 1;
                else hi = m;
            }
            c = lo;
        }
        cuts[i] = c;
    }
    pdl_trigger();
}

}  // namespace gns
