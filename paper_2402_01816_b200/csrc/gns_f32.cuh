// gns_f32.cuh — NEXT f3: the binary32 key path on its own 4-byte kernels
// (footprint-native: buffer n keys (+ n u32 vals), %RAM 2.0 like the f64
// path).  Same method as the f64 path (PAPER.md:150/219/221: one tile-sort
// pass with every level on chip, then one HBM pass per merge level, ping-pong
// between the data and the buffer, the left run winning ties), simpler
// kernels: no TMA, one CTA per output tile, the tile's splits searched in
// global memory by 32-lane groups.
//   F1  f32_tile_sort_kernel  stable sort of 8192-key tiles (registers + smem)
//   F2  f32_merge_kernel      one merge level, 4096 outputs per CTA
// DESC selects the descending key order; ties always keep input order.
#pragma once

namespace gns {

constexpr int F_NT = 256;                 // threads per CTA
constexpr int F_VT = 32;                  // keys per thread in the tile sort
constexpr int F_TILE = F_NT * F_VT;       // 8192 keys per tile (level-0 run)
constexpr int F_MVT = 16;                 // outputs per thread in a merge pass
constexpr int F_MTILE = F_NT * F_MVT;     // 4096 outputs per merge CTA
constexpr size_t f_tile_smem(bool hv) { return (size_t)F_TILE * (hv ? 8 : 4); }
static_assert(F_TILE % F_MTILE == 0, "pair boundaries on merge-tile boundaries");
static_assert(F_TILE == TILE, "the f32 path shares the f64 path's level count (merge_passes_for)");

template <bool DESC>
__device__ __forceinline__ bool fbefore(float a, float b) { return DESC ? (a > b) : (a < b); }

// key pads after every real key (the stable sort keeps real infinities first)
template <bool DESC>
__device__ __forceinline__ float fpad() { return DESC ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000); }

// shared-memory slot of tile element e: the 32-element row index XORed into
// the column, so the blocked accesses (thread t, element 32t + x) and the
// stride-16 merge reads spread over the 32 banks
__device__ __forceinline__ int fswz(int e) { return e ^ ((e >> 5) & 31); }

// ------------------------------------------------------------------ F1
template <bool HV, bool DESC>
__global__ void __launch_bounds__(F_NT, HV ? 2 : 3)
f32_tile_sort_kernel(const float *src_k, const uint32_t *src_v, float *dst_k, uint32_t *dst_v, long long n)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char f_smem[];      // keys [8192] (+ vals [8192])
    float *sk = reinterpret_cast<float *>(f_smem);
    uint32_t *sv = reinterpret_cast<uint32_t *>(f_smem + F_TILE * sizeof(float));
    const int tid = threadIdx.x;
    const long long base = (long long)blockIdx.x * F_TILE;
    const int cnt = (int)min((long long)F_TILE, n - base);
    const int e0 = tid * F_VT;
    float k[F_VT];
    uint32_t v[F_VT];
    // coalesced loads, all issued before the shared stores
#pragma unroll
    for (int u = 0; u < F_VT; ++u) {
        const int e = tid + u * F_NT;
        k[u] = e < cnt ? src_k[base + e] : fpad<DESC>();
        if (HV) v[u] = e < cnt ? src_v[base + e] : 0u;
    }
#pragma unroll
    for (int u = 0; u < F_VT; ++u) {
        const int e = tid + u * F_NT;
        sk[fswz(e)] = k[u];
        if (HV) sv[fswz(e)] = v[u];
    }
    __syncthreads();
#pragma unroll
    for (int x = 0; x < F_VT; ++x) {
        k[x] = sk[fswz(e0 + x)];
        if (HV) v[x] = sv[fswz(e0 + x)];
    }
    // stable odd-even transposition sort of the thread's 32 keys
#pragma unroll
    for (int r = 0; r < F_VT; ++r) {
#pragma unroll
        for (int i = r & 1; i + 1 < F_VT; i += 2) {
            const bool p = fbefore<DESC>(k[i + 1], k[i]);
            const float lo = p ? k[i + 1] : k[i], hi = p ? k[i] : k[i + 1];
            k[i] = lo;
            k[i + 1] = hi;
            if (HV) {
                const uint32_t vl = p ? v[i + 1] : v[i], vh = p ? v[i] : v[i + 1];
                v[i] = vl;
                v[i + 1] = vh;
            }
        }
    }
    // shared-memory merge rounds: runs of 32 -> 8192 (merge path + serial merge)
#pragma unroll 1
    for (int coop = 2; coop <= F_NT; coop <<= 1) {
        // (a pair of <= 32 threads lies inside one warp: warp-level sync)
        const bool wsync = GNS_K1_WSYNC && coop <= 32;
        if (wsync) __syncwarp();
        else __syncthreads();
#pragma unroll
        for (int x = 0; x < F_VT; ++x) {
            sk[fswz(e0 + x)] = k[x];
            if (HV) sv[fswz(e0 + x)] = v[x];
        }
        if (wsync) __syncwarp();
        else __syncthreads();
        const int local = tid & (coop - 1);
        const int a0 = (tid - local) * F_VT;
        const int run = (coop >> 1) * F_VT;
        const int b0 = a0 + run;
        const int d = local * F_VT;
        int lo = max(0, d - run), hi = min(d, run);
        while (lo < hi) {                                // co-rank: A[m] <= B[d-1-m]
            const int m = (lo + hi) >> 1;
            if (!fbefore<DESC>(sk[fswz(b0 + d - 1 - m)], sk[fswz(a0 + m)])) lo = m + 1;
            else hi = m;
        }
        int ai = a0 + lo, bi = b0 + d - lo;
        const int aend = a0 + run, bend = b0 + run;
#pragma unroll
        for (int x = 0; x < F_VT; ++x) {
            const float ka = ai < aend ? sk[fswz(ai)] : 0.f, kb = bi < bend ? sk[fswz(bi)] : 0.f;
            const bool p = (bi < bend) && ((ai >= aend) || fbefore<DESC>(kb, ka));
            k[x] = p ? kb : ka;
            if (HV) v[x] = sv[fswz(p ? bi : ai)];
            if (p) ++bi;
            else ++ai;
        }
    }
    // the thread's 32 outputs are elements e0.. of the sorted tile
    if (cnt == F_TILE) {
        float4 *dk = reinterpret_cast<float4 *>(dst_k + base + e0);
#pragma unroll
        for (int c = 0; c < F_VT / 4; ++c) dk[c] = make_float4(k[4 * c], k[4 * c + 1], k[4 * c + 2], k[4 * c + 3]);
        if (HV) {
            uint4 *dv = reinterpret_cast<uint4 *>(dst_v + base + e0);
#pragma unroll
            for (int c = 0; c < F_VT / 4; ++c) dv[c] = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        }
    } else {
#pragma unroll
        for (int x = 0; x < F_VT; ++x)
            if (e0 + x < cnt) {
                dst_k[base + e0 + x] = k[x];
                if (HV) dst_v[base + e0 + x] = v[x];
            }
    }
    pdl_trigger();
}

// Stable co-rank of output position d of the merge of A[0:na) and B[0:nb)
// (A wins ties) by the 32 lanes of a warp, in global memory.
template <bool DESC>
__device__ __forceinline__ int f32_corank(const float *A, int na, const float *B, int nb, int d, int lane)
{
    const int lo = max(0, d - nb), hi = min(d, na);
    if (lo >= hi) return lo;
    return lo + group_count_true<32>(lo, hi - 1, lane, 0xFFFFFFFFu, 0,
                                     [&](int m) { return !fbefore<DESC>(B[d - 1 - m], A[m]); });
}

// F2a: the split (A keys among the pair's first k0 outputs) of every merge
// tile's first output, one warp per tile (all tiles in one wave: the
// latency-bound searches overlap).
template <bool DESC>
__global__ void __launch_bounds__(256)
f32_partition_kernel(const float *src_k, long long n, long long L, int ntiles, int *corank)
{
    pdl_wait();
    pdl_trigger();
    const int t = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= ntiles) return;
    const long long t0 = (long long)t * F_MTILE;
    const long long pb = (t0 / (2 * L)) * (2 * L);
    const int na = (int)min(L, n - pb);
    const int nb = (int)max(0LL, min(L, n - pb - L));
    const int c = f32_corank<DESC>(src_k + pb, na, src_k + pb + L, nb, (int)(t0 - pb), lane);
    if (lane == 0) corank[t] = c;
}

// ------------------------------------------------------------------ F2
// One merge level: pair q = runs [2qL, 2qL+L) and [2qL+L, 2qL+2L) of src
// (clipped to n) into the same range of dst; CTA t writes outputs
// [4096 t, 4096 t + 4096), its splits from the partition.
// merge stage: A slots [0, F_SEG), B slots [F_SEG, 2 F_SEG) (+ vals alike);
// each part arrives by one 16-byte aligned 1-D bulk copy, `off` elements in
constexpr int F_SEG = F_MTILE + 8;
constexpr size_t f_merge_smem(bool hv) { return (size_t)2 * F_SEG * 4 * (hv ? 2 : 1); }

template <bool HV, bool DESC>
__global__ void __launch_bounds__(F_NT)
f32_merge_kernel(const float *src_k, const uint32_t *src_v, float *dst_k, uint32_t *dst_v, long long n, long long L,
                 const int *corank)
{
    pdl_wait();
    extern __shared__ __align__(16) unsigned char fm_smem[];
    float *SA = reinterpret_cast<float *>(fm_smem);
    float *SB = SA + F_SEG;
    uint32_t *VA = reinterpret_cast<uint32_t *>(fm_smem + 2 * F_SEG * 4);
    uint32_t *VB = VA + F_SEG;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    const long long t0 = (long long)blockIdx.x * F_MTILE;
    const long long pb = (t0 / (2 * L)) * (2 * L);          // the pair's first element
    const int na = (int)min(L, n - pb);
    const int nb = (int)max(0LL, min(L, n - pb - L));
    const int k0 = (int)(t0 - pb);
    const int k1 = (int)min((long long)k0 + F_MTILE, (long long)na + nb);
    // Split points clamped to the feasible co-ranks: with NaN keys (a
    // precondition violation, R1) the searches may return
    // non-monotone splits; clamping keeps 0 <= ca, cb and ca + cb = k1 - k0
    // <= F_MTILE, so every copy stays inside its F_SEG slots.
    const int i0 = min(max(corank[blockIdx.x], max(0, k0 - nb)), min(k0, na));
    int i1 = (k1 == na + nb) ? na : corank[blockIdx.x + 1];         // (the pair's last tile ends at na)
    i1 = min(max(max(i1, i0), k1 - nb), min(i0 + (k1 - k0), na));
    const int j0 = k0 - i0, j1 = k1 - i1;
    const int ca = i1 - i0, cb = j1 - j0, cnt = ca + cb;
    GNS_DASSERT(ca >= 0 && cb >= 0 && cnt == k1 - k0 && cnt <= F_MTILE);
    // global element ranges of the two parts, the 16-byte aligned bulk range
    // inside [0, n & ~3), and the elements past it (at most 3, loaded by hand)
    const long long ga = pb + i0, gb = pb + L + j0;
    const long long nal = n & ~3LL;
    auto span = [&](long long g, int c, long long &s0, long long &s1) {
        s0 = g & ~3LL;
        s1 = min((g + c + 3) & ~3LL, nal);
        if (s1 < s0) s1 = s0;
    };
    long long sa0, sa1, sb0, sb1;
    span(ga, ca, sa0, sa1);
    span(gb, cb, sb0, sb1);
    if (ca == 0) sa1 = sa0;                                  // (nothing to copy: no bytes expected)
    if (cb == 0) sb1 = sb0;
    const int oa = (int)(ga - sa0), ob = (int)(gb - sb0);
    GNS_DASSERT(oa + ca <= F_SEG && ob + cb <= F_SEG && (sa1 - sa0) <= F_SEG && (sb1 - sb0) <= F_SEG);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        const uint32_t bytes = (uint32_t)((sa1 - sa0) + (sb1 - sb0)) * 4u * (HV ? 2u : 1u);
        mbar_expect_tx(&bar, bytes);
        const uint64_t pol = policy_evict_first();
        if (sa1 > sa0) {
            tma_load_1d(SA, src_k + sa0, (uint32_t)(sa1 - sa0) * 4u, &bar, pol);
            if (HV) tma_load_1d(VA, src_v + sa0, (uint32_t)(sa1 - sa0) * 4u, &bar, pol);
        }
        if (sb1 > sb0) {
            tma_load_1d(SB, src_k + sb0, (uint32_t)(sb1 - sb0) * 4u, &bar, pol);
            if (HV) tma_load_1d(VB, src_v + sb0, (uint32_t)(sb1 - sb0) * 4u, &bar, pol);
        }
        mbar_arrive(&bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    // the tails past the last aligned group of the array (only at its end)
    if (tid < 8) {
        const bool fa = tid < 4;
        const long long g = (fa ? sa1 : sb1) + (tid & 3);
        const long long gend = fa ? ga + ca : gb + cb;
        if (g < gend) {
            const int slot = (int)(g - (fa ? sa0 : sb0));
            (fa ? SA : SB)[slot] = src_k[g];
            if (HV) (fa ? VA : VB)[slot] = src_v[g];
        }
    }
    __syncthreads();
    const int d = tid * F_MVT;
    if (d < cnt) {
        int lo = max(0, d - cb), hi = min(d, ca);
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if (!fbefore<DESC>(SB[ob + d - 1 - m], SA[oa + m])) lo = m + 1;
            else hi = m;
        }
        int ai = lo, bj = d - lo;
        float k[F_MVT];
        uint32_t v[F_MVT];
#pragma unroll
        for (int x = 0; x < F_MVT; ++x) {
            const float ka = ai < ca ? SA[oa + ai] : 0.f, kb = bj < cb ? SB[ob + bj] : 0.f;
            const bool p = (bj < cb) && ((ai >= ca) || fbefore<DESC>(kb, ka));
            k[x] = p ? kb : ka;
            if (HV) v[x] = p ? VB[ob + bj] : VA[oa + ai];
            if (p) ++bj;
            else ++ai;
        }
        const long long o = t0 + d;
        if (d + F_MVT <= cnt && (o & 3) == 0) {
            float4 *ok = reinterpret_cast<float4 *>(dst_k + o);
#pragma unroll
            for (int c = 0; c < F_MVT / 4; ++c) ok[c] = make_float4(k[4 * c], k[4 * c + 1], k[4 * c + 2], k[4 * c + 3]);
            if (HV) {
                uint4 *ov = reinterpret_cast<uint4 *>(dst_v + o);
#pragma unroll
                for (int c = 0; c < F_MVT / 4; ++c) ov[c] = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            }
        } else {
#pragma unroll
            for (int x = 0; x < F_MVT; ++x)
                if (d + x < cnt) {
                    dst_k[o + x] = k[x];
                    if (HV) dst_v[o + x] = v[x];
                }
        }
    }
    pdl_trigger();
}

// ------------------------------------------------------------------ F2 v2
// One merge level of binary32 keys (key-only) as a persistent, warp-
// specialised pipeline like the f64 pass (merge_tstore_kernel): each CTA owns a
// contiguous run of 4096-output tiles;
//   warps 0-7  merge: per thread the merge path of its 16 outputs in the
//              staged slices, 16-step serial merge (left run wins ties,
//              PAPER.md:221); the tile's outputs are staged in shared memory
//              and leave by one 1-D bulk store (TMA engine);
//   warp 8     producer (one lane): per tile one 1-D bulk copy (16-byte
//              aligned superset) of A's and of B's slice into a double-
//              buffered stage (A then B, packed), mbarrier tx-count completion;
//   warps 9-12 search: the tiles' co-ranks (A keys among the pair's first
//              k0 outputs) ahead into a shared ring, two 16-lane 17-ary
//              searches per warp in global memory (no separate partition
//              launch); at kernel start every warp computes one.
constexpr int F2_NS = 2;
#ifndef GNS_F2_SW
#define GNS_F2_SW 2
#endif
constexpr int F2_SW = GNS_F2_SW;                     // search warps
constexpr int F2_THREADS = F_NT + 32 + 32 * F2_SW;   // 352
constexpr int F2_RING = 64;
constexpr int F2_VT = 16;                            // outputs per merge thread
constexpr int F2_MT = F_NT * F2_VT;                  // 4096 outputs per tile (8192: 47 vs 41 us per 2^24-key level)
static_assert(F_TILE % F2_MT == 0, "pair boundaries on tile boundaries");
#ifndef GNS_F2_NET
#define GNS_F2_NET 0
#endif
constexpr bool F2_NET = GNS_F2_NET != 0;             // key-only: register bitonic merge of a thread's outputs
constexpr int F2_SLOTS = F2_MT + 16;                 // A (+ <= 6 alignment slots), then B (+ <= 6)
constexpr size_t f2_smem(bool hv = false) { return (size_t)F2_NS * F2_SLOTS * 4 * (hv ? 2 : 1) + 16; }

struct F2Meta {
    int t, ca, cb, oa, ob;    // tile, slice lengths, slots of A[0] / B[0] in the stage
};

template <bool DESC, int W = 16>
__device__ __forceinline__ int f2_corank(const float *src, long long n, long long L, int t, int gl, unsigned mask,
                                         int gbase)
{
    const long long t0 = (long long)t * F2_MT;
    const long long pb = (t0 / (2 * L)) * (2 * L);
    const int na = (int)min(L, n - pb);
    const int nb = (int)max(0LL, min(L, n - pb - L));
    const int d = (int)(t0 - pb);
    const float *A = src + pb, *B = src + pb + L;
    const int lo = max(0, d - nb), hi = min(d, na);
    if (lo >= hi) return lo;
    return lo + group_count_true<W>(lo, hi - 1, gl, mask, gbase,
                                    [&](int m) { return !fbefore<DESC>(B[d - 1 - m], A[m]); });
}

// HV: u32 payload staged at the same slots as its key (vals stage after the
// key stages), carried through the merge, stored with 16-byte stores.
template <bool HV, bool DESC>
__global__ void __launch_bounds__(F2_THREADS, HV ? 2 : 3)
f32_merge2_kernel(const float *src, const uint32_t *srcv, float *dst, uint32_t *dstv, long long n, long long L,
                  int ntiles, int per_cta)
{
    if (!GNS_LATE_PDL_WAIT) pdl_wait();
    extern __shared__ __align__(16) unsigned char f2_smem_raw[];
    float *stage = reinterpret_cast<float *>(f2_smem_raw);
    uint32_t *vstage = reinterpret_cast<uint32_t *>(stage + F2_NS * F2_SLOTS);
    __shared__ __align__(8) uint64_t full[F2_NS];
    __shared__ __align__(8) uint64_t freed[F2_NS];
    __shared__ F2Meta meta[F2_NS];
    __shared__ int spl[F2_RING];
    __shared__ volatile int spl_tag[F2_RING];
    __shared__ volatile int spl_used;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int first = blockIdx.x * per_cta;
    const int last = min(first + per_cta, ntiles);
    const int m = last - first;
    if (m <= 0) return;
    const int nspl = (last < ntiles) ? m + 1 : m;      // split of tile `last` ends the CTA's last tile
    for (int j = tid; j < F2_RING; j += F2_THREADS) spl_tag[j] = -1;
    if (tid == 0) {
        for (int b = 0; b < F2_NS; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&freed[b], F_NT / 32);
        }
        fence_mbar_init();
        spl_used = 0;
    }
    __syncthreads();
    if (GNS_LATE_PDL_WAIT) pdl_wait();       // (the prologue above reads nothing of the previous launch)
    auto publish = [&](int j, int c) {
        spl[j % F2_RING] = c;
        __threadfence_block();
        spl_tag[j % F2_RING] = j;
    };
    const int init = min(nspl, F2_THREADS / 32);
    if (warp < init) {
        // (the start-up splits by whole warps: one 33-ary round fewer than a 16-lane group)
        const int c = f2_corank<DESC, 32>(src, n, L, first + warp, lane, 0xFFFFFFFFu, 0);
        if (lane == 0) publish(warp, c);
    }
    __syncthreads();
    if (warp > F_NT / 32) {
        // ------------------------------------------------ search warps
        const int sw = warp - F_NT / 32 - 1;
        const int h = lane >> 4, gl = lane & 15;
        const unsigned mask = 0xFFFFu << (16 * h);
        for (int j0 = init + 2 * sw; j0 < nspl; j0 += 2 * F2_SW) {
            const int j = j0 + h;
            while (j0 + 1 - spl_used >= F2_RING) __nanosleep(64);
            if (j < nspl) {
                const int c = f2_corank<DESC>(src, n, L, first + j, gl, mask, 16 * h);
                if (gl == 0) publish(j, c);
            }
            __syncwarp();
        }
        return;
    }
    if (warp == F_NT / 32) {
        // ------------------------------------------------ producer (one lane)
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        const long long nal = n & ~3LL;
        auto get = [&](int j) -> int {
            while (spl_tag[j % F2_RING] != j) { }
            return spl[j % F2_RING];
        };
        auto issue = [&](int i) {
            const int st = i % F2_NS;
            const int t = first + i;
            const long long t0 = (long long)t * F2_MT;
            const long long pb = (t0 / (2 * L)) * (2 * L);
            const int na = (int)min(L, n - pb);
            const int nb = (int)max(0LL, min(L, n - pb - L));
            const int k0 = (int)(t0 - pb);
            const int k1 = (int)min((long long)k0 + F2_MT, (long long)na + nb);
            // split points clamped to the feasible co-ranks (NaN keys: DESIGN.md R1)
            const int i0 = min(max(get(i), max(0, k0 - nb)), min(k0, na));
            int i1 = (k1 == na + nb) ? na : get(i + 1);
            i1 = min(max(max(i1, i0), k1 - nb), min(i0 + (k1 - k0), na));
            spl_used = i;
            const int ca = i1 - i0, cb = (k1 - k0) - ca;
            const long long ga = pb + i0, gb = pb + L + (k0 - i0);
            long long sa0 = ga & ~3LL, sa1 = min((ga + ca + 3) & ~3LL, nal);
            long long sb0 = gb & ~3LL, sb1 = min((gb + cb + 3) & ~3LL, nal);
            if (sa1 < sa0 || ca == 0) sa1 = sa0;
            if (sb1 < sb0 || cb == 0) sb1 = sb0;
            const int oa = (int)(ga - sa0);
            const int rb = (oa + ca + 3) & ~3;                 // B's region: after all of A's slots, 16-byte aligned
            const int ob = rb + (int)(gb - sb0);
            float *S = stage + st * F2_SLOTS;
            GNS_DASSERT(oa + ca <= rb && sa1 - sa0 <= rb && ob + cb + 1 <= F2_SLOTS && rb + (sb1 - sb0) <= F2_SLOTS);
            uint32_t *V = vstage + st * F2_SLOTS;
            mbar_expect_tx(&full[st], (uint32_t)((sa1 - sa0) + (sb1 - sb0)) * 4u * (HV ? 2u : 1u));
            if (sa1 > sa0) {
                tma_load_1d(S, src + sa0, (uint32_t)(sa1 - sa0) * 4u, &full[st], pol);
                if (HV) tma_load_1d(V, srcv + sa0, (uint32_t)(sa1 - sa0) * 4u, &full[st], pol);
            }
            if (sb1 > sb0) {
                tma_load_1d(S + rb, src + sb0, (uint32_t)(sb1 - sb0) * 4u, &full[st], pol);
                if (HV) tma_load_1d(V + rb, srcv + sb0, (uint32_t)(sb1 - sb0) * 4u, &full[st], pol);
            }
            // the <= 3 keys past the array's last aligned group, by hand
            for (long long g = max(sa1, ga); g < ga + ca; ++g) {
                S[g - sa0] = src[g];
                if (HV) V[g - sa0] = srcv[g];
            }
            for (long long g = max(sb1, gb); g < gb + cb; ++g) {
                S[rb + (g - sb0)] = src[g];
                if (HV) V[rb + (g - sb0)] = srcv[g];
            }
            F2Meta mt;
            mt.t = t;
            mt.ca = ca;
            mt.cb = cb;
            mt.oa = oa;
            mt.ob = ob;
            meta[st] = mt;
            mbar_arrive(&full[st]);
        };
        for (int i = 0; i < F2_NS && i < m; ++i) issue(i);
        for (int i = F2_NS; i < m; ++i) {
            const int st = i % F2_NS;
            mbar_wait(&freed[st], (uint32_t)(((i - F2_NS) / F2_NS) & 1));   // tile i - NS merged out of stage st
            issue(i);
        }
        pdl_trigger();
        return;
    }
    // ---------------------------------------------------- merge warps 0-7
    for (int i = 0; i < m; ++i) {
        const int st = i % F2_NS;
        mbar_wait(&full[st], (uint32_t)((i / F2_NS) & 1));
        const F2Meta mt = meta[st];
        const float *S = stage + st * F2_SLOTS;
        const float *SA = S + mt.oa, *SB = S + mt.ob;
        const uint32_t *VA = vstage + st * F2_SLOTS + mt.oa, *VB = vstage + st * F2_SLOTS + mt.ob;
        const int cnt = mt.ca + mt.cb;
        const int d = tid * F2_VT;
        float k[F2_VT];
        uint32_t v[F2_VT];
        bool merged = false;
        int lo = 0;
        if (!HV && F2_NET) {
            // Key-only: the thread's 16 outputs merged by a bitonic network in
            // registers instead of 16 dependent shared-memory steps.  Its A
            // count is the next thread's co-rank minus its own (lane 31: the
            // warp's end co-rank, searched by all 32 lanes together); the A
            // keys ascending followed by the B keys descending are a bitonic
            // sequence, which 4 stages of fmin / fmax sort.  Keys that compare
            // equal are bit-identical unless they are zeros of both signs, so
            // the result equals the stable merge's whenever the
            // warp's inputs hold no -0.0; a warp that sees one (or a partial
            // tile) takes the serial merge below.
            const int dd = min(d, cnt);
            // the warp's last diagonal by a 33-ary search of all 32 lanes
            // (three rounds for 4096 keys); it bounds every lane's own range
            const int de = min((warp + 1) * 32 * F2_VT, cnt);
            int ce;
            {
                const int l0 = max(0, de - mt.cb), h0 = min(de, mt.ca);
                ce = l0;
                if (l0 < h0)
                    ce = l0 + group_count_true<32>(l0, h0 - 1, lane, 0xffffffffu, 0,
                                                   [&](int x) { return !fbefore<DESC>(SB[de - 1 - x], SA[x]); });
            }
            // co-rank(d) <= co-rank(de) and d - co-rank(d) <= de - co-rank(de)
            int hi = min(min(dd, mt.ca), ce);
            lo = min(max(max(0, dd - mt.cb), ce - (de - dd)), hi);
            while (lo < hi) {
                const int x = (lo + hi) >> 1;
                if (!fbefore<DESC>(SB[dd - 1 - x], SA[x])) lo = x + 1;
                else hi = x;
            }
            int nlo = __shfl_down_sync(0xffffffffu, lo, 1);
            if (lane == 31) nlo = ce;
            const bool fullt = d + F2_VT <= cnt;
            // A count, clamped to what both slices hold (a no-op unless NaN
            // keys made the searches inconsistent: DESIGN.md R1)
            const int ai = lo, bj = dd - lo;
            int an = min(max(nlo - lo, 0), F2_VT);
            an = max(min(an, mt.ca - ai), F2_VT - (mt.cb - bj));
            bool zero = false;
            if (fullt) {
                GNS_DASSERT(an >= 0 && an <= F2_VT && ai + an <= mt.ca && bj + (F2_VT - an) <= mt.cb);
                const float *pa = SA + ai, *pb = SB + bj + (F2_VT - 1);
#pragma unroll
                for (int x = 0; x < F2_VT; ++x) {
                    k[x] = *(x < an ? pa + x : pb - x);
                    zero |= (__float_as_uint(k[x]) == 0x80000000u);     // -0.0
                }
            }
            if (__all_sync(0xffffffffu, fullt && !zero)) {
#pragma unroll
                for (int s = F2_VT / 2; s > 0; s >>= 1) {
#pragma unroll
                    for (int x = 0; x < F2_VT; ++x) {
                        if ((x & s) == 0) {
                            const float a = k[x], b = k[x + s];
                            k[x] = DESC ? fmaxf(a, b) : fminf(a, b);
                            k[x + s] = DESC ? fminf(a, b) : fmaxf(a, b);
                        }
                    }
                }
                merged = true;
            }
        }
        if (!merged && d < cnt) {
            if (HV || !F2_NET) {
                int hi = min(d, mt.ca);
                lo = max(0, d - mt.cb);
                while (lo < hi) {
                    const int x = (lo + hi) >> 1;
                    if (!fbefore<DESC>(SB[d - 1 - x], SA[x])) lo = x + 1;
                    else hi = x;
                }
            }
            int ai = lo, bj = d - lo;
            float ka = SA[ai], kb = SB[bj];          // (one slot past a run end is inside the stage)
#pragma unroll
            for (int x = 0; x < F2_VT; ++x) {
                const bool p = (bj < mt.cb) && ((ai >= mt.ca) || fbefore<DESC>(kb, ka));
                k[x] = p ? kb : ka;
                if (HV) v[x] = p ? VB[bj] : VA[ai];
                if (p) kb = SB[++bj];
                else ka = SA[++ai];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&freed[st]);             // this warp is done reading stage st
        if (d < cnt) {
            const long long o = (long long)mt.t * F2_MT + d;
            if (d + F2_VT <= cnt && (o & 3) == 0) {
                float4 *ok = reinterpret_cast<float4 *>(dst + o);
#pragma unroll
                for (int c = 0; c < F2_VT / 4; ++c) ok[c] = make_float4(k[4 * c], k[4 * c + 1], k[4 * c + 2], k[4 * c + 3]);
                if (HV) {
                    uint4 *ov = reinterpret_cast<uint4 *>(dstv + o);
#pragma unroll
                    for (int c = 0; c < F2_VT / 4; ++c) ov[c] = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                }
            } else {
#pragma unroll
                for (int x = 0; x < F2_VT; ++x)
                    if (d + x < cnt) {
                        dst[o + x] = k[x];
                        if (HV) dstv[o + x] = v[x];
                    }
            }
        }
    }
    pdl_trigger();
}

// reversal of a binary32 array (+ vals) in place (the Right targets)
template <bool HV>
__global__ void __launch_bounds__(256) f32_reverse_kernel(float *k, uint32_t *v, long long n)
{
    pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n / 2; i += (long long)gridDim.x * blockDim.x) {
        const long long j = n - 1 - i;
        const float a = k[i], b = k[j];
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

}  // namespace gns
