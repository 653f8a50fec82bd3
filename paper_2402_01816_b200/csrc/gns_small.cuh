// gns_small.cuh — the whole sort of a small array (n <= 16 x 4096 = 65536,
// e.g. BASELINE config 1) in ONE thread-block cluster, on chip.
//
// Why: with the tile sort + one launch per merge level, a small sort is pure
// latency -- one wave of single-tile sorts (~33 us) plus ~10 us per merge
// level of launch, co-rank search and load (2^16 pairs: 68.6 us).  Here a
// cluster of C = 1..16 CTAs (the 16 needs the non-portable cluster size)
// holds the array in shared memory, 4096 elements per CTA:
//   1. each CTA loads its 4096 keys (+ vals; the last CTA padded with the
//      order's maximum key, placed after every real key) and sorts them
//      stably: an SM_VT-key transposition sort per thread (512 threads x 8
//      keys; 256 x 16 measured 4 % slower at 2^16 pairs, 1024 x 4 8 % slower),
//      then log2(SM_NT) shared-memory merge-path rounds (runs 8 -> 4096, left
//      run wins ties);
//   2. log2(C) merge levels across the cluster through distributed shared
//      memory: CTA c produces outputs [4096 (c - g0), +4096) of its group's
//      two runs (A = the group's first half of CTAs, B = the second): two
//      warps find the co-ranks of the first and the one-past-last output by
//      33-ary searches over the remote keys, all threads copy A[i0:i1) and
//      B[j0:j1) from the remote CTAs into local staging, then a local merge
//      path + SM_VT-step serial merge per thread; cluster barriers separate the
//      remote reads from the overwrite of each CTA's buffer;
//   3. each CTA writes its first real outputs back.
// One read and one write of the data in HBM; no buffer (%RAM 1.0).
#pragma once
#include <cooperative_groups.h>

namespace gns {

namespace cg = cooperative_groups;

#ifndef GNS_SM_NT
#define GNS_SM_NT 512
#endif
#ifndef GNS_SM_VT
#define GNS_SM_VT 8
#endif
constexpr int SM_NT = GNS_SM_NT;             // threads per CTA
constexpr int SM_VT = GNS_SM_VT;             // elements per thread
constexpr int SM_TILE = SM_NT * SM_VT;       // 4096 elements per CTA
constexpr int SM_MAXC = 16;                  // CTAs per cluster (non-portable above 8)
constexpr long long SMALL_MAX_N = (long long)SM_MAXC * SM_TILE;   // 65536
// shared memory: the CTA's run (keys, vals) and the merge staging (A then B)
constexpr size_t sm_smem(bool hv)
{
    return (size_t)SM_TILE * 8 * 2 + (hv ? (size_t)SM_TILE * 4 * 2 : 0) + 64 * 8 + 1024;
}

// Shared slot of element e: the 8-byte slot within each 16-element (128-byte)
// line XORed with the line index, so a thread's 16 consecutive elements
// (blocked spills) and stride-16 data-dependent merge reads spread over the
// banks (without it every lane of a warp hits the same bank).
__device__ __forceinline__ int swz16(int e) { return e ^ ((e >> 4) & 15); }

template <int ORD>
__device__ __forceinline__ void sm_transpose16(double (&k)[SM_VT], uint32_t (&v)[SM_VT], bool hv)
{
#pragma unroll
    for (int r = 0; r < SM_VT; ++r) {
#pragma unroll
        for (int i = r & 1; i + 1 < SM_VT; i += 2) {
            const bool p = before<ORD>(k[i + 1], k[i]);
            const double lo = p ? k[i + 1] : k[i], hi = p ? k[i] : k[i + 1];
            k[i] = lo;
            k[i + 1] = hi;
            if (hv) {
                const uint32_t vl = p ? v[i + 1] : v[i], vh = p ? v[i] : v[i + 1];
                v[i] = vl;
                v[i + 1] = vh;
            }
        }
    }
}

// Serial merge of SM_VT outputs from two runs in a swizzled local array
// (A: elements [oa, oa + na), B: [ob, ob + nb) of k / v), starting at co-rank
// (ia, ib); one slot past a run end is readable (padding), its value unused.
template <bool HV, int ORD>
__device__ __forceinline__ void sm_serial(const double *ks, const uint32_t *vs, int oa, int na, int ob, int nb,
                                          int ia, int ib, double (&k)[SM_VT], uint32_t (&v)[SM_VT])
{
    double ka = ks[swz16(oa + ia)], kb = ks[swz16(ob + ib)];
#pragma unroll
    for (int x = 0; x < SM_VT; ++x) {
        const bool p = (ib < nb) && ((ia >= na) || before<ORD>(kb, ka));
        k[x] = p ? kb : ka;
        if (HV) v[x] = p ? vs[swz16(ob + ib)] : vs[swz16(oa + ia)];
        if (p) kb = ks[swz16(ob + (++ib))];
        else ka = ks[swz16(oa + (++ia))];
    }
}

template <int ORD>
__device__ __forceinline__ int sm_corank_local(const double *ks, int oa, int na, int ob, int nb, int d)
{
    int lo = max(0, d - nb), hi = min(d, na);
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (!before<ORD>(ks[swz16(ob + d - 1 - m)], ks[swz16(oa + m)])) lo = m + 1;
        else hi = m;
    }
    return lo;
}

template <bool HV, int ORD>
__global__ void __launch_bounds__(SM_NT, 1)
small_sort_kernel(double *keys, uint32_t *vals, long long n)
{
#ifdef GNS_PROF
    // phase clocks of CTA 0 (tools/prof_small.py): g_prof[0..8]
    const long long pt0 = clock64();
#define SM_PT(q) do { if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&g_prof[q], (unsigned long long)(clock64() - pt0)); } while (0)
#else
#define SM_PT(q) do {} while (0)
#endif
    pdl_wait();
    SM_PT(0);
    cg::cluster_group cluster = cg::this_cluster();
    const int C = (int)cluster.num_blocks();
    const int c = (int)cluster.block_rank();
    extern __shared__ __align__(16) unsigned char sm_raw[];
    double *rk = reinterpret_cast<double *>(sm_raw);                  // this CTA's run (linear)
    double *sk = rk + SM_TILE + 32;                                   // staging: A then B (+ a pad slot each)
    uint32_t *rv = reinterpret_cast<uint32_t *>(sk + SM_TILE + 32);
    uint32_t *sv = rv + SM_TILE + 32;
    const int tid = threadIdx.x;
    const long long base = (long long)c * SM_TILE;
    double k[SM_VT];
    uint32_t v[SM_VT];
    // ---- 1. load (blocked: thread t owns elements 16t..16t+15; the load is
    // coalesced through the staging buffer) and sort the CTA's 4096 elements
    // (all 16 loads of a thread issued before any use: one DRAM latency, not 16)
#pragma unroll
    for (int x = 0; x < SM_VT; ++x) {
        const long long g = base + tid + x * SM_NT;
        k[x] = g < n ? keys[g] : pad_key<ORD>();
        if (HV) v[x] = g < n ? vals[g] : 0u;
    }
#pragma unroll
    for (int x = 0; x < SM_VT; ++x) {
        sk[swz16(tid + x * SM_NT)] = k[x];
        if (HV) sv[swz16(tid + x * SM_NT)] = v[x];
    }
    __syncthreads();
#pragma unroll
    for (int x = 0; x < SM_VT; ++x) {
        k[x] = sk[swz16(tid * SM_VT + x)];
        if (HV) v[x] = sv[swz16(tid * SM_VT + x)];
    }
    SM_PT(1);
    sm_transpose16<ORD>(k, v, HV);
    SM_PT(2);
#pragma unroll 1
    for (int coop = 2; coop <= SM_NT; coop <<= 1) {
        // a pair of <= 32 threads lies inside one warp (spills, reads and the
        // 16-element swizzle): those rounds synchronise the warp only
        const bool wsync = GNS_K1_WSYNC && coop <= 32;
        if (wsync) __syncwarp();
        else __syncthreads();
#pragma unroll
        for (int x = 0; x < SM_VT; ++x) {
            rk[swz16(tid * SM_VT + x)] = k[x];
            if (HV) rv[swz16(tid * SM_VT + x)] = v[x];
        }
        if (wsync) __syncwarp();
        else __syncthreads();
        const int local = tid & (coop - 1);
        const int a0 = (tid - local) * SM_VT;
        const int run = (coop >> 1) * SM_VT;
        const int d = local * SM_VT;
        const int i = sm_corank_local<ORD>(rk, a0, run, a0 + run, run, d);
        sm_serial<HV, ORD>(rk, rv, a0, run, a0 + run, run, i, d - i, k, v);
    }
    __syncthreads();
#pragma unroll
    for (int x = 0; x < SM_VT; ++x) {
        rk[swz16(tid * SM_VT + x)] = k[x];
        if (HV) rv[swz16(tid * SM_VT + x)] = v[x];
    }
    SM_PT(3);
    // ---- 2. merge levels across the cluster
    __shared__ int s_co[2];
    const int warp = tid >> 5, lane = tid & 31;
#pragma unroll 1
    for (int G = 2; G <= C; G <<= 1) {
        cluster.sync();                                  // every CTA's run is written (and readable remotely)
        if (G == 2) SM_PT(4);
        const int g0 = c & ~(G - 1), half = G >> 1;
        const int la = half * SM_TILE, lb = half * SM_TILE;
        auto A = [&](int m) -> double {
            return *cluster.map_shared_rank(rk + swz16(m & (SM_TILE - 1)), g0 + (m >> 12));
        };
        auto B = [&](int m) -> double {
            return *cluster.map_shared_rank(rk + swz16(m & (SM_TILE - 1)), g0 + half + (m >> 12));
        };
        if (warp < 2) {
            const int d = (c - g0) * SM_TILE + warp * SM_TILE;
            const int lo = max(0, d - lb), hi = min(d, la);
            int r = lo;
            if (lo < hi)
                r = lo + group_count_true<32>(lo, hi - 1, lane, 0xFFFFFFFFu, 0,
                                              [&](int m) { return !before<ORD>(B(d - 1 - m), A(m)); });
            if (lane == 0) s_co[warp] = r;
        }
        __syncthreads();
        if (G == 2) SM_PT(5);
        const int d0 = (c - g0) * SM_TILE;
        const int i0 = s_co[0], i1 = s_co[1];
        const int j0 = d0 - i0, j1 = d0 + SM_TILE - i1;
        const int ca = i1 - i0, cb = j1 - j0;
        // remote slices -> local staging (A at elements [0, ca), B at [ca + 1, ...), swizzled)
        const int ob = ca + 1;
        // the 4096 inputs [A slice, B slice], 16 per thread, all remote loads
        // issued before the local stores (one DSMEM latency, not 16)
#pragma unroll
        for (int x = 0; x < SM_VT; ++x) {
            const int e = tid + x * SM_NT;
            const bool fa = e < ca;
            const int m = fa ? i0 + e : j0 + (e - ca);
            const int r = (fa ? g0 : g0 + half) + (m >> 12);
            const int sl = swz16(m & (SM_TILE - 1));
            k[x] = *cluster.map_shared_rank(rk + sl, r);
            if (HV) v[x] = *cluster.map_shared_rank(rv + sl, r);
        }
#pragma unroll
        for (int x = 0; x < SM_VT; ++x) {
            const int e = tid + x * SM_NT;
            const int dst = swz16(e < ca ? e : e + 1);     // (B after A's pad slot)
            sk[dst] = k[x];
            if (HV) sv[dst] = v[x];
        }
        if (tid == 0) {
            sk[swz16(ca)] = pad_key<ORD>();              // (readable pad slots past each run)
            sk[swz16(ob + cb)] = pad_key<ORD>();
        }
        __syncthreads();
        if (G == 2) SM_PT(6);
        const int d = tid * SM_VT;
        const int i = sm_corank_local<ORD>(sk, 0, ca, ob, cb, d);
        sm_serial<HV, ORD>(sk, sv, 0, ca, ob, cb, i, d - i, k, v);
        cluster.sync();                                  // every remote read of this level is done
#pragma unroll
        for (int x = 0; x < SM_VT; ++x) {
            rk[swz16(tid * SM_VT + x)] = k[x];
            if (HV) rv[swz16(tid * SM_VT + x)] = v[x];
        }
    }
    // ---- 3. the CTA's real outputs back to HBM (coalesced)
    __syncthreads();
    SM_PT(7);
    for (int e = tid; e < SM_TILE; e += SM_NT) {
        const long long g = base + e;
        if (g < n) {
            keys[g] = rk[swz16(e)];
            if (HV) vals[g] = rv[swz16(e)];
        }
    }
    SM_PT(8);
    pdl_trigger();
#undef SM_PT
}

}  // namespace gns
