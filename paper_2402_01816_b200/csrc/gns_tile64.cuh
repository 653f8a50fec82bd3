// gns_tile64.cuh — K1 for key-only sorts: the stable
// sort of one 8192-key tile per CTA with NT3 threads x VT3 keys (default
// 256 x 32, three CTAs per SM; GNS_VT3=64 gives round 2's 128 x 64).
//
// Why a second K1 for key-only: the 256 x 32 kernel with payload
// (tile_sort2_kernel) is bound by shared-memory wavefronts (ncu: l1tex 91 %
// busy, 3.7 wavefronts per key, half of them bank conflicts of the
// data-dependent merge reads) and spends ~77 instructions per key on its
// 32-key transposition sort.  Here:
//   * one VT3-key sorting network per thread in registers (Batcher's odd-even
//     merge sort: 191 compare-exchanges for 32 keys, 543 for 64, instead of
//     496 / 2016 for a transposition sort) -- unstable, which is harmless for
//     key-only input because equal keys are bit-identical, except -0.0 / +0.0
//     (equal under IEEE <, different bits): a thread holding a zero records
//     the signs of its zeros in input order, sorts canonical +0.0 and writes
//     the signs back in that order, which is exactly the stable order
//     (R2);
//   * GNS_K1_BITONIC warp-level bitonic merge rounds in registers + shuffles
//     (default 2: runs 32 -> 128) unless the CTA holds a -0.0 or NaN key, then
//     shared-memory merge-path rounds up to 8192 (all of them in the -0.0 /
//     NaN case), each thread producing VT3 outputs as two independent chains
//     (merge path + serial merge, left run wins ties); rounds
//     inside one warp synchronise that warp only, wider rounds the CTA, and
//     there the warp's end co-rank is one 33-ary search by all 32 lanes;
//   * the tile arrives by one-dimensional bulk copies (one VT3-key segment
//     per thread, TMA engine, one mbarrier) into a padded layout whose 16-byte
//     register transfers are conflict-free, and leaves the same way.
// Measured (B200, 2^24 f64, event-timed): 128 x 64: 246 -> 223-229 us (ncu:
// 61.5 M -> ~31 M shared wavefronts, 154 M -> ~120 M instructions); 256 x 32
// (24 warps per SM instead of 12): whole sort 0.807 -> 0.794 ms, 24 tie
// values 0.783 -> 0.752 ms (DESIGN.md 8b lists the variants tried: one-load
// merge steps, 16384-key tiles, 0-5 bitonic rounds, 16 keys per thread,
// four chains).  One read-scan and one write-scan of HBM per tile
// (PAPER.md:150); the 13 merge levels inside the tile cost no HBM traffic.
#pragma once

namespace gns {

// warp-level bitonic merge rounds before the merge-path rounds (0..5)
#ifndef GNS_K1_BITONIC
#define GNS_K1_BITONIC 2
#endif
#ifndef GNS_K1_ONELDS
#define GNS_K1_ONELDS 0
#endif
// keys per thread: 32 (256 threads, 3 CTAs per SM = 24 warps, Batcher's
// 191-comparator network of 32 keys) -- measured against 64 (128 threads,
// 12 warps, 543 comparators): 2^24 keys 0.794 vs 0.804 ms, 24 heavy-tie
// values 0.750 vs 0.780 ms
#ifndef GNS_VT3
#define GNS_VT3 32
#endif
constexpr int VT3 = GNS_VT3;              // keys per thread (64: 2^6, the finest sample spacing of K1)
constexpr int NT3 = TILE / VT3;           // threads per CTA (128)
constexpr int VT3_LOG2 = VT3 == 64 ? 6 : VT3 == 32 ? 5 : 4;
static_assert((1 << VT3_LOG2) == VT3, "VT3_LOG2");
#ifndef GNS_T3_MINB
#define GNS_T3_MINB 3             // CTAs per SM (shared memory allows three 8192-key tiles)
#endif
#ifndef GNS_T3F_MINB
#define GNS_T3F_MINB 4            // binary32 keys: four (half the shared memory per tile)
#endif
static_assert(NT3 * VT3 == TILE, "K1 key-only tile must equal TILE");
template <typename K = double, int NT = 128> constexpr size_t t3_smem() { return (size_t)NT * (VT3 * sizeof(K) + 16) + 128; }
constexpr int SEG3_BYTES = VT3 * 8 + 16;  // padded 512-byte segment per thread (+16)
constexpr size_t T3_SMEM = (size_t)NT3 * SEG3_BYTES + 128;   // 67,712 B: 3 CTAs per SM
static_assert(256 + TILE * 8 + 8 <= NT3 * SEG3_BYTES, "merge layout + guard slots fit the padded segments");

// ---- Batcher's odd-even merge sort network for N keys (Knuth 5.3.4,
// exercise 5.2.2-12 form), as a compile-time comparator list.
template <int N>
struct OddEvenNet {
    static constexpr int count()
    {
        int c = 0;
        for (int p = 1; p < N; p <<= 1)
            for (int k = p; k >= 1; k >>= 1)
                for (int j = k % p; j + k < N; j += 2 * k)
                    for (int i = 0; i < k && i + j + k < N; ++i)
                        if ((i + j) / (2 * p) == (i + j + k) / (2 * p)) ++c;
        return c;
    }
    static constexpr int NC = count();
    unsigned char a[NC], b[NC];
    constexpr OddEvenNet() : a(), b()
    {
        int c = 0;
        for (int p = 1; p < N; p <<= 1)
            for (int k = p; k >= 1; k >>= 1)
                for (int j = k % p; j + k < N; j += 2 * k)
                    for (int i = 0; i < k && i + j + k < N; ++i)
                        if ((i + j) / (2 * p) == (i + j + k) / (2 * p)) {
                            a[c] = (unsigned char)(i + j);
                            b[c] = (unsigned char)(i + j + k);
                            ++c;
                        }
    }
};
static_assert(OddEvenNet<64>::NC == 543, "Batcher odd-even merge sort of 64 keys has 543 comparators");
static_assert(OddEvenNet<32>::NC == 191, "Batcher odd-even merge sort of 32 keys has 191 comparators");

// ---- key width: binary64 (and the 8-byte integer key types) or binary32
// (NEXT f3).  kbef<K, ORD>: x must be output strictly before y (ORD = DESC |
// key type << 1 for 8-byte keys, DESC for binary32).
template <typename K, int ORD>
__device__ __forceinline__ bool kbef(K x, K y)
{
    if constexpr (sizeof(K) == 8) return before<ORD>((double)x, (double)y);
    else return (ORD & 1) ? (x > y) : (x < y);
}
template <typename K, int ORD>
__device__ __forceinline__ K kpad()
{
    if constexpr (sizeof(K) == 8) return pad_key<ORD>();
    else return (ORD & 1) ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000);
}
template <typename K>
__device__ __forceinline__ K lds_k(uint32_t a)
{
    if constexpr (sizeof(K) == 8) return lds_f64(a);
    else {
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
        return v;
    }
}
// 16-byte shared transfers of 16 / sizeof(K) consecutive keys
template <typename K>
__device__ __forceinline__ void lds16_k(uint32_t a, K *v)
{
    if constexpr (sizeof(K) == 8)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(a));
    else
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                     : "r"(a));
}
template <typename K>
__device__ __forceinline__ void sts16_k(uint32_t a, const K *v)
{
    if constexpr (sizeof(K) == 8)
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" :: "r"(a), "d"(v[0]), "d"(v[1]) : "memory");
    else
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" :: "r"(a), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3])
                     : "memory");
}
// key bits: -0.0 (the one key equal to another key with different bits)
template <typename K>
__device__ __forceinline__ bool neg_zero(K x)
{
    if constexpr (sizeof(K) == 8) return __double_as_longlong(x) == (long long)0x8000000000000000ULL;
    else return __float_as_uint(x) == 0x80000000u;
}
template <typename K>
__device__ __forceinline__ bool sign_set(K x)
{
    if constexpr (sizeof(K) == 8) return __double_as_longlong(x) < 0;
    else return (int)__float_as_uint(x) < 0;
}

template <typename K, int N, int ORD>
__device__ __forceinline__ void network_sort(K (&k)[N])
{
    constexpr OddEvenNet<N> net{};
#pragma unroll
    for (int c = 0; c < OddEvenNet<N>::NC; ++c) {
        const int i = net.a[c], j = net.b[c];
        const bool p = kbef<K, ORD>(k[j], k[i]);
        const K lo = p ? k[j] : k[i];
        const K hi = p ? k[i] : k[j];
        k[i] = lo;
        k[j] = hi;
    }
}

// Merge-round layout: byte address a -> a with its 16-byte chunk (bits 4-6)
// XORed with bits 9-11 (the thread's 512-byte block), so the blocked 16-byte
// spill (lane t writes chunk c of its own block) hits 8 distinct chunk
// positions per 8 lanes: conflict-free.  A bijection on every 128-byte line.
// (binary32: 256-byte blocks, bits 4-6 XORed with bits 8-10)
template <typename K = double>
__device__ __forceinline__ uint32_t sw3(uint32_t a)
{
    // bits 4-6 XOR the thread-block index bits: block = VT3 * sizeof(K) bytes
    constexpr int SH = (VT3 * (int)sizeof(K) == 512) ? 5 : (VT3 * (int)sizeof(K) == 256) ? 4 : 3;
    return a ^ ((a >> SH) & 0x70u);
}

// Stable co-rank of diagonal d (A wins ties; predicate A[m] <= B[d-1-m]) and,
// if `two`, of diagonal d + VT3 in the same loop (independent probes).
template <typename K, int ORD>
__device__ __forceinline__ void merge_path3x2(uint32_t base, int a0, int na, int b0, int nb, int d, bool two,
                                              int &r1, int &r2)
{
    int lo = max(0, d - nb), hi = min(d, na);
    const int d2 = d + VT3;
    int lo2 = two ? max(0, d2 - nb) : 0, hi2 = two ? min(d2, na) : 0;
    while (lo < hi || lo2 < hi2) {
        if (lo < hi) {
            const int m = (lo + hi) >> 1;
            const K b = lds_k<K>(sw3<K>(base + (uint32_t)sizeof(K) * (b0 + d - 1 - m)));
            const K a = lds_k<K>(sw3<K>(base + (uint32_t)sizeof(K) * (a0 + m)));
            if (!kbef<K, ORD>(b, a)) lo = m + 1;
            else hi = m;
        }
        if (lo2 < hi2) {
            const int m = (lo2 + hi2) >> 1;
            const K b = lds_k<K>(sw3<K>(base + (uint32_t)sizeof(K) * (b0 + d2 - 1 - m)));
            const K a = lds_k<K>(sw3<K>(base + (uint32_t)sizeof(K) * (a0 + m)));
            if (!kbef<K, ORD>(b, a)) lo2 = m + 1;
            else hi2 = m;
        }
    }
    r1 = lo;
    r2 = lo2;
}

// Serial merge of the thread's VT3 outputs as two independent chains (twice
// the instruction-level parallelism of one chain; the kernel runs 12 warps per
// SM and is bound by the shared-memory load latency of each merge step):
//   forward  from co-rank (ai, bi) of the thread's first output: outputs
//            k[0 .. VT3/2), B's head taken only if strictly before A's (left
//            wins ties);
//   backward from co-rank (qa, qb) of the output after the thread's last
//            (exclusive ends): outputs k[VT3-1 .. VT3/2], A's tail taken only
//            if strictly after B's (a tie puts B's element later).
// By the merge-path property both chains meet exactly at the midpoint.
template <typename K, int ORD>
__device__ __forceinline__ void serial_merge3(uint32_t base, int a0, int ai, int aend, int bi, int bend, int qa,
                                              int qb, K (&k)[VT3])
{
    constexpr uint32_t SZ = sizeof(K);
    uint32_t pa = base + SZ * ai, pb = base + SZ * bi;
    const uint32_t pae = base + SZ * aend, pbe = base + SZ * bend;
    // backward chain: ra / rb = addresses of the next A / B key to take from
    // the back; A's run starts at a0, B's run starts at aend
    uint32_t ra = base + SZ * (qa - 1), rb = base + SZ * (qb - 1);
    const uint32_t ras = base + SZ * a0, rbs = pae;
    K ka = lds_k<K>(sw3<K>(pa)), kb = lds_k<K>(sw3<K>(pb));
    K ta = lds_k<K>(sw3<K>(ra)), tb = lds_k<K>(sw3<K>(rb));
#pragma unroll
    for (int x = 0; x < VT3 / 2; ++x) {
        const bool p = (pb < pbe) && ((pa >= pae) || kbef<K, ORD>(kb, ka));
        k[x] = p ? kb : ka;
        const uint32_t nxt = (p ? pb : pa) + SZ;
        GNS_DASSERT(nxt >= base && nxt <= base + SZ * 2 * TILE + SZ);
        const uint32_t a = sw3<K>(nxt);
        // backward: take A's tail iff it exists and (B is exhausted or B's
        // tail is strictly before it)
        const bool q = (ra >= ras) && ((rb < rbs) || kbef<K, ORD>(tb, ta));
        k[VT3 - 1 - x] = q ? ta : tb;
        const uint32_t prv = (q ? ra : rb) - SZ;
        GNS_DASSERT(prv + SZ >= base && prv < base + SZ * 2 * TILE);
        const uint32_t b = sw3<K>(prv);
#if GNS_K1_ONELDS
        // one full-warp load per chain step (fewer shared wavefronts than two
        // predicated half-warp loads), routed into the consumed side's head
        const K u = lds_k<K>(a), w = lds_k<K>(b);
        if (p) pb = nxt; else pa = nxt;
        kb = p ? u : kb;
        ka = p ? ka : u;
        if (q) ra = prv; else rb = prv;
        ta = q ? w : ta;
        tb = q ? tb : w;
#else
        if (p) {
            pb = nxt;
            kb = lds_k<K>(a);
        } else {
            pa = nxt;
            ka = lds_k<K>(a);
        }
        if (q) {
            ra = prv;
            ta = lds_k<K>(b);
        } else {
            rb = prv;
            tb = lds_k<K>(b);
        }
#endif
    }
}

// Network merge of the thread's VT3 outputs (no dependent shared-memory
// chain): its an A keys ascending followed by its VT3 - an B keys descending
// are a bitonic sequence, sorted by log2(VT3) half-cleaner stages in
// registers (binary32: fmin / fmax).  Unstable, so only used when no key of
// the CTA is -0.0 or NaN (equal keys are then bit-identical and the result is
// the stable merge's) -- the same condition as the warp-level
// bitonic rounds.  GNS_K1_NET: bit 0 = binary32 keys, bit 1 = 8-byte keys.
#ifndef GNS_K1_NET
#define GNS_K1_NET 0
#endif
// merge-path rounds over more than one warp: the warp's end co-rank by a
// 33-ary search of the whole warp (1) or by lane 31's second search (0)
// merge-path round synchronisation: rounds inside one warp synchronise that
// warp only (GNS_K1_WSYNC); rounds over 2 or 4 warps synchronise those warps on
// a named barrier (GNS_K1_GSYNC); only the last round needs the whole CTA
#ifndef GNS_K1_WSYNC
#define GNS_K1_WSYNC 1
#endif
#ifndef GNS_K1_GSYNC
#define GNS_K1_GSYNC 0
#endif
// Barrier of the coop threads that merge one pair (coop a power of two).
__device__ __forceinline__ void pair_sync(int tid, int coop, int nt)
{
    if (GNS_K1_WSYNC && coop <= 32) __syncwarp();
    else if (GNS_K1_GSYNC && GNS_K1_WSYNC && coop < nt && coop <= 128) {
        // ids 1-4: pairs of 64 threads, 5-6: pairs of 128 threads (id 0 = __syncthreads)
        const int id = (coop == 64 ? 1 : 5) + tid / coop;
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(coop) : "memory");
    } else __syncthreads();
}
#ifndef GNS_K1_COOPEND
#define GNS_K1_COOPEND 1
#endif
template <typename K, int ORD>
__device__ __forceinline__ void net_merge3(uint32_t base, int ai, int an, int bi, K (&k)[VT3])
{
    constexpr uint32_t SZ = sizeof(K);
    GNS_DASSERT(an >= 0 && an <= VT3 && ai >= 0 && bi >= 0 && ai + an <= TILE && bi + (VT3 - an) <= TILE + VT3);
    const uint32_t pa = base + SZ * ai, pb = base + SZ * (bi + VT3 - 1);
#pragma unroll
    for (int x = 0; x < VT3; ++x) k[x] = lds_k<K>(sw3<K>(x < an ? pa + SZ * x : pb - SZ * x));
#pragma unroll
    for (int s = VT3 / 2; s > 0; s >>= 1) {
#pragma unroll
        for (int x = 0; x < VT3; ++x) {
            if ((x & s) == 0) {
                const K a = k[x], b = k[x + s];
                if constexpr (sizeof(K) == 4) {
                    k[x] = (ORD & 1) ? fmaxf(a, b) : fminf(a, b);
                    k[x + s] = (ORD & 1) ? fminf(a, b) : fmaxf(a, b);
                } else {
                    const bool p = kbef<K, ORD>(b, a);
                    k[x] = p ? b : a;
                    k[x + s] = p ? a : b;
                }
            }
        }
    }
}

// One merge-path round: spill the thread's sorted run block, synchronise
// (the warp, or the CTA if `cta`), then merge pair (A, B) of runs of
// (coop / 2) * VT3 keys; the thread produces outputs [d, d + VT3) of its pair.
template <typename K, int ORD>
__device__ __forceinline__ void merge_round3(uint32_t sbase, int tid, int e0, int coop, K (&k)[VT3],
                                             bool cta = false, bool net = false)
{
    constexpr int PER = 16 / (int)sizeof(K);          // keys per 16-byte transfer
#pragma unroll
    for (int c = 0; c < VT3 / PER; ++c) sts16_k<K>(sw3<K>(sbase + (uint32_t)sizeof(K) * (e0 + PER * c)), &k[PER * c]);
    if (cta) pair_sync(tid, coop, NT3);
    else __syncwarp();
    const int local = tid & (coop - 1);
    const int a0 = (tid - local) * VT3;
    const int run = (coop >> 1) * VT3;
    const int b0 = a0 + run;
    const int d = local * VT3;
    // co-ranks of the thread's first output (d) and of the output after its
    // last (d + VT3): the latter is the next thread's first (a shuffle),
    // searched here only by lane 31, or the pair's end
    int i, inext;
    if (GNS_K1_COOPEND && coop > 32) {
        // the warp's last diagonal lies inside the pair: all 32 lanes search
        // its co-rank together (33-ary, 2-3 rounds) instead of lane 31 running
        // a second binary search beside its own; it also bounds every lane's
        // own range (co-rank(d) <= co-rank(de), d - co-rank(d) <= de - co-rank(de))
        const int lane = lane_id();
        const int de = (local - lane + 32) * VT3;
        int ce = run;
        if (de < 2 * run) {
            const int l0 = max(0, de - run), h0 = min(de, run);
            ce = l0;
            if (l0 < h0)
                ce = l0 + group_count_true<32>(l0, h0 - 1, lane, 0xFFFFFFFFu, 0, [&](int m) {
                    const K b = lds_k<K>(sw3<K>(sbase + (uint32_t)sizeof(K) * (b0 + de - 1 - m)));
                    const K a = lds_k<K>(sw3<K>(sbase + (uint32_t)sizeof(K) * (a0 + m)));
                    return !kbef<K, ORD>(b, a);
                });
        }
        int hi = min(min(d, run), ce);
        int lo = min(max(max(0, d - run), ce - (de - d)), hi);
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            const K b = lds_k<K>(sw3<K>(sbase + (uint32_t)sizeof(K) * (b0 + d - 1 - m)));
            const K a = lds_k<K>(sw3<K>(sbase + (uint32_t)sizeof(K) * (a0 + m)));
            if (!kbef<K, ORD>(b, a)) lo = m + 1;
            else hi = m;
        }
        i = lo;
        inext = __shfl_down_sync(0xFFFFFFFFu, i, 1);
        if (lane == 31) inext = ce;
    } else {
        merge_path3x2<K, ORD>(sbase, a0, run, b0, run, d, (lane_id() == 31 && local + 1 < coop), i, inext);
        const int up = __shfl_down_sync(0xFFFFFFFFu, i, 1);
        if (lane_id() != 31) inext = up;
        if (local + 1 == coop) inext = run;
    }
    const int dn = d + VT3;
    if ((GNS_K1_NET & (sizeof(K) == 4 ? 1 : 2)) && net) {
        net_merge3<K, ORD>(sbase, a0 + i, inext - i, b0 + d - i, k);
        return;
    }
    serial_merge3<K, ORD>(sbase, a0, a0 + i, b0, b0 + d - i, b0 + run, a0 + inext, b0 + dn - inext, k);
}

// ---- warp-level bitonic merge rounds (runs of 64 keys in 2^r lanes, r = 1..5)
// A data-independent merge of two sorted runs held in registers across lanes:
// one compare of A[i] with B[R-1-i] (partner lane ^ (2^r - 1), register
// reversed), then half-cleaners across lanes (lane ^ d, same register) and
// in registers (distances 32..1).  Shuffles cost one shared-memory wavefront
// per 32-bit warp transfer (measured), a quarter of what a data-dependent
// merge-path round costs here (random 8-byte loads, ~4 wavefronts per
// half-warp), and there is no spill, search or barrier.  Unstable: used only
// by warps without -0.0/+0.0 or NaN keys (key-only, equal keys are
// bit-identical), the others take the stable merge-path rounds.
template <typename K, int ORD>
__device__ __forceinline__ K bce(K own, K oth, bool up)
{
    // the lower lane keeps the earlier key, the upper lane the later one
    return (kbef<K, ORD>(oth, own) != up) ? oth : own;
}

template <typename K, int ORD>
__device__ __forceinline__ void incore_halfcleaners(K (&k)[VT3])
{
#pragma unroll
    for (int dist = VT3 / 2; dist >= 1; dist >>= 1) {
#pragma unroll
        for (int i = 0; i < VT3; ++i) {
            if ((i & dist) == 0) {
                const bool p = kbef<K, ORD>(k[i + dist], k[i]);
                const K lo = p ? k[i + dist] : k[i];
                const K hi = p ? k[i] : k[i + dist];
                k[i] = lo;
                k[i + dist] = hi;
            }
        }
    }
}

template <typename K, int ORD>
__device__ __forceinline__ void warp_bitonic_rounds(K (&k)[VT3], int lane)
{
#pragma unroll 1
    for (int h = 1; h < (1 << GNS_K1_BITONIC); h <<= 1) {   // runs of 64 h keys in h lanes -> 128 h in 2 h lanes
        const int mask = 2 * h - 1;
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int x = 0; x < VT3 / 2; ++x) {
            const K lo = k[x], hi = k[VT3 - 1 - x];
            const K olo = __shfl_xor_sync(0xFFFFFFFFu, lo, mask);
            const K ohi = __shfl_xor_sync(0xFFFFFFFFu, hi, mask);
            k[x] = bce<K, ORD>(lo, ohi, up);
            k[VT3 - 1 - x] = bce<K, ORD>(hi, olo, up);
        }
#pragma unroll 1
        for (int d = h >> 1; d >= 1; d >>= 1) {
            const bool u = (lane & d) != 0;
#pragma unroll
            for (int x = 0; x < VT3; ++x) {
                const K o = __shfl_xor_sync(0xFFFFFFFFu, k[x], d);
                k[x] = bce<K, ORD>(k[x], o, u);
            }
        }
        incore_halfcleaners<K, ORD>(k);
    }
}

// 1-D bulk copy shared -> global (TMA engine), bulk-group completion
__device__ __forceinline__ void bulk_store_1d(void *gdst, const void *ssrc, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}

// ---- distributed shared memory (thread-block cluster) access
__device__ __forceinline__ uint32_t cl_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_size()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address a of this CTA -> the same offset in cluster CTA `rank`
__device__ __forceinline__ uint32_t cl_map(uint32_t a, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
template <typename K>
__device__ __forceinline__ void sts_k(uint32_t a, K v)
{
    if constexpr (sizeof(K) == 8) asm volatile("st.shared.f64 [%0], %1;" :: "r"(a), "d"(v) : "memory");
    else asm volatile("st.shared.f32 [%0], %1;" :: "r"(a), "f"(v) : "memory");
}
template <typename K>
__device__ __forceinline__ K ldc_k(uint32_t a)
{
    if constexpr (sizeof(K) == 8) {
        double v;
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
        return v;
    } else {
        float v;
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
        return v;
    }
}

// Cluster extension of K1 (CLU): the C CTAs of a thread-block cluster hold
// their sorted tiles in shared memory (linear sw3 layout at sbase, identical
// addresses in every CTA) and merge them on chip into one run of C x TL keys
// in log2(C) levels: at level G (groups of G CTAs, runs of G/2 tiles), CTA c
// produces outputs [(c - g0) TL, +TL) of its group's pair (A = the first G/2
// tiles, B = the rest): warps 0 / 1 find the co-ranks of its first and
// one-past-last output by 33-ary searches over the remote keys (left run
// wins ties), every thread loads 64 of the TL inputs A[i0:i1),
// B[j0:j1) from the remote CTAs into registers, a cluster barrier ends the
// remote reads, the inputs go to the CTA's own shared memory and one
// merge-path round (merge_path3x2 + serial_merge3) merges them.  Pads (the
// order's largest key) of a ragged or empty last tile stay behind every real
// key.  No HBM traffic; the merge passes that follow start at C x TL keys.
template <typename K, int ORD, int NT3>
__device__ __forceinline__ void cluster_levels(uint32_t sbase, int tid, K (&k)[VT3])
{
    constexpr int TL = NT3 * VT3;
    constexpr int PER = 16 / (int)sizeof(K);
    constexpr uint32_t SZ = sizeof(K);
    __shared__ int s_co[2];
    const int C = (int)cl_size(), c = (int)cl_rank();
    const int e0 = tid * VT3;
    const int warp = tid >> 5, lane = tid & 31;
#pragma unroll 1
    for (int G = 2; G <= C; G <<= 1) {
        __syncthreads();                              // (the previous merge's reads of the staging are done)
#pragma unroll
        for (int q = 0; q < VT3 / PER; ++q) sts16_k<K>(sw3<K>(sbase + SZ * (e0 + PER * q)), &k[PER * q]);
        cl_sync();                                    // every CTA's run is in its shared memory
        const int g0 = c & ~(G - 1), half = G >> 1;
        const int run = half * TL;
        const int d0 = (c - g0) * TL;
        auto A = [&](int m) -> K {
            return ldc_k<K>(cl_map(sw3<K>(sbase + SZ * (uint32_t)(m & (TL - 1))), (uint32_t)(g0 + m / TL)));
        };
        auto B = [&](int m) -> K {
            return ldc_k<K>(cl_map(sw3<K>(sbase + SZ * (uint32_t)(m & (TL - 1))), (uint32_t)(g0 + half + m / TL)));
        };
        if (warp < 2) {
            const int d = d0 + warp * TL;
            const int lo = max(0, d - run), hi = min(d, run);
            int r = lo;
            if (lo < hi)
                r = lo + group_count_true<32>(lo, hi - 1, lane, 0xFFFFFFFFu, 0,
                                              [&](int m) { return !kbef<K, ORD>(B(d - 1 - m), A(m)); });
            if (lane == 0) s_co[warp] = r;
        }
        __syncthreads();
        const int i0 = s_co[0], i1 = s_co[1];
        const int j0 = d0 - i0;
        const int ca = i1 - i0, cb = TL - ca;
        // the TL inputs [A slice, B slice]: element e = x NT3 + tid (consecutive
        // lanes, consecutive remote slots), all loads issued before any use
#pragma unroll
        for (int x = 0; x < VT3; ++x) {
            const int e = x * NT3 + tid;
            const bool fa = e < ca;
            const int m = fa ? i0 + e : j0 + (e - ca);
            const int r = (fa ? g0 : g0 + half) + m / TL;
            k[x] = ldc_k<K>(cl_map(sw3<K>(sbase + SZ * (uint32_t)(m & (TL - 1))), (uint32_t)r));
        }
        cl_sync();                                    // every remote read of this level is done
#pragma unroll
        for (int x = 0; x < VT3; ++x) {
            const int e = x * NT3 + tid;
            sts_k<K>(sw3<K>(sbase + SZ * e), k[x]);
        }
        __syncthreads();
        int i, inext;
        merge_path3x2<K, ORD>(sbase, 0, ca, ca, cb, e0, (lane == 31 && tid + 1 < NT3), i, inext);
        const int up = __shfl_down_sync(0xFFFFFFFFu, i, 1);
        if (lane != 31) inext = up;
        if (tid + 1 == NT3) inext = ca;
        const int dn = e0 + VT3;
        serial_merge3<K, ORD>(sbase, 0, i, ca, ca + e0 - i, TL, inext, ca + dn - inext, k);
    }
    __syncthreads();                                  // (the caller reuses the shared memory)
}

// K1 key-only.  Same contract as tile_sort2_kernel<false, ORD> (flags,
// samples, Omitsort tile descriptors; the tensor maps are unused).  K = double
// (every 8-byte key type, ORD = DESC | key type << 1) or float (NEXT f3
// binary32 keys, ORD = DESC; flags / samples / descriptors unused).
// CLU: launched in thread-block clusters of C CTAs, the output runs are
// C x TL keys (cluster_levels); no Omitsort descriptors (tdesc == nullptr).
template <typename K, int ORD, int NT3 = gns::NT3, bool CLU = false>
__global__ void __launch_bounds__(NT3, NT3 == gns::NT3 ? (sizeof(K) == 4 ? GNS_T3F_MINB : GNS_T3_MINB) : 1)
tile_sort3_kernel(const K *src_k, K *dst_k, long long n, unsigned *unsorted, K *smp,
                  unsigned char *tdesc, K *smp_src, int smp_log2)
{
    constexpr int TL = NT3 * VT3;                // keys per tile
    constexpr int SZ = sizeof(K);
    constexpr int SEG = VT3 * SZ + 16;           // padded segment per thread
    constexpr int PER = 16 / SZ;                 // keys per 16-byte transfer
    pdl_wait();
    GNS_TL_START(0);
    extern __shared__ __align__(16) unsigned char smem3[];
    unsigned char *smem = smem3 + ((128u - (smem_u32(smem3) & 127u)) & 127u);
    __shared__ __align__(8) uint64_t bar;
    __shared__ unsigned s_flags;
    const int tid = threadIdx.x;
    const long long tile = blockIdx.x;
    const long long base = tile * TL;
    const int cnt = (int)min((long long)TL, n - base);
    const bool full = cnt == TL;
    const int e0 = tid * VT3;
    unsigned char *seg = smem + tid * SEG;              // this thread's padded segment
    K k[VT3];
    if (tid == 0) {
        s_flags = 0;
        if (full) {
            mbar_init(&bar, 1);
            fence_mbar_init();
            mbar_expect_tx(&bar, (uint32_t)TL * SZ);
        }
    }
    __syncthreads();
    if (full) {
        tma_load_1d(seg, src_k + base + e0, VT3 * SZ, &bar, policy_evict_first());
        if (tid == 0) mbar_arrive(&bar);
        mbar_wait(&bar, 0);
#pragma unroll
        for (int c = 0; c < VT3 / PER; ++c) lds16_k<K>(smem_u32(seg) + 16 * c, &k[PER * c]);
    } else {
#pragma unroll
        for (int x = 0; x < VT3; ++x) {
            const int e = e0 + x;
            // pads sort after every real key; they are bit-identical to the
            // largest key, so an unstable order among them changes nothing
            k[x] = e < cnt ? src_k[base + e] : kpad<K, ORD>();
        }
    }
    // ---- NEXT f2 per-tile order tests (as in tile_sort2_kernel): in order
    // (Omitsort) or strictly reversed (Octosort)
    int mode = 0;
    {
        int pairs = 0, desc = 0;
#pragma unroll
        for (int x = 0; x + 1 < VT3; ++x) {
            if (e0 + x + 1 < cnt) {
                ++pairs;
                desc += kbef<K, ORD>(k[x + 1], k[x]) ? 1 : 0;
            }
        }
        unsigned fl = 0;
        const long long nx = base + e0 + VT3;
        if (nx < n) {
            const K kn = (full && e0 + VT3 < TL) ? *reinterpret_cast<const K *>(seg + SEG) : src_k[nx];
            const bool d = kbef<K, ORD>(kn, k[VT3 - 1]);
            fl |= (e0 + VT3 < cnt) ? (d ? 1u : 2u) : (d ? 4u : 8u);
        }
        fl |= (desc > 0 ? 1u : 0u) | (desc < pairs ? 2u : 0u);
        fl = __reduce_or_sync(0xFFFFFFFFu, fl);
        if (lane_id() == 0 && fl) atomicOr(&s_flags, fl);
        __syncthreads();
        fl = s_flags;
        mode = !(fl & 1u) ? 1 : (!(fl & 2u) && full) ? 2 : 0;
        if (unsorted && tid == 0) {
            const unsigned g = ((fl | (fl >> 2)) & 3u);
            if (g) atomicOr(unsorted, g);
        }
    }
    if (mode == 0) {
        // ---- the thread's 64 keys: sorting network in registers
        // floating-point keys (binary64 / binary32): the zero-sign fix-up and
        // the -0.0 / NaN check; the integer key types have neither
        constexpr bool F64 = sizeof(K) == 4 || (ORD >> 1) == KT_F64;
        unsigned long long zsign = 0;      // signs of the thread's zeros, input order
        bool zero = false, special = false;
        if (F64) {
#pragma unroll
            for (int x = 0; x < VT3; ++x) {
                zero |= (k[x] == (K)0);
            }
            if (zero) {
                int z = 0;
#pragma unroll
                for (int x = 0; x < VT3; ++x) {
                    if (k[x] == (K)0) {
                        zsign |= (unsigned long long)sign_set<K>(k[x]) << z;
                        ++z;
                        k[x] = (K)0;
                    }
                }
            }
        }
        network_sort<K, VT3, ORD>(k);
        if (F64 && zero) {
            int z = 0;
#pragma unroll
            for (int x = 0; x < VT3; ++x) {
                if (k[x] == (K)0) {
                    k[x] = ((zsign >> z) & 1ull) ? -(K)0 : (K)0;
                    ++z;
                }
            }
        }
        const uint32_t sbase = smem_u32(smem) + 256u;   // (one slot before the array is readable)
        // ---- rounds 1-3 (runs 64 -> 512, inside each warp): bitonic unless
        // some key of the CTA is -0.0 or NaN (then all 7 rounds merge-path)
        if (F64) {
            // (computed after the network, which permutes the keys: a flag
            // live across it costs registers)
#pragma unroll
            for (int x = 0; x < VT3; ++x)       // -0.0 (unequal bits among equal keys) or NaN
                special |= !(k[x] >= (K)0 || k[x] < (K)0) || neg_zero<K>(k[x]);
        }
        const bool cta_special = __syncthreads_or(special) != 0;
        if (!cta_special) warp_bitonic_rounds<K, ORD>(k, lane_id());
        // ---- merge-path rounds (runs 2048 -> 8192, or 64 -> 8192)
#pragma unroll 1
        for (int coop = cta_special ? 2 : (2 << GNS_K1_BITONIC); coop <= NT3; coop <<= 1) {
            // rounds inside one warp (coop <= 32: a pair's threads, their spills
            // and their reads all belong to that warp) synchronise the warp only
            merge_round3<K, ORD>(sbase, tid, e0, coop, k, true, F64 && !cta_special);
            pair_sync(tid, coop, NT3);
        }
    } else {
        __syncthreads();
    }
    // Omitsort schedule (tdesc != nullptr): bit 0 = kept as a descending run,
    // bit 1 = written to dst
    if (tdesc != nullptr && tid == 0)
        tdesc[tile] = (unsigned char)((mode == 2 ? 1 : 0) | ((mode == 0 && dst_k != src_k) ? 2 : 0));
    if (tdesc != nullptr && mode != 0) {
        if (smp_src != nullptr && e0 < cnt && (tid & (SMP_G / VT3 - 1)) == 0)
            smp_src[(base + e0) >> SMP_LOG2] = k[0];
        GNS_TL_END(0);
        pdl_trigger();
        return;
    }
    if (CLU) {
        const uint32_t sbase = smem_u32(smem) + 256u;
        if (mode == 2) {
            // strictly reversed full tile: sorted order = the reversal (thread
            // t's keys go to the other end), through shared memory
            __syncthreads();
#pragma unroll
            for (int c = 0; c < VT3 / PER; ++c) {
                K r[PER];
#pragma unroll
                for (int j = 0; j < PER; ++j) r[j] = k[PER * c + PER - 1 - j];
                sts16_k<K>(sw3<K>(sbase + (uint32_t)SZ * (TL - e0 - PER * (c + 1))), r);
            }
            __syncthreads();
#pragma unroll
            for (int c = 0; c < VT3 / PER; ++c) lds16_k<K>(sw3<K>(sbase + (uint32_t)SZ * (e0 + PER * c)), &k[PER * c]);
        }
        cluster_levels<K, ORD, NT3>(sbase, tid, k);
    }
    if (!CLU && mode == 2) {
        // full tile, strictly reversed: output TL-1-e <- input e; thread t
        // fills segment 127-t backwards and stores it
        const int ot = NT3 - 1 - tid;
        unsigned char *oseg = smem + ot * SEG;
#pragma unroll
        for (int c = 0; c < VT3 / PER; ++c) {
            K r[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) r[j] = k[PER * c + PER - 1 - j];
            sts16_k<K>(smem_u32(oseg) + 16 * (VT3 / PER - 1 - c), r);
        }
        // (samples of dst every 1 << smp_log2 keys, smp_log2 >= log2(VT3); 6 before 4-way passes)
        if (smp != nullptr && (ot & ((1 << (smp_log2 - VT3_LOG2)) - 1)) == 0)
            smp[(base + (long long)ot * VT3) >> smp_log2] = k[VT3 - 1];
        fence_proxy_async();
        bulk_store_1d(dst_k + base + (long long)ot * VT3, oseg, VT3 * SZ);
        bulk_commit();
        bulk_wait_read0();
        GNS_TL_END(0);
        pdl_trigger();
        return;
    }
    if (smp != nullptr && e0 < cnt && (tid & ((1 << (smp_log2 - VT3_LOG2)) - 1)) == 0)
        smp[(base + e0) >> smp_log2] = k[0];
    if (!CLU && mode == 1 && dst_k == src_k) {
        GNS_TL_END(0);
        pdl_trigger();
        return;
    }
    if (full) {
#pragma unroll
        for (int c = 0; c < VT3 / PER; ++c) sts16_k<K>(smem_u32(seg) + 16 * c, &k[PER * c]);
        fence_proxy_async();
        bulk_store_1d(dst_k + base + e0, seg, VT3 * SZ);
        bulk_commit();
        bulk_wait_read0();
    } else {
#pragma unroll
        for (int x = 0; x < VT3; ++x)
            if (e0 + x < cnt) dst_k[base + e0 + x] = k[x];
    }
    GNS_TL_END(0);
    pdl_trigger();
}

}  // namespace gns
