// gns_tile64.cuh — K1 for key-only sorts: the stable
// sort of one 8192-key tile per CTA with 128 threads x 64 keys.
//
// Why a second K1 for key-only: the 256 x 32 kernel (tile_sort2_kernel) is
// bound by shared-memory wavefronts (ncu: l1tex 91 % busy, 3.7 wavefronts per
// key, half of them bank conflicts of the data-dependent merge reads) and
// spends ~77 instructions per key on its 32-key transposition sort.  Here:
//   * one 64-key sorting network per thread in registers (Batcher's odd-even
//     merge sort: 543 compare-exchanges instead of 2016 for a 64-key
//     transposition sort) -- unstable, which is harmless for key-only input
//     because equal keys are bit-identical, except -0.0 / +0.0 (equal under
//     IEEE <, different bits): a thread holding a zero records the signs of its
//     zeros in input order, sorts canonical +0.0 and writes the signs back in
//     that order, which is exactly the stable order (R2);
//   * 3 warp-level bitonic merge rounds in registers + shuffles (runs 64 ->
//     512) unless the CTA holds a -0.0 or NaN key, then 4 shared-memory
//     merge-path rounds (runs 512 -> 8192; all 7 in the -0.0 / NaN case), each
//     thread producing 64 outputs as two independent chains (merge path +
//     serial merge, left run wins ties);
//   * the tile arrives by 128 one-dimensional bulk copies (one 512-byte
//     segment per thread, TMA engine, one mbarrier) into a padded layout whose
//     16-byte register transfers are conflict-free, and leaves the same way.
// Measured (B200, 2^24 f64 U(0,1), event-timed): 246 -> 223 us; ncu: 61.5 M ->
// ~31 M shared wavefronts, 154 M -> ~120 M instructions (DESIGN.md 8b lists
// the variants tried: one-load merge steps, 16384-key tiles, 0-5 bitonic rounds).
// One read-scan and one write-scan of HBM per tile; the 13
// merge levels inside the tile cost no HBM traffic.
#pragma once

namespace gns {

// warp-level bitonic merge rounds before the merge-path rounds (0..5)
#ifndef GNS_K1_BITONIC
#define GNS_K1_BITONIC 3
#endif
#ifndef GNS_K1_ONELDS
#define GNS_K1_ONELDS 0
#endif
constexpr int NT3 = 128;                  // threads per CTA
constexpr int VT3 = 64;                   // keys per thread
static_assert(NT3 * VT3 == TILE, "K1 key-only tile must equal TILE");
template <int NT> constexpr size_t t3_smem() { return (size_t)NT * (VT3 * 8 + 16) + 128; }
constexpr int SEG3_BYTES = VT3 * 8 + 16;  // padded 512-byte segment per thread
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

template <int N, int ORD>
__device__ __forceinline__ void network_sort(double (&k)[N])
{
    constexpr OddEvenNet<N> net{};
#pragma unroll
    for (int c = 0; c < OddEvenNet<N>::NC; ++c) {
        const int i = net.a[c], j = net.b[c];
        const bool p = before<ORD>(k[j], k[i]);
        const double lo = p ? k[j] : k[i];
        const double hi = p ? k[i] : k[j];
        k[i] = lo;
        k[j] = hi;
    }
}

// Merge-round layout: byte address a -> a with its 16-byte chunk (bits 4-6)
// XORed with bits 9-11 (the thread's 512-byte block), so the blocked 16-byte
// spill (lane t writes chunk c of its own block) hits 8 distinct chunk
// positions per 8 lanes: conflict-free.  A bijection on every 128-byte line.
__device__ __forceinline__ uint32_t sw3(uint32_t a) { return a ^ ((a >> 5) & 0x70u); }

// Stable co-rank of diagonal d (A wins ties; predicate A[m] <= B[d-1-m]) and,
// if `two`, of diagonal d + VT3 in the same loop (independent probes).
template <int ORD>
__device__ __forceinline__ void merge_path3x2(uint32_t base, int a0, int na, int b0, int nb, int d, bool two,
                                              int &r1, int &r2)
{
    int lo = max(0, d - nb), hi = min(d, na);
    const int d2 = d + VT3;
    int lo2 = two ? max(0, d2 - nb) : 0, hi2 = two ? min(d2, na) : 0;
    while (lo < hi || lo2 < hi2) {
        if (lo < hi) {
            const int m = (lo + hi) >> 1;
            const double b = lds_f64(sw3(base + 8u * (b0 + d - 1 - m)));
            const double a = lds_f64(sw3(base + 8u * (a0 + m)));
            if (!before<ORD>(b, a)) lo = m + 1;
            else hi = m;
        }
        if (lo2 < hi2) {
            const int m = (lo2 + hi2) >> 1;
            const double b = lds_f64(sw3(base + 8u * (b0 + d2 - 1 - m)));
            const double a = lds_f64(sw3(base + 8u * (a0 + m)));
            if (!before<ORD>(b, a)) lo2 = m + 1;
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
template <int ORD>
__device__ __forceinline__ void serial_merge3(uint32_t base, int a0, int ai, int aend, int bi, int bend, int qa,
                                              int qb, double (&k)[VT3])
{
    uint32_t pa = base + 8u * ai, pb = base + 8u * bi;
    const uint32_t pae = base + 8u * aend, pbe = base + 8u * bend;
    // backward chain: ra / rb = addresses of the next A / B key to take from
    // the back; A's run starts at a0, B's run starts at aend
    uint32_t ra = base + 8u * (qa - 1), rb = base + 8u * (qb - 1);
    const uint32_t ras = base + 8u * a0, rbs = pae;
    double ka = lds_f64(sw3(pa)), kb = lds_f64(sw3(pb));
    double ta = lds_f64(sw3(ra)), tb = lds_f64(sw3(rb));
#pragma unroll
    for (int x = 0; x < VT3 / 2; ++x) {
        const bool p = (pb < pbe) && ((pa >= pae) || before<ORD>(kb, ka));
        k[x] = p ? kb : ka;
        const uint32_t nxt = (p ? pb : pa) + 8u;
        GNS_DASSERT(nxt >= base && nxt <= base + 8u * 2 * TILE + 8u);
        const uint32_t a = sw3(nxt);
        // backward: take A's tail iff it exists and (B is exhausted or B's
        // tail is strictly before it)
        const bool q = (ra >= ras) && ((rb < rbs) || before<ORD>(tb, ta));
        k[VT3 - 1 - x] = q ? ta : tb;
        const uint32_t prv = (q ? ra : rb) - 8u;
        GNS_DASSERT(prv + 8u >= base && prv < base + 8u * 2 * TILE);
        const uint32_t b = sw3(prv);
#if GNS_K1_ONELDS
        // one full-warp load per chain step (fewer shared wavefronts than two
        // predicated half-warp loads), routed into the consumed side's head
        const double u = lds_f64(a), w = lds_f64(b);
        if (p) pb = nxt; else pa = nxt;
        kb = p ? u : kb;
        ka = p ? ka : u;
        if (q) ra = prv; else rb = prv;
        ta = q ? w : ta;
        tb = q ? tb : w;
#else
        if (p) {
            pb = nxt;
            kb = lds_f64(a);
        } else {
            pa = nxt;
            ka = lds_f64(a);
        }
        if (q) {
            ra = prv;
            ta = lds_f64(b);
        } else {
            rb = prv;
            tb = lds_f64(b);
        }
#endif
    }
}

// One merge-path round: spill the thread's sorted run block, synchronise
// (the warp, or the CTA if `cta`), then merge pair (A, B) of runs of
// (coop / 2) * VT3 keys; the thread produces outputs [d, d + VT3) of its pair.
template <int ORD>
__device__ __forceinline__ void merge_round3(uint32_t sbase, int tid, int e0, int coop, double (&k)[VT3],
                                             bool cta = false)
{
#pragma unroll
    for (int c = 0; c < VT3 / 2; ++c)
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};"
                     :: "r"(sw3(sbase + 8u * (e0 + 2 * c))), "d"(k[2 * c]), "d"(k[2 * c + 1]) : "memory");
    if (cta) __syncthreads();
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
    merge_path3x2<ORD>(sbase, a0, run, b0, run, d, (lane_id() == 31 && local + 1 < coop), i, inext);
    const int up = __shfl_down_sync(0xFFFFFFFFu, i, 1);
    if (lane_id() != 31) inext = up;
    if (local + 1 == coop) inext = run;
    const int dn = d + VT3;
    serial_merge3<ORD>(sbase, a0, a0 + i, b0, b0 + d - i, b0 + run, a0 + inext, b0 + dn - inext, k);
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
template <int ORD>
__device__ __forceinline__ double bce(double own, double oth, bool up)
{
    // the lower lane keeps the earlier key, the upper lane the later one
    return (before<ORD>(oth, own) != up) ? oth : own;
}

template <int ORD>
__device__ __forceinline__ void incore_halfcleaners(double (&k)[VT3])
{
#pragma unroll
    for (int dist = VT3 / 2; dist >= 1; dist >>= 1) {
#pragma unroll
        for (int i = 0; i < VT3; ++i) {
            if ((i & dist) == 0) {
                const bool p = before<ORD>(k[i + dist], k[i]);
                const double lo = p ? k[i + dist] : k[i];
                const double hi = p ? k[i] : k[i + dist];
                k[i] = lo;
                k[i + dist] = hi;
            }
        }
    }
}

template <int ORD>
__device__ __forceinline__ void warp_bitonic_rounds(double (&k)[VT3], int lane)
{
#pragma unroll 1
    for (int h = 1; h < (1 << GNS_K1_BITONIC); h <<= 1) {   // runs of 64 h keys in h lanes -> 128 h in 2 h lanes
        const int mask = 2 * h - 1;
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int x = 0; x < VT3 / 2; ++x) {
            const double lo = k[x], hi = k[VT3 - 1 - x];
            const double olo = __shfl_xor_sync(0xFFFFFFFFu, lo, mask);
            const double ohi = __shfl_xor_sync(0xFFFFFFFFu, hi, mask);
            k[x] = bce<ORD>(lo, ohi, up);
            k[VT3 - 1 - x] = bce<ORD>(hi, olo, up);
        }
#pragma unroll 1
        for (int d = h >> 1; d >= 1; d >>= 1) {
            const bool u = (lane & d) != 0;
#pragma unroll
            for (int x = 0; x < VT3; ++x) {
                const double o = __shfl_xor_sync(0xFFFFFFFFu, k[x], d);
                k[x] = bce<ORD>(k[x], o, u);
            }
        }
        incore_halfcleaners<ORD>(k);
    }
}

// 1-D bulk copy shared -> global (TMA engine), bulk-group completion
__device__ __forceinline__ void bulk_store_1d(void *gdst, const void *ssrc, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}

// K1 key-only.  Same contract as tile_sort2_kernel<false, ORD> (flags,
// samples, Omitsort tile descriptors; the tensor maps are unused).
template <int ORD, int NT3 = gns::NT3>
__global__ void __launch_bounds__(NT3, NT3 == 128 ? 3 : 1)
tile_sort3_kernel(const double *src_k, double *dst_k, long long n, unsigned *unsorted, double *smp,
                  unsigned char *tdesc, double *smp_src)
{
    constexpr int TL = NT3 * VT3;                // keys per tile
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
    unsigned char *seg = smem + tid * SEG3_BYTES;       // this thread's padded segment
    double k[VT3];
    if (tid == 0) {
        s_flags = 0;
        if (full) {
            mbar_init(&bar, 1);
            fence_mbar_init();
            mbar_expect_tx(&bar, (uint32_t)TL * 8u);
        }
    }
    __syncthreads();
    if (full) {
        tma_load_1d(seg, src_k + base + e0, VT3 * 8, &bar, policy_evict_first());
        if (tid == 0) mbar_arrive(&bar);
        mbar_wait(&bar, 0);
#pragma unroll
        for (int c = 0; c < VT3 / 2; ++c) lds128(seg + 16 * c, k[2 * c], k[2 * c + 1]);
    } else {
#pragma unroll
        for (int x = 0; x < VT3; ++x) {
            const int e = e0 + x;
            // pads sort after every real key; they are bit-identical to the
            // largest key, so an unstable order among them changes nothing
            k[x] = e < cnt ? src_k[base + e] : pad_key<ORD>();
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
                desc += before<ORD>(k[x + 1], k[x]) ? 1 : 0;
            }
        }
        unsigned fl = 0;
        const long long nx = base + e0 + VT3;
        if (nx < n) {
            const double kn = (full && e0 + VT3 < TL) ? *reinterpret_cast<const double *>(seg + SEG3_BYTES)
                                                        : src_k[nx];
            const bool d = before<ORD>(kn, k[VT3 - 1]);
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
        constexpr bool F64 = (ORD >> 1) == KT_F64;
        unsigned long long zsign = 0;      // signs of the thread's zeros, input order
        bool zero = false, special = false;
        if (F64) {
#pragma unroll
            for (int x = 0; x < VT3; ++x) {
                zero |= (k[x] == 0.0);
            }
            if (zero) {
                int z = 0;
#pragma unroll
                for (int x = 0; x < VT3; ++x) {
                    if (k[x] == 0.0) {
                        zsign |= (unsigned long long)(__double_as_longlong(k[x]) < 0) << z;
                        ++z;
                        k[x] = 0.0;
                    }
                }
            }
        }
        network_sort<VT3, ORD>(k);
        if (F64 && zero) {
            int z = 0;
#pragma unroll
            for (int x = 0; x < VT3; ++x) {
                if (k[x] == 0.0) {
                    k[x] = ((zsign >> z) & 1ull) ? -0.0 : 0.0;
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
                special |= !(k[x] >= 0.0 || k[x] < 0.0) || __double_as_longlong(k[x]) == (long long)0x8000000000000000ULL;
        }
        const bool cta_special = __syncthreads_or(special) != 0;
        if (!cta_special) warp_bitonic_rounds<ORD>(k, lane_id());
        // ---- merge-path rounds (runs 2048 -> 8192, or 64 -> 8192)
#pragma unroll 1
        for (int coop = cta_special ? 2 : (2 << GNS_K1_BITONIC); coop <= NT3; coop <<= 1) {
            merge_round3<ORD>(sbase, tid, e0, coop, k, true);
            __syncthreads();
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
    if (mode == 2) {
        // full tile, strictly reversed: output TL-1-e <- input e; thread t
        // fills segment 127-t backwards and stores it
        const int ot = NT3 - 1 - tid;
        unsigned char *oseg = smem + ot * SEG3_BYTES;
#pragma unroll
        for (int c = 0; c < VT3 / 2; ++c) sts128(oseg + 16 * (VT3 / 2 - 1 - c), k[2 * c + 1], k[2 * c]);
        if (smp != nullptr && (ot & (SMP_G / VT3 - 1)) == 0)
            smp[(base + (long long)ot * VT3) >> SMP_LOG2] = k[VT3 - 1];
        fence_proxy_async();
        bulk_store_1d(dst_k + base + (long long)ot * VT3, oseg, VT3 * 8);
        bulk_commit();
        bulk_wait_read0();
        GNS_TL_END(0);
        pdl_trigger();
        return;
    }
    if (smp != nullptr && e0 < cnt && (tid & (SMP_G / VT3 - 1)) == 0)
        smp[(base + e0) >> SMP_LOG2] = k[0];
    if (mode == 1 && dst_k == src_k) {
        GNS_TL_END(0);
        pdl_trigger();
        return;
    }
    if (full) {
#pragma unroll
        for (int c = 0; c < VT3 / 2; ++c) sts128(seg + 16 * c, k[2 * c], k[2 * c + 1]);
        fence_proxy_async();
        bulk_store_1d(dst_k + base + e0, seg, VT3 * 8);
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
