// gns_merge4.cuh — two merge levels per HBM pass (SURVEY.md §8 rows a3 + a4):
// groups of four runs R0..R3 of length L are merged into one run of 4L in
// one read-scan and one write-scan of HBM, as (R0 ⊕ R1) ⊕ (R2 ⊕ R3) on chip.
//
// Why: the merge passes are HBM-bound (a 2-way pass streams at ~0.8 of the
// copy peak) and the tile sort leaves 11 of them at 2^24 keys; a 4-way pass
// does two merge levels for the bytes of one (every level costs one
// read-scan and one write-scan -- here two levels share them).
//
// Splits without a nested search.  An exact 4-way co-rank of an arbitrary
// output position needs a search inside a search; instead the pass splits at
// PIVOTS: every PIV-th key of every run.  For pivot v = R_r[p] the keys that
// precede v in the stable order (key, run, position) are, per run s,
//   s < r: the keys <= v (upper bound),  s = r: the first p,  s > r: the keys < v,
// so its split vector (c0, c1, c2, c3) needs three independent binary searches
// (rank4_kernel, sample-guided) and its output position is c0+c1+c2+c3.
// Consecutive pivots in output order are at most 4 * (PIV - 1) + 1 positions
// apart, so choosing for chunk j the pivot with the largest position <= j*T4
// gives chunks of T4 - 508 .. T4 + 508 outputs with exact split vectors.
//
// Per chunk the merge CTA loads the four slices R_s[c_s(j), c_s(j+1)) by 1-D
// bulk copies (TMA, mbarrier), merges S0 ⊕ S1 -> X' and S2 ⊕ S3 -> Y' into a
// shared buffer (merge path + serial merge, the left run wins ties,
// PAPER.md:221), then X' ⊕ Y' (X' wins ties: runs 0, 1 precede runs 2, 3)
// into the staging area, which leaves by one 1-D bulk store.  The result is
// the unique stable merge of the four runs.
#pragma once

namespace gns {

constexpr int FS_LOG2 = 6;                // fine samples: every 64th key of the runs (written by the previous pass)
constexpr int FS = 1 << FS_LOG2;
#ifndef GNS_M4_VT
#define GNS_M4_VT 11
#endif
#ifndef GNS_M4_T
#define GNS_M4_T 2048
#endif
#ifndef GNS_M4_CTAS
#define GNS_M4_CTAS 3
#endif
constexpr int T4 = GNS_M4_T;              // target outputs per chunk
constexpr int NT4 = 256;                  // merge threads per CTA
constexpr int VT4 = GNS_M4_VT;            // outputs per merge thread and level
constexpr int CAP4 = NT4 * VT4;           // 2816
// chunk sizes: T4 -+ (4 (FS - 1) + 1 + 3 (FS - 1)) (see chunk4_kernel)
constexpr int C4_DEV = 4 * (FS - 1) + 1 + 3 * (FS - 1);
static_assert(CAP4 >= T4 + C4_DEV + VT4, "chunk capacity");
constexpr int STG4_SLOTS = (T4 + C4_DEV + 16 + 63) / 64 * 64;   // input stage: four slices + parity / guard slots
static_assert(STG4_SLOTS >= T4 + C4_DEV + 16, "stage capacity");
constexpr int MID4_SLOTS = CAP4 + 8;
constexpr int M4_WARPS = NT4 / 32;        // 8 merge warps
constexpr int M4_THREADS = NT4 + 32;      // + producer warp
constexpr size_t M4_SMEM = 2 * (size_t)STG4_SLOTS * 8 + (size_t)MID4_SLOTS * 8 + 256;

struct Geo4 {
    const double *src;      // runs of length L; group q = runs 4q .. 4q+3
    double *dst;
    long long n;
    long long L;
    const double *fsmp;     // fine samples of src: fsmp[g >> FS_LOG2] = src[g] for g % FS == 0
    double *smp_out;        // samples of dst (every 1 << so_log2 -th key), or nullptr (last pass)
    int so_log2;
    int *apx;               // per fine sample: a lower bound of its output position (rank4_kernel)
    int4 *vec;              // per chunk: the split vector of its first output (chunk4_kernel)
    long long cpg;          // chunks per full group: ceil(4L / T4)
    long long nchunks;
};

__device__ __forceinline__ long long run_len4(const Geo4 &g, long long q, int s)
{
    const long long b = q * 4 * g.L + s * g.L;
    return max(0LL, min(g.L, g.n - b));
}

// x precedes the pivot v (of run r) in the stable order, x in run s != r
template <int ORD>
__device__ __forceinline__ bool precedes4(double x, double v, int s, int r)
{
    return s < r ? !before<ORD>(v, x) : before<ORD>(x, v);
}

// ------------------------------------------------ pivot positions, approximate
// Pivots = the fine samples (every FS-th key of every run).  For pivot
// v = R_r[p] the keys preceding it are, per run s != r, c_s = the keys <= v
// (s < r) or < v (s > r); with cnt_s = the fine samples of R_s preceding v,
// c_s lies in [FS (cnt_s - 1) + 1, FS cnt_s] (0 if cnt_s = 0).  rank4_kernel
// stores p + sum of the lower ends: the output position of v minus at most
// 3 (FS - 1).  Only the fine samples (L2-resident) are read.
template <int ORD>
__global__ void __launch_bounds__(256) rank4_kernel(Geo4 g, const unsigned *flag)
{
    pdl_wait();
    pdl_trigger();
    if (flag != nullptr) {
        const unsigned f = *(volatile const unsigned *)flag;
        if ((f & 1u) == 0u || (f & 2u) == 0u) return;      // NEXT f2: no merge in this pass
    }
    const long long np = (g.n + FS - 1) >> FS_LOG2;
    for (long long pi = blockIdx.x * (long long)blockDim.x + threadIdx.x; pi < np;
         pi += (long long)gridDim.x * blockDim.x) {
        const long long gp = pi << FS_LOG2;
        const long long q = gp / (4 * g.L);
        const long long gb = q * 4 * g.L;
        const int r = (int)((gp - gb) / g.L);
        const double v = g.fsmp[pi];
        int lo[4], hi[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            lo[s] = 0;
            hi[s] = 0;
            if (s != r) hi[s] = (int)((run_len4(g, q, s) + FS - 1) >> FS_LOG2);
        }
        bool busy = true;
        while (busy) {
            busy = false;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                if (lo[s] >= hi[s]) continue;
                busy = true;
                const int m = (lo[s] + hi[s]) >> 1;
                if (precedes4<ORD>(g.fsmp[((gb + s * g.L) >> FS_LOG2) + m], v, s, r)) lo[s] = m + 1;
                else hi[s] = m;
            }
        }
        int a = (int)(gp - gb - r * g.L);
#pragma unroll
        for (int s = 0; s < 4; ++s)
            if (s != r && lo[s] > 0) a += ((lo[s] - 1) << FS_LOG2) + 1;
        g.apx[pi] = a;
    }
}

// ------------------------------------------------------- chunk split vectors
// One warp per chunk j of group q (jj = j - q cpg): the pivot with the largest
// approximate position <= jj T4 (lanes 8s .. 8s+7 search run s's, 9-ary; the
// approximate positions of a run's pivots increase), then its exact split
// vector (per run s != r: the fine-sample count, then the exact count inside
// that FS window of R_s).  Chunk starts: consecutive pivots in output order
// are <= 4 (FS - 1) + 1 apart, the approximation is <= 3 (FS - 1) low, so the
// start lies in (jj T4 - 4(FS-1) - 1 - 3(FS-1), jj T4 + 3(FS-1)]: chunks of
// T4 -+ C4_DEV outputs, exact split vectors (jj = 0: the group start).
template <int ORD>
__global__ void __launch_bounds__(256) chunk4_kernel(Geo4 g, const unsigned *flag)
{
    pdl_wait();
    pdl_trigger();
    if (flag != nullptr) {
        const unsigned f = *(volatile const unsigned *)flag;
        if ((f & 1u) == 0u || (f & 2u) == 0u) return;
    }
    const long long j = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= g.nchunks) return;
    const long long q = j / g.cpg;
    const long long jj = j - q * g.cpg;
    if (jj == 0) {
        if (lane == 0) g.vec[j] = make_int4(0, 0, 0, 0);
        return;
    }
    const int k = (int)(jj * T4);
    const long long gb = q * 4 * g.L;
    const int s = lane >> 3, gl = lane & 7;
    const unsigned mask = 0xFFu << (8 * s);
    const long long ls = run_len4(g, q, s);
    const int nsmp = (int)((ls + FS - 1) >> FS_LOG2);
    const long long sb = (gb + s * g.L) >> FS_LOG2;       // run s's first fine sample
    // (1) the candidate of run s: its last pivot with approximate position <= k
    int cnt = 0;
    if (nsmp > 0) cnt = group_count_true<8>(0, nsmp - 1, gl, mask, 8 * s, [&](int i) { return g.apx[sb + i] <= k; });
    int best = cnt > 0 ? g.apx[sb + cnt - 1] : -1;
    int r = s, pi = cnt - 1;
#pragma unroll
    for (int off = 8; off <= 16; off <<= 1) {
        const int ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
        const int orr = __shfl_xor_sync(0xFFFFFFFFu, r, off);
        const int op = __shfl_xor_sync(0xFFFFFFFFu, pi, off);
        if (ob > best || (ob == best && orr < r)) {
            best = ob;
            r = orr;
            pi = op;
        }
    }
    // (2) the exact split vector of pivot v = R_r[FS pi]
    const double v = g.fsmp[((gb + r * g.L) >> FS_LOG2) + pi];
    int c = 0;
    if (s == r) {
        c = pi << FS_LOG2;
    } else if (nsmp > 0) {
        const int cs = group_count_true<8>(0, nsmp - 1, gl, mask, 8 * s,
                                           [&](int m) { return precedes4<ORD>(g.fsmp[sb + m], v, s, r); });
        if (cs > 0) {
            const int lo = ((cs - 1) << FS_LOG2) + 1;
            const int hi = (int)min((long long)cs << FS_LOG2, ls);
            const double *R = g.src + gb + s * g.L;
            c = lo + group_count_true<8>(lo, hi - 1, gl, mask, 8 * s,
                                         [&](int x) { return precedes4<ORD>(R[x], v, s, r); });
        }
    }
    const int c0 = __shfl_sync(0xFFFFFFFFu, c, 0), c1 = __shfl_sync(0xFFFFFFFFu, c, 8);
    const int c2 = __shfl_sync(0xFFFFFFFFu, c, 16), c3 = __shfl_sync(0xFFFFFFFFu, c, 24);
    if (lane == 0) g.vec[j] = make_int4(c0, c1, c2, c3);
}

struct Meta4 {
    int o[4];            // stage slot of slice s's first key
    int len[4];
    long long gout;      // dst index of the chunk's first output
    int cnt;
    int last;            // 1: end marker
};

// smem helpers (byte addresses)
__device__ __forceinline__ double lds4(uint32_t a) { return lds_f64(a); }
__device__ __forceinline__ void sts4(uint32_t a, double v)
{
    asm volatile("st.shared.f64 [%0], %1;" :: "r"(a), "d"(v) : "memory");
}

// merge path: number of A keys among the first d outputs (A wins ties)
template <int ORD>
__device__ __forceinline__ int mpath4(uint32_t A, int na, uint32_t B, int nb, int d)
{
    int lo = max(0, d - nb), hi = min(d, na);
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        const double b = lds4(B + 8u * (uint32_t)(d - 1 - m));
        const double a = lds4(A + 8u * (uint32_t)m);
        if (!before<ORD>(b, a)) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// up to VT4 outputs of the merge of A[ai..na) and B[bi..nb) (A wins ties);
// reads at most one slot past each run's end (never used)
template <int ORD>
__device__ __forceinline__ void serial4(uint32_t A, int ai, int na, uint32_t B, int bi, int nb, double (&k)[VT4])
{
    double ka = lds4(A + 8u * (uint32_t)ai), kb = lds4(B + 8u * (uint32_t)bi);
#pragma unroll
    for (int x = 0; x < VT4; ++x) {
        const bool p = (bi < nb) && ((ai >= na) || before<ORD>(kb, ka));
        k[x] = p ? kb : ka;
        if (p) {
            ++bi;
            kb = lds4(B + 8u * (uint32_t)bi);
        } else {
            ++ai;
            ka = lds4(A + 8u * (uint32_t)ai);
        }
    }
}

// Persistent 4-way merge pass.  CTA c owns global chunks [c N / G, (c+1) N / G).
//   warps 0-7  merge (two levels per chunk)
//   warp 8     producer (one lane): bulk copies of the four slices, bulk store of the staged chunk
template <int ORD>
__global__ void __launch_bounds__(M4_THREADS, GNS_M4_CTAS)
merge4_kernel(Geo4 g, Adapt ad)
{
    pdl_wait();
    const unsigned f_adapt = ad.flag ? *(volatile const unsigned *)ad.flag : 3u;
    const long long c0 = (long long)blockIdx.x * g.nchunks / gridDim.x;
    const long long c1 = (long long)(blockIdx.x + 1) * g.nchunks / gridDim.x;
    if ((f_adapt & 1u) == 0u || (f_adapt & 2u) == 0u) {
        // NEXT f2: ordered / strictly reversed input: only the scheduled moves
        const bool pre = (f_adapt & 1u) == 0u;
        const double *ck = pre ? ad.pre_k : ad.rev_k;
        if (ck) {
            MergeGeo mg{};
            mg.ok = g.dst;
            mg.n = g.n;
            const int ntl = (int)((g.n + MTILE - 1) / MTILE);
            adapt_move<false>(mg, (ntl + (int)gridDim.x - 1) / (int)gridDim.x, ck, nullptr, !pre && ad.rev_gather,
                              ad.run_log2);
        }
        pdl_trigger();
        return;
    }
    const int m = (int)(c1 - c0);
    extern __shared__ __align__(16) unsigned char smem4[];
    unsigned char *sm = smem4 + ((128u - (smem_u32(smem4) & 127u)) & 127u);
    auto stage = [&](int st) { return reinterpret_cast<double *>(sm + st * (STG4_SLOTS * 8)); };
    double *mid = reinterpret_cast<double *>(sm + 2 * STG4_SLOTS * 8);
    __shared__ __align__(8) uint64_t full[2];
    __shared__ __align__(8) uint64_t staged[2];
    __shared__ Meta4 meta[2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (m <= 0) {
        pdl_trigger();
        return;
    }
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&staged[b], M4_WARPS);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == M4_WARPS) {
        // ---------------------------------------------------- producer (one lane)
        if (lane != 0) return;
        const uint64_t policy = policy_evict_first();
        auto issue = [&](int i) {
            const int st = i & 1;
            const long long j = c0 + i;
            const long long q = j / g.cpg;
            const long long jj = j - q * g.cpg;
            const int4 a = g.vec[j];
            int4 b;
            const long long gq = q * 4 * g.L;
            const bool grp_end = (jj + 1 == g.cpg) || (j + 1 == g.nchunks);
            if (grp_end)
                b = make_int4((int)run_len4(g, q, 0), (int)run_len4(g, q, 1), (int)run_len4(g, q, 2),
                              (int)run_len4(g, q, 3));
            else
                b = g.vec[j + 1];
            const int av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
            Meta4 mt;
            uint32_t total = 0;
            int o = 0;
            long long lo_[4];
            int nn[4];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const long long gs = gq + s * g.L + av[s];
                const int ln = bv[s] - av[s];
                GNS_DASSERT(ln >= 0);
                o = ((o + 1) & ~1) + (int)(gs & 1);
                mt.o[s] = o;
                mt.len[s] = ln;
                lo_[s] = gs;
                nn[s] = ln;
                o += ln + 1;            // (+1: a guard slot between slices)
            }
            GNS_DASSERT(o + 2 <= STG4_SLOTS);
            // bytes: [align_down(gs, 2), align_up(gs + ln, 2)) clipped at n (an odd last key: plain load)
            long long bs[4], be[4];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                bs[s] = lo_[s] & ~1LL;
                be[s] = (lo_[s] + nn[s] + 1) & ~1LL;
                if (be[s] > g.n) be[s] -= 2;
                if (nn[s] > 0 && be[s] > bs[s]) total += (uint32_t)(be[s] - bs[s]) * 8u;
            }
            mbar_expect_tx(&full[st], total);
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                if (nn[s] > 0 && be[s] > bs[s])
                    tma_load_1d(stage(st) + mt.o[s] - (lo_[s] & 1), g.src + bs[s], (uint32_t)(be[s] - bs[s]) * 8u,
                                &full[st], policy);
                if (nn[s] > 0 && lo_[s] + nn[s] > be[s]) {      // the array's odd last key
                    const long long e = be[s] > lo_[s] ? be[s] : lo_[s];
                    for (long long x = e; x < lo_[s] + nn[s]; ++x) stage(st)[mt.o[s] + (x - lo_[s])] = g.src[x];
                }
            }
            mt.gout = gq + a.x + a.y + a.z + a.w;
            mt.cnt = nn[0] + nn[1] + nn[2] + nn[3];
            mt.last = 0;
            meta[st] = mt;
            mbar_arrive(&full[st]);
        };
        issue(0);
        if (m > 1) issue(1);
        for (int i = 0; i < m; ++i) {
            const int st = i & 1;
            mbar_wait(&staged[st], (uint32_t)((i >> 1) & 1));
            const Meta4 &mt = meta[st];
            const long long G0 = mt.gout;
            const long long ga = (G0 + 1) & ~1LL, ge = (G0 + mt.cnt) & ~1LL;
            if (ge > ga) {
                bulk_store_1d(g.dst + ga, stage(st) + (G0 & 1) + (ga - G0), (uint32_t)(ge - ga) * 8u);
                bulk_commit();
            }
            if (i + 2 < m) {
                bulk_wait_read0();
                issue(i + 2);
            }
        }
        bulk_wait0();
        pdl_trigger();
        return;
    }

    // -------------------------------------------------------- merge warps
    const uint32_t mbase = smem_u32(mid);
    for (int i = 0; i < m; ++i) {
        const int st = i & 1;
        mbar_wait(&full[st], (uint32_t)((i >> 1) & 1));
        const Meta4 mt = meta[st];
        const uint32_t sbase = smem_u32(stage(st));
        const int nx = mt.len[0] + mt.len[1], ny = mt.len[2] + mt.len[3];
        const int ybase = (nx + VT4 - 1) / VT4 * VT4;
        // ---- level 1: S0 ⊕ S1 -> mid[0, nx), S2 ⊕ S3 -> mid[ybase, ybase + ny)
        bar_merge_warps();                  // the previous chunk's level-2 reads of mid are done
        double k[VT4];
        const int d = tid * VT4;
        if (d < nx) {
            const uint32_t A = sbase + 8u * mt.o[0], B = sbase + 8u * mt.o[1];
            const int ii = mpath4<ORD>(A, mt.len[0], B, mt.len[1], d);
            serial4<ORD>(A, ii, mt.len[0], B, d - ii, mt.len[1], k);
            const int mo = min(VT4, nx - d);
#pragma unroll
            for (int x = 0; x < VT4; ++x)
                if (x < mo) sts4(mbase + 8u * (uint32_t)(d + x), k[x]);
        } else if (d >= ybase && d - ybase < ny) {
            const int dy = d - ybase;
            const uint32_t A = sbase + 8u * mt.o[2], B = sbase + 8u * mt.o[3];
            const int ii = mpath4<ORD>(A, mt.len[2], B, mt.len[3], dy);
            serial4<ORD>(A, ii, mt.len[2], B, dy - ii, mt.len[3], k);
            const int mo = min(VT4, ny - dy);
#pragma unroll
            for (int x = 0; x < VT4; ++x)
                if (x < mo) sts4(mbase + 8u * (uint32_t)(d + x), k[x]);
        }
        bar_merge_warps();                  // mid complete; the stage's inputs are dead
        // ---- level 2: X' ⊕ Y' -> staging (stage st, slot (gout & 1) + output)
        const int cnt = mt.cnt;
        const int par = (int)(mt.gout & 1);
        if (d < cnt) {
            const uint32_t A = mbase, B = mbase + 8u * (uint32_t)ybase;
            const int ii = mpath4<ORD>(A, nx, B, ny, d);
            serial4<ORD>(A, ii, nx, B, d - ii, ny, k);
            const int mv = min(VT4, cnt - d);
#pragma unroll
            for (int x = 0; x < VT4; ++x)
                if (x < mv) sts4(sbase + 8u * (uint32_t)(par + d + x), k[x]);
            // the chunk's unaligned first / last output: plain global stores
            if (par && d == 0) g.dst[mt.gout] = k[0];
            const long long gend = mt.gout + cnt;
            // (values at a run-time index are read back from this thread's own staging slots)
            if ((gend & 1) && d + mv == cnt && !(par && cnt == 1))
                g.dst[gend - 1] = lds4(sbase + 8u * (uint32_t)(par + cnt - 1));
            // samples of the output (every SMP_G-th dst index)
            if (g.smp_out != nullptr) {
                const long long g0 = mt.gout + d;
                const long long sm_ = (1LL << g.so_log2) - 1;
                const long long sg = (g0 + sm_) & ~sm_;
                if (sg < g0 + mv) g.smp_out[sg >> g.so_log2] = lds4(sbase + 8u * (uint32_t)(par + (int)(sg - mt.gout)));
            }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&staged[st]);
    }
    pdl_trigger();
}

}  // namespace gns
