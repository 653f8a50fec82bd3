// gns_multipass.cuh — every merge pass of a full-buffer sort in ONE persistent
// launch (SURVEY.md §8 rows a3 + a4, the "Nocopy" ping-pong of PAPER.md:219),
// pipelined across levels.
//
// Why: with one launch per level each pass paid a start-up (launch gap, PDL
// wait, the first co-rank searches, the first TMA load: ~8 us) and a drain
// (CTAs finishing unevenly) around ~41 us of HBM streaming -- the merge pass
// ran at 0.75 of the copy peak at 2^24 keys.  Here:
//   * work items are merge tiles (4096 outputs) of all passes, claimed in one
//     global ticket order (pass-major, tile-minor) by persistent CTAs;
//   * a tile of pass p may start as soon as the pass-(p-1) tiles of its pair's
//     input region [q 2L, (q+1) 2L) have been stored -- per-region completion
//     counters (red.release / ld.acquire at gpu scope), so pass p+1 streams
//     while pass p drains its later regions; the region also covers the
//     write-after-read hazard (pass p overwrites what pass p-1 read there);
//   * deadlock-free: a CTA claims tickets in order and only waits on smaller
//     tickets, held by running CTAs that wait on still smaller ones;
//   * per tile the search warps compute both co-ranks (start and end, two
//     concurrent 8-lane sample-guided searches) ahead into a shared ring; the
//     producer lane issues the TMA loads / tensor stores, the 8 merge warps
//     merge (merge path + serial merge, left run wins ties).
// NEXT f2 (presorted input, decided from the tile sort's flag word): the
// whole input in order or strictly reversed -- the kernel moves the tile-sorted
// data to where the sort ends instead (copy, or tile-order reversal), as one
// or two phases of ticketed 4096-element moves.
#pragma once

namespace gns {

#ifndef GNS_MP_SIGFENCE
#define GNS_MP_SIGFENCE 0
#endif
#ifndef GNS_MP_CHUNK
#define GNS_MP_CHUNK 4
#endif
constexpr int MP_CHUNK = GNS_MP_CHUNK;        // merge tiles per work item
constexpr int MP_RING = 16;                   // chunk entries in the split ring
#ifndef GNS_MP_AHEAD
#define GNS_MP_AHEAD 2
#endif
// chunks a CTA may claim beyond the one its producer is issuing: enough to
// hide the co-rank searches, few enough that claim order stays processing
// order (a deep claim-ahead queues dependencies behind other CTAs' backlogs)
constexpr int MP_AHEAD = GNS_MP_AHEAD;
#ifndef GNS_MP_SWARPS
#define GNS_MP_SWARPS 4
#endif
constexpr int MP_SWARPS = GNS_MP_SWARPS;      // search warps (one chunk each at a time)
constexpr int MP_THREADS = NT + 32 + 32 * MP_SWARPS + 32;   // 448 (+ the signal warp)
constexpr int MP_SIGNAL_WARP = MERGE_WARPS + 1 + MP_SWARPS;   // 13
constexpr int MP_DQ = 16;                     // completed-tile queue (producer -> signal warp)
static_assert(MP_CHUNK * MTILE <= 4 * TILE, "a chunk must lie inside one pair region of pass 1");

struct MultiGeo {
    double *xk;            // array X: the tile sort's output = source of pass 0
    uint32_t *xv;
    double *yk;            // array Y: the other one
    uint32_t *yv;
    double *xs;            // split-search samples of X's / Y's regions (every SMP_G-th key)
    double *ys;
    long long n;
    int passes;            // merge passes M (>= 1)
    int ntiles;            // merge tiles per pass
    int blk;               // the first `blk` passes run block-major (blocks of TILE << blk keys: L2-resident), 0: pass-major
    unsigned *ticket;      // [0] work ticket (zeroed by the host)
    unsigned *done;        // completion counters (zeroed by the host)
    long long x_idx0, y_idx0;   // element index of xk[0] / yk[0] in its load map (0 or 1)
    long long x_rows, y_rows;   // full 16-key rows of the X / Y load maps
    // NEXT f2: flag word of the tile sort (bit 0 some descent, bit 1 some
    // pair not strictly reversed) and the moves an ordered / strictly
    // reversed input needs instead of the merges (phase 2 reads phase 1's
    // output range after it is stored)
    const unsigned *flag;
    const double *ord_src;  // ordered: copy ord_src -> ord_dst (or nullptr: nothing moves)
    const uint32_t *ord_srcv;
    double *ord_dst;
    uint32_t *ord_dstv;
    const double *rev_src;  // reversed: tile-order reversal rev_src -> rev_dst
    const uint32_t *rev_srcv;
    double *rev_dst;
    uint32_t *rev_dstv;
    const double *rev2_src; // reversed, second phase: copy rev2_src -> rev2_dst (or nullptr)
    const uint32_t *rev2_srcv;
    double *rev2_dst;
    uint32_t *rev2_dstv;
};

// pass p's merge geometry (source = X for even p)
__device__ __forceinline__ MergeGeo mp_geo(const MultiGeo &G, int p)
{
    const bool ev = (p & 1) == 0;
    MergeGeo g;
    const long long L = (long long)TILE << p;
    g.ak = ev ? G.xk : G.yk;
    g.av = ev ? G.xv : G.yv;
    g.bk = g.ak + L;
    g.bv = g.av ? g.av + L : nullptr;
    g.ok = ev ? G.yk : G.xk;
    g.ov = ev ? G.yv : G.xv;
    g.n = G.n;
    g.L = L;
    g.single = 0;
    g.tpp = (int)(2 * L / MTILE);
    g.tpp_log2 = p + TILE_LOG2 + 1 - MTILE_LOG2;
    g.sa = ev ? G.xs : G.ys;
    g.so = (p + 1 < G.passes) ? (ev ? G.ys : G.xs) : nullptr;
    g.sb = nullptr;
    return g;
}

__device__ __forceinline__ PipeGeo mp_pipe(const MultiGeo &G, int p)
{
    PipeGeo pg;
    pg.g = mp_geo(G, p);
    const bool ev = (p & 1) == 0;
    pg.a_lim = (ev ? G.xk : G.yk) + G.n;     // end of the source array
    pg.b_lim = pg.a_lim;
    pg.a_idx0 = ev ? G.x_idx0 : G.y_idx0;
    pg.b_idx0 = pg.a_idx0 + pg.g.L;          // B = the same array, L keys on
    pg.a_rows = ev ? G.x_rows : G.y_rows;
    pg.b_rows = pg.a_rows;
    return pg;
}

// completion counter of pass p for the pass-(p+1) pair region q, and the
// number of pass-p tiles in that region
__device__ __forceinline__ unsigned *mp_counter(const MultiGeo &G, int p, long long q)
{
    long long off = 0;
    for (int i = 0; i < p; ++i) off += (G.n + ((long long)TILE << (i + 2)) - 1) / ((long long)TILE << (i + 2));
    return G.done + off + q;
}
__device__ __forceinline__ unsigned mp_target(const MultiGeo &G, int p, long long q)
{
    const long long span = (long long)TILE << (p + 2);
    const long long lo = q * span, hi = min(G.n, lo + span);
    return (unsigned)((hi - lo + MTILE - 1) / MTILE);
}
// stored tiles whose completion is signalled once their bulk group is done:
// at most MP_PEND groups stay in flight, so the producer never waits for a
// store's global write except when it has nothing else to do
constexpr int MP_PEND = 2;
__device__ __forceinline__ void bulk_wait_pend() { asm volatile("cp.async.bulk.wait_group %0;" :: "n"(MP_PEND - 1) : "memory"); }
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}

// Ticket order.  Pass-major: ticket tk = p * cpp + chunk.  With G.blk > 0 the
// first blk passes are claimed block by block (all blk passes of block b, a
// block = TILE << blk keys, before block b+1), so a block's intermediate runs
// stay in L2 between its passes; the remaining passes follow pass-major.
// Every chunk still depends only on smaller tickets (its pair region of the
// previous pass): deadlock-free.
__device__ __forceinline__ void mp_item(const MultiGeo &G, int cpp, int tk, int &p, int &c)
{
    const int blk = min(G.blk, G.passes);
    if (blk > 0) {
        const int cpb = (int)(((long long)TILE << blk) / (MP_CHUNK * MTILE));   // chunks per block and pass
        const int nb = (cpp + cpb - 1) / cpb;
        const int tb = blk * cpp;
        if (tk < tb) {
            const int b = tk / (blk * cpb);
            if (b < nb - 1) {
                const int r = tk - b * blk * cpb;
                p = r / cpb;
                c = b * cpb + r % cpb;
            } else {
                const int lc = cpp - (nb - 1) * cpb;                    // chunks of the last (partial) block
                const int r = tk - (nb - 1) * blk * cpb;
                p = r / lc;
                c = (nb - 1) * cpb + r % lc;
            }
            return;
        }
        tk -= tb;
        p = blk + tk / cpp;
        c = tk % cpp;
        return;
    }
    p = tk / cpp;
    c = tk % cpp;
}

struct MpEntry {
    int p, t0, nt;                 // pass, first tile, tiles (p < 0: end)
    int spl[MP_CHUNK + 1];         // co-ranks of the tiles' first outputs and of the output after the last
};
struct MpMeta {
    PipeMeta pm;
    int p;
};

// NEXT f2 moves of an ordered / strictly reversed input (see MultiGeo), one
// ticketed 4096-element chunk at a time; the second phase's chunk c waits on
// the first phase's chunk c.
template <bool HV>
__device__ void mp_adapt(const MultiGeo &G, bool ordered)
{
    __shared__ int s_item;
    const long long n = G.n;
    const int nt = G.ntiles;
    const int phases = ordered ? (G.ord_src ? 1 : 0) : (G.rev2_src ? 2 : 1);
    for (;;) {
        if (threadIdx.x == 0) s_item = (int)atomicAdd(G.ticket, 1u);
        __syncthreads();
        const int item = s_item;
        __syncthreads();
        if (item >= phases * nt) break;
        const int ph = item / nt, c = item % nt;
        const long long lo = (long long)c * MTILE, hi = min(n, lo + MTILE);
        if (ph == 1) {
            if (threadIdx.x == 0)
                while (ld_acquire(G.done + c) == 0u) __nanosleep(64);
            __syncthreads();
        }
        const double *sk = ordered ? G.ord_src : (ph == 0 ? G.rev_src : G.rev2_src);
        const uint32_t *sv = ordered ? G.ord_srcv : (ph == 0 ? G.rev_srcv : G.rev2_srcv);
        double *dk = ordered ? G.ord_dst : (ph == 0 ? G.rev_dst : G.rev2_dst);
        uint32_t *dv = ordered ? G.ord_dstv : (ph == 0 ? G.rev_dstv : G.rev2_dstv);
        const bool gather = !ordered && ph == 0;
        for (long long j = lo + threadIdx.x; j < hi; j += blockDim.x) {
            long long s = j;
            if (gather) {
                // the stable sort of a strictly reversed input is its reversal;
                // tile t of src holds input tile t sorted (= reversed)
                const long long t = (n - 1 - j) >> TILE_LOG2;
                const long long ct = min((long long)TILE, n - (t << TILE_LOG2));
                s = 2 * (t << TILE_LOG2) + ct - n + j;
            }
            dk[j] = sk[s];
            if (HV) dv[j] = sv[s];
        }
        if (phases == 2 && ph == 0) {
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                red_release_add(G.done + c, 1u);
            }
        }
    }
}

template <bool HV, int ORD>
__global__ void __launch_bounds__(MP_THREADS, 2)
merge_multi_kernel(MultiGeo G, const __grid_constant__ CUtensorMap xload, const __grid_constant__ CUtensorMap yload,
                   const __grid_constant__ CUtensorMap xstore, const __grid_constant__ CUtensorMap ystore)
{
    constexpr int NS = 2;
    pdl_wait();
    const unsigned f = G.flag ? *(volatile const unsigned *)G.flag : 3u;
    if ((f & 1u) == 0u || (f & 2u) == 0u) {
        // NEXT f2: in order (every merge an omission) or
        // strictly reversed (the stable sort is the reversal)
        mp_adapt<HV>(G, (f & 1u) == 0u);
        pdl_trigger();
        return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw0[];
    unsigned char *smem_raw = smem_raw0 + ((1024u - (smem_u32(smem_raw0) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t full[NS];
    __shared__ __align__(8) uint64_t staged[NS];
    __shared__ MpMeta meta[NS];
    __shared__ MpEntry ring[MP_RING];
    __shared__ volatile int ring_tag[MP_RING];
    __shared__ volatile int ring_used;      // the producer has consumed chunks < ring_used
    __shared__ volatile int next_claim;     // CTA-local chunk index to claim next
    __shared__ volatile int end_h;          // CTA-local index of the first claim past the last ticket
    __shared__ int dq_p[MP_DQ], dq_t[MP_DQ];
    __shared__ volatile int dq_head;        // completed tiles posted by the producer (-1 - count: no more)
    __shared__ volatile int dq_tail;
    auto skb = [&](int st) { return reinterpret_cast<double *>(smem_raw + st * ts_stage_bytes(HV)); };
    auto svb = [&](int st) {
        return reinterpret_cast<uint32_t *>(smem_raw + st * ts_stage_bytes(HV) + ts_key_bytes(HV));
    };
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int cpp = (G.ntiles + MP_CHUNK - 1) / MP_CHUNK;      // chunks per pass
    const int total = G.passes * cpp;
    for (int j = tid; j < MP_RING; j += MP_THREADS) ring_tag[j] = -1;
    if (tid == 0) {
#pragma unroll
        for (int b = 0; b < NS; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&staged[b], MERGE_WARPS);
        }
        fence_mbar_init();
        ring_used = 0;
        next_claim = 0;
        end_h = 0x7FFFFFFF;
        dq_head = 0;
        dq_tail = 0;
    }
    __syncthreads();

    if (warp == MP_SIGNAL_WARP) {
        // ------------------------------------------------ signal warp (one lane)
        // Publishes the completion of stored tiles (counter of the pass-(p+1)
        // pair region) with a gpu-scope release.  Kept off the producer: its
        // fences would wait for the producer's in-flight TMA loads (~2.4 us).
        if (lane != 0) return;
        int tail = 0;
        for (;;) {
            const int hd = dq_head;
            const int cnt = hd < 0 ? -1 - hd : hd;
            if (tail == cnt) {
                if (hd < 0) break;
                __nanosleep(64);
                continue;
            }
            __threadfence_block();
            const int p = dq_p[tail % MP_DQ], t = dq_t[tail % MP_DQ];
            ++tail;
            dq_tail = tail;
#ifdef GNS_PROF
            atomicMax(&g_tl[1 + p][1], gtimer());
#endif
#ifdef GNS_MP_NOSIG
            if (false) {
#else
            if (p + 1 < G.passes) {            // the last pass has no dependents
#endif
                const long long q = ((long long)t * MTILE) / ((long long)TILE << (p + 2));
                // (the producer's bulk groups are complete and released to this
                // lane through the queue; the gpu-scope release is cumulative)
#if GNS_MP_SIGFENCE == 2
                fence_proxy_async_global();
                __threadfence();
#elif GNS_MP_SIGFENCE == 1
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
                red_release_add(mp_counter(G, p, q), 1u);
            }
        }
        return;
    }

    if (warp > PRODUCER_WARP) {
        // ------------------------------------------------ search warps
        // warp sw handles CTA-local chunks h = sw, sw + MP_SWARPS, ...: claims
        // the chunk's ticket (in h order), waits for its input region, then
        // computes the co-ranks of its tiles' first outputs (four 8-lane
        // sample-guided searches at once) and of the output after its last
        const int sw = warp - PRODUCER_WARP - 1;
        const int gj = lane >> 3, gl = lane & 7;
        const unsigned gmask = 0xFFu << (8 * gj);
        for (int h = sw;; h += MP_SWARPS) {
            int tk = 0;
            if (lane == 0) {
                // (past the first end marker the producer stops consuming: leave)
                while (h - ring_used > MP_AHEAD && h <= end_h) __nanosleep(64);
                while (next_claim != h && h <= end_h) __nanosleep(32);
                if (h > end_h) tk = -1;
                else {
                    tk = (int)atomicAdd(G.ticket, 1u);
                    if (tk >= total) end_h = h;
                    next_claim = h + 1;
                }
            }
            tk = __shfl_sync(0xFFFFFFFFu, tk, 0);
            if (tk < 0) break;
            if (tk >= total) {
                if (lane == 0) {
                    ring[h % MP_RING].p = -1;
                    __threadfence_block();
                    ring_tag[h % MP_RING] = h;
                }
                break;
            }
            int p, cidx;
            mp_item(G, cpp, tk, p, cidx);
            const int t0 = cidx * MP_CHUNK;
            const int nt = min(MP_CHUNK, G.ntiles - t0);
            const MergeGeo g = mp_geo(G, p);
#ifdef GNS_PROF
            const long long pc0 = clock64();
            if (lane == 0) atomicMin(&g_tl[1 + p][0], gtimer());
#endif
            if (p > 0 && lane == 0) {
                // the pass-(p-1) tiles of this pair's region must be stored
                const long long q = ((long long)t0 * MTILE) / (2 * g.L);
                const unsigned *c = mp_counter(G, p - 1, q);
                const unsigned want = mp_target(G, p - 1, q);
#ifndef GNS_MP_NODEP
                while (ld_acquire(c) < want) __nanosleep(100);
#endif
            }
            __syncwarp();
#ifdef GNS_PROF
            const long long pc1 = clock64();
#endif
            int c = 0, c2 = 0;
            if (gj < nt) c = tile_corank<8, ORD>(g, t0 + gj, gl, gmask, 8 * gj);
            if (MP_CHUNK > 4 && gj + 4 < nt) c2 = tile_corank<8, ORD>(g, t0 + gj + 4, gl, gmask, 8 * gj);
            const TileSpan sl = tile_span(g, t0 + nt - 1);
            int ce = 0;
            if (sl.k1 < sl.na + sl.nb) ce = tile_corank<32, ORD>(g, t0 + nt, lane, 0xFFFFFFFFu, 0);
#ifdef GNS_PROF
            if (lane == 0) {
                atomicAdd(&g_prof[0], (unsigned long long)(pc1 - pc0));    // dependency wait
                atomicAdd(&g_prof[1], (unsigned long long)(clock64() - pc1)); // the searches
                atomicAdd(&g_prof[2], 1ull);
            }
#endif
            if (gl == 0) ring[h % MP_RING].spl[gj] = c;
            if (MP_CHUNK > 4 && gl == 0 && gj + 4 < MP_CHUNK) ring[h % MP_RING].spl[gj + 4] = c2;
            if (lane == 0) {
                ring[h % MP_RING].p = p;
                ring[h % MP_RING].t0 = t0;
                ring[h % MP_RING].nt = nt;
                ring[h % MP_RING].spl[nt] = ce;
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                ring_tag[h % MP_RING] = h;
            }
        }
        return;
    }

    if (warp == PRODUCER_WARP) {
        // ------------------------------------------------ producer (one lane)
        if (lane != 0) return;
        const uint64_t policy = policy_evict_first();
        int pq_p[MP_PEND], pq_t[MP_PEND];    // stored tiles whose completion is not yet signalled (FIFO)
        int pq_n = 0, pq_h = 0;
        // post a stored tile (its bulk group complete) to the signal warp
        auto signal = [&](int p, int t) {
            while (dq_head - dq_tail >= MP_DQ) { }
            const int hd = dq_head;
            dq_p[hd % MP_DQ] = p;
            dq_t[hd % MP_DQ] = t;
            __threadfence_block();
            dq_head = hd + 1;
        };
        // Event loop: issue tile `issued` when its ring entry is ready and a
        // stage is free; store tile `stored` once the merge warps staged it;
        // never block on a ring entry while a tile of ours is unstored or its
        // completion unsignalled (the entry's search may wait on that tile).
        int issued = 0, stored = 0;
        int ch = 0, cj = 0;                  // current chunk (CTA-local) and its next tile
        bool more = true;
        for (;;) {
            bool progress = false;
            if (more && issued - stored < NS && ring_tag[ch % MP_RING] == ch) {
                const int st = issued % NS;
                const MpEntry &e = ring[ch % MP_RING];
                if (e.p < 0) {
                    meta[st].p = -1;                                   // end marker for the merge warps
                    mbar_arrive(&full[st]);
                    more = false;
                } else {
                    if (cj == 0) fence_proxy_async_global();   // the region's stores (acquired by a search lane) before our loads
                    const PipeGeo pg = mp_pipe(G, e.p);
                    const bool ev = (e.p & 1) == 0;
                    meta[st].p = e.p;
#ifdef GNS_PROF
                    const long long z1 = clock64();
#endif
                    pipe_issue<HV>(pg, ev ? xload : yload, ev ? xload : yload, e.t0 + cj, e.spl[cj], e.spl[cj + 1],
                                   skb(st), svb(st), &full[st], &meta[st].pm, policy);
#ifdef GNS_PROF
                    atomicAdd(&g_prof[5], (unsigned long long)(clock64() - z1));
#endif
                    if (++cj == e.nt) {
                        cj = 0;
                        ++ch;
                        ring_used = ch;                                // chunk entry consumed
                    }
                }
                ++issued;
                progress = true;
            }
            if (stored < issued && mbar_test(&staged[stored % NS], (uint32_t)((stored / NS) & 1))) {
                const int st = stored % NS;
                const int p = meta[st].p;
                if (p < 0) break;                                      // every tile before the end marker is stored
                const int t = meta[st].pm.t;
                if (G.n >= 16) {
                    tma_store_2d((p & 1) == 0 ? &ystore : &xstore, skb(st), 0, t * (MTILE / 16));
                    bulk_commit();
                }
                // queue tile t; once MP_PEND stores are in flight, the oldest
                // is complete (bulk groups complete in order): signal it
                pq_p[(pq_h + pq_n) % MP_PEND] = p;
                pq_t[(pq_h + pq_n) % MP_PEND] = t;
                if (++pq_n == MP_PEND) {
#ifdef GNS_PROF
                    const long long z2 = clock64();
                    bulk_wait_pend();
                    atomicAdd(&g_prof[6], (unsigned long long)(clock64() - z2));
#else
                    bulk_wait_pend();
#endif
                    signal(pq_p[pq_h], pq_t[pq_h]);
                    pq_h = (pq_h + 1) % MP_PEND;
                    --pq_n;
                }
#ifdef GNS_PROF
                const long long z3 = clock64();
                bulk_wait_read0();                                     // stage st read out -> reusable
                atomicAdd(&g_prof[7], (unsigned long long)(clock64() - z3));
#else
                bulk_wait_read0();                                     // stage st read out -> reusable
#endif
                ++stored;
                progress = true;
            }
            if (!progress) {
                if (pq_n > 0) {
                    bulk_wait0();
                    for (; pq_n > 0; --pq_n, pq_h = (pq_h + 1) % MP_PEND) signal(pq_p[pq_h], pq_t[pq_h]);
                } else {
#ifdef GNS_PROF
                    const long long z0 = clock64();
                    __nanosleep(32);
                    atomicAdd(&g_prof[3], (unsigned long long)(clock64() - z0));
#else
                    __nanosleep(32);
#endif
                }
            }
        }
        bulk_wait0();
        for (; pq_n > 0; --pq_n, pq_h = (pq_h + 1) % MP_PEND) signal(pq_p[pq_h], pq_t[pq_h]);
        __threadfence_block();
        dq_head = -1 - dq_head;                                        // no more tiles
        pdl_trigger();
        return;
    }

    // ---------------------------------------------------- merge warps 0-7
    const long long n = G.n;
    const long long full_rows = n >> 4;
    for (int i = 0;; ++i) {
        const int st = i % NS;
        mbar_wait(&full[st], (uint32_t)((i / NS) & 1));
        const int p = meta[st].p;
        if (p < 0) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&staged[st]);
            break;
        }
        const PipeMeta mt = meta[st].pm;
        const MergeGeo G_ = mp_geo(G, p);
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
        const long long row = (long long)mt.t * (MTILE / 16) + tid;
        if (G_.so != nullptr && (tid & (SMP_G / VT - 1)) == 0 && d < cnt)
            G_.so[(row * 16) >> SMP_LOG2] = k[0];
        bar_merge_warps();                                         // stage st fully read
        unsigned char *rowp = reinterpret_cast<unsigned char *>(sk) + tid * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) sts128(rowp + ((c ^ (tid & 7)) << 4), k[2 * c], k[2 * c + 1]);
        fence_proxy_async();
        if (HV) {
            const int mv = cnt - d;
            if (mv >= VT) {
#pragma unroll
                for (int x = 0; x < VT; x += 8) st_v8(G_.ov + row * 16 + x, &v[x]);
            } else {
#pragma unroll
                for (int x = 0; x < VT; ++x)
                    if (x < mv) G_.ov[row * 16 + x] = v[x];
            }
        }
        if (row == full_rows && d < cnt) {
#pragma unroll
            for (int x = 0; x < VT; ++x)
                if (x < cnt - d) G_.ok[row * 16 + x] = k[x];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&staged[st]);
    }
    pdl_trigger();
}

}  // namespace gns
