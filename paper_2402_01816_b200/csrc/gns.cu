// gns.cu — host planner, launcher and C-ABI (include/gns.h) of the B200-native
// stable f64 mergesort hot path (greeNsort, arXiv 2402.01816).
//
// Row a1 (validate & plan), a5 (0.5-mode orchestration), a7 (buffer
// allocation and %RAM accounting) of SURVEY.md §8 live here; the kernels are in
// gns_kernels.cuh.  Everything is enqueued on the caller's stream; nothing here
// calls into the oracle or any CPU sort.
#include "../../include/gns.h"
#include "gns_kernels.cuh"
#include "gns_f32.cuh"
#include "gns_tile64.cuh"
#include "gns_multipass.cuh"
#include "gns_merge4.cuh"
#include "gns_peel.cuh"
#include "gns_small.cuh"

#include <cuda_runtime.h>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

using namespace gns;

namespace {

thread_local std::string g_last_error;

gns_status fail(gns_status s, const char *msg)
{
    g_last_error = msg;
    return s;
}

gns_status check(cudaError_t e, const char *where)
{
    if (e == cudaSuccess) return GNS_OK;
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return GNS_ERR_CUDA;
}

#define GNS_TRY(expr)                        \
    do {                                     \
        gns_status _s = (expr);              \
        if (_s != GNS_OK) return _s;         \
    } while (0)

inline size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t a, size_t b) { return ceil_div(a, b) * b; }

int merge_passes_for(size_t n, size_t run = TILE)
{
    if (n <= run) return 0;
    size_t runs = ceil_div(n, run);
    int p = 0;
    while (((size_t)1 << p) < runs) ++p;
    return p;
}

bool k1_v3();
bool multi_on();
bool chain_on();
// K1 cluster size C (key-only, 8-byte keys): the tile sort merges the C tiles
// of a thread-block cluster on chip (cluster_levels, gns_tile64.cuh), so the
// merge passes start at runs of C x TILE keys.  GNS_K1_CL = 1, 2, 4, 8, 16;
// default 1: measured slower at every C (2^24 keys 0.80 / 0.83 / 0.87 / 0.96
// / 1.09 ms for C = 1 / 2 / 4 / 8 / 16, DESIGN.md 8b -- a distributed
// shared memory merge level costs more than the HBM pass it saves).  1 for
// pairs, the A/B kernels and arrays of at most one tile.
int k1_cluster(size_t len, bool hv)
{
    static const int cl = [] {
        const char *e = std::getenv("GNS_K1_CL");
        const int v = e ? std::atoi(e) : 1;
        return (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) ? v : 1;
    }();
    if (hv || !k1_v3() || multi_on() || chain_on() || len <= (size_t)TILE) return 1;
    int c = 1;
    while (c < cl && (size_t)c * TILE < len) c <<= 1;
    return c;
}
size_t k1_run(size_t len, bool hv) { return (size_t)TILE * k1_cluster(len, hv); }

// 0.5 mode split: the left (larger) half goes to the buffer.  Rounded up to 32
// elements so that data + nl stays 256-byte (keys) / 128-byte (vals) aligned.
size_t left_len(size_t n)
{
    size_t nl = align_up(ceil_div(n, 2), 32);
    return nl < n ? nl : n;
}

bool is_aligned(const void *p, size_t a) { return ((uintptr_t)p % a) == 0; }

// Workspace layout (one allocation = the whole bufferRAM of a call).
struct Layout {
    size_t buf_elems = 0;   // buffer key(+val) slots
    size_t off_k = 0, off_v = 0, off_corank = 0, off_deps = 0, off_flags = 0, off_adapt = 0, off_smp = 0, total = 0;
    size_t nsmp = 0;        // keys per sample array (two arrays: data-side and buffer-side regions)
    size_t off_piv = 0;     // 4-way passes: approximate pivot positions + chunk split vectors, or none
    int ntiles = 0;         // merge tiles over the whole array
    // NEXT f2 Omitsort (full buffer only): run state of two levels (location,
    // first and last key), per level and pair the copy flag, per level the
    // merge tile list and its length (+ the sorted run's region)
    size_t off_loc = 0, off_fl = 0, off_fix = 0, off_pre = 0, off_list = 0, off_cnt = 0, off_tdesc = 0;
    size_t nruns = 0, npairs = 0;
};

// Buffer mode (row a5 and NEXT f1): FULL = 100 % buffer (ping-pong with the
// data), LIMITED = a buffer of `buf` elements (multiple of 32); fraction 0.5
// gives buf = left_len(n) (the 0.5 mode), smaller fractions recurse.
struct Mode {
    bool limited = false;
    size_t buf = 0;
    bool omit = false;      // NEXT f2: Omitsort schedule (full buffer; gns_sort_omit)
};

// words of the multi-pass launch: [0] flag (NEXT f2), [1] ticket, then the
// per-region completion counters of all passes (<= ntiles/4 + passes) or the
// per-chunk counters of a two-phase reversal (ntiles)
size_t mp_words(int ntiles) { return 2 + (size_t)ntiles + 64; }

bool small_on();
bool four_on();

Layout layout(size_t n, const Mode &m, bool hv)
{
    Layout L;
    if (n <= (size_t)TILE) return L;   // one tile, sorted in place, no buffer
    if (n <= (size_t)SMALL_MAX_N && small_on()) return L;   // one cluster, on chip, no buffer
    L.buf_elems = m.limited ? m.buf : n;
    L.ntiles = (int)ceil_div(n, MTILE);
    size_t o = 0;
    L.off_k = o;
    o = align_up(o + L.buf_elems * sizeof(double), 256);
    L.off_v = o;
    if (hv) o = align_up(o + L.buf_elems * sizeof(uint32_t), 256);
    L.off_corank = o;
    o = align_up(o + (size_t)(L.ntiles + 1) * sizeof(int), 256);
    L.off_deps = o;
    if (m.limited) o = align_up(o + (size_t)L.ntiles * sizeof(int2), 256);
    L.off_flags = o;
    if (m.limited) o = align_up(o + (size_t)(L.ntiles + 1) * sizeof(unsigned), 256);
    L.off_adapt = o;                   // the "input not presorted" word (NEXT f2); full buffer: + the
                                       // multi-pass ticket and completion counters (mp_words)
    o = align_up(o + (m.limited ? 1 : mp_words(L.ntiles)) * sizeof(unsigned), 256);
    // split-search samples of each region: every SMP_G-th key, or every FS-th
    // (fine samples) when 4-way passes run (gns_merge4.cuh)
    const bool four = !hv && four_on();
    L.off_smp = o;
    L.nsmp = n / (four ? FS : SMP_G) + 2;
    o = align_up(o + 2 * L.nsmp * sizeof(double), 256);
    if (four) {
        L.off_piv = o;                 // 4-way passes: per fine sample its approximate position, per chunk its split vector
        o = align_up(o + (ceil_div(n, FS) + 2) * sizeof(int), 256);
        o = align_up(o + (3 * ceil_div(n, T4) + 8) * sizeof(int4), 256);
    }
    if (!m.limited) {
        L.nruns = ceil_div(n, TILE);
        L.npairs = ceil_div(n, 2 * (size_t)TILE);
        const size_t M = (size_t)merge_passes_for(n);
        L.off_tdesc = o;                                    // per tile: kept as a descending run (Octosort)
        o = align_up(o + L.nruns, 256);
        L.off_loc = o;
        o = align_up(o + 2 * L.nruns, 256);
        L.off_fl = o;
        o = align_up(o + 4 * L.nruns * sizeof(double), 256);
        L.off_fix = o;                                      // action bytes, all levels' pairs (<= nruns + M)
        o = align_up(o + L.nruns + M, 256);
        L.off_pre = o;                                      // merge-tile prefixes, all levels' pairs
        o = align_up(o + (L.nruns + M) * sizeof(int), 256);
        L.off_list = o;                                     // one level's merge-tile list
        o = align_up(o + (size_t)L.ntiles * sizeof(int), 256);
        L.off_cnt = o;
        o = align_up(o + (M + 1) * sizeof(int), 256);
    }
    L.total = o;
    return L;
}

// Size of the co-rank array only (gns_merge_pass / gns_merge_inplace_top).
size_t merge_ws(size_t n)
{
    size_t nt = ceil_div(n, MTILE);
    return align_up((nt + 1) * sizeof(int), 256) + align_up(nt * sizeof(int2), 256) +
           align_up((nt + 1) * sizeof(unsigned), 256);
}

// Kernel instances by payload (hv) and order ORD = DESC | key type << 1
// (ord_of): 3 key types x 2 directions.
constexpr int NORD = 6;
using TileK = decltype(&tile_sort2_kernel<false, 0>);
using MergeK = decltype(&merge_tstore_kernel<false, 0>);
using MergeOLK = decltype(&merge_tstore_kernel<false, 0, 2, true>);
using OmitPlanK = decltype(&omit_plan_kernel<0>);
using InplK = decltype(&merge_inplace_kernel<false, 0>);
using PartK = decltype(&partition_kernel<0>);
#define GNS_ORDS(K, HV) {&K<HV, 0>, &K<HV, 1>, &K<HV, 2>, &K<HV, 3>, &K<HV, 4>, &K<HV, 5>}
TileK tile_kern(bool hv, int o)
{
    static const TileK t[2][NORD] = {GNS_ORDS(tile_sort2_kernel, false), GNS_ORDS(tile_sort2_kernel, true)};
    return t[hv][o];
}
using Rank4K = decltype(&rank4_kernel<0>);
using Merge4K = decltype(&merge4_kernel<0>);
Rank4K rank4_kern(int o)
{
    static const Rank4K t[NORD] = {&rank4_kernel<0>, &rank4_kernel<1>, &rank4_kernel<2>,
                                   &rank4_kernel<3>, &rank4_kernel<4>, &rank4_kernel<5>};
    return t[o];
}
using Chunk4K = decltype(&chunk4_kernel<0>);
Chunk4K chunk4_kern(int o)
{
    static const Chunk4K t[NORD] = {&chunk4_kernel<0>, &chunk4_kernel<1>, &chunk4_kernel<2>,
                                    &chunk4_kernel<3>, &chunk4_kernel<4>, &chunk4_kernel<5>};
    return t[o];
}
Merge4K merge4_kern(int o)
{
    static const Merge4K t[NORD] = {&merge4_kernel<0>, &merge4_kernel<1>, &merge4_kernel<2>,
                                    &merge4_kernel<3>, &merge4_kernel<4>, &merge4_kernel<5>};
    return t[o];
}
using SmallK = decltype(&small_sort_kernel<false, 0>);
SmallK small_kern(bool hv, int o)
{
    static const SmallK t[2][NORD] = {
        {&small_sort_kernel<false, 0>, &small_sort_kernel<false, 1>, &small_sort_kernel<false, 2>,
         &small_sort_kernel<false, 3>, &small_sort_kernel<false, 4>, &small_sort_kernel<false, 5>},
        {&small_sort_kernel<true, 0>, &small_sort_kernel<true, 1>, &small_sort_kernel<true, 2>,
         &small_sort_kernel<true, 3>, &small_sort_kernel<true, 4>, &small_sort_kernel<true, 5>}};
    return t[hv][o];
}
// Small arrays (n <= SMALL_MAX_N) on one thread-block cluster (gns_small.cuh)
// unless GNS_SMALL=0 (A/B).
bool small_on()
{
    static const bool on = [] {
        const char *e = std::getenv("GNS_SMALL");
        return !(e && e[0] == '0');
    }();
    return on;
}
// 4-way merge passes (gns_merge4.cuh) for key-only sorts only with GNS_FOUR=1:
// bit-exact, but measured slower at 2^23 .. 2^27 keys (2^24: 0.92 vs 0.80 ms,
// the on-chip merge is bound by shared-memory wavefronts, so a
// 4-way pass costs about two 2-way passes, plus the pivot ranking).
bool four_on()
{
    static const bool on = [] {
        const char *e = std::getenv("GNS_FOUR");
        return e && e[0] == '1';
    }();
    return on;
}
// whether a range of len keys (runs of R after K1) merges by 4-way passes
bool use_four(bool hv, size_t len, size_t R)
{
    return !hv && four_on() && !multi_on() && !chain_on() && merge_passes_for(len, R) >= 2;
}
using MHeadK = decltype(&merge_head_kernel<false, 0>);
MHeadK mhead_kern(bool hv, int o)
{
    static const MHeadK t[2][NORD] = {
        {&merge_head_kernel<false, 0>, &merge_head_kernel<false, 1>, &merge_head_kernel<false, 2>,
         &merge_head_kernel<false, 3>, &merge_head_kernel<false, 4>, &merge_head_kernel<false, 5>},
        {&merge_head_kernel<true, 0>, &merge_head_kernel<true, 1>, &merge_head_kernel<true, 2>,
         &merge_head_kernel<true, 3>, &merge_head_kernel<true, 4>, &merge_head_kernel<true, 5>}};
    return t[hv][o];
}
using PeelK = decltype(&peel_merge_kernel<false, 0>);
PeelK peel_kern(bool hv, int o)
{
    static const PeelK t[2][NORD] = {
        {&peel_merge_kernel<false, 0>, &peel_merge_kernel<false, 1>, &peel_merge_kernel<false, 2>,
         &peel_merge_kernel<false, 3>, &peel_merge_kernel<false, 4>, &peel_merge_kernel<false, 5>},
        {&peel_merge_kernel<true, 0>, &peel_merge_kernel<true, 1>, &peel_merge_kernel<true, 2>,
         &peel_merge_kernel<true, 3>, &peel_merge_kernel<true, 4>, &peel_merge_kernel<true, 5>}};
    return t[hv][o];
}
using PeelHK = decltype(&peel_head_kernel<false, 0>);
PeelHK peel_head_kern(bool hv, int o)
{
    static const PeelHK t[2][NORD] = {
        {&peel_head_kernel<false, 0>, &peel_head_kernel<false, 1>, &peel_head_kernel<false, 2>,
         &peel_head_kernel<false, 3>, &peel_head_kernel<false, 4>, &peel_head_kernel<false, 5>},
        {&peel_head_kernel<true, 0>, &peel_head_kernel<true, 1>, &peel_head_kernel<true, 2>,
         &peel_head_kernel<true, 3>, &peel_head_kernel<true, 4>, &peel_head_kernel<true, 5>}};
    return t[hv][o];
}
using MultiK = decltype(&merge_multi_kernel<false, 0>);
MultiK multi_kern(bool hv, int o)
{
    static const MultiK t[2][NORD] = {
        {&merge_multi_kernel<false, 0>, &merge_multi_kernel<false, 1>, &merge_multi_kernel<false, 2>,
         &merge_multi_kernel<false, 3>, &merge_multi_kernel<false, 4>, &merge_multi_kernel<false, 5>},
        {&merge_multi_kernel<true, 0>, &merge_multi_kernel<true, 1>, &merge_multi_kernel<true, 2>,
         &merge_multi_kernel<true, 3>, &merge_multi_kernel<true, 4>, &merge_multi_kernel<true, 5>}};
    return t[hv][o];
}
// Full-buffer merge passes: one launch per level (merge_tstore_kernel), or,
// with GNS_MULTI=1, one pipelined launch for all levels (merge_multi_kernel;
// measured slower at 2^24 keys: dependency stalls of the
// whole-array regions of the last passes).
bool multi_on()
{
    static const bool on = [] {
        const char *e = std::getenv("GNS_MULTI");
        return e && e[0] == '1';
    }();
    return on;
}
// Chained uniform passes (no griddepcontrol.wait between merge levels, region
// counters instead) only with GNS_CHAIN=1: measured 809 vs 798 us per 2^24-key
// sort, bit-exact either way.
bool chain_on()
{
    static const bool on = [] {
        const char *e = std::getenv("GNS_CHAIN");
        return e && e[0] == '1';
    }();
    return on;
}
// The merge pass's producer warp issues a tile's TMA boxes one per lane
// (PipeGeo::coop) instead of all from one lane.  GNS_COOP=0: one lane (A/B).
bool coop_on()
{
    static const bool on = [] {
        const char *e = std::getenv("GNS_COOP");
        return !(e && e[0] == '0');
    }();
    return on;
}
using Tile3K = decltype(&tile_sort3_kernel<double, 0>);
Tile3K tile3_kern(int o)
{
    static const Tile3K t[NORD] = {&tile_sort3_kernel<double, 0>, &tile_sort3_kernel<double, 1>,
                                   &tile_sort3_kernel<double, 2>, &tile_sort3_kernel<double, 3>,
                                   &tile_sort3_kernel<double, 4>, &tile_sort3_kernel<double, 5>};
    return t[o];
}
using Tile3FK = decltype(&tile_sort3_kernel<float, 0>);
Tile3K tile3c_kern(int o)
{
    static const Tile3K t[NORD] = {
        &tile_sort3_kernel<double, 0, NT3, true>, &tile_sort3_kernel<double, 1, NT3, true>,
        &tile_sort3_kernel<double, 2, NT3, true>, &tile_sort3_kernel<double, 3, NT3, true>,
        &tile_sort3_kernel<double, 4, NT3, true>, &tile_sort3_kernel<double, 5, NT3, true>};
    return t[o];
}
Tile3FK tile3f_kern(int desc)
{
    static const Tile3FK t[2] = {&tile_sort3_kernel<float, 0>, &tile_sort3_kernel<float, 1>};
    return t[desc];
}
// Key-only K1: the 128 x 64 kernel (tile_sort3_kernel) unless GNS_K1=2
// forces the 256 x 32 one (A/B).
bool k1_v3()
{
    static const bool on = [] {
        const char *e = std::getenv("GNS_K1");
        return !(e && e[0] == '2');
    }();
    return on;
}
MergeK merge_kern(bool hv, int o)
{
    static const MergeK t[2][NORD] = {GNS_ORDS(merge_tstore_kernel, false), GNS_ORDS(merge_tstore_kernel, true)};
    return t[hv][o];
}
#define GNS_ORDS_OL(K, HV) {&K<HV, 0, 2, true>, &K<HV, 1, 2, true>, &K<HV, 2, 2, true>, \
                           &K<HV, 3, 2, true>, &K<HV, 4, 2, true>, &K<HV, 5, 2, true>}
MergeOLK merge_kern_ol(bool hv, int o)
{
    static const MergeOLK t[2][NORD] = {GNS_ORDS_OL(merge_tstore_kernel, false),
                                        GNS_ORDS_OL(merge_tstore_kernel, true)};
    return t[hv][o];
}
#undef GNS_ORDS_OL
OmitPlanK omit_plan_kern(int o)
{
    static const OmitPlanK t[NORD] = {&omit_plan_kernel<0>, &omit_plan_kernel<1>, &omit_plan_kernel<2>,
                                      &omit_plan_kernel<3>, &omit_plan_kernel<4>, &omit_plan_kernel<5>};
    return t[o];
}
using F32TileK = decltype(&f32_tile_sort_kernel<false, false>);
using F32MergeK = decltype(&f32_merge_kernel<false, false>);
F32TileK f32_tile_kern(bool hv, int desc)
{
    static const F32TileK t[2][2] = {{&f32_tile_sort_kernel<false, false>, &f32_tile_sort_kernel<false, true>},
                                     {&f32_tile_sort_kernel<true, false>, &f32_tile_sort_kernel<true, true>}};
    return t[hv][desc];
}
using F32M2K = decltype(&f32_merge2_kernel<false, false>);
F32M2K f32_merge2_kern(bool hv, int desc)
{
    static const F32M2K t[2][2] = {{&f32_merge2_kernel<false, false>, &f32_merge2_kernel<false, true>},
                                   {&f32_merge2_kernel<true, false>, &f32_merge2_kernel<true, true>}};
    return t[hv][desc];
}
using F32PartK = decltype(&f32_partition_kernel<false>);
F32PartK f32_part_kern(int desc)
{
    static const F32PartK t[2] = {&f32_partition_kernel<false>, &f32_partition_kernel<true>};
    return t[desc];
}
F32MergeK f32_merge_kern(bool hv, int desc)
{
    static const F32MergeK t[2][2] = {{&f32_merge_kernel<false, false>, &f32_merge_kernel<false, true>},
                                      {&f32_merge_kernel<true, false>, &f32_merge_kernel<true, true>}};
    return t[hv][desc];
}
InplK inplace_kern(bool hv, int o)
{
    static const InplK t[2][NORD] = {GNS_ORDS(merge_inplace_kernel, false), GNS_ORDS(merge_inplace_kernel, true)};
    return t[hv][o];
}
// Lanes per tile of the partition search: 4 (eight tiles per warp; 2^27
// pairs 10.22 -> 9.81 ms, keys 7.14 -> 6.72 ms against one warp per tile,
// 8 lanes 9.90 / 6.80: the searches are latency-bound, fewer waves of warps
// win over fewer search rounds).  GNS_PART_W = 32 / 16 / 8 / 4 (A/B).
int part_w()
{
    static const int w = [] {
        const char *e = std::getenv("GNS_PART_W");
        const int v = e ? std::atoi(e) : 4;
        return (v == 8 || v == 16 || v == 32) ? v : 4;
    }();
    return w;
}
PartK partition_kern(int o)
{
#define GNS_PW(W) {&partition_kernel<0, W>, &partition_kernel<1, W>, &partition_kernel<2, W>, \
                   &partition_kernel<3, W>, &partition_kernel<4, W>, &partition_kernel<5, W>}
    static const PartK t[4][NORD] = {GNS_PW(32), GNS_PW(16), GNS_PW(8), GNS_PW(4)};
#undef GNS_PW
    const int w = part_w();
    return t[w == 32 ? 0 : w == 16 ? 1 : w == 8 ? 2 : 3][o];
}
#undef GNS_ORDS

// Per-device one-time kernel attributes (dynamic shared memory > 48 KB).
std::mutex g_attr_mu;
unsigned long long g_attr_done = 0;   // bit per device ordinal
int g_num_sms[64];

gns_status ensure_attrs()
{
    int dev = 0;
    GNS_TRY(check(cudaGetDevice(&dev), "cudaGetDevice"));
    if (dev >= 64) return fail(GNS_ERR_CUDA, "device ordinal >= 64");
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (g_attr_done & (1ull << dev)) return GNS_OK;
#define GNS_ATTR(K, BYTES) \
    GNS_TRY(check(cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(BYTES)), "attr"))
    for (int o = 0; o < NORD; ++o) {
        for (int hv = 0; hv < 2; ++hv) {
            GNS_ATTR(merge_kern(hv, o), ts_smem(hv));
            GNS_ATTR(merge_kern_ol(hv, o), ts_smem(hv));
            if (o < 2) GNS_ATTR(f32_tile_kern(hv, o), f_tile_smem(hv));
            if (o < 2) GNS_ATTR(f32_merge_kern(hv, o), f_merge_smem(hv));
            if (o < 2) GNS_ATTR(f32_merge2_kern(hv, o), f2_smem(hv));
            if (!hv) GNS_ATTR(omit_plan_kern(o), OMIT_SMEM);
            GNS_ATTR(inplace_kern(hv, o), ts_smem(hv));
            GNS_ATTR(tile_kern(hv, o), t1_smem(hv));
            if (!hv) GNS_ATTR(tile3_kern(o), T3_SMEM);
            if (!hv) {
                GNS_ATTR(tile3c_kern(o), T3_SMEM);
                GNS_TRY(check(cudaFuncSetAttribute(tile3c_kern(o), cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                              "cudaFuncSetAttribute"));
            }
            if (!hv && o < 2) GNS_ATTR(tile3f_kern(o), (t3_smem<float, NT3>()));
            GNS_ATTR(multi_kern(hv, o), ts_smem(hv));
            if (!hv) GNS_ATTR(merge4_kern(o), M4_SMEM);
            GNS_ATTR(small_kern(hv, o), sm_smem(hv));
            GNS_TRY(check(cudaFuncSetAttribute(small_kern(hv, o), cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                          "attr"));
        }
    }
#undef GNS_ATTR
    GNS_TRY(check(cudaDeviceGetAttribute(&g_num_sms[dev], cudaDevAttrMultiProcessorCount, dev), "sm count"));
    g_attr_done |= (1ull << dev);
    return GNS_OK;
}

int num_sms()
{
    int dev = 0;
    cudaGetDevice(&dev);
    return (dev >= 0 && dev < 64 && g_num_sms[dev] > 0) ? g_num_sms[dev] : 148;
}

// ------------------------------------------------------------------ launches
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}

// 2-D tensor map for TMA: an array of n keys (f64, 16 per 128-byte row) or
// vals (u32, 32 per row) viewed as [n / per_row][per_row], box [box_rows][per_row],
// 128-byte swizzle.  A partial last row is outside the map (handled by hand).
gns_status row_map(void *base, size_t n, bool f64, int box_rows, CUtensorMap *map)
{
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(GNS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int per_row = f64 ? 16 : 32;
    // n < per_row: a 1-row map that no kernel stores through (they check n)
    cuuint64_t dims[2] = {(cuuint64_t)per_row, (cuuint64_t)std::max<size_t>(1, n / per_row)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {(cuuint32_t)per_row, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, base, dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(GNS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return GNS_OK;
}

// Key map of a merge input run for the stage loads: rows of 16 keys starting
// at ptr rounded down to 16 bytes (idx0 = 0 or 1 keys before ptr), boxes of
// krows(hv) rows, 128-byte swizzle; `rows` = full rows (the partial last row is
// patched by the merge warps).
gns_status key_map(const double *ptr, size_t count, bool hv, CUtensorMap *map, long long *idx0, long long *rows)
{
    const uintptr_t a = (uintptr_t)ptr;
    const double *base = (const double *)(a & ~(uintptr_t)15);
    *idx0 = (long long)(ptr - base);
    *rows = (long long)((count + (size_t)*idx0) / 16);
    return row_map((void *)base, (size_t)(*rows) * 16, true, krows(hv), map);
}

// Programmatic dependent launch: every kernel of a sort is launched with
// programmatic stream serialization; it may be scheduled while its predecessor
// drains and waits in griddepcontrol.wait until the predecessor's writes are
// visible.  Measured -3 % per 2^24 sort on B200.  GNS_PDL=0 disables it (A/B).
bool pdl_enabled()
{
    static const bool on = [] {
        const char *e = std::getenv("GNS_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Launch timing (gns_timing_begin/end): one CUDA event on the launching stream
// before the first launch and after every launch of the calling thread.
struct Timing {
    bool on = false;
    int cap = 0;
    std::vector<cudaEvent_t> ev;     // pool
    std::vector<int> kind;           // kind of launch i (between ev[i] and ev[i+1])
    int used = 0;                    // events recorded
};
thread_local Timing g_timing;

int launch_kind(const char *what)
{
    static const char *names[] = {"tile_sort2_kernel", "merge_tstore_kernel", "partition_kernel",
                                  "inplace_deps_kernel", "merge_inplace_kernel", "reverse_kernel",
                                  "split_cuts_kernel", "gather_samples_kernel", "omit_plan_kernel",
                                  "omit_prep_kernel", "omit_final_kernel", "iota_u32_kernel", "gather_u64_kernel",
                                  "f32_tile_sort_kernel", "f32_merge_kernel", "f32_reverse_kernel",
                                  "f32_partition_kernel", "merge_multi_kernel", "peel_head_kernel",
                                  "peel_merge_kernel", "small_sort_kernel", "rank4_kernel", "merge4_kernel", "chunk4_kernel"};
    for (int i = 0; i < 24; ++i)
        if (std::strcmp(what, names[i]) == 0) return i + 1;
    return 0;
}

// Which kernel runs a uniform merge pass: the fused one (search warps) or
// partition + ticket-scheduled merge.  GNS_MERGE_MODE=0/1 forces one (A/B).
bool ticket_pass(bool hv, int ntiles)
{
    static const int forced = [] {
        const char *e = std::getenv("GNS_MERGE_MODE");
        return e ? std::atoi(e) : -1;
    }();
    if (forced == 0 || forced == 1) return forced == 1;
    return ntiles >= (hv ? 8192 : 16384);   // >= 2^25 elements with payload, >= 2^26 key-only (measured)
}

template <typename... KArgs, typename... Args>
gns_status launch_pdl(const char *what, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t st, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    Timing &T = g_timing;
    const bool timed = T.on && T.used + 2 <= T.cap;
    if (timed && T.used == 0) cudaEventRecord(T.ev[T.used++], st);
    gns_status r = check(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), what);
    if (timed && r == GNS_OK) {
        T.kind[T.used - 1] = launch_kind(what);
        cudaEventRecord(T.ev[T.used++], st);
    }
    return r;
}

// Row a2 (K1).
gns_status launch_tile_sort(const double *sk, const uint32_t *sv, double *dk, uint32_t *dv, size_t n, int ord,
                            cudaStream_t st, unsigned *unsorted = nullptr, double *smp = nullptr,
                            unsigned char *tdesc = nullptr, double *smp_src = nullptr, int cl = 1,
                            int smp_log2 = SMP_LOG2)
{
    if (n == 0) return GNS_OK;
    const unsigned grid = (unsigned)ceil_div(n, TILE);
    const bool hv = sv != nullptr;
    if (!hv && k1_v3() && cl > 1) {
        // thread-block clusters of cl CTAs (the grid padded to whole clusters;
        // CTAs past the array hold pads only)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)align_up(grid, (size_t)cl));
        cfg.blockDim = dim3(NT3);
        cfg.dynamicSmemBytes = T3_SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl_enabled() ? 2 : 1;
        Timing &T = g_timing;
        const bool timed = T.on && T.used + 2 <= T.cap;
        if (timed && T.used == 0) cudaEventRecord(T.ev[T.used++], st);
        const gns_status r = check(cudaLaunchKernelEx(&cfg, tile3c_kern(ord), sk, dk, (long long)n, unsorted, smp,
                                                      (unsigned char *)nullptr, (double *)nullptr, smp_log2),
                                   "tile_sort2_kernel");
        if (timed && r == GNS_OK) {
            T.kind[T.used - 1] = launch_kind("tile_sort2_kernel");
            cudaEventRecord(T.ev[T.used++], st);
        }
        return r;
    }
    if (!hv && k1_v3())
        return launch_pdl("tile_sort2_kernel", tile3_kern(ord), grid, NT3, T3_SMEM, st, sk, dk, (long long)n, unsorted,
                          smp, tdesc, smp_src, smp_log2);
    CUtensorMap m[4];
    std::memset(m, 0, sizeof(m));
    if (n >= (size_t)TILE) {          // full tiles move by TMA tensor copies; a ragged last tile by plain loads
        GNS_TRY(row_map((void *)sk, n, true, 256, &m[0]));
        GNS_TRY(row_map(dk, n, true, 256, &m[2]));
        if (hv) {
            GNS_TRY(row_map((void *)sv, n, false, 256, &m[1]));
            GNS_TRY(row_map(dv, n, false, 256, &m[3]));
        }
    }
    const uint32_t *svv = hv ? sv : nullptr;
    uint32_t *dvv = hv ? dv : nullptr;
    auto kern = tile_kern(hv, ord);
    return launch_pdl("tile_sort2_kernel", kern, grid, NT1, t1_smem(hv), st, sk, svv, dk, dvv, (long long)n, m[0],
                      m[1], m[2], m[3], unsorted, smp, tdesc, smp_src);
}

// Rows a3+a4 (fused K2+K3, persistent TMA pipeline) or, in place, a6 (K2 +
// dependency ranges + K4 with the ticket/flag protocol).
gns_status launch_merge(const MergeGeo &g, const double *lim_a, const double *lim_b, int *corank, int2 *deps,
                        unsigned *flags, bool inplace, int ord, cudaStream_t st, Adapt ad = Adapt{},
                        Chain chain = Chain{nullptr, nullptr})
{
    const int ntiles = (int)ceil_div((size_t)g.n, MTILE);
    const bool hv = g.av != nullptr;
    PipeGeo pg;
    pg.g = g;
    pg.a_lim = lim_a;
    pg.b_lim = lim_b;
    pg.coop = coop_on();
    CUtensorMap map, amap, bmap;
    GNS_TRY(row_map(g.ok, (size_t)g.n, true, MTILE / 16, &map));
    // (B may start past the array end when the last pair has no B run: empty map, never loaded)
    GNS_TRY(key_map(g.ak, (size_t)std::max<long long>(0, lim_a - g.ak), hv, &amap, &pg.a_idx0, &pg.a_rows));
    GNS_TRY(key_map(g.bk, (size_t)std::max<long long>(0, lim_b - g.bk), hv, &bmap, &pg.b_idx0, &pg.b_rows));
    if (!inplace && ticket_pass(hv, ntiles)) {
        // Large passes: a partition kernel (sample-guided splits of every
        // tile) + the ticket-scheduled merge (K4's kernel without
        // dependencies; dynamic tile order balances the tail) beat the fused
        // search warps (2^27 pairs 10.2 vs 10.8 ms, 2^27 keys 7.37 vs 7.60 ms
        // per sort); smaller passes keep the fused kernel (the partition
        // launch costs more than it saves).
        unsigned *ticket = reinterpret_cast<unsigned *>(corank + ntiles);
        GNS_TRY(check(cudaMemsetAsync(ticket, 0, sizeof(unsigned), st), "memset"));
        GNS_TRY(launch_pdl("partition_kernel", partition_kern(ord),
                           (unsigned)ceil_div((size_t)ntiles * part_w(), 256), 256, 0, st, g, ntiles, corank));
        const int grid = std::min(ntiles, 2 * num_sms());
        auto kern = inplace_kern(hv, ord);
        return launch_pdl("merge_inplace_kernel", kern, grid, NT + 32, ts_smem(hv), st, pg, ntiles,
                          (const int *)corank, (const int2 *)nullptr, (unsigned *)nullptr, ticket, map, amap, bmap,
                          ad);
    }
    if (!inplace) {
        const int ctas = std::min(ntiles, 2 * num_sms());
        const int per = (int)ceil_div(ntiles, ctas);
        const int grid = (int)ceil_div(ntiles, per);
        auto kern = merge_kern(hv, ord);
        return launch_pdl("merge_tstore_kernel", kern, grid, WS_THREADS, ts_smem(hv), st, pg, ntiles, per, map, amap,
                          bmap, ad, OmitList{}, map, amap, bmap, chain);
    }
    GNS_TRY(launch_pdl("partition_kernel", partition_kern(ord),
                       (unsigned)ceil_div((size_t)ntiles * part_w(), 256), 256, 0, st, g, ntiles, corank));
    GNS_TRY(launch_pdl("inplace_deps_kernel", inplace_deps_kernel, (unsigned)ceil_div(ntiles + 1, 256), 256, 0, st,
                       (const int *)corank, ntiles, g.L, g.n, deps, flags));
    unsigned *ticket = flags + ntiles;
    const int grid = std::min(ntiles, 2 * num_sms());
    auto kern = inplace_kern(hv, ord);
    return launch_pdl("merge_inplace_kernel", kern, grid, NT + 32, ts_smem(hv), st, pg, ntiles, (const int *)corank,
                      (const int2 *)deps, flags, ticket, map, amap, bmap, Adapt{});
}

gns_status launch_reverse(double *k, uint32_t *v, size_t n, cudaStream_t st)
{
    if (n < 2) return GNS_OK;
    const unsigned grid = (unsigned)std::min<size_t>(ceil_div(n / 2, 256), (size_t)num_sms() * 8);
    if (v) return launch_pdl("reverse_kernel", reverse_kernel<true>, grid, 256, 0, st, k, v, (long long)n);
    return launch_pdl("reverse_kernel", reverse_kernel<false>, grid, 256, 0, st, k, (uint32_t *)nullptr,
                      (long long)n);
}

MergeGeo uniform_geo(const double *sk, const uint32_t *sv, double *dk, uint32_t *dv, size_t n, size_t L,
                     const double *sa = nullptr, double *so = nullptr)
{
    MergeGeo g;
    g.ak = sk;
    g.av = sv;
    g.bk = sk + L;
    g.bv = sv ? sv + L : nullptr;
    g.ok = dk;
    g.ov = dv;
    g.n = (long long)n;
    g.L = (long long)L;
    g.single = 0;
    g.tpp = (int)(2 * L / MTILE);
    g.tpp_log2 = (g.tpp & (g.tpp - 1)) ? -1 : __builtin_ctz((unsigned)g.tpp);
    g.sa = (L % SMP_G == 0) ? sa : nullptr;
    g.so = so;
    g.sb = nullptr;
    return g;
}

// One 4-way merge pass (gns_merge4.cuh): the pivots' split vectors
// (rank4_kernel), then the persistent merge of the chunks (merge4_kernel).
gns_status launch_merge4(const double *src, double *dst, size_t n, size_t L, const double *fsmp, double *smp_out,
                         int so_log2, unsigned char *wsp, int ord, cudaStream_t st, const Adapt &ad)
{
    Geo4 g;
    g.src = src;
    g.dst = dst;
    g.n = (long long)n;
    g.L = (long long)L;
    g.fsmp = fsmp;
    g.smp_out = smp_out;
    g.so_log2 = so_log2;
    g.apx = reinterpret_cast<int *>(wsp);
    g.vec = reinterpret_cast<int4 *>(wsp + align_up((ceil_div(n, FS) + 2) * sizeof(int), 256));
    g.cpg = (long long)ceil_div(4 * L, T4);
    const size_t ng = ceil_div(n, 4 * L);
    const size_t last_len = n - (ng - 1) * 4 * L;
    g.nchunks = (long long)((ng - 1) * (size_t)g.cpg + ceil_div(last_len, T4));
    const size_t np = ceil_div(n, FS);
    const unsigned rgrid = (unsigned)std::max<size_t>(1, std::min<size_t>(ceil_div(np, 256), (size_t)num_sms() * 8));
    GNS_TRY(launch_pdl("rank4_kernel", rank4_kern(ord), rgrid, 256, 0, st, g, ad.flag));
    GNS_TRY(launch_pdl("chunk4_kernel", chunk4_kern(ord), (unsigned)ceil_div((size_t)g.nchunks * 32, 256), 256, 0, st,
                       g, ad.flag));
    const int grid = (int)std::min<long long>(g.nchunks, (long long)GNS_M4_CTAS * num_sms());
    return launch_pdl("merge4_kernel", merge4_kern(ord), std::max(grid, 1), M4_THREADS, M4_SMEM, st, g, ad);
}

// Sorts region R = (rk, rv)[0:len) using partner region P of >= len slots as
// ping-pong buffer (Nocopy-Mergesort).  The result ends in P if
// `final_in_partner`, else in R.  Parity picks the tile-sort destination so
// no copy pass is ever needed (an odd number of merge levels starts from P).
// smp: two sample arrays of >= len/SMP_G + 2 keys (R's and P's), or nullptr.
// All M merge passes of a full-buffer sort as one pipelined launch
// (merge_multi_kernel): X = the tile sort's output, Y = the other region;
// words = mp_words(ntiles) zeroed words ([0] = the NEXT f2 flag, written by
// the tile sort).  `fin` = where the sort must end (X or Y).
gns_status launch_multi(double *xk, uint32_t *xv, double *yk, uint32_t *yv, double *xs, double *ys, size_t n, int M,
                        unsigned *words, double *fin, int ord, cudaStream_t st)
{
    const bool hv = xv != nullptr;
    const int ntiles = (int)ceil_div(n, MTILE);
    MultiGeo G;
    std::memset(&G, 0, sizeof(G));
    G.xk = xk;
    G.xv = xv;
    G.yk = yk;
    G.yv = yv;
    G.xs = xs;
    G.ys = ys;
    G.n = (long long)n;
    G.passes = M;
    G.ntiles = ntiles;
    {
        const char *e = std::getenv("GNS_MP_BLK");
        G.blk = e ? std::atoi(e) : 0;
    }
    G.flag = words;
    G.ticket = words + 1;
    G.done = words + 2;
    CUtensorMap xl, yl, xs_map, ys_map;
    GNS_TRY(key_map(xk, n, hv, &xl, &G.x_idx0, &G.x_rows));
    GNS_TRY(key_map(yk, n, hv, &yl, &G.y_idx0, &G.y_rows));
    GNS_TRY(row_map(xk, n, true, MTILE / 16, &xs_map));
    GNS_TRY(row_map(yk, n, true, MTILE / 16, &ys_map));
    // NEXT f2: the moves of an ordered / strictly reversed input
    const bool fin_x = fin == xk;
    if (!fin_x) {
        G.ord_src = xk;
        G.ord_srcv = xv;
        G.ord_dst = yk;
        G.ord_dstv = yv;
    }
    G.rev_src = xk;
    G.rev_srcv = xv;
    G.rev_dst = yk;
    G.rev_dstv = yv;
    if (fin_x) {                 // reversal into Y, then back to X
        G.rev2_src = yk;
        G.rev2_srcv = yv;
        G.rev2_dst = xk;
        G.rev2_dstv = xv;
    }
    const int grid = (int)std::min<long long>((long long)M * ntiles, 2LL * num_sms());
    return launch_pdl("merge_multi_kernel", multi_kern(hv, ord), std::max(grid, 1), MP_THREADS, ts_smem(hv), st, G, xl,
                      yl, xs_map, ys_map);
}

gns_status sort_range(double *rk, uint32_t *rv, double *pk_, uint32_t *pv_, size_t len,
                      bool final_in_partner, int *corank, int ord, cudaStream_t st, unsigned *unsorted = nullptr,
                      double *smp_r = nullptr, double *smp_p = nullptr, unsigned *mpw = nullptr,
                      unsigned char *piv = nullptr)
{
    if (len == 0) return GNS_OK;
    const int cl = k1_cluster(len, rv != nullptr);
    const size_t R = (size_t)TILE * cl;                 // run length after K1
    const int M = merge_passes_for(len, R);
    // 4-way passes (gns_merge4.cuh): two merge levels per HBM pass; an odd
    // level count starts with one 2-way pass.  P = HBM passes after K1.
    const bool four = use_four(rv != nullptr, len, R) && piv && smp_r && smp_p && !multi_on() && !chain_on();
    const int two_first = four ? (M & 1) : M;          // leading 2-way passes
    const int P = four ? two_first + M / 2 : M;
    const bool tile_to_partner = final_in_partner ^ (bool)(P & 1);
    double *ck = tile_to_partner ? pk_ : rk;
    uint32_t *cv = tile_to_partner ? pv_ : rv;
    double *ok = tile_to_partner ? rk : pk_;
    uint32_t *ov = tile_to_partner ? rv : pv_;
    double *tile_k = ck;
    uint32_t *tile_v = cv;
    double *cs = tile_to_partner ? smp_p : smp_r;      // samples of the region holding the current runs
    double *os = tile_to_partner ? smp_r : smp_p;
    if (mpw && unsorted == mpw && M > 0 && multi_on() && smp_r && smp_p) {
        // one pipelined launch for all merge levels (flag word + counters zeroed together)
        GNS_TRY(check(cudaMemsetAsync(mpw, 0, mp_words((int)ceil_div(len, MTILE)) * sizeof(unsigned), st), "memset"));
        GNS_TRY(launch_tile_sort(rk, rv, ck, cv, len, ord, st, unsorted, cs));
        return launch_multi(ck, cv, ok, ov, cs, os, len, M, mpw, final_in_partner ? pk_ : rk, ord, st);
    }
    // Chained passes (Chain, gns_kernels.cuh): every uniform pass after the
    // first starts as the previous one drains, tile by tile on region
    // counters (mp_words: [0] flag, [1] spare, then the counters of every
    // pass).  Only when every pass is the fused kernel (no ticket passes).
    const int ntl = (int)ceil_div(len, MTILE);
    const bool chain = mpw && unsorted == mpw && M > 1 && chain_on() && !ticket_pass(rv != nullptr, ntl);
    // NEXT f2: with `unsorted` the tile sort also tests whether the input is
    // already in order; if it is, every merge pass is omitted on the device.
    if (chain) GNS_TRY(check(cudaMemsetAsync(mpw, 0, mp_words(ntl) * sizeof(unsigned), st), "memset"));
    else if (unsorted && M > 0) GNS_TRY(check(cudaMemsetAsync(unsorted, 0, sizeof(unsigned), st), "memset"));
    unsigned *cnt_prev = nullptr;
    unsigned *cnt_next = chain ? mpw + 2 : nullptr;
    // samples of each pass's output for the next pass: fine (every FS-th key) before a 4-way pass
    auto smp_log2_before = [&](int p) { return (four && p >= two_first) ? FS_LOG2 : SMP_LOG2; };
    GNS_TRY(launch_tile_sort(rk, rv, ck, cv, len, ord, st, M > 0 ? unsorted : nullptr, M > 0 ? cs : nullptr,
                             nullptr, nullptr, cl, smp_log2_before(0)));
    int lvl = 0;                                       // merge levels done
    for (int p = 0; p < P; ++p) {
        const size_t L = R << lvl;
        const bool last = p == P - 1;
        const bool four_pass = four && p >= two_first;
        lvl += four_pass ? 2 : 1;
        MergeGeo g = uniform_geo(ck, cv, ok, ov, len, L, cs, last ? nullptr : os);
        g.so_log2 = smp_log2_before(p + 1);
        Adapt ad{};
        ad.flag = unsorted;
        ad.run_log2 = TILE_LOG2 + __builtin_ctz((unsigned)cl);
        if (unsorted) {
            // ordered input: the tile sort's output must end where the sort ends
            if (last && tile_k != ok) {
                ad.pre_k = tile_k;
                ad.pre_v = tile_v;
            }
            // strictly reversed input: tile-order reversal into the final
            // array in the last pass, or (tile output already there, even M)
            // reversal into the other array in pass M-2, then a copy back
            const bool tile_final = tile_k == (final_in_partner ? pk_ : rk);
            if (!tile_final && last) {
                ad.rev_k = tile_k;
                ad.rev_v = tile_v;
                ad.rev_gather = 1;
            } else if (tile_final && p == P - 2) {
                ad.rev_k = tile_k;
                ad.rev_v = tile_v;
                ad.rev_gather = 1;
            } else if (tile_final && last) {
                ad.rev_k = ck;
                ad.rev_v = cv;
                ad.rev_gather = 0;
            }
        }
        Chain chn{nullptr, nullptr};
        if (chain) {
            chn.dep = cnt_prev;                        // (pass 0: griddepcontrol.wait on the tile sort)
            chn.sig = last ? nullptr : cnt_next;
            cnt_prev = cnt_next;
            cnt_next += ceil_div(len, 4 * L);          // next-pass regions of this pass
        }
        if (four_pass)
            GNS_TRY(launch_merge4(ck, ok, len, L, cs, last ? nullptr : os, smp_log2_before(p + 1), piv, ord, st, ad));
        else GNS_TRY(launch_merge(g, ck + len, ck + len, corank, nullptr, nullptr, false, ord, st, ad, chn));
        std::swap(ck, ok);
        std::swap(cv, ov);
        std::swap(cs, os);
    }
    return GNS_OK;
}

// One list-driven merge launch (Omitsort): the listed tiles, data -> buffer
// (g0) or buffer -> data (g1) per the entry's direction bit.
gns_status launch_merge_list(const MergeGeo &g0, const MergeGeo &g1, const int *list, const int *count, int ord,
                             cudaStream_t st)
{
    const int ntiles = (int)ceil_div((size_t)g0.n, MTILE);
    const bool hv = g0.av != nullptr;
    PipeGeo pg[2];
    CUtensorMap map[2], amap[2], bmap[2];
    const MergeGeo *gs[2] = {&g0, &g1};
    for (int d = 0; d < 2; ++d) {
        const MergeGeo &g = *gs[d];
        const double *lim = g.ak + g.n;
        pg[d].g = g;
        pg[d].a_lim = lim;
        pg[d].b_lim = lim;
        GNS_TRY(row_map(g.ok, (size_t)g.n, true, MTILE / 16, &map[d]));
        GNS_TRY(key_map(g.ak, (size_t)g.n, hv, &amap[d], &pg[d].a_idx0, &pg[d].a_rows));
        GNS_TRY(key_map(g.bk, (size_t)std::max<long long>(0, lim - g.bk), hv, &bmap[d], &pg[d].b_idx0,
                        &pg[d].b_rows));
    }
    OmitList ol{list, count, pg[1]};
    const int grid = std::min(ntiles, 2 * num_sms());
    return launch_pdl("merge_tstore_kernel", merge_kern_ol(hv, ord), grid, WS_THREADS, ts_smem(hv), st, pg[0], ntiles,
                      0, map[0], amap[0], bmap[0], Adapt{}, ol, map[1], amap[1], bmap[1], Chain{nullptr, nullptr});
}

// NEXT f2: Omitsort on the full buffer.  The tile sort leaves
// tiles in order (and strictly reversed ones, Octosort) where they are and
// writes the others to the region that makes an all-merging input end in
// the data array; one plan launch decides every level; per level the copies
// and one list-driven merge launch; a final copy if the sorted run ends in
// the buffer.  Presorted input: no key moves.
gns_status sort_omit(double *keys, uint32_t *vals, size_t n, unsigned char *ws, const Layout &Lo, int ord,
                     cudaStream_t st)
{
    const bool hv = vals != nullptr;
    double *bk = reinterpret_cast<double *>(ws + Lo.off_k);
    uint32_t *bv = hv ? reinterpret_cast<uint32_t *>(ws + Lo.off_v) : nullptr;
    double *smp_d = reinterpret_cast<double *>(ws + Lo.off_smp);
    double *smp_b = smp_d + Lo.nsmp;
    OmitState S;
    S.st[0] = ws + Lo.off_loc;
    S.st[1] = S.st[0] + Lo.nruns;
    double *fl = reinterpret_cast<double *>(ws + Lo.off_fl);
    S.lo[0] = fl;
    S.lo[1] = fl + Lo.nruns;
    S.hi[0] = fl + 2 * Lo.nruns;
    S.hi[1] = fl + 3 * Lo.nruns;
    unsigned char *tdesc = ws + Lo.off_tdesc;
    unsigned char *act = ws + Lo.off_fix;
    int *pre = reinterpret_cast<int *>(ws + Lo.off_pre);
    int *list = reinterpret_cast<int *>(ws + Lo.off_list);
    int *cnt = reinterpret_cast<int *>(ws + Lo.off_cnt);
    const int M = merge_passes_for(n);
    // Tiles that need sorting go to the buffer when the number of merge
    // levels is odd (random input then ends in the data region with no copy
    // back); tiles in order or strictly reversed stay in place either way.
    const bool to_buf = (M & 1) != 0;
    GNS_TRY(launch_tile_sort(keys, vals, to_buf ? bk : keys, to_buf ? bv : vals, n, ord, st, nullptr,
                             to_buf ? smp_b : smp_d, tdesc, smp_d));
    GNS_TRY(launch_pdl("omit_plan_kernel", omit_plan_kern(ord), 1, OMIT_THREADS,
                       Lo.nruns <= (size_t)OMIT_SMEM_RUNS ? OMIT_SMEM : 0, st, (const double *)keys,
                       (const double *)bk, (const unsigned char *)tdesc, (long long)n, M, S, act, pre, cnt));
    const unsigned cgrid = (unsigned)std::min<size_t>(ceil_div(n, MTILE), (size_t)num_sms() * 4);
    size_t off = 0;
    for (int p = 0; p < M; ++p) {
        const size_t L = (size_t)TILE << p;
        const unsigned char *ap = act + off;
        const int *pp = pre + off;
        off += ceil_div(n, 2 * L);
        if (hv)
            GNS_TRY(launch_pdl("omit_prep_kernel", omit_prep_kernel<true>, cgrid, 256, 0, st, keys, vals, bk, bv,
                               smp_d, smp_b, (long long)n, TILE_LOG2 + p, ap, pp, list));
        else
            GNS_TRY(launch_pdl("omit_prep_kernel", omit_prep_kernel<false>, cgrid, 256, 0, st, keys,
                               (uint32_t *)nullptr, bk, (uint32_t *)nullptr, smp_d, smp_b, (long long)n,
                               TILE_LOG2 + p, ap, pp, list));
        MergeGeo g0 = uniform_geo(keys, vals, bk, bv, n, L, smp_d, smp_b);
        MergeGeo g1 = uniform_geo(bk, bv, keys, vals, n, L, smp_b, smp_d);
        GNS_TRY(launch_merge_list(g0, g1, list, cnt + p, ord, st));
    }
    const unsigned grid = (unsigned)std::min<size_t>(ceil_div(n, 2 * 256), (size_t)num_sms() * 8);
    if (hv)
        return launch_pdl("omit_final_kernel", omit_final_kernel<true>, grid, 256, 0, st, keys, vals,
                          (const double *)bk, (const uint32_t *)bv, (long long)n, (const int *)(cnt + M));
    return launch_pdl("omit_final_kernel", omit_final_kernel<false>, grid, 256, 0, st, keys, (uint32_t *)nullptr,
                      (const double *)bk, (const uint32_t *)nullptr, (long long)n, (const int *)(cnt + M));
}

constexpr double GNS_MIN_FRACTION = 1.0 / 64.0;

// buffer_fraction: exactly 1.0 (100 % buffer, %RAM 2.0), or p in [1/64, 0.5]:
// a buffer of ceil(p*n) elements rounded up to 32 (%RAM ~ 1 + p).
gns_status mode_for(double f, size_t n, Mode *m)
{
    if (f == 1.0) {
        m->limited = false;
        m->buf = n;
        return GNS_OK;
    }
    if (!(f >= GNS_MIN_FRACTION && f <= 0.5))
        return fail(GNS_ERR_UNSUPPORTED_FRACTION, "buffer_fraction must be 1.0 or in [1/64, 0.5]");
    m->limited = true;
    const size_t b = align_up((size_t)std::ceil(f * (double)n), 32);
    m->buf = b < n ? b : n;
    if (f == 0.5) m->buf = left_len(n);
    return GNS_OK;
}

gns_status validate_data(const double *keys, const uint32_t *vals, bool hv, size_t n, bool strict = false)
{
    if (n > GNS_MAX_N) return fail(GNS_ERR_INVALID_ARGUMENT, "n > GNS_MAX_N");
    if (n == 0) return GNS_OK;
    if (!keys || (hv && !vals)) return fail(GNS_ERR_INVALID_ARGUMENT, "NULL keys/vals with n > 0");
    // the per-step entry points launch the 32-byte kernels directly
    if (strict && (!is_aligned(keys, 32) || (hv && !is_aligned(vals, 32))))
        return fail(GNS_ERR_MISALIGNED, "keys/vals of the per-step entry points must be 32-byte aligned");
    // natural alignment; other 8-byte / 4-byte alignments take the peel path (run_sort)
    if (!is_aligned(keys, 8) || (hv && !is_aligned(vals, 4)))
        return fail(GNS_ERR_MISALIGNED, "keys must be 8-byte and vals 4-byte aligned");
    return GNS_OK;
}

// Ordered in-place merge of A = buffer[0:nl) and B = data[lo+nl : lo+len)
// into data[lo : lo+len) (row a6, K2 + deps + K4).
// s0, s1: two sample arrays (>= n/SMP_G + 2 keys each; free at this point),
// or nullptr: the partition then searches without samples.
gns_status top_merge(double *keys, uint32_t *vals, double *bk, uint32_t *bv, size_t lo, size_t len, size_t nl,
                     int *corank, int2 *deps, unsigned *flags, int ord, cudaStream_t st, double *s0 = nullptr,
                     double *s1 = nullptr)
{
    const bool hv = vals != nullptr;
    MergeGeo g;
    g.ak = bk;
    g.av = bv;
    g.bk = keys + lo + nl;
    g.bv = hv ? vals + lo + nl : nullptr;
    g.ok = keys + lo;
    g.ov = hv ? vals + lo : nullptr;
    g.n = (long long)len;
    g.L = (long long)nl;
    g.single = 1;
    g.tpp = 1;
    g.tpp_log2 = 0;
    g.sa = nullptr;
    g.so = nullptr;
    g.sb = nullptr;
    if (s0 && s1 && nl % SMP_G == 0) {
        // every SMP_G-th key of both runs -> sample-guided partition
        const long long nb = (long long)(len - nl);
        const size_t cnt = ceil_div(nl, SMP_G) + ceil_div((size_t)nb, SMP_G);
        GNS_TRY(launch_pdl("gather_samples_kernel", gather_samples_kernel,
                           (unsigned)std::max<size_t>(1, std::min<size_t>(ceil_div(cnt, 256), 1024)), 256, 0, st,
                           (const double *)bk, (long long)nl, s0, (const double *)g.bk, nb, s1));
        g.sa = s0;
        g.sb = s1;
    }
    return launch_merge(g, bk + nl, keys + lo + len, corank, deps, flags, true, ord, st);
}

// One step of a limited-buffer sort, also used by gns_plan to count element passes.
struct Sched {
    double elem_passes = 0;     // sum over steps of (HBM passes of the step x elements) / n
    int launches = 0;
    bool hv = false;
};

void count_sort_range(size_t len, Sched *sc, size_t n)
{
    if (!len) return;
    const size_t R = k1_run(len, sc->hv);
    const int M = merge_passes_for(len, R);
    if (use_four(sc->hv, len, R)) {
        // 4-way passes (two levels each, rank + merge launch), an odd level count starts 2-way
        const int P = (M & 1) + M / 2;
        sc->elem_passes += (double)(1 + P) * (double)len / (double)n;
        sc->launches += 1 + (M & 1) * (ticket_pass(false, (int)ceil_div(len, MTILE)) ? 2 : 1) + 2 * (M / 2);
        return;
    }
    sc->elem_passes += (double)(1 + M) * (double)len / (double)n;
    // tile sort + per pass one fused launch, or partition + ticket merge
    sc->launches += 1 + M * (ticket_pass(sc->hv, (int)ceil_div(len, MTILE)) ? 2 : 1);
}

// Limited-buffer sort of data[lo : lo+len) with a buffer of b elements
// (Frogsort2/3-style imbalanced split): if the 0.5 scheme
// fits (b >= left_len(len)), left half -> buffer, right half in place using the
// dead left region, in-place top merge.  Otherwise the right part
// data[lo+b : lo+len) is sorted first (recursively, same buffer), then the
// left b elements are sorted into the buffer and merged in place.
gns_status sort_limited(double *keys, uint32_t *vals, size_t lo, size_t len, size_t b, double *bk, uint32_t *bv,
                        int *corank, int2 *deps, unsigned *flags, int ord, cudaStream_t st, Sched *sc, size_t n,
                        double *s0 = nullptr, double *s1 = nullptr, unsigned char *piv = nullptr)
{
    const bool hv = vals != nullptr;
    double *dk = keys + lo;
    uint32_t *dv = hv ? vals + lo : nullptr;
    if (len <= (size_t)TILE) {
        if (sc) {
            count_sort_range(len, sc, n);
            return GNS_OK;
        }
        return launch_tile_sort(dk, dv, dk, dv, len, ord, st);
    }
    const size_t nl = left_len(len);
    if (b >= nl) {
        const size_t nr = len - nl;
        if (sc) {
            count_sort_range(nl, sc, n);
            count_sort_range(nr, sc, n);
            sc->elem_passes += (double)len / (double)n;
            sc->launches += 3 + (nl % SMP_G == 0 ? 1 : 0);   // (+ sample gather)
            return GNS_OK;
        }
        GNS_TRY(sort_range(dk, dv, bk, bv, nl, true, corank, ord, st, nullptr, s0, s1, nullptr, piv));
        GNS_TRY(sort_range(dk + nl, hv ? dv + nl : nullptr, dk, dv, nr, false, corank, ord, st, nullptr, s0, s1, nullptr,
                           piv));
        return top_merge(keys, vals, bk, bv, lo, len, nl, corank, deps, flags, ord, st, s0, s1);
    }
    GNS_TRY(sort_limited(keys, vals, lo + b, len - b, b, bk, bv, corank, deps, flags, ord, st, sc, n, s0, s1, piv));
    if (sc) {
        count_sort_range(b, sc, n);
        sc->elem_passes += (double)len / (double)n;
        sc->launches += 3 + (b % SMP_G == 0 ? 1 : 0);
        return GNS_OK;
    }
    GNS_TRY(sort_range(dk, dv, bk, bv, b, true, corank, ord, st, nullptr, s0, s1, nullptr, piv));
    return top_merge(keys, vals, bk, bv, lo, len, b, corank, deps, flags, ord, st, s0, s1);
}

// The sort proper (rows a1..a7).  ws already validated and sized.
// target: 0 AscLeft, 1 AscRight, 2 DescLeft, 3 DescRight (NEXT f3).
// AscRight = reverse(DescLeft), DescRight = reverse(AscLeft).
// kt: key type (0 f64, 1 i64, 2 u64; NEXT f3).
// One cluster of C CTAs (cluster dimension C, non-portable above 8).
gns_status launch_small(double *keys, uint32_t *vals, size_t n, int ord, int C, cudaStream_t st)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)C);
    cfg.blockDim = dim3(SM_NT);
    cfg.dynamicSmemBytes = sm_smem(vals != nullptr);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    Timing &T = g_timing;
    const bool timed = T.on && T.used + 2 <= T.cap;
    if (timed && T.used == 0) cudaEventRecord(T.ev[T.used++], st);
    const gns_status r = check(cudaLaunchKernelEx(&cfg, small_kern(vals != nullptr, ord), keys, vals, (long long)n),
                               "small_sort_kernel");
    if (timed && r == GNS_OK) {
        T.kind[T.used - 1] = launch_kind("small_sort_kernel");
        cudaEventRecord(T.ev[T.used++], st);
    }
    return r;
}

gns_status run_sort_aligned(double *keys, uint32_t *vals, size_t n, const Mode &m, unsigned char *ws, int target, int kt,
                    cudaStream_t st, bool reverse_right = true)
{
    if (n <= 1) return GNS_OK;
    GNS_TRY(ensure_attrs());
    const bool hv = vals != nullptr;
    const bool right = target == 1 || target == 3;
    const int ord = ord_of((target == 2) || (target == 1), kt);   // AscRight is reverse(DescLeft)
    if (small_on() && n <= (size_t)SMALL_MAX_N) {
        // on one thread-block cluster, no buffer (gns_small.cuh)
        int C = 1;
        while ((size_t)C * SM_TILE < n) C <<= 1;
        GNS_TRY(launch_small(keys, vals, n, ord, C, st));
    } else if (n <= (size_t)TILE) {   // one tile: in place, no buffer
        GNS_TRY(launch_tile_sort(keys, vals, keys, vals, n, ord, st));
    } else {
        const Layout Lo = layout(n, m, hv);
        double *bk = reinterpret_cast<double *>(ws + Lo.off_k);
        uint32_t *bv = hv ? reinterpret_cast<uint32_t *>(ws + Lo.off_v) : nullptr;
        int *corank = reinterpret_cast<int *>(ws + Lo.off_corank);
        double *smp = reinterpret_cast<double *>(ws + Lo.off_smp);
        unsigned char *piv = Lo.off_piv ? ws + Lo.off_piv : nullptr;
        if (m.omit) {
            GNS_TRY(sort_omit(keys, vals, n, ws, Lo, ord, st));
        } else if (!m.limited) {
            unsigned *unsorted = reinterpret_cast<unsigned *>(ws + Lo.off_adapt);
            GNS_TRY(sort_range(keys, vals, bk, bv, n, false, corank, ord, st, unsorted, smp, smp + Lo.nsmp, unsorted,
                               piv));
        } else {
            int2 *deps = reinterpret_cast<int2 *>(ws + Lo.off_deps);
            unsigned *flags = reinterpret_cast<unsigned *>(ws + Lo.off_flags);
            GNS_TRY(sort_limited(keys, vals, 0, n, m.buf, bk, bv, corank, deps, flags, ord, st, nullptr, n, smp,
                                 smp + Lo.nsmp, piv));
        }
    }
    if (right && reverse_right) GNS_TRY(launch_reverse(keys, vals, n, st));
    return GNS_OK;
}

// Natural alignment: head elements before the first
// 32-byte boundary of keys (and vals) -- 0..7 -- or -1 if keys and vals
// are misaligned relative to each other (no common boundary).
int peel_count(const double *keys, const uint32_t *vals)
{
    const int hk = (int)((4 - (((uintptr_t)keys >> 3) & 3)) & 3);
    if (!vals) return hk;
    const int hv = (int)((8 - (((uintptr_t)vals >> 2) & 7)) & 7);
    return (hv & 3) == hk ? hv : -1;
}

// The sort of keys[0:n) (+ vals) whatever their natural alignment: 32-byte
// aligned arrays go straight to run_sort_aligned; otherwise the aligned
// middle is sorted and the <= 7 head elements are merged in (gns_peel.cuh).
gns_status run_sort(double *keys, uint32_t *vals, size_t n, const Mode &m, unsigned char *ws, int target, int kt,
                    cudaStream_t st)
{
    if (n <= 1) return GNS_OK;
    const int h = peel_count(keys, vals);
    if (h == 0) return run_sort_aligned(keys, vals, n, m, ws, target, kt, st);
    GNS_TRY(ensure_attrs());
    const bool hv = vals != nullptr;
    if (h < 0) {
        // keys and vals with no common 32-byte boundary: the vals go through
        // a temporary placed so that it shares the keys' boundary (4n extra
        // bytes for the call)
        uint32_t *tbase = nullptr;
        cudaError_t e = cudaMallocAsync((void **)&tbase, (n + 8) * sizeof(uint32_t), st);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return e == cudaErrorMemoryAllocation ? fail(GNS_ERR_OUT_OF_MEMORY, "cudaMallocAsync: out of memory")
                                                  : check(e, "cudaMallocAsync");
        }
        const int hk = peel_count(keys, nullptr);
        uint32_t *tv = tbase + ((8 - hk) & 7);          // peel_count(keys, tv) == hk
        gns_status r = check(cudaMemcpyAsync(tv, vals, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st), "copy");
        if (r == GNS_OK) r = run_sort(keys, tv, n, m, ws, target, kt, st);
        if (r == GNS_OK)
            r = check(cudaMemcpyAsync(vals, tv, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st), "copy");
        const gns_status f = check(cudaFreeAsync(tbase, st), "cudaFreeAsync");
        return r != GNS_OK ? r : f;
    }
    const bool right = target == 1 || target == 3;
    const int ord = ord_of((target == 2) || (target == 1), kt);
    const size_t hh = std::min<size_t>((size_t)h, n);
    if (n > hh) {
        // the middle in the target's merge order (a Right target is the
        // reversal of the opposite-direction Left one: the whole array is
        // reversed at the end, not the middle)
        GNS_TRY(run_sort_aligned(keys + hh, hv ? vals + hh : nullptr, n - hh, m, ws, target, kt, st, false));
    }
    const Layout Lo = layout(n, m, hv);
    if (n <= (size_t)PEEL_CHUNK * 2 || Lo.total == 0) {
        // one CTA merges in order (no flags; the head sorted by the kernel)
        if (hv)
            GNS_TRY(launch_pdl("peel_merge_kernel", peel_kern(true, ord), 1, PEEL_NT, 0, st, keys, vals, (long long)n,
                               (int)hh, (const double *)nullptr, (const uint32_t *)nullptr, (unsigned *)nullptr,
                               (unsigned *)nullptr));
        else
            GNS_TRY(launch_pdl("peel_merge_kernel", peel_kern(false, ord), 1, PEEL_NT, 0, st, keys, (uint32_t *)nullptr,
                               (long long)n, (int)hh, (const double *)nullptr, (const uint32_t *)nullptr,
                               (unsigned *)nullptr, (unsigned *)nullptr));
    } else {
        // free workspace regions after the middle's sort: the co-rank array
        // (>= n / 4096 + 1 words) holds the chunk flags and the ticket, the
        // sample region the sorted head
        unsigned *flags = reinterpret_cast<unsigned *>(ws + Lo.off_corank);
        const size_t nch = ceil_div(n, PEEL_CHUNK);
        double *hk = reinterpret_cast<double *>(ws + Lo.off_smp);
        uint32_t *hvp = reinterpret_cast<uint32_t *>(hk + 8);
        GNS_TRY(check(cudaMemsetAsync(flags, 0, (nch + 1) * sizeof(unsigned), st), "memset"));
        if (hv)
            GNS_TRY(launch_pdl("peel_head_kernel", peel_head_kern(true, ord), 1, 32, 0, st, (const double *)keys,
                               (const uint32_t *)vals, (int)hh, hk, hvp));
        else
            GNS_TRY(launch_pdl("peel_head_kernel", peel_head_kern(false, ord), 1, 32, 0, st, (const double *)keys,
                               (const uint32_t *)nullptr, (int)hh, hk, (uint32_t *)nullptr));
        const int grid = (int)std::min<size_t>(nch, (size_t)num_sms() * 4);
        GNS_TRY(launch_pdl("peel_merge_kernel", peel_kern(hv, ord), grid, PEEL_NT, 0, st, keys,
                           hv ? vals : (uint32_t *)nullptr, (long long)n, (int)hh, (const double *)hk,
                           (const uint32_t *)(hv ? hvp : nullptr), flags, flags + nch));
    }
    if (right) GNS_TRY(launch_reverse(keys, vals, n, st));
    return GNS_OK;
}

// GNS_DEBUG=1: reject NaN keys (a precondition, R1) with
// GNS_ERR_INVALID_ARGUMENT before sorting; costs one pass and a host sync.
gns_status nan_guard(const double *keys, size_t n, int kt, cudaStream_t st)
{
    const char *e = std::getenv("GNS_DEBUG");
    if (kt != KT_F64 || n == 0 || !e || e[0] != '1') return GNS_OK;
    unsigned *dcnt = nullptr;
    GNS_TRY(check(cudaMallocAsync((void **)&dcnt, sizeof(unsigned), st), "cudaMallocAsync"));
    unsigned hcnt = 0;
    gns_status r = check(cudaMemsetAsync(dcnt, 0, sizeof(unsigned), st), "memset");
    if (r == GNS_OK) {
        const unsigned grid = (unsigned)std::min<size_t>(ceil_div(n, 256), (size_t)num_sms() * 8);
        nan_count_kernel<<<grid, 256, 0, st>>>(keys, (long long)n, dcnt);
        r = check(cudaGetLastError(), "nan_count_kernel");
    }
    if (r == GNS_OK) r = check(cudaMemcpyAsync(&hcnt, dcnt, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "memcpy");
    if (r == GNS_OK) r = check(cudaStreamSynchronize(st), "sync");
    cudaFreeAsync(dcnt, st);
    if (r != GNS_OK) return r;
    if (hcnt) return fail(GNS_ERR_INVALID_ARGUMENT, "NaN key (GNS_DEBUG=1 pre-scan)");
    return GNS_OK;
}

gns_status sort_alloc(double *keys, uint32_t *vals, bool hv, size_t n, double frac, int target, cudaStream_t st,
                      int kt = KT_F64, bool omit = false)
{
    Mode m;
    GNS_TRY(mode_for(frac, n, &m));
    m.omit = omit && !m.limited;
    GNS_TRY(validate_data(keys, vals, hv, n));
    if (n <= 1) return GNS_OK;
    GNS_TRY(ensure_attrs());
    GNS_TRY(nan_guard(keys, n, kt, st));
    const Layout Lo = layout(n, m, hv);
    unsigned char *ws = nullptr;
    if (Lo.total) {
        cudaError_t e = cudaMallocAsync((void **)&ws, Lo.total, st);
        if (e != cudaSuccess) {
            cudaGetLastError();
            if (e == cudaErrorMemoryAllocation) return fail(GNS_ERR_OUT_OF_MEMORY, "cudaMallocAsync: out of memory");
            return check(e, "cudaMallocAsync");
        }
    }
    gns_status s = run_sort(keys, hv ? vals : nullptr, n, m, ws, target, kt, st);
    if (ws) {
        gns_status f = check(cudaFreeAsync(ws, st), "cudaFreeAsync");
        if (s == GNS_OK) s = f;
    }
    return s;
}

gns_status sort_ws(double *keys, uint32_t *vals, bool hv, size_t n, double frac, void *ws, size_t ws_bytes,
                   int target, cudaStream_t st, int kt = KT_F64, bool omit = false)
{
    Mode m;
    GNS_TRY(mode_for(frac, n, &m));
    m.omit = omit && !m.limited;
    GNS_TRY(validate_data(keys, vals, hv, n));
    if (n <= 1) return GNS_OK;
    const Layout Lo = layout(n, m, hv);
    if (Lo.total) {
        if (!ws || ws_bytes < Lo.total) return fail(GNS_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
        if (!is_aligned(ws, 32)) return fail(GNS_ERR_MISALIGNED, "ws must be 32-byte aligned");
    }
    GNS_TRY(ensure_attrs());
    GNS_TRY(nan_guard(keys, n, kt, st));
    return run_sort(keys, hv ? vals : nullptr, n, m, (unsigned char *)ws, target, kt, st);
}

}  // namespace

// ======================================================================= C-ABI
extern "C" {

gns_status gns_sort_f64(double *keys, size_t n, double buffer_fraction, gns_stream_t stream)
{
    return sort_alloc(keys, nullptr, false, n, buffer_fraction, 0, (cudaStream_t)stream);
}

gns_status gns_sort_pairs_f64_u32(double *keys, uint32_t *vals, size_t n, double buffer_fraction,
                                  gns_stream_t stream)
{
    return sort_alloc(keys, vals, true, n, buffer_fraction, 0, (cudaStream_t)stream);
}

size_t gns_workspace_bytes(size_t n, double buffer_fraction, int with_vals)
{
    Mode m;
    if (mode_for(buffer_fraction, n, &m) != GNS_OK || n > GNS_MAX_N) return 0;
    return layout(n, m, with_vals != 0).total;
}

gns_status gns_sort_f64_ws(double *keys, size_t n, double buffer_fraction, void *ws, size_t ws_bytes,
                           gns_stream_t stream)
{
    return sort_ws(keys, nullptr, false, n, buffer_fraction, ws, ws_bytes, 0, (cudaStream_t)stream);
}

gns_status gns_sort_pairs_f64_u32_ws(double *keys, uint32_t *vals, size_t n, double buffer_fraction,
                                     void *ws, size_t ws_bytes, gns_stream_t stream)
{
    return sort_ws(keys, vals, true, n, buffer_fraction, ws, ws_bytes, 0, (cudaStream_t)stream);
}

gns_status gns_sort_target_f64(double *keys, uint32_t *vals, size_t n, double buffer_fraction, gns_target target,
                               void *ws, size_t ws_bytes, gns_stream_t stream)
{
    if ((int)target < 0 || (int)target > 3) return fail(GNS_ERR_INVALID_ARGUMENT, "target must be 0..3");
    if (ws) return sort_ws(keys, vals, vals != nullptr, n, buffer_fraction, ws, ws_bytes, (int)target,
                           (cudaStream_t)stream);
    return sort_alloc(keys, vals, vals != nullptr, n, buffer_fraction, (int)target, (cudaStream_t)stream);
}

gns_status gns_sort_keys(void *keys, gns_key_type key_type, uint32_t *vals, size_t n, double buffer_fraction,
                         gns_target target, void *ws, size_t ws_bytes, gns_stream_t stream)
{
    if ((int)target < 0 || (int)target > 3) return fail(GNS_ERR_INVALID_ARGUMENT, "target must be 0..3");
    if ((int)key_type < 0 || (int)key_type > 2) return fail(GNS_ERR_INVALID_ARGUMENT, "key_type must be 0..2");
    double *k = (double *)keys;
    if (ws) return sort_ws(k, vals, vals != nullptr, n, buffer_fraction, ws, ws_bytes, (int)target,
                           (cudaStream_t)stream, (int)key_type);
    return sort_alloc(k, vals, vals != nullptr, n, buffer_fraction, (int)target, (cudaStream_t)stream,
                      (int)key_type);
}

size_t gns_workspace_bytes_u64(size_t n)
{
    Mode m;
    if (mode_for(1.0, n, &m) != GNS_OK || n > GNS_MAX_N) return 0;
    if (n <= 1) return 0;
    return align_up(n * sizeof(uint32_t), 256) +
           std::max(layout(n, m, true).total, align_up(n * sizeof(uint64_t), 256));
}

gns_status gns_sort_keys_u64(void *keys, gns_key_type key_type, uint64_t *vals, size_t n, gns_target target,
                             void *ws, size_t ws_bytes, gns_stream_t stream)
{
    if ((int)target < 0 || (int)target > 3) return fail(GNS_ERR_INVALID_ARGUMENT, "target must be 0..3");
    if ((int)key_type < 0 || (int)key_type > 2) return fail(GNS_ERR_INVALID_ARGUMENT, "key_type must be 0..2");
    double *k = (double *)keys;
    if (n > GNS_MAX_N) return fail(GNS_ERR_INVALID_ARGUMENT, "n > GNS_MAX_N");
    if (n && (!keys || !vals)) return fail(GNS_ERR_INVALID_ARGUMENT, "NULL keys/vals with n > 0");
    if (n && (!is_aligned(keys, 32) || !is_aligned(vals, 32)))
        return fail(GNS_ERR_MISALIGNED, "keys/vals must be 32-byte aligned");
    if (n <= 1) return GNS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t need = gns_workspace_bytes_u64(n);
    unsigned char *w = (unsigned char *)ws;
    if (w) {
        if (ws_bytes < need) return fail(GNS_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
        if (!is_aligned(w, 32)) return fail(GNS_ERR_MISALIGNED, "ws must be 32-byte aligned");
    }
    GNS_TRY(ensure_attrs());
    GNS_TRY(nan_guard(k, n, (int)key_type, st));
    bool own = false;
    if (!w) {
        cudaError_t e = cudaMallocAsync((void **)&w, need, st);
        if (e != cudaSuccess) {
            cudaGetLastError();
            if (e == cudaErrorMemoryAllocation) return fail(GNS_ERR_OUT_OF_MEMORY, "cudaMallocAsync: out of memory");
            return check(e, "cudaMallocAsync");
        }
        own = true;
    }
    uint32_t *idx = reinterpret_cast<uint32_t *>(w);
    unsigned char *rest = w + align_up(n * sizeof(uint32_t), 256);     // pairs workspace, then the gather buffer
    Mode m;
    gns_status r = mode_for(1.0, n, &m);
    const unsigned grid = (unsigned)std::min<size_t>(ceil_div(n, 256), (size_t)num_sms() * 8);
    if (r == GNS_OK) r = launch_pdl("iota_u32_kernel", iota_u32_kernel, grid, 256, 0, st, idx, (long long)n);
    if (r == GNS_OK) r = run_sort(k, idx, n, m, rest, (int)target, (int)key_type, st);
    uint64_t *tmp = reinterpret_cast<uint64_t *>(rest);
    if (r == GNS_OK)
        r = launch_pdl("gather_u64_kernel", gather_u64_kernel, grid, 256, 0, st, tmp, (const uint64_t *)vals,
                       (const uint32_t *)idx, (long long)n);
    if (r == GNS_OK) r = check(cudaMemcpyAsync(vals, tmp, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st), "copy");
    if (own) {
        gns_status f = check(cudaFreeAsync(w, st), "cudaFreeAsync");
        if (r == GNS_OK) r = f;
    }
    return r;
}

size_t gns_workspace_bytes_f32(size_t n, int with_vals)
{
    // the buffer: n keys (+ n vals), the merge tiles' splits; none for one tile
    if (n > GNS_MAX_N || n <= (size_t)F_TILE) return 0;
    return (with_vals ? 2 : 1) * align_up(n * sizeof(float), 256) +
           align_up((ceil_div(n, F_MTILE) + 1) * sizeof(int), 256);
}

gns_status gns_sort_f32(float *keys, uint32_t *vals, size_t n, gns_target target, void *ws, size_t ws_bytes,
                        gns_stream_t stream)
{
    if ((int)target < 0 || (int)target > 3) return fail(GNS_ERR_INVALID_ARGUMENT, "target must be 0..3");
    if (n > GNS_MAX_N) return fail(GNS_ERR_INVALID_ARGUMENT, "n > GNS_MAX_N");
    if (n && !keys) return fail(GNS_ERR_INVALID_ARGUMENT, "NULL keys with n > 0");
    if (n && (!is_aligned(keys, 32) || (vals && !is_aligned(vals, 32))))
        return fail(GNS_ERR_MISALIGNED, "keys/vals must be 32-byte aligned");
    if (n <= 1) return GNS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const bool hv = vals != nullptr;
    const size_t need = gns_workspace_bytes_f32(n, hv ? 1 : 0);
    unsigned char *w = (unsigned char *)ws;
    if (need && w) {
        if (ws_bytes < need) return fail(GNS_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
        if (!is_aligned(w, 32)) return fail(GNS_ERR_MISALIGNED, "ws must be 32-byte aligned");
    }
    GNS_TRY(ensure_attrs());
    bool own = false;
    if (need && !w) {
        cudaError_t e = cudaMallocAsync((void **)&w, need, st);
        if (e != cudaSuccess) {
            cudaGetLastError();
            if (e == cudaErrorMemoryAllocation) return fail(GNS_ERR_OUT_OF_MEMORY, "cudaMallocAsync: out of memory");
            return check(e, "cudaMallocAsync");
        }
        own = true;
    }
    const bool right = target == 1 || target == 3;
    const int desc = (target == 2 || target == 1) ? 1 : 0;      // AscRight = reverse(DescLeft)
    float *bk = reinterpret_cast<float *>(w);
    uint32_t *bv = hv ? reinterpret_cast<uint32_t *>(w + align_up(n * sizeof(float), 256)) : nullptr;
    const int M = merge_passes_for(n);                // (F_TILE == TILE: the same level count)
    // the tile sort's destination by the parity of the merge levels: the last pass lands in keys
    float *ck = (M & 1) ? bk : keys, *ok = (M & 1) ? keys : bk;
    uint32_t *cv = (M & 1) ? bv : vals, *ov = (M & 1) ? vals : bv;
    // key-only: the 128 x 64 K1 (gns_tile64.cuh) on 4-byte keys; with payload
    // the 256 x 32 binary32 tile sort (gns_f32.cuh)
    gns_status r = (!hv && k1_v3())
        ? launch_pdl("f32_tile_sort_kernel", tile3f_kern(desc), (unsigned)ceil_div(n, F_TILE), NT3,
                     t3_smem<float, NT3>(), st, (const float *)keys, ck, (long long)n, (unsigned *)nullptr,
                     (float *)nullptr, (unsigned char *)nullptr, (float *)nullptr, (int)SMP_LOG2)
        : launch_pdl("f32_tile_sort_kernel", f32_tile_kern(hv, desc), (unsigned)ceil_div(n, F_TILE), F_NT,
                     f_tile_smem(hv), st, (const float *)keys, (const uint32_t *)vals, ck, cv, (long long)n);
    int *corank = reinterpret_cast<int *>(w + (hv ? 2 : 1) * align_up(n * sizeof(float), 256));
    const int ntiles = (int)ceil_div(n, F_MTILE);
    for (int p = 0; p < M && r == GNS_OK && k1_v3(); ++p) {
        // the pipelined pass with in-kernel co-rank searches (with payload: 2 CTAs per SM)
        const long long L = (long long)F_TILE << p;
        const int nt2 = (int)ceil_div(n, F2_MT);
        const int ctas = std::min(nt2, (hv ? 2 : 3) * num_sms());
        const int per = (int)ceil_div(nt2, ctas);
        r = launch_pdl("f32_merge_kernel", f32_merge2_kern(hv, desc), (unsigned)ceil_div(nt2, per), F2_THREADS,
                       f2_smem(hv), st, (const float *)ck, (const uint32_t *)cv, ok, ov, (long long)n, L, nt2, per);
        std::swap(ck, ok);
        std::swap(cv, ov);
    }
    for (int p = 0; p < M && r == GNS_OK && !k1_v3(); ++p) {
        const long long L = (long long)F_TILE << p;
        r = launch_pdl("f32_partition_kernel", f32_part_kern(desc), (unsigned)ceil_div((size_t)ntiles * 32, 256), 256,
                       0, st, (const float *)ck, (long long)n, L, ntiles, corank);
        if (r == GNS_OK)
            r = launch_pdl("f32_merge_kernel", f32_merge_kern(hv, desc), (unsigned)ntiles, F_NT, f_merge_smem(hv), st,
                           (const float *)ck, (const uint32_t *)cv, ok, ov, (long long)n, L, (const int *)corank);
        std::swap(ck, ok);
        std::swap(cv, ov);
    }
    if (r == GNS_OK && right) {
        const unsigned grid = (unsigned)std::min<size_t>(ceil_div(n / 2, 256), (size_t)num_sms() * 8);
        r = hv ? launch_pdl("f32_reverse_kernel", f32_reverse_kernel<true>, std::max(1u, grid), 256, 0, st, keys,
                            vals, (long long)n)
               : launch_pdl("f32_reverse_kernel", f32_reverse_kernel<false>, std::max(1u, grid), 256, 0, st, keys,
                            (uint32_t *)nullptr, (long long)n);
    }
    if (own) {
        gns_status f = check(cudaFreeAsync(w, st), "cudaFreeAsync");
        if (r == GNS_OK) r = f;
    }
    return r;
}

gns_status gns_sort_omit(void *keys, gns_key_type key_type, uint32_t *vals, size_t n, gns_target target, void *ws,
                         size_t ws_bytes, gns_stream_t stream)
{
    if ((int)target < 0 || (int)target > 3) return fail(GNS_ERR_INVALID_ARGUMENT, "target must be 0..3");
    if ((int)key_type < 0 || (int)key_type > 2) return fail(GNS_ERR_INVALID_ARGUMENT, "key_type must be 0..2");
    double *k = (double *)keys;
    if (ws) return sort_ws(k, vals, vals != nullptr, n, 1.0, ws, ws_bytes, (int)target, (cudaStream_t)stream,
                           (int)key_type, true);
    return sort_alloc(k, vals, vals != nullptr, n, 1.0, (int)target, (cudaStream_t)stream, (int)key_type, true);
}

gns_status gns_plan(size_t n, double buffer_fraction, int with_vals, gns_plan_info *out)
{
    Mode m;
    GNS_TRY(mode_for(buffer_fraction, n, &m));
    if (!out) return fail(GNS_ERR_INVALID_ARGUMENT, "out == NULL");
    if (n > GNS_MAX_N) return fail(GNS_ERR_INVALID_ARGUMENT, "n > GNS_MAX_N");
    const Layout Lo = layout(n, m, with_vals != 0);
    const size_t s = with_vals ? 12 : 8;
    std::memset(out, 0, sizeof(*out));
    out->tile = TILE;
    out->merge_tile = MTILE;
    out->merge_passes = merge_passes_for(n, k1_run(n, with_vals != 0));
    Sched sc;
    sc.hv = with_vals != 0;
    if (n <= 1) {
        sc.elem_passes = 0;
    } else if (n <= (size_t)SMALL_MAX_N && small_on()) {
        sc.elem_passes = 1;                           // one read + one write, every level on chip
        sc.launches = 1;
        out->merge_passes = 0;
    } else if (n <= (size_t)TILE || !m.limited) {
        count_sort_range(n, &sc, n);
    } else {
        sort_limited(nullptr, nullptr, 0, n, m.buf, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, &sc, n);
    }
    out->element_passes = sc.elem_passes;
    out->launches = sc.launches;
    out->hbm_passes = (int)std::ceil(sc.elem_passes - 1e-9);
    out->left_len = (m.limited && n > (size_t)TILE) ? std::min(m.buf, left_len(n)) : 0;
    out->workspace_bytes = Lo.total;
    out->buffer_elems = Lo.buf_elems;
    out->bytes_lower_bound = (size_t)std::llround(sc.elem_passes * (double)n) * 2 * s;
    return GNS_OK;
}

gns_status gns_tile_sort(const double *src_keys, const uint32_t *src_vals, double *dst_keys,
                         uint32_t *dst_vals, size_t n, gns_stream_t stream)
{
    const bool hv = src_vals != nullptr || dst_vals != nullptr;
    if (hv && (!src_vals || !dst_vals)) return fail(GNS_ERR_INVALID_ARGUMENT, "src_vals/dst_vals: both or neither");
    GNS_TRY(validate_data(src_keys, src_vals, hv, n, true));
    GNS_TRY(validate_data(dst_keys, dst_vals, hv, n, true));
    if (n == 0) return GNS_OK;
    GNS_TRY(ensure_attrs());
    return launch_tile_sort(src_keys, src_vals, dst_keys, dst_vals, n, 0, (cudaStream_t)stream);
}

size_t gns_merge_workspace_bytes(size_t n) { return merge_ws(n); }

gns_status gns_merge_pass(const double *src_keys, const uint32_t *src_vals, double *dst_keys,
                          uint32_t *dst_vals, size_t n, size_t run_len, void *ws, size_t ws_bytes,
                          gns_stream_t stream)
{
    const bool hv = src_vals != nullptr || dst_vals != nullptr;
    if (hv && (!src_vals || !dst_vals)) return fail(GNS_ERR_INVALID_ARGUMENT, "src_vals/dst_vals: both or neither");
    GNS_TRY(validate_data(src_keys, src_vals, hv, n, true));
    GNS_TRY(validate_data(dst_keys, dst_vals, hv, n, true));
    if (run_len == 0 || run_len % (MTILE / 2) != 0 || run_len > (size_t)1 << 30)
        return fail(GNS_ERR_INVALID_ARGUMENT, "run_len must be a positive multiple of gns_merge_tile_elems()/2, <= 2^30");
    if (n == 0) return GNS_OK;
    if (!ws || ws_bytes < merge_ws(n)) return fail(GNS_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
    GNS_TRY(ensure_attrs());
    MergeGeo g = uniform_geo(src_keys, src_vals, dst_keys, dst_vals, n, run_len);
    return launch_merge(g, src_keys + n, src_keys + n, (int *)ws, nullptr, nullptr, false, 0, (cudaStream_t)stream);
}

gns_status gns_merge_two(const void *a_keys, const uint32_t *a_vals, size_t la, const void *b_keys,
                         const uint32_t *b_vals, size_t lb, void *dst_keys, uint32_t *dst_vals, gns_key_type key_type,
                         gns_stream_t stream)
{
    const bool hv = dst_vals != nullptr;      // an empty run's vals may be NULL
    if ((!hv && (a_vals || b_vals)) || (hv && ((la && !a_vals) || (lb && !b_vals))))
        return fail(GNS_ERR_INVALID_ARGUMENT, "vals: dst_vals and the non-empty runs' vals, or none");
    if ((int)key_type < 0 || (int)key_type > 2) return fail(GNS_ERR_INVALID_ARGUMENT, "key_type must be 0..2");
    const size_t n = la + lb;
    if (n > GNS_MAX_N) return fail(GNS_ERR_INVALID_ARGUMENT, "la + lb > GNS_MAX_N");
    if (n == 0) return GNS_OK;
    if ((la && !a_keys) || (lb && !b_keys) || !dst_keys)
        return fail(GNS_ERR_INVALID_ARGUMENT, "NULL keys with a non-empty run");
    if (!is_aligned(a_keys, 8) || !is_aligned(b_keys, 8) || !is_aligned(a_vals, 4) || !is_aligned(b_vals, 4))
        return fail(GNS_ERR_MISALIGNED, "a/b keys must be 8-byte, vals 4-byte aligned");
    GNS_TRY(validate_data((const double *)dst_keys, dst_vals, hv, n));
    // dst at natural alignment: the first `off` outputs go through a one-thread
    // head kernel so that the pipelined merge stores from a 16-byte aligned
    // key row / 32-byte aligned vals (the distributed sort merges runs at any
    // element offset)
    int off = (int)(((uintptr_t)dst_keys >> 3) & 1);
    if (hv) {
        off = (int)((8 - (((uintptr_t)dst_vals >> 2) & 7)) & 7);
        if (((((uintptr_t)dst_keys >> 3) + off) & 1) != 0)
            return fail(GNS_ERR_MISALIGNED, "dst keys and vals have no common aligned element");
    }
    off = (int)std::min<size_t>((size_t)off, n);
    GNS_TRY(ensure_attrs());
    cudaStream_t st = (cudaStream_t)stream;
    if (la == 0 || lb == 0) {          // one run: a copy
        const void *sk = la ? a_keys : b_keys;
        const uint32_t *sv = la ? a_vals : b_vals;
        GNS_TRY(check(cudaMemcpyAsync(dst_keys, sk, n * 8, cudaMemcpyDeviceToDevice, st), "copy"));
        if (hv) GNS_TRY(check(cudaMemcpyAsync(dst_vals, sv, n * 4, cudaMemcpyDeviceToDevice, st), "copy"));
        return GNS_OK;
    }
    const int ordm = ord_of(false, (int)key_type);
    if (off > 0) {
        if (hv)
            GNS_TRY(launch_pdl("merge_head_kernel", mhead_kern(true, ordm), 1, 32, 0, st, (const double *)a_keys, a_vals,
                               (long long)la, (const double *)b_keys, b_vals, (long long)lb, (double *)dst_keys,
                               dst_vals, off));
        else
            GNS_TRY(launch_pdl("merge_head_kernel", mhead_kern(false, ordm), 1, 32, 0, st, (const double *)a_keys,
                               (const uint32_t *)nullptr, (long long)la, (const double *)b_keys,
                               (const uint32_t *)nullptr, (long long)lb, (double *)dst_keys, (uint32_t *)nullptr,
                               off));
        if ((size_t)off == n) return GNS_OK;
    }
    MergeGeo g;
    g.ak = (const double *)a_keys;
    g.av = hv ? a_vals : nullptr;
    g.bk = (const double *)b_keys;
    g.bv = hv ? b_vals : nullptr;
    g.ok = (double *)dst_keys + off;
    g.ov = hv ? dst_vals + off : nullptr;
    g.n = (long long)n;
    g.L = (long long)la;
    g.single = 1;
    g.tpp = 1;
    g.tpp_log2 = 0;
    g.sa = nullptr;
    g.so = nullptr;
    g.sb = nullptr;
    g.off = off;
    const int ntiles = (int)ceil_div(n - off, MTILE);
    PipeGeo pg;
    pg.g = g;
    pg.a_lim = g.ak + la;
    pg.b_lim = g.bk + lb;
    CUtensorMap map, amap, bmap;
    GNS_TRY(row_map(g.ok, n - off, true, MTILE / 16, &map));
    GNS_TRY(key_map(g.ak, la, hv, &amap, &pg.a_idx0, &pg.a_rows));
    GNS_TRY(key_map(g.bk, lb, hv, &bmap, &pg.b_idx0, &pg.b_rows));
    const int ctas = std::min(ntiles, 2 * num_sms());
    const int per = (int)ceil_div(ntiles, ctas);
    const int grid = (int)ceil_div(ntiles, per);
    auto kern = merge_kern(hv, ordm);
    return launch_pdl("merge_tstore_kernel", kern, grid, WS_THREADS, ts_smem(hv), st, pg, ntiles, per, map, amap, bmap,
                      Adapt{}, OmitList{}, map, amap, bmap, Chain{nullptr, nullptr});
}

gns_status gns_split_cuts(const void *sorted_keys, gns_key_type key_type, size_t n, const void *spl_keys,
                          const int32_t *spl_rank, const int64_t *spl_pos, int nsplit, int my_rank, int64_t *cuts,
                          gns_stream_t stream)
{
    if ((int)key_type < 0 || (int)key_type > 2) return fail(GNS_ERR_INVALID_ARGUMENT, "key_type must be 0..2");
    if (nsplit < 0 || n > GNS_MAX_N) return fail(GNS_ERR_INVALID_ARGUMENT, "nsplit < 0 or n > GNS_MAX_N");
    if (nsplit == 0) return GNS_OK;
    if ((n && !sorted_keys) || !spl_keys || !spl_rank || !spl_pos || !cuts)
        return fail(GNS_ERR_INVALID_ARGUMENT, "NULL pointer");
    GNS_TRY(ensure_attrs());
    static const decltype(&split_cuts_kernel<0>) tab[3] = {&split_cuts_kernel<0>, &split_cuts_kernel<2>,
                                                          &split_cuts_kernel<4>};
    return launch_pdl("split_cuts_kernel", tab[(int)key_type], (unsigned)ceil_div((size_t)nsplit, 128), 128, 0,
                      (cudaStream_t)stream, (const double *)sorted_keys, (long long)n, (const double *)spl_keys,
                      (const int *)spl_rank, (const long long *)spl_pos, nsplit, my_rank, (long long *)cuts);
}

gns_status gns_merge_inplace_top(double *keys, uint32_t *vals, const double *left_keys,
                                 const uint32_t *left_vals, size_t nl, size_t n, void *ws, size_t ws_bytes,
                                 gns_stream_t stream)
{
    const bool hv = vals != nullptr || left_vals != nullptr;
    if (hv && (!vals || !left_vals)) return fail(GNS_ERR_INVALID_ARGUMENT, "vals/left_vals: both or neither");
    GNS_TRY(validate_data(keys, vals, hv, n, true));
    GNS_TRY(validate_data(left_keys, left_vals, hv, nl, true));
    if (nl > n || nl % 32 != 0 || nl == 0)
        return fail(GNS_ERR_INVALID_ARGUMENT, "need 0 < nl <= n, nl % 32 == 0");
    if (!ws || ws_bytes < merge_ws(n)) return fail(GNS_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
    GNS_TRY(ensure_attrs());
    const size_t nt = ceil_div(n, MTILE);
    unsigned char *w = (unsigned char *)ws;
    int *corank = (int *)w;
    int2 *deps = (int2 *)(w + align_up((nt + 1) * sizeof(int), 256));
    unsigned *flags = (unsigned *)((unsigned char *)deps + align_up(nt * sizeof(int2), 256));
    MergeGeo g;
    g.ak = left_keys;
    g.av = left_vals;
    g.bk = keys + nl;
    g.bv = hv ? vals + nl : nullptr;
    g.ok = keys;
    g.ov = vals;
    g.n = (long long)n;
    g.L = (long long)nl;
    g.single = 1;
    g.tpp = 1;
    g.tpp_log2 = 0;
    g.sa = nullptr;
    g.so = nullptr;
    g.sb = nullptr;
    return launch_merge(g, left_keys + nl, keys + n, corank, deps, flags, true, 0, (cudaStream_t)stream);
}

#ifdef GNS_PROF
void gns_prof_reset(void)
{
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    unsigned long long tl[32][2];
    for (int i = 0; i < 32; ++i) {
        tl[i][0] = ~0ull;
        tl[i][1] = 0;
    }
    cudaMemcpyToSymbol(g_tl, tl, sizeof(tl));
}
void gns_prof_timeline(unsigned long long *out)
{
    cudaMemcpyFromSymbol(out, g_tl, 64 * sizeof(unsigned long long));
}
void gns_prof_read(unsigned long long *out)
{
    cudaMemcpyFromSymbol(out, g_prof, 16 * sizeof(unsigned long long));
}
#endif

size_t gns_pool_high_water(int reset)
{
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess)
        return (size_t)-1;
    cuuint64_t v = 0;
    if (reset) {
        if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &v) != cudaSuccess) return (size_t)-1;
        return 0;
    }
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &v) != cudaSuccess) return (size_t)-1;
    return (size_t)v;
}

gns_status gns_timing_begin(int max_launches)
{
    Timing &T = g_timing;
    if (T.on) return fail(GNS_ERR_INVALID_ARGUMENT, "timing already on");
    if (max_launches <= 0 || max_launches > 4096) return fail(GNS_ERR_INVALID_ARGUMENT, "max_launches in 1..4096");
    const int need = max_launches + 1;
    while ((int)T.ev.size() < need) {
        cudaEvent_t e;
        GNS_TRY(check(cudaEventCreate(&e), "cudaEventCreate"));
        T.ev.push_back(e);
    }
    T.kind.assign(need, 0);
    T.cap = need;
    T.used = 0;
    T.on = true;
    return GNS_OK;
}

int gns_timing_end(float *ms, int *kind, int cap)
{
    Timing &T = g_timing;
    if (!T.on) return -1;
    T.on = false;
    const int n = T.used > 0 ? T.used - 1 : 0;
    if (n > 0 && cudaEventSynchronize(T.ev[T.used - 1]) != cudaSuccess) return -1;
    for (int i = 0; i < n && i < cap; ++i) {
        float t = 0.f;
        cudaEventElapsedTime(&t, T.ev[i], T.ev[i + 1]);
        if (ms) ms[i] = t;
        if (kind) kind[i] = T.kind[i];
    }
    return n;
}

int gns_tile_elems(void) { return TILE; }
int gns_merge_tile_elems(void) { return MTILE; }

const char *gns_status_string(gns_status s)
{
    switch (s) {
    case GNS_OK: return "GNS_OK";
    case GNS_ERR_INVALID_ARGUMENT: return "GNS_ERR_INVALID_ARGUMENT";
    case GNS_ERR_UNSUPPORTED_FRACTION: return "GNS_ERR_UNSUPPORTED_FRACTION";
    case GNS_ERR_OUT_OF_MEMORY: return "GNS_ERR_OUT_OF_MEMORY";
    case GNS_ERR_CUDA: return "GNS_ERR_CUDA";
    case GNS_ERR_WORKSPACE_TOO_SMALL: return "GNS_ERR_WORKSPACE_TOO_SMALL";
    case GNS_ERR_MISALIGNED: return "GNS_ERR_MISALIGNED";
    }
    return "GNS_ERR_UNKNOWN";
}

const char *gns_last_error_string(void) { return g_last_error.c_str(); }

}  // extern "C"
