// gns_peel.cuh — the natural-alignment path of the C-ABI (SURVEY.md §8(b):
// "Natural alignment is required ... other pointers take a slower correct
// path"): sorting applies to any contiguous sequence (PAPER.md:121,
// §Definition of sorting), e.g. a sliced tensor t[1:].
//
// The TMA / 256-bit kernels need 32-byte aligned arrays.  For keys that are
// 8-byte (vals 4-byte) aligned but not 32-byte aligned, the sort peels the
// h <= 7 head elements before the first 32-byte boundary:
//   1. the aligned middle [h, n) is sorted by the normal path (any buffer mode);
//   2. peel_head_kernel sorts the h head elements (stable insertion, one
//      thread) into a small scratch area;
//   3. peel_merge_kernel merges head (first: it wins ties) and
//      middle in place into [0, n): output k takes middle element
//      k - i(k) (i(k) <= h head elements before it) from position
//      h + k - i(k) in [k, k + h] -- a left shift by at most h.  Chunks of
//      4096 outputs, claimed in ticket order: each loads its inputs into
//      registers, publishes "read" (st.release), waits until the previous
//      chunk has read (its inputs reach up to h elements into our output
//      range), then writes.  Deadlock-free (a chunk only waits on a smaller
//      ticket that never waits on a larger one).  One extra read + write pass.
// With a single CTA (n small, no workspace) the chunks run in order inside the
// CTA and no flags are needed.
#pragma once

namespace gns {

constexpr int PEEL_MAX = 7;
constexpr int PEEL_NT = 256, PEEL_VT = 16, PEEL_CHUNK = PEEL_NT * PEEL_VT;   // 4096 outputs

template <bool HV, int ORD>
__device__ __forceinline__ int peel_sort_head(const double *k, const uint32_t *v, int h, double *hk, uint32_t *hv)
{
    // stable insertion sort (shift while the previous key is strictly after)
    for (int i = 0; i < h; ++i) {
        const double x = k[i];
        const uint32_t y = HV ? v[i] : 0u;
        int j = i;
        while (j > 0 && before<ORD>(x, hk[j - 1])) {
            hk[j] = hk[j - 1];
            if (HV) hv[j] = hv[j - 1];
            --j;
        }
        hk[j] = x;
        if (HV) hv[j] = y;
    }
    return h;
}

template <bool HV, int ORD>
__global__ void peel_head_kernel(const double *keys, const uint32_t *vals, int h, double *hk, uint32_t *hv)
{
    pdl_wait();
    if (threadIdx.x == 0 && blockIdx.x == 0) peel_sort_head<HV, ORD>(keys, vals, h, hk, hv);
    pdl_trigger();
}

// flags == nullptr: single CTA (grid 1), the head is sorted by the kernel itself
template <bool HV, int ORD>
__global__ void __launch_bounds__(PEEL_NT)
peel_merge_kernel(double *keys, uint32_t *vals, long long n, int h, const double *hk_g, const uint32_t *hv_g,
                  unsigned *flags, unsigned *ticket)
{
    pdl_wait();
    __shared__ double hk[PEEL_MAX + 1];
    __shared__ uint32_t hvs[PEEL_MAX + 1];
    __shared__ int s_chunk;
    const int tid = threadIdx.x;
    if (tid == 0) {
        if (flags == nullptr) {
            peel_sort_head<HV, ORD>(keys, vals, h, hk, hvs);
        } else {
            for (int i = 0; i < h; ++i) {
                hk[i] = hk_g[i];
                if (HV) hvs[i] = hv_g[i];
            }
        }
    }
    __syncthreads();
    const double *M = keys + h;             // the sorted middle, m keys
    const uint32_t *MV = HV ? vals + h : nullptr;
    const long long m = n - h;
    const long long nchunks = (n + PEEL_CHUNK - 1) / PEEL_CHUNK;
    for (long long it = 0;; ++it) {
        long long b;
        if (flags == nullptr) {
            b = it;
        } else {
            if (tid == 0) s_chunk = (int)atomicAdd(ticket, 1u);
            __syncthreads();
            b = s_chunk;
            __syncthreads();
        }
        if (b >= nchunks) break;
        const long long k0 = b * PEEL_CHUNK + (long long)tid * PEEL_VT;
        double ok[PEEL_VT];
        uint32_t ov[PEEL_VT];
        int cnt = 0;
        if (k0 < n) {
            cnt = (int)min((long long)PEEL_VT, n - k0);
            // co-rank: head elements among the first k0 outputs (head first, wins ties)
            int lo = (int)max(0LL, k0 - m), hi = (int)min(k0, (long long)h);
            while (lo < hi) {
                const int x = (lo + hi) >> 1;
                if (!before<ORD>(M[k0 - 1 - x], hk[x])) lo = x + 1;
                else hi = x;
            }
            int i = lo;
            long long j = k0 - i;
            for (int x = 0; x < PEEL_VT; ++x) {
                if (x < cnt) {
                    const bool tb = (j < m) && (i >= h || before<ORD>(M[j], hk[i]));
                    if (tb) {
                        ok[x] = M[j];
                        if (HV) ov[x] = MV[j];
                        ++j;
                    } else {
                        ok[x] = hk[i];
                        if (HV) ov[x] = hvs[i];
                        ++i;
                    }
                }
            }
        }
        __syncthreads();                                   // the whole chunk's inputs are read
        if (flags != nullptr) {
            if (tid == 0) {
                __threadfence();
                st_release(flags + b, 1u);
                if (b > 0)
                    while (ld_acquire(flags + b - 1) == 0u) __nanosleep(32);
            }
            __syncthreads();
        }
        for (int x = 0; x < cnt; ++x) {
            keys[k0 + x] = ok[x];
            if (HV) vals[k0 + x] = ov[x];
        }
        __syncthreads();                                   // (single CTA: next chunk reads after these writes)
    }
    pdl_trigger();
}

}  // namespace gns
