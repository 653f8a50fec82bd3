// Microbenchmark (tools only, not product code): a random 8-byte gather
// out[i] = vals[idx[i]] over n = 2^24 elements with a random permutation idx,
// in several load flavours, against a plain sequential copy.  Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gather_bench tools/gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ uint64_t ld(const uint64_t *p)
{
    uint64_t v;
    if (MODE == 0) v = __ldg(p);
    else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else if (MODE == 2) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else if (MODE == 3) asm volatile("ld.global.nc.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(0ull));
    return v;
}

template <int MODE, int U>
__global__ void __launch_bounds__(256) gather(uint64_t *out, const uint64_t *vals, const uint32_t *idx, long long n)
{
    const long long nu = n / U;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < nu; g += stride) {
        uint32_t ix[U];
#pragma unroll
        for (int u = 0; u < U; u += 4) {
            const uint4 a = reinterpret_cast<const uint4 *>(idx)[(g * U + u) / 4];
            ix[u] = a.x; ix[u + 1] = a.y; ix[u + 2] = a.z; ix[u + 3] = a.w;
        }
        uint64_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld<MODE>(vals + ix[u]);
#pragma unroll
        for (int u = 0; u < U; u += 2)
            reinterpret_cast<ulonglong2 *>(out + g * U)[u / 2] = make_ulonglong2(v[u], v[u + 1]);
    }
}

__global__ void copyk(uint4 *o, const uint4 *i, long long n16)
{
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n16; g += (long long)gridDim.x * blockDim.x)
        o[g] = i[g];
}

template <class F>
float timeit(F f)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
    }
    return best;
}

int main()
{
    const long long n = 1LL << 24;
    std::vector<uint32_t> h(n);
    for (long long i = 0; i < n; ++i) h[i] = (uint32_t)i;
    std::mt19937_64 rng(7);
    std::shuffle(h.begin(), h.end(), rng);
    uint64_t *vals, *out;
    uint32_t *idx;
    cudaMalloc(&vals, n * 8);
    cudaMalloc(&out, n * 8);
    cudaMalloc(&idx, n * 4);
    cudaMemset(vals, 1, n * 8);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("copy 128 MB: %.1f us\n", 1e3 * timeit([&] { copyk<<<sms * 8, 256>>>((uint4 *)out, (const uint4 *)vals, n / 2); }));
    for (int bpsm : {4, 8, 16}) {
        const int g = sms * bpsm;
        printf("blocks/SM %d: ldg8 %.1f  nc_noalloc8 %.1f  cg8 %.1f  L2_64B8 %.1f  ldg16 %.1f  nc_noalloc16 %.1f us\n", bpsm,
               1e3 * timeit([&] { gather<0, 8><<<g, 256>>>(out, vals, idx, n); }),
               1e3 * timeit([&] { gather<1, 8><<<g, 256>>>(out, vals, idx, n); }),
               1e3 * timeit([&] { gather<2, 8><<<g, 256>>>(out, vals, idx, n); }),
               1e3 * timeit([&] { gather<3, 8><<<g, 256>>>(out, vals, idx, n); }),
               1e3 * timeit([&] { gather<0, 16><<<g, 256>>>(out, vals, idx, n); }),
               1e3 * timeit([&] { gather<1, 16><<<g, 256>>>(out, vals, idx, n); }));
    }
    // sorted index: the sequential-gather bound
    std::sort(h.begin(), h.end());
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    printf("identity idx ldg8: %.1f us\n", 1e3 * timeit([&] { gather<0, 8><<<sms * 8, 256>>>(out, vals, idx, n); }));
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
