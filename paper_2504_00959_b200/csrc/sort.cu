// Exclusive scan and stable LSD radix sort (8-bit digits) for the K1
// bucketing stage. Stability is what makes the per-cell accumulation order
// of the gridder the global record order (gindex), independent of the GPU
// count -- the property gridder.py:262-269 guarantees for the reference.
#include "wsb_internal.cuh"

namespace wsb {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;                        // per thread
constexpr int kScanTile = kScanThreads * kScanItems; // 4096

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Block-wide exclusive scan of one value per thread (blockDim.x == 1024).
__device__ uint32_t block_excl_scan(uint32_t x, uint32_t *total) {
    __shared__ uint32_t warp_sums[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = warp_incl_scan(x);
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = warp_sums[lane];
        uint32_t si = warp_incl_scan(s);
        warp_sums[lane] = si - s;
        if (lane == 31 && total) *total = si;
    }
    __syncthreads();
    uint32_t r = warp_sums[warp] + incl - x;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t *__restrict__ in,
                                                              int64_t n, uint32_t *sums) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) s += in[base + i];
    __shared__ uint32_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_sums(uint32_t *sums, int nb,
                                                            uint32_t *total) {
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += kScanThreads) {
        int i = base + threadIdx.x;
        uint32_t x = i < nb ? sums[i] : 0;
        __shared__ uint32_t tot;
        uint32_t ex = block_excl_scan(x, &tot);
        uint32_t c = carry;
        if (i < nb) sums[i] = c + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry = c + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_final(const uint32_t *__restrict__ in,
                                                             uint32_t *out, int64_t n,
                                                             const uint32_t *sums) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    uint32_t ex = block_excl_scan(s, nullptr) + sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = ex;
        ex += v[i];
    }
}

// ---------------------------------------------------------------------------
// radix sort
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsIpt = 16;                      // rounds of 32 per warp
constexpr int kRsItems = kRsThreads * kRsIpt;   // 4096 per block
constexpr int kRsPerWarp = 32 * kRsIpt;         // 512

__global__ void __launch_bounds__(kRsThreads) k_radix_hist(const uint32_t *__restrict__ keys,
                                                           int64_t n, int shift,
                                                           uint32_t *hist, int nb) {
    // one sub-histogram per warp (shared-memory atomics, little contention),
    // all loads of a thread issued up front
    __shared__ uint32_t h[kRsWarps][256];
    const int warp = threadIdx.x >> 5;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) h[w][threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRsItems;
    uint32_t d[kRsIpt];
#pragma unroll
    for (int r = 0; r < kRsIpt; ++r) {
        const int64_t i = base + (int64_t)r * kRsThreads + threadIdx.x;
        d[r] = i < n ? (__ldg(&keys[i]) >> shift) & 255u : 256u;
    }
#pragma unroll
    for (int r = 0; r < kRsIpt; ++r)
        if (d[r] < 256u) atomicAdd(&h[warp][d[r]], 1u);
    __syncthreads();
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) s += h[w][threadIdx.x];
    hist[(int64_t)threadIdx.x * nb + blockIdx.x] = s;
}

__global__ void __launch_bounds__(kRsThreads) k_radix_scatter(
    const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint32_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, int shift, const uint32_t *__restrict__ offs, int nb) {
    __shared__ uint32_t wc[kRsWarps][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < 8; ++i) wc[warp][lane + 32 * i] = 0;
    __syncwarp();
    const int64_t base = (int64_t)blockIdx.x * kRsItems + warp * kRsPerWarp;
    uint32_t k[kRsIpt], v[kRsIpt], pm[kRsIpt];
#pragma unroll
    for (int r = 0; r < kRsIpt; ++r) {
        int64_t i = base + r * 32 + lane;
        bool ok = i < n;
        k[r] = ok ? kin[i] : 0u;
        v[r] = ok ? vin[i] : 0u;
    }
#pragma unroll
    for (int r = 0; r < kRsIpt; ++r) {
        const bool ok = base + r * 32 + lane < n;
        const uint32_t d = ok ? (k[r] >> shift) & 255u : 256u;
        pm[r] = __match_any_sync(0xffffffffu, d);
        if (d < 256u && lane == __ffs(pm[r]) - 1) wc[warp][d] += __popc(pm[r]);
        __syncwarp();
    }
    __syncthreads();
    // block-local start of each digit run (exclusive scan over the 256
    // digits of the block totals) and the start of each warp inside it
    __shared__ uint32_t bstart[256], goff[256], wsum[kRsWarps];
    {
        const int d = threadIdx.x;  // 256 threads == 256 digits
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) {
            const uint32_t c = wc[w][d];
            wc[w][d] = tot;
            tot += c;
        }
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        uint32_t wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += wsum[w];
        bstart[d] = wbase + incl - tot;
        goff[d] = offs[(int64_t)d * nb + blockIdx.x];
    }
    __syncthreads();
    // stable rank inside the block -> shared-memory staging in digit order
    __shared__ uint32_t ks[kRsItems], vs[kRsItems];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < kRsIpt; ++r) {
        int64_t i = base + r * 32 + lane;
        bool ok = i < n;
        uint32_t d = ok ? (k[r] >> shift) & 255u : 256u;
        const uint32_t peers = pm[r];
        uint32_t pos = 0;
        if (ok) pos = bstart[d] + wc[warp][d] + __popc(peers & lt);
        __syncwarp();
        if (ok && lane == __ffs(peers) - 1) wc[warp][d] += __popc(peers);
        __syncwarp();
        if (ok) {
            ks[pos] = k[r];
            vs[pos] = v[r];
        }
    }
    __syncthreads();
    // consecutive threads write consecutive positions of each digit run
    const int64_t nblk = min((int64_t)kRsItems, n - (int64_t)blockIdx.x * kRsItems);
    for (int p = threadIdx.x; p < nblk; p += kRsThreads) {
        const uint32_t key = ks[p];
        const uint32_t d = (key >> shift) & 255u;
        const uint32_t gpos = goff[d] + (p - bstart[d]);
        kout[gpos] = key;
        vout[gpos] = vs[p];
    }
}

}  // namespace

int exclusive_scan_u32(wsb_ctx *ctx, const uint32_t *in, uint32_t *out, int64_t n,
                       uint32_t *total_host) {
    if (n <= 0) {
        if (total_host) *total_host = 0;
        return WSB_OK;
    }
    const int nb = ceil_div(n, kScanTile);
    uint32_t *sums;
    WSB_TRY(ensure(ctx, kSlotScanTmp, sizeof(uint32_t) * (nb + 1), (void **)&sums));
    k_scan_reduce<<<nb, kScanThreads, 0, ctx->stream>>>(in, n, sums);
    k_scan_sums<<<1, kScanThreads, 0, ctx->stream>>>(sums, nb, sums + nb);
    k_scan_final<<<nb, kScanThreads, 0, ctx->stream>>>(in, out, n, sums);
    ctx->launches += 3;
    WSB_CUDA_TRY(cudaGetLastError());
    if (total_host) {
        WSB_CUDA_TRY(cudaMemcpyAsync(ctx->flag_host, sums + nb, sizeof(uint32_t),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        *total_host = (uint32_t)ctx->flag_host[0];
    }
    return WSB_OK;
}

int radix_sort_pairs(wsb_ctx *ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                     uint32_t *vals_alt, int64_t n, int bits, uint32_t **keys_out,
                     uint32_t **vals_out) {
    *keys_out = keys;
    *vals_out = vals;
    if (n <= 1 || bits <= 0) return WSB_OK;
    const int nb = ceil_div(n, kRsItems);
    uint32_t *hist;
    WSB_TRY(ensure(ctx, kSlotRadixHist, sizeof(uint32_t) * 256 * (size_t)nb, (void **)&hist));
    uint32_t *ka = keys, *kb = keys_alt, *va = vals, *vb = vals_alt;
    for (int shift = 0; shift < bits; shift += 8) {
        k_radix_hist<<<nb, kRsThreads, 0, ctx->stream>>>(ka, n, shift, hist, nb);
        ctx->launches += 1;
        WSB_TRY(exclusive_scan_u32(ctx, hist, hist, (int64_t)256 * nb, nullptr));
        k_radix_scatter<<<nb, kRsThreads, 0, ctx->stream>>>(ka, va, kb, vb, n, shift, hist, nb);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
        uint32_t *t = ka; ka = kb; kb = t;
        t = va; va = vb; vb = t;
    }
    *keys_out = ka;
    *vals_out = va;
    return WSB_OK;
}

}  // namespace wsb
