// K1b: bucketing of a slab's records by (w plane, 32-column tile, anchor row).
//
// The reference gives every slab the records of exchange_to_space_order in
// (time_index, gindex) order (comms.py:534-545) and grids them tap-major
// (gridder.py:160-183). The sweep gridder (grid.cu) instead walks each
// 32-column strip of a plane down its rows, so it needs the strip's records
// sorted by anchor row floor(gv). This file builds that order with a
// counting sort over the dense key
//     key = (plane * n_tc + tc) * RS + (floor(gv) - v_start + S),
//     RS  = v_count + 2S (anchor rows that can touch the slab),
// a record being listed once per tile column its footprint reaches.
// Slots are claimed with atomics, then every bucket is sorted by record
// index, so the final order is (key, record index): deterministic and, since
// the record index follows gindex, independent of the GPU count.
#include "wsb_internal.cuh"

namespace wsb {
namespace {

constexpr int kThreads = 256;
constexpr int kSmallBucket = 32;     // insertion-sorted by one thread
constexpr int kMidBucket = 8192;     // bitonic-sorted in shared memory by one CTA

struct KeyGeom {
    int n_u, v_start, v_count, S, n_tc, rs;
};

// Inclusive tap range of one axis: {i : |g - i| <= S} (gridder.py:171,177),
// clipped to [lo, hi]. For in-range taps g - i is exact, so the rounded
// test below is the reference's test. Returns false if empty.
__device__ __forceinline__ bool tap_range(double g, int S, int lo, int hi, int *a, int *b) {
    const double fl = floor(g);
    int i0 = (int)fl - S;
    if (__dsub_rn(g, (double)i0) > (double)S) ++i0;
    int i1 = (int)fl + S;
    *a = max(i0, lo);
    *b = min(i1, hi);
    return *a <= *b;
}

// Returns the number of tile columns (0, 1 or 2) and the first key.
__device__ __forceinline__ int record_keys(const double4 &r, uint32_t plane, const KeyGeom &k,
                                           uint32_t *key0) {
    int i0, i1, j0, j1;
    if (!tap_range(r.x, k.S, 0, k.n_u - 1, &i0, &i1)) return 0;
    if (!tap_range(r.y, k.S, k.v_start, k.v_start + k.v_count - 1, &j0, &j1)) return 0;
    const int rel = (int)floor(r.y) - k.v_start + k.S;
    if (rel < 0 || rel >= k.rs) return 0;
    const int tc0 = i0 >> 5, tc1 = i1 >> 5;
    *key0 = ((uint32_t)plane * k.n_tc + tc0) * (uint32_t)k.rs + rel;
    return tc1 - tc0 + 1;
}

__global__ void __launch_bounds__(kThreads) k_bkt_count(const double4 *__restrict__ rec,
                                                        const uint32_t *__restrict__ plane,
                                                        int64_t m, KeyGeom k,
                                                        uint32_t *__restrict__ cnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t key;
        const int n = record_keys(rec[i], plane[i], k, &key);
        for (int t = 0; t < n; ++t) atomicAdd(&cnt[key + t * k.rs], 1u);
    }
}

__global__ void __launch_bounds__(kThreads) k_bkt_scatter(const double4 *__restrict__ rec,
                                                          const uint32_t *__restrict__ plane,
                                                          int64_t m, KeyGeom k,
                                                          const uint32_t *__restrict__ off,
                                                          uint32_t *__restrict__ fill,
                                                          uint32_t *__restrict__ idx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t key;
        const int n = record_keys(rec[i], plane[i], k, &key);
        for (int t = 0; t < n; ++t) {
            const uint32_t kk = key + t * k.rs;
            idx[off[kk] + atomicAdd(&fill[kk], 1u)] = (uint32_t)i;
        }
    }
}

// Small buckets: insertion sort by one thread. Larger ones are listed.
__global__ void __launch_bounds__(kThreads) k_bkt_fix(const uint32_t *__restrict__ off,
                                                      int64_t n_keys, uint32_t *__restrict__ idx,
                                                      uint32_t *__restrict__ big,
                                                      uint32_t *__restrict__ n_big) {
    const int64_t key = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (key >= n_keys) return;
    const uint32_t b = off[key], e = off[key + 1], n = e - b;
    if (n < 2) return;
    if (n > kSmallBucket) {
        big[atomicAdd(n_big, 1u)] = (uint32_t)key;
        return;
    }
    uint32_t *p = idx + b;
    for (uint32_t i = 1; i < n; ++i) {
        const uint32_t x = p[i];
        uint32_t j = i;
        while (j > 0 && p[j - 1] > x) {
            p[j] = p[j - 1];
            --j;
        }
        p[j] = x;
    }
}

// Mid buckets (<= kMidBucket): bitonic sort in shared memory, one CTA each.
__global__ void __launch_bounds__(1024) k_bkt_fix_mid(const uint32_t *__restrict__ off,
                                                      const uint32_t *__restrict__ big,
                                                      uint32_t *__restrict__ idx) {
    __shared__ uint32_t s[kMidBucket];
    const uint32_t key = big[blockIdx.x];
    const uint32_t b = off[key], n = off[key + 1] - b;
    if (n > kMidBucket) return;  // handled on the host path
    uint32_t p2 = 1;
    while (p2 < n) p2 <<= 1;
    for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) s[i] = i < n ? idx[b + i] : 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t size = 2; size <= p2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < p2; i += blockDim.x) {
                const uint32_t j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const uint32_t a = s[i], c = s[j];
                    if ((a > c) == up) {
                        s[i] = c;
                        s[j] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) idx[b + i] = s[i];
}

}  // namespace

int bucket_rows(wsb_ctx *ctx, const wsb_grid *g, int S, int v_start, int v_count,
                const double *rec, const uint32_t *plane, int64_t m, RowBuckets *out) {
    KeyGeom k;
    k.n_u = g->n_u;
    k.v_start = v_start;
    k.v_count = v_count;
    k.S = S;
    k.n_tc = ceil_div(g->n_u, 32);
    k.rs = v_count + 2 * S;
    const int64_t n_keys = (int64_t)g->n_w * k.n_tc * k.rs;
    if (n_keys >= 0xFFFFFFFFll) return fail(WSB_EUNSUPPORTED, "bucket key space exceeds 32 bits");
    uint32_t *cnt, *off, *fill, *idx, *big;
    WSB_TRY(ensure(ctx, kSlotTileCount, sizeof(uint32_t) * (n_keys + 1), (void **)&cnt));
    WSB_TRY(ensure(ctx, kSlotTileOff, sizeof(uint32_t) * (n_keys + 1), (void **)&off));
    WSB_TRY(ensure(ctx, kSlotKeysA, sizeof(uint32_t) * (n_keys + 1), (void **)&fill));
    WSB_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (n_keys + 1), ctx->stream));
    WSB_CUDA_TRY(cudaMemsetAsync(fill, 0, sizeof(uint32_t) * (n_keys + 1), ctx->stream));
    const int grid = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(m, kThreads)), 148 * 16);
    if (m > 0) {
        k_bkt_count<<<grid, kThreads, 0, ctx->stream>>>((const double4 *)rec, plane, m, k, cnt);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
    }
    uint32_t total = 0;
    WSB_TRY(exclusive_scan_u32(ctx, cnt, off, n_keys + 1, &total));
    const int64_t ne = std::max<uint32_t>(total, 1);
    WSB_TRY(ensure(ctx, kSlotIdxA, sizeof(uint32_t) * ne, (void **)&idx));
    WSB_TRY(ensure(ctx, kSlotIdxB, sizeof(uint32_t) * (ne / (kSmallBucket + 1) + 2), (void **)&big));
    uint32_t *n_big;
    WSB_TRY(ensure(ctx, kSlotU64, 64, (void **)&n_big));
    n_big += 2;  // bytes 8..11 of the u64 slot (0..7 hold the update counter)
    WSB_CUDA_TRY(cudaMemsetAsync(n_big, 0, sizeof(uint32_t), ctx->stream));
    if (total > 0) {
        k_bkt_scatter<<<grid, kThreads, 0, ctx->stream>>>((const double4 *)rec, plane, m, k, off,
                                                          fill, idx);
        k_bkt_fix<<<ceil_div(n_keys, kThreads), kThreads, 0, ctx->stream>>>(off, n_keys, idx, big,
                                                                           n_big);
        ctx->launches += 2;
        WSB_CUDA_TRY(cudaGetLastError());
        uint32_t nb = 0;
        WSB_CUDA_TRY(cudaMemcpyAsync(ctx->flag_host, n_big, 4, cudaMemcpyDeviceToHost, ctx->stream));
        WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        nb = (uint32_t)ctx->flag_host[0];
        if (nb > 0) {
            k_bkt_fix_mid<<<nb, 1024, 0, ctx->stream>>>(off, big, idx);
            ctx->launches += 1;
            WSB_CUDA_TRY(cudaGetLastError());
            // buckets beyond kMidBucket: stable radix sort of the segment by record index
            std::vector<uint32_t> keys(nb);
            WSB_CUDA_TRY(cudaMemcpyAsync(keys.data(), big, 4 * nb, cudaMemcpyDeviceToHost, ctx->stream));
            WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
            for (uint32_t kk : keys) {
                uint32_t be[2];
                WSB_CUDA_TRY(cudaMemcpy(be, off + kk, 8, cudaMemcpyDeviceToHost));
                const uint32_t n = be[1] - be[0];
                if (n <= (uint32_t)kMidBucket) continue;
                uint32_t *ka, *kb, *va, *vb, *ko, *vo;
                WSB_TRY(ensure(ctx, kSlotKeysB, 4 * (size_t)n, (void **)&ka));
                WSB_TRY(ensure(ctx, kSlotRadixTmpA, 4 * (size_t)n, (void **)&kb));
                WSB_TRY(ensure(ctx, kSlotRadixTmpB, 4 * (size_t)n, (void **)&va));
                WSB_TRY(ensure(ctx, kSlotRadixTmpC, 4 * (size_t)n, (void **)&vb));
                WSB_CUDA_TRY(cudaMemcpyAsync(ka, idx + be[0], 4 * (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
                WSB_CUDA_TRY(cudaMemcpyAsync(va, idx + be[0], 4 * (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
                WSB_TRY(radix_sort_pairs(ctx, ka, kb, va, vb, n, 32, &ko, &vo));
                WSB_CUDA_TRY(cudaMemcpyAsync(idx + be[0], ko, 4 * (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
            }
        }
    }
    out->idx = idx;
    out->off = off;
    out->n_entries = total;
    out->n_keys = n_keys;
    out->n_tc = k.n_tc;
    out->rs = k.rs;
    ctx->last_idx = idx;
    ctx->last_off = off;
    ctx->last_entries = total;
    ctx->last_tiles = n_keys;
    return WSB_OK;
}

}  // namespace wsb
