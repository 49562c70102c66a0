// K1b: bucketing of a slab's records by (w plane, 32-column strip, anchor row).
//
// The reference gives every slab the records of exchange_to_space_order in
// (time_index, gindex) order (comms.py:534-545) and grids them tap-major
// (gridder.py:160-183). The sweep gridder (grid.cu) instead walks each
// 32-column strip of a plane down its rows, so it needs the strip's records
// sorted by anchor row floor(gv). Every (record, strip) pair becomes one
// entry with the dense key
//     key = (plane * n_tc + tc) * RS + (floor(gv) - v_start + S),
//     RS  = v_count + 2S (anchor rows that can touch the slab),
// written in record order (block-stable compaction), then sorted by a
// stable LSD radix sort (sort.cu). The final order is (key, record index):
// deterministic, independent of how skewed the buckets are (LOFAR-like
// tracks put millions of records into a few buckets), and -- the record
// index following gindex -- independent of the GPU count. Bucket offsets
// come from a key histogram.
#include "wsb_internal.cuh"

namespace wsb {
namespace {

constexpr int kThreads = 256;
constexpr int kBlockItems = 2048;  // records per block

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

// Number of strips (0, 1 or 2) a record reaches and its first key.
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

__device__ __forceinline__ uint32_t block_excl_sum(uint32_t x, uint32_t *total, uint32_t *smem) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) smem[warp] = incl;
    __syncthreads();
    uint32_t base = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < kThreads / 32; ++k) {
        const uint32_t s = smem[k];
        if (k < warp) base += s;
        tot += s;
    }
    __syncthreads();
    *total = tot;
    return base + incl - x;
}

// entries per block (for the compaction) and the key histogram
__global__ void __launch_bounds__(kThreads) k_keys_count(const double4 *__restrict__ rec,
                                                         const uint32_t *__restrict__ plane,
                                                         int64_t m, KeyGeom k,
                                                         uint32_t *__restrict__ block_cnt,
                                                         uint32_t *__restrict__ key_cnt) {
    __shared__ uint32_t c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    uint32_t local = 0;
    for (int it = 0; it < kBlockItems / kThreads; ++it) {
        const int64_t i = base + it * kThreads + threadIdx.x;
        if (i < m) {
            uint32_t key;
            const int n = record_keys(rec[i], plane[i], k, &key);
            for (int t = 0; t < n; ++t) atomicAdd(&key_cnt[key + t * k.rs], 1u);
            local += n;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&c, local);
    __syncthreads();
    if (threadIdx.x == 0) block_cnt[blockIdx.x] = c;
}

// (key, record) entries in record order
__global__ void __launch_bounds__(kThreads) k_keys_write(const double4 *__restrict__ rec,
                                                         const uint32_t *__restrict__ plane,
                                                         int64_t m, KeyGeom k,
                                                         const uint32_t *__restrict__ block_off,
                                                         uint32_t *__restrict__ keys,
                                                         uint32_t *__restrict__ idx) {
    __shared__ uint32_t wsum[kThreads / 32];
    uint32_t run = block_off[blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    for (int it = 0; it < kBlockItems / kThreads; ++it) {
        const int64_t i = base + it * kThreads + threadIdx.x;
        uint32_t key = 0;
        int n = 0;
        if (i < m) n = record_keys(rec[i], plane[i], k, &key);
        uint32_t tot;
        uint32_t pos = run + block_excl_sum((uint32_t)n, &tot, wsum);
        for (int t = 0; t < n; ++t) {
            keys[pos + t] = key + t * k.rs;
            idx[pos + t] = (uint32_t)i;
        }
        run += tot;
    }
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
    uint32_t *cnt, *off;
    WSB_TRY(ensure(ctx, kSlotTileCount, sizeof(uint32_t) * (n_keys + 1), (void **)&cnt));
    WSB_TRY(ensure(ctx, kSlotTileOff, sizeof(uint32_t) * (n_keys + 1), (void **)&off));
    WSB_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (n_keys + 1), ctx->stream));
    const int nb = std::max(1, ceil_div(m, kBlockItems));
    uint32_t *bcnt, *boff;
    WSB_TRY(ensure(ctx, kSlotBlockCounts, sizeof(uint32_t) * (nb + 1), (void **)&bcnt));
    WSB_TRY(ensure(ctx, kSlotBlockOffsets, sizeof(uint32_t) * (nb + 1), (void **)&boff));
    uint32_t total = 0;
    if (m > 0) {
        k_keys_count<<<nb, kThreads, 0, ctx->stream>>>((const double4 *)rec, plane, m, k, bcnt, cnt);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
        WSB_TRY(exclusive_scan_u32(ctx, bcnt, boff, nb, &total));
    }
    WSB_TRY(exclusive_scan_u32(ctx, cnt, off, n_keys + 1, nullptr));
    const size_t eb = sizeof(uint32_t) * std::max<int64_t>(1, total);
    uint32_t *ka, *kb, *ia, *ib;
    WSB_TRY(ensure(ctx, kSlotKeysA, eb, (void **)&ka));
    WSB_TRY(ensure(ctx, kSlotKeysB, eb, (void **)&kb));
    WSB_TRY(ensure(ctx, kSlotIdxA, eb, (void **)&ia));
    WSB_TRY(ensure(ctx, kSlotIdxB, eb, (void **)&ib));
    if (total > 0) {
        k_keys_write<<<nb, kThreads, 0, ctx->stream>>>((const double4 *)rec, plane, m, k, boff, ka, ia);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
    }
    uint32_t *ks, *is;
    WSB_TRY(radix_sort_pairs(ctx, ka, kb, ia, ib, total, ilog2(n_keys), &ks, &is));
    out->idx = is;
    out->off = off;
    out->n_entries = total;
    out->n_keys = n_keys;
    out->n_tc = k.n_tc;
    out->rs = k.rs;
    ctx->last_idx = is;
    ctx->last_off = off;
    ctx->last_entries = total;
    ctx->last_tiles = n_keys;
    return WSB_OK;
}

}  // namespace wsb
