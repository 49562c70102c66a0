// K1: record preparation, exchange routing and (plane, tile) bucketing.
//
//  k_prepare       prepare_chunk (comms.py:477-492) + VisChunk.validate
//                  (visdata.py:178-184), bit-exact FP64 arithmetic.
//  k_route_*       destination slabs of exchange_to_space_order
//                  (comms.py:516-523), packed in record (gindex) order.
//  k_bucket_*      (record, 64x64 tile) entries in record order, then a
//                  stable radix sort by tile key (sort.cu) and tile offsets.
#include "wsb_internal.cuh"

namespace wsb {
namespace {

constexpr int kThreads = 256;
constexpr int kBlockItems = 2048;  // records per block in the count/pack kernels

enum : int { kErrUV = 1, kErrW = 2, kErrWeight = 4 };

// complex128(vis) * float32 weight with NumPy's full complex multiply
// (ar*br - ai*bi, ar*bi + ai*br), bi = 0: keeps the sign of zero bit-exact.
__device__ __forceinline__ double2 vis_times_weight(float2 a, float wt) {
    const double ar = a.x, ai = a.y, br = wt;
    return make_double2(__dsub_rn(__dmul_rn(ar, br), __dmul_rn(ai, 0.0)),
                        __dadd_rn(__dmul_rn(ar, 0.0), __dmul_rn(ai, br)));
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// NumPy's pairwise complex summation (numpy/_core/src/umath/loops_utils.h,
// CDOUBLE_pairwise_sum) over products p[0..m): the order of
// (vis * weight).sum(axis=1) in comms.py:491.
__device__ double2 pairwise_sum(const float2 *vis, const float *wt, int m) {
    if (m < 4) {
        double2 t = make_double2(-0.0, -0.0);
        for (int i = 0; i < m; ++i) t = cadd(t, vis_times_weight(vis[i], wt[i]));
        return t;
    }
    if (m <= 64) {
        double2 r0 = vis_times_weight(vis[0], wt[0]);
        double2 r1 = vis_times_weight(vis[1], wt[1]);
        double2 r2 = vis_times_weight(vis[2], wt[2]);
        double2 r3 = vis_times_weight(vis[3], wt[3]);
        int i = 4;
        const int lim = m - (m % 4);
        for (; i < lim; i += 4) {
            r0 = cadd(r0, vis_times_weight(vis[i + 0], wt[i + 0]));
            r1 = cadd(r1, vis_times_weight(vis[i + 1], wt[i + 1]));
            r2 = cadd(r2, vis_times_weight(vis[i + 2], wt[i + 2]));
            r3 = cadd(r3, vis_times_weight(vis[i + 3], wt[i + 3]));
        }
        double2 t = cadd(cadd(r0, r1), cadd(r2, r3));
        for (; i < m; ++i) t = cadd(t, vis_times_weight(vis[i], wt[i]));
        return t;
    }
    const int n2 = (m - (m % 8)) / 2;
    return cadd(pairwise_sum(vis, wt, n2), pairwise_sum(vis + n2, wt + n2, m - n2));
}

__global__ void __launch_bounds__(kThreads) k_prepare(
    const double *__restrict__ u, const double *__restrict__ v, const double *__restrict__ w,
    const float2 *__restrict__ vis, const float *__restrict__ wt, int64_t n, int n_chan,
    double n_u, double n_v, int n_w, double4 *__restrict__ rec, uint32_t *__restrict__ plane,
    int *err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double uu = u[i], vv = v[i], ww = w[i];
    int e = 0;
    // validate(): u,v in [0,1), w in [0,1]; NaN coordinates are rejected too.
    if (!(uu >= 0.0 && uu < 1.0 && vv >= 0.0 && vv < 1.0)) e |= kErrUV;
    if (!(ww >= 0.0 && ww <= 1.0)) e |= kErrW;
    double2 val;
    if (n_chan == 1) {
        const float wv = wt[i];
        if (!isfinite(wv) || wv < 0.0f) e |= kErrWeight;
        // reduce identity 0.0 + pairwise(-0.0 + p0)
        val = cadd(make_double2(0.0, 0.0), cadd(make_double2(-0.0, -0.0),
                                                vis_times_weight(vis[i], wv)));
    } else {
        const float2 *vr = vis + i * n_chan;
        const float *wr = wt + i * n_chan;
        for (int c = 0; c < n_chan; ++c)
            if (!isfinite(wr[c]) || wr[c] < 0.0f) e |= kErrWeight;
        val = cadd(make_double2(0.0, 0.0), pairwise_sum(vr, wr, n_chan));
    }
    if (e) atomicOr(err, e);
    uint32_t p = 0;
    if (n_w > 1) {
        // floor(w*(n_w-1) + 0.5), two rounded FP64 ops, then clip
        double k = floor(__dadd_rn(__dmul_rn(ww, (double)(n_w - 1)), 0.5));
        k = fmin(fmax(k, 0.0), (double)(n_w - 1));
        p = (uint32_t)(k == k ? k : 0.0);
    }
    rec[i] = make_double4(__dmul_rn(uu, n_u), __dmul_rn(vv, n_v), val.x, val.y);
    plane[i] = p;
}

// ---------------------------------------------------------------------------
// block-level stable compaction helper (256 threads)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t block_excl_sum256(uint32_t x, uint32_t *total,
                                                      uint32_t *smem /*[8]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) smem[warp] = incl;
    __syncthreads();
    uint32_t base = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < kThreads / 32; ++k) {
        uint32_t s = smem[k];
        if (k < warp) base += s;
        tot += s;
    }
    __syncthreads();
    *total = tot;
    return base + incl - x;
}

// ---------------------------------------------------------------------------
// exchange routing
// ---------------------------------------------------------------------------
struct Slabs {
    int start[8];
    int count[8];
};

__device__ __forceinline__ uint32_t dest_mask(double gv, double S, const Slabs &sl, int R) {
    uint32_t m = 0;
    for (int d = 0; d < R; ++d) {
        // comms.py:521-523, rounded FP64 adds
        bool in = (__dadd_rn(gv, S) >= (double)sl.start[d]) &&
                  (__dsub_rn(gv, S) <= (double)(sl.start[d] + sl.count[d] - 1));
        m |= (uint32_t)in << d;
    }
    return m;
}

__global__ void __launch_bounds__(kThreads) k_route_count(const double4 *__restrict__ rec,
                                                          int64_t n, double S, Slabs sl, int R,
                                                          uint32_t *counts /*[R][nb]*/, int nb) {
    __shared__ uint32_t c[8];
    if (threadIdx.x < 8) c[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    uint32_t local[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < kBlockItems / kThreads; ++it) {
        int64_t i = base + it * kThreads + threadIdx.x;
        if (i < n) {
            uint32_t m = dest_mask(rec[i].y, S, sl, R);
            for (int d = 0; d < R; ++d) local[d] += (m >> d) & 1u;
        }
    }
    for (int d = 0; d < R; ++d) {
        uint32_t x = local[d];
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(&c[d], x);
    }
    __syncthreads();
    if (threadIdx.x < R) counts[(int64_t)threadIdx.x * nb + blockIdx.x] = c[threadIdx.x];
}

__global__ void __launch_bounds__(kThreads) k_route_pack(
    const double4 *__restrict__ rec, const uint32_t *__restrict__ plane, int64_t n, double S,
    Slabs sl, int R, const uint32_t *__restrict__ offs /*[R][nb] exclusive*/, int nb,
    double4 *__restrict__ send_rec, uint32_t *__restrict__ send_plane, int64_t *src_index) {
    __shared__ uint32_t wsum[8];
    __shared__ uint32_t run[8];
    if (threadIdx.x < 8) run[threadIdx.x] = threadIdx.x < R ? offs[(int64_t)threadIdx.x * nb + blockIdx.x] : 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    for (int it = 0; it < kBlockItems / kThreads; ++it) {
        int64_t i = base + it * kThreads + threadIdx.x;
        double4 r = make_double4(0, 0, 0, 0);
        uint32_t p = 0, m = 0;
        if (i < n) {
            r = rec[i];
            p = plane[i];
            m = dest_mask(r.y, S, sl, R);
        }
        for (int d = 0; d < R; ++d) {
            uint32_t tot;
            uint32_t f = (m >> d) & 1u;
            uint32_t ex = block_excl_sum256(f, &tot, wsum);
            if (f) {
                uint32_t pos = run[d] + ex;
                send_rec[pos] = r;
                send_plane[pos] = p;
                if (src_index) src_index[pos] = i;
            }
            __syncthreads();
            if (threadIdx.x == 0) run[d] += tot;
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// tile bucketing
// ---------------------------------------------------------------------------
struct TileGeom {
    int n_u, v_start, v_count, S, n_tu, n_tv;
};

// Inclusive tap range of one axis: {i : |g - i| <= S} (gridder.py:171,177),
// clipped to [lo, hi]. Returns false if empty.
__device__ __forceinline__ bool tap_range(double g, int S, int lo, int hi, int *a, int *b) {
    const double fl = floor(g);
    int i0 = (int)fl - S;
    if (__dsub_rn(g, (double)i0) > (double)S) ++i0;
    int i1 = (int)fl + S;
    i0 = max(i0, lo);
    i1 = min(i1, hi);
    *a = i0;
    *b = i1;
    return i0 <= i1;
}

__device__ __forceinline__ int record_tiles(const double4 &r, const TileGeom &t, int *tu0,
                                            int *tu1, int *tv0, int *tv1) {
    int i0, i1, j0, j1;
    if (!tap_range(r.x, t.S, 0, t.n_u - 1, &i0, &i1)) return 0;
    if (!tap_range(r.y, t.S, t.v_start, t.v_start + t.v_count - 1, &j0, &j1)) return 0;
    *tu0 = i0 / kTile;
    *tu1 = i1 / kTile;
    *tv0 = (j0 - t.v_start) / kTile;
    *tv1 = (j1 - t.v_start) / kTile;
    return (*tu1 - *tu0 + 1) * (*tv1 - *tv0 + 1);
}

__global__ void __launch_bounds__(kThreads) k_bucket_count(const double4 *__restrict__ rec,
                                                           int64_t m, TileGeom t,
                                                           uint32_t *counts) {
    __shared__ uint32_t c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    uint32_t local = 0;
    for (int it = 0; it < kBlockItems / kThreads; ++it) {
        int64_t i = base + it * kThreads + threadIdx.x;
        if (i < m) {
            int a, b, cc, d;
            local += record_tiles(rec[i], t, &a, &b, &cc, &d);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&c, local);
    __syncthreads();
    if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

__global__ void __launch_bounds__(kThreads) k_bucket_write(
    const double4 *__restrict__ rec, const uint32_t *__restrict__ plane, int64_t m, TileGeom t,
    const uint32_t *__restrict__ offs, uint32_t *__restrict__ keys, uint32_t *__restrict__ idx,
    uint32_t *__restrict__ tile_count) {
    __shared__ uint32_t wsum[8];
    uint32_t run = offs[blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    for (int it = 0; it < kBlockItems / kThreads; ++it) {
        int64_t i = base + it * kThreads + threadIdx.x;
        int tu0 = 0, tu1 = -1, tv0 = 0, tv1 = -1, cnt = 0;
        uint32_t p = 0;
        if (i < m) {
            cnt = record_tiles(rec[i], t, &tu0, &tu1, &tv0, &tv1);
            p = plane[i];
        }
        uint32_t tot;
        uint32_t pos = run + block_excl_sum256((uint32_t)cnt, &tot, wsum);
        if (cnt) {
            for (int tv = tv0; tv <= tv1; ++tv)
                for (int tu = tu0; tu <= tu1; ++tu) {
                    uint32_t key = ((uint32_t)p * t.n_tv + tv) * t.n_tu + tu;
                    keys[pos] = key;
                    idx[pos] = (uint32_t)i;
                    ++pos;
                    atomicAdd(&tile_count[key], 1u);
                }
        }
        run += tot;
    }
}

}  // namespace

int prepare(wsb_ctx *ctx, const wsb_grid *g, const double *u, const double *v, const double *w,
            const float *vis, const float *weight, int64_t n, int32_t n_chan, double *rec,
            uint32_t *plane) {
    if (n <= 0) return WSB_OK;
    int *err;
    WSB_TRY(ensure(ctx, kSlotFlag, 64, (void **)&err));
    WSB_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
    k_prepare<<<ceil_div(n, kThreads), kThreads, 0, ctx->stream>>>(
        u, v, w, (const float2 *)vis, weight, n, n_chan, (double)g->n_u, (double)g->n_v, g->n_w,
        (double4 *)rec, plane, err);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    WSB_CUDA_TRY(cudaMemcpyAsync(ctx->flag_host, err, sizeof(int), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    const int e = ctx->flag_host[0];
    if (e & kErrUV) return fail(WSB_EINVAL, "u and v must lie in [0, 1)");
    if (e & kErrW) return fail(WSB_EINVAL, "w must lie in [0, 1]");
    if (e & kErrWeight) return fail(WSB_EINVAL, "weights must be finite and >= 0");
    return WSB_OK;
}

static int make_slabs(int n_v, int R, Slabs *sl) {
    if (R < 1 || R > 8) return fail(WSB_EINVAL, "n_ranks must be in [1, 8]");
    if (R > n_v) return fail(WSB_EINVAL, "n_ranks exceeds n_v");
    const int q = n_v / R, r = n_v % R;  // partition_1d (mesh.py:34-45)
    for (int d = 0; d < R; ++d) {
        sl->start[d] = d < r ? d * (q + 1) : r * (q + 1) + (d - r) * q;
        sl->count[d] = d < r ? q + 1 : q;
    }
    return WSB_OK;
}

int route_count(wsb_ctx *ctx, const wsb_grid *g, int S, int R, const double *rec, int64_t n,
                int64_t *counts_host, uint32_t **offs_out, int *nb_out) {
    Slabs sl;
    WSB_TRY(make_slabs(g->n_v, R, &sl));
    const int nb = std::max(1, ceil_div(n, kBlockItems));
    uint32_t *cnt, *off;
    WSB_TRY(ensure(ctx, kSlotBlockCounts, sizeof(uint32_t) * R * (size_t)nb, (void **)&cnt));
    WSB_TRY(ensure(ctx, kSlotBlockOffsets, sizeof(uint32_t) * (R * (size_t)nb + 1), (void **)&off));
    if (n > 0) {
        k_route_count<<<nb, kThreads, 0, ctx->stream>>>((const double4 *)rec, n, (double)S, sl, R,
                                                        cnt, nb);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
    } else {
        WSB_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * R * (size_t)nb, ctx->stream));
    }
    uint32_t total = 0;
    WSB_TRY(exclusive_scan_u32(ctx, cnt, off, (int64_t)R * nb, counts_host ? &total : nullptr));
    if (counts_host) {
        // first offset of each destination's block row; totals by difference
        std::vector<uint32_t> firsts(R + 1);
        WSB_CUDA_TRY(cudaMemcpy2DAsync(firsts.data(), sizeof(uint32_t), off, sizeof(uint32_t) * nb,
                                       sizeof(uint32_t), R, cudaMemcpyDeviceToHost, ctx->stream));
        WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        firsts[R] = total;
        for (int d = 0; d < R; ++d) counts_host[d] = (int64_t)firsts[d + 1] - firsts[d];
    }
    if (offs_out) *offs_out = off;
    if (nb_out) *nb_out = nb;
    return WSB_OK;
}

int route_pack(wsb_ctx *ctx, const wsb_grid *g, int S, int R, const double *rec,
               const uint32_t *plane, int64_t n, double *send_rec, uint32_t *send_plane,
               int64_t *src_index) {
    uint32_t *off;
    int nb;
    WSB_TRY(route_count(ctx, g, S, R, rec, n, nullptr, &off, &nb));
    if (n <= 0) return WSB_OK;
    Slabs sl;
    WSB_TRY(make_slabs(g->n_v, R, &sl));
    k_route_pack<<<nb, kThreads, 0, ctx->stream>>>((const double4 *)rec, plane, n, (double)S, sl,
                                                   R, off, nb, (double4 *)send_rec, send_plane,
                                                   src_index);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

int bucket_tiles(wsb_ctx *ctx, const wsb_grid *g, int S, int v_start, int v_count,
                 const double *rec, const uint32_t *plane, int64_t m, uint32_t **sorted_idx,
                 uint32_t **tile_off, int64_t *n_entries, int64_t *n_tiles) {
    TileGeom t;
    t.n_u = g->n_u;
    t.v_start = v_start;
    t.v_count = v_count;
    t.S = S;
    t.n_tu = ceil_div(g->n_u, kTile);
    t.n_tv = ceil_div(v_count, kTile);
    const int64_t tiles = (int64_t)g->n_w * t.n_tu * t.n_tv;
    if (tiles >= (int64_t(1) << 31)) return fail(WSB_EUNSUPPORTED, "too many tiles");
    *n_tiles = tiles;
    uint32_t *tcount, *toff;
    WSB_TRY(ensure(ctx, kSlotTileCount, sizeof(uint32_t) * (tiles + 1), (void **)&tcount));
    WSB_TRY(ensure(ctx, kSlotTileOff, sizeof(uint32_t) * (tiles + 1), (void **)&toff));
    WSB_CUDA_TRY(cudaMemsetAsync(tcount, 0, sizeof(uint32_t) * (tiles + 1), ctx->stream));
    const int nb = std::max(1, ceil_div(m, kBlockItems));
    uint32_t *cnt, *off;
    WSB_TRY(ensure(ctx, kSlotBlockCounts, sizeof(uint32_t) * nb, (void **)&cnt));
    WSB_TRY(ensure(ctx, kSlotBlockOffsets, sizeof(uint32_t) * (nb + 1), (void **)&off));
    uint32_t total = 0;
    if (m > 0) {
        k_bucket_count<<<nb, kThreads, 0, ctx->stream>>>((const double4 *)rec, m, t, cnt);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
        WSB_TRY(exclusive_scan_u32(ctx, cnt, off, nb, &total));
    }
    *n_entries = total;
    uint32_t *ka, *kb, *ia, *ib;
    const size_t eb = sizeof(uint32_t) * std::max<int64_t>(1, total);
    WSB_TRY(ensure(ctx, kSlotKeysA, eb, (void **)&ka));
    WSB_TRY(ensure(ctx, kSlotKeysB, eb, (void **)&kb));
    WSB_TRY(ensure(ctx, kSlotIdxA, eb, (void **)&ia));
    WSB_TRY(ensure(ctx, kSlotIdxB, eb, (void **)&ib));
    if (m > 0 && total > 0) {
        k_bucket_write<<<nb, kThreads, 0, ctx->stream>>>((const double4 *)rec, plane, m, t, off,
                                                         ka, ia, tcount);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
    }
    uint32_t *ks, *is;
    WSB_TRY(radix_sort_pairs(ctx, ka, kb, ia, ib, total, ilog2(tiles), &ks, &is));
    WSB_TRY(exclusive_scan_u32(ctx, tcount, toff, tiles + 1, nullptr));
    *sorted_idx = is;
    *tile_off = toff;
    ctx->last_keys = ks;
    ctx->last_idx = is;
    ctx->last_off = toff;
    ctx->last_entries = total;
    ctx->last_tiles = tiles;
    return WSB_OK;
}

}  // namespace wsb
