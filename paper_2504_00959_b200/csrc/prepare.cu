// K1: record preparation and exchange routing.
//
//  k_prepare[_multichan]  prepare_chunk (comms.py:477-492) + VisChunk.validate
//                         (visdata.py:178-184), bit-exact FP64 arithmetic.
//  k_route_*              destination slabs of exchange_to_space_order
//                         (comms.py:516-523), packed in record (gindex) order.
// The (plane, tile column, row) bucketing of the slab records lives in bucket.cu.
#include "wsb_internal.cuh"

namespace wsb {
namespace {

constexpr int kThreads = 256;
constexpr int kBlockItems = 2048;  // records per block in the count/pack kernels

enum : int { kErrUV = 1, kErrW = 2, kErrWeight = 4, kErrTime = 8 };

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
__device__ __noinline__ double2 pairwise_sum(const float2 *vis, const float *wt, int m) {
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

__device__ __forceinline__ int check_uvw(double uu, double vv, double ww) {
    int e = 0;
    // validate(): u,v in [0,1), w in [0,1]; NaN coordinates are rejected too.
    if (!(uu >= 0.0 && uu < 1.0 && vv >= 0.0 && vv < 1.0)) e |= kErrUV;
    if (!(ww >= 0.0 && ww <= 1.0)) e |= kErrW;
    return e;
}

__device__ __forceinline__ uint32_t plane_of(double ww, int n_w) {
    if (n_w <= 1) return 0;
    // floor(w*(n_w-1) + 0.5), two rounded FP64 ops, then clip
    double k = floor(__dadd_rn(__dmul_rn(ww, (double)(n_w - 1)), 0.5));
    k = fmin(fmax(k, 0.0), (double)(n_w - 1));
    return (uint32_t)(k == k ? k : 0.0);
}

// single channel: value = 0.0 + (-0.0 + vis*weight), the reduce identity plus
// NumPy's pairwise start, bit-exact
__global__ void __launch_bounds__(kThreads) k_prepare(
    const double *__restrict__ u, const double *__restrict__ v, const double *__restrict__ w,
    const float2 *__restrict__ vis, const float *__restrict__ wt, int64_t n, double n_u,
    double n_v, int n_w, double4 *__restrict__ rec, uint32_t *__restrict__ plane, int *err,
    const uint32_t *__restrict__ tidx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double uu = u[i], vv = v[i], ww = w[i];
    const float wv = wt[i];
    int e = check_uvw(uu, vv, ww);
    if (tidx && i + 1 < n && tidx[i] > tidx[i + 1]) e |= kErrTime;
    if (!isfinite(wv) || wv < 0.0f) e |= kErrWeight;
    if (e) atomicOr(err, e);
    const double2 val = cadd(make_double2(0.0, 0.0),
                             cadd(make_double2(-0.0, -0.0), vis_times_weight(vis[i], wv)));
    rec[i] = make_double4(__dmul_rn(uu, n_u), __dmul_rn(vv, n_v), val.x, val.y);
    plane[i] = plane_of(ww, n_w);
}

__global__ void __launch_bounds__(kThreads) k_prepare_multichan(
    const double *__restrict__ u, const double *__restrict__ v, const double *__restrict__ w,
    const float2 *__restrict__ vis, const float *__restrict__ wt, int64_t n, int n_chan,
    double n_u, double n_v, int n_w, double4 *__restrict__ rec, uint32_t *__restrict__ plane,
    int *err, const uint32_t *__restrict__ tidx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double uu = u[i], vv = v[i], ww = w[i];
    int e = check_uvw(uu, vv, ww);
    if (tidx && i + 1 < n && tidx[i] > tidx[i + 1]) e |= kErrTime;
    const float2 *vr = vis + i * n_chan;
    const float *wr = wt + i * n_chan;
    for (int c = 0; c < n_chan; ++c)
        if (!isfinite(wr[c]) || wr[c] < 0.0f) e |= kErrWeight;
    if (e) atomicOr(err, e);
    const double2 val = cadd(make_double2(0.0, 0.0), pairwise_sum(vr, wr, n_chan));
    rec[i] = make_double4(__dmul_rn(uu, n_u), __dmul_rn(vv, n_v), val.x, val.y);
    plane[i] = plane_of(ww, n_w);
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
    int by_plane;   // 1: ranges of w planes (each record to the one owner of its plane)
};

__device__ __forceinline__ uint32_t dest_mask(double gv, uint32_t p, double S, const Slabs &sl,
                                              int R) {
    uint32_t m = 0;
    if (sl.by_plane) {
#pragma unroll
        for (int d = 0; d < 8; ++d)
            m |= (uint32_t)(d < R && (int)p >= sl.start[d] && (int)p < sl.start[d] + sl.count[d]) << d;
        return m;
    }
    const double hi = __dadd_rn(gv, S), lo = __dsub_rn(gv, S);  // comms.py:521-523
#pragma unroll
    for (int d = 0; d < 8; ++d) {
        const bool in = d < R && hi >= (double)sl.start[d] &&
                        lo <= (double)(sl.start[d] + sl.count[d] - 1);
        m |= (uint32_t)in << d;
    }
    return m;
}

__global__ void __launch_bounds__(kThreads) k_route_count(const double4 *__restrict__ rec,
                                                          const uint32_t *__restrict__ plane,
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
            uint32_t m = dest_mask(rec[i].y, sl.by_plane ? plane[i] : 0u, S, sl, R);
#pragma unroll
            for (int d = 0; d < 8; ++d) local[d] += (m >> d) & 1u;
        }
    }
#pragma unroll
    for (int d = 0; d < 8; ++d) {
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
    // Per 256 records: one ballot per destination ranks each lane inside its
    // warp; the warps' counts go through shared memory once (double-buffered)
    // and every thread advances its own copy of the running offsets, so a
    // round costs one barrier instead of 2R.
    constexpr int kW = kThreads / 32;
    __shared__ uint32_t wc[2][8][kW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t run[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) run[d] = d < R ? offs[(int64_t)d * nb + blockIdx.x] : 0u;
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    for (int it = 0; it < kBlockItems / kThreads; ++it) {
        const int buf = it & 1;
        const int64_t i = base + it * kThreads + threadIdx.x;
        double4 r = make_double4(0, 0, 0, 0);
        uint32_t p = 0, m = 0;
        if (i < n) {
            r = rec[i];
            p = plane[i];
            m = dest_mask(r.y, p, S, sl, R);
        }
        uint32_t in_warp[8];
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            if (d < R) {
                const uint32_t b = __ballot_sync(0xffffffffu, (m >> d) & 1u);
                in_warp[d] = __popc(b & lt);
                if (lane == 0) wc[buf][d][warp] = __popc(b);
            }
        }
        __syncthreads();
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            if (d < R) {
                uint32_t before = 0, tot = 0;
#pragma unroll
                for (int k = 0; k < kW; ++k) {
                    const uint32_t c = wc[buf][d][k];
                    before += k < warp ? c : 0u;
                    tot += c;
                }
                if ((m >> d) & 1u) {
                    const uint32_t pos = run[d] + before + in_warp[d];
                    send_rec[pos] = r;
                    send_plane[pos] = sl.by_plane ? p - (uint32_t)sl.start[d] : p;
                    if (src_index) src_index[pos] = i;
                }
                run[d] += tot;
            }
        }
    }
}

// Records per anchor row floor(gv) (load balancing of the slabs): a block
// histogram in shared memory, flushed with one global atomic per non-zero bin.
__global__ void __launch_bounds__(kThreads) k_row_hist(const double4 *__restrict__ rec, int64_t n,
                                                       int n_v, uint32_t *__restrict__ hist) {
    extern __shared__ uint32_t h[];
    for (int i = threadIdx.x; i < n_v; i += kThreads) h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    for (int it = 0; it < kBlockItems / kThreads; ++it) {
        const int64_t i = base + it * kThreads + threadIdx.x;
        if (i < n) {
            const int row = min(max((int)floor(rec[i].y), 0), n_v - 1);
            atomicAdd(&h[row], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_v; i += kThreads)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// Records per w plane (load balancing of the plane ranges), as k_row_hist.
__global__ void __launch_bounds__(kThreads) k_plane_hist(const uint32_t *__restrict__ plane,
                                                         int64_t n, int n_w,
                                                         uint32_t *__restrict__ hist) {
    extern __shared__ uint32_t h[];
    for (int i = threadIdx.x; i < n_w; i += kThreads) h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kBlockItems;
    for (int it = 0; it < kBlockItems / kThreads; ++it) {
        const int64_t i = base + it * kThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[min(plane[i], (uint32_t)(n_w - 1))], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_w; i += kThreads)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

}  // namespace

int plane_histogram(wsb_ctx *ctx, const wsb_grid *g, const uint32_t *plane, int64_t n,
                    uint32_t *hist) {
    WSB_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * g->n_w, ctx->stream));
    if (n <= 0) return WSB_OK;
    const size_t smem = sizeof(uint32_t) * g->n_w;
    if (smem > 200 * 1024) return fail(WSB_EUNSUPPORTED, "plane histogram above 51200 planes");
    WSB_CUDA_TRY(cudaFuncSetAttribute(k_plane_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    k_plane_hist<<<ceil_div(n, kBlockItems), kThreads, smem, ctx->stream>>>(plane, n, g->n_w, hist);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

int row_histogram(wsb_ctx *ctx, const wsb_grid *g, const double *rec, int64_t n, uint32_t *hist) {
    WSB_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * g->n_v, ctx->stream));
    if (n <= 0) return WSB_OK;
    const size_t smem = sizeof(uint32_t) * g->n_v;
    if (smem > 200 * 1024) return fail(WSB_EUNSUPPORTED, "row histogram above 51200 rows");
    WSB_CUDA_TRY(cudaFuncSetAttribute(k_row_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    k_row_hist<<<ceil_div(n, kBlockItems), kThreads, smem, ctx->stream>>>((const double4 *)rec, n,
                                                                          g->n_v, hist);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

int prepare(wsb_ctx *ctx, const wsb_grid *g, const double *u, const double *v, const double *w,
            const float *vis, const float *weight, int64_t n, int32_t n_chan, double *rec,
            uint32_t *plane, const uint32_t *time_index) {
    ctx->route.valid = false;   // records are (re)written
    if (n <= 0) return WSB_OK;
    int *err;
    WSB_TRY(ensure(ctx, kSlotFlag, 64, (void **)&err));
    WSB_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
    if (n_chan == 1)
        k_prepare<<<ceil_div(n, kThreads), kThreads, 0, ctx->stream>>>(
            u, v, w, (const float2 *)vis, weight, n, (double)g->n_u, (double)g->n_v, g->n_w,
            (double4 *)rec, plane, err, time_index);
    else
        k_prepare_multichan<<<ceil_div(n, kThreads), kThreads, 0, ctx->stream>>>(
            u, v, w, (const float2 *)vis, weight, n, n_chan, (double)g->n_u, (double)g->n_v,
            g->n_w, (double4 *)rec, plane, err, time_index);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    WSB_CUDA_TRY(cudaMemcpyAsync(ctx->flag_host, err, sizeof(int), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    const int e = ctx->flag_host[0];
    if (e & kErrUV) return fail(WSB_EINVAL, "u and v must lie in [0, 1)");
    if (e & kErrW) return fail(WSB_EINVAL, "w must lie in [0, 1]");
    if (e & kErrWeight) return fail(WSB_EINVAL, "weights must be finite and >= 0");
    // partition_time_ordered (visdata.py:354-355), reached by run_pipeline
    // through _partition_for_ranks (pipeline.py:47-52)
    if (e & kErrTime) return fail(WSB_EINVAL, "records must be sorted by time_index");
    return WSB_OK;
}

// Slab rows: partition_1d (mesh.py:34-45) or explicit starts (load-balanced
// slabs: starts[0] = 0 < starts[1] < ... < starts[R] = n_v).
static int make_slabs(int n_v, int R, const int32_t *starts, Slabs *sl) {
    sl->by_plane = 0;
    if (R < 1 || R > 8) return fail(WSB_EINVAL, "n_ranks must be in [1, 8]");
    if (R > n_v) return fail(WSB_EINVAL, "n_ranks exceeds n_v");
    if (starts) {
        if (starts[0] != 0 || starts[R] != n_v) return fail(WSB_EINVAL, "slab starts must span [0, n_v]");
        for (int d = 0; d < R; ++d) {
            if (starts[d + 1] <= starts[d]) return fail(WSB_EINVAL, "slab starts must increase");
            sl->start[d] = starts[d];
            sl->count[d] = starts[d + 1] - starts[d];
        }
        return WSB_OK;
    }
    const int q = n_v / R, r = n_v % R;
    for (int d = 0; d < R; ++d) {
        sl->start[d] = d < r ? d * (q + 1) : r * (q + 1) + (d - r) * q;
        sl->count[d] = d < r ? q + 1 : q;
    }
    return WSB_OK;
}

// Plane ranges [starts[d], starts[d+1]) over [0, n_w] (w-plane decomposition).
static int make_plane_ranges(int n_w, int R, const int32_t *starts, Slabs *sl) {
    if (R < 1 || R > 8) return fail(WSB_EINVAL, "n_ranks must be in [1, 8]");
    if (R > n_w) return fail(WSB_EINVAL, "n_ranks exceeds n_w");
    if (!starts) return fail(WSB_EINVAL, "plane_starts is NULL");
    if (starts[0] != 0 || starts[R] != n_w) return fail(WSB_EINVAL, "plane starts must span [0, n_w]");
    for (int d = 0; d < R; ++d) {
        if (starts[d + 1] <= starts[d]) return fail(WSB_EINVAL, "plane starts must increase");
        sl->start[d] = starts[d];
        sl->count[d] = starts[d + 1] - starts[d];
    }
    sl->by_plane = 1;
    return WSB_OK;
}

static int make_routing(const wsb_grid *g, int R, const int32_t *starts, int by_plane, Slabs *sl) {
    return by_plane ? make_plane_ranges(g->n_w, R, starts, sl) : make_slabs(g->n_v, R, starts, sl);
}

int route_count(wsb_ctx *ctx, const wsb_grid *g, int S, int R, const int32_t *starts,
                const double *rec, int64_t n, int64_t *counts_host, uint32_t **offs_out,
                int *nb_out, const uint32_t *plane, int by_plane) {
    Slabs sl;
    WSB_TRY(make_routing(g, R, starts, by_plane, &sl));
    if (by_plane && n > 0 && !plane) return fail(WSB_EINVAL, "plane is NULL");
    const int nb = std::max(1, ceil_div(n, kBlockItems));
    uint32_t *cnt, *off;
    WSB_TRY(ensure(ctx, kSlotRouteCnt, sizeof(uint32_t) * R * (size_t)nb, (void **)&cnt));
    WSB_TRY(ensure(ctx, kSlotRouteOff, sizeof(uint32_t) * (R * (size_t)nb + 1), (void **)&off));
    ctx->route.valid = false;
    if (n > 0) {
        k_route_count<<<nb, kThreads, 0, ctx->stream>>>((const double4 *)rec, plane, n, (double)S,
                                                        sl, R, cnt, nb);
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
    auto &c = ctx->route;
    c.rec = rec;
    c.plane = plane;
    c.by_plane = by_plane;
    c.n = n;
    c.S = S;
    c.R = R;
    c.n_v = by_plane ? -g->n_w : g->n_v;
    c.nb = nb;
    for (int d = 0; d < 8; ++d) c.starts[d] = sl.start[d];
    c.starts[8] = R;
    c.valid = true;
    return WSB_OK;
}

int route_pack(wsb_ctx *ctx, const wsb_grid *g, int S, int R, const int32_t *starts,
               const double *rec, const uint32_t *plane, int64_t n, double *send_rec,
               uint32_t *send_plane, int64_t *src_index, int by_plane) {
    uint32_t *off;
    int nb;
    Slabs sl;
    WSB_TRY(make_routing(g, R, starts, by_plane, &sl));
    auto &c = ctx->route;
    // the cache key covers every input of the destination mask: records,
    // their planes (plane mode), mode, halo, slabs
    bool hit = c.valid && c.rec == rec && c.plane == plane && c.by_plane == by_plane &&
               c.n == n && c.S == S && c.R == R &&
               c.n_v == (by_plane ? -g->n_w : g->n_v) &&
               c.starts[8] == R;
    for (int d = 0; hit && d < R; ++d) hit = c.starts[d] == sl.start[d];
    if (hit) {   // the counts of the preceding route_count on these records
        void *p;
        WSB_TRY(ensure(ctx, kSlotRouteOff, 0, &p));
        off = (uint32_t *)p;
        nb = c.nb;
    } else {
        WSB_TRY(route_count(ctx, g, S, R, starts, rec, n, nullptr, &off, &nb, plane, by_plane));
    }
    c.valid = false;
    if (n <= 0) return WSB_OK;
    k_route_pack<<<nb, kThreads, 0, ctx->stream>>>((const double4 *)rec, plane, n, (double)S, sl,
                                                   R, off, nb, (double4 *)send_rec, send_plane,
                                                   src_index);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

}  // namespace wsb
