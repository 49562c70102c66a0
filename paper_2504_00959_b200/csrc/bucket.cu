// K1b: bucketing of a slab's records into the gridder's work items.
//
// The reference gives every slab the records of exchange_to_space_order in
// (time_index, gindex) order (comms.py:534-545) and grids them tap-major
// (gridder.py:160-183). The GPU gridder (grid.cu) sweeps work items
// item = (w plane, 16-column strip (WSB_ITEM_COLS), 128-row block of the slab), so
// every (record, item) pair the record's taps reach becomes one entry
//     key = item << 8 | rowrel,   rowrel = anchor row - (R0 - 2S) < 128 + 2S
// (anchor row = floor(gv) - S, R0 = the block's first row), written in
// record order (k_count: entries per tile; k_keys: prepare_chunk fused in
// when it starts from the visibility columns, the tile's entries compacted
// at its offset), then stably radix-sorted on the whole key (sort.cu). Each
// item's entries are thus a contiguous run in (anchor row, record) order --
// the per-cell accumulation order of the gridder -- independent of how
// skewed the items are and of the GPU count. Item offsets come from the
// boundaries of the sorted keys (no histogram atomics: Earth-rotation tracks
// send millions of entries to single items).
#include "wsb_internal.cuh"

namespace wsb {
namespace {

constexpr int kThreads = 256;
constexpr int kPer = 4;                    // consecutive records per thread
constexpr int kTile = kThreads * kPer;     // 1024 records per block

enum : int { kErrUV = 1, kErrW = 2, kErrWeight = 4, kErrTime = 8 };

struct KeyGeom {
    int n_u, n_v, n_w, v_start, v_count, S;
    int n_ss, n_rb, item_bits;
};

// Inclusive tap range of one axis: {i : |g - i| <= S} (gridder.py:171,177),
// clipped to [lo, hi]. For in-range taps g - i is exact, so the rounded
// test below is the reference's test. Returns false if empty.
__device__ __forceinline__ bool tap_range(double g, int S, int lo, int hi, int *a, int *b) {
    const double fl = floor(g);
    int i0 = (int)fl - S;
    if (__dsub_rn(g, (double)i0) > (double)S) ++i0;
    const int i1 = (int)fl + S;
    *a = max(i0, lo);
    *b = min(i1, hi);
    return *a <= *b;
}

// Entries of one record (at most 4: two column blocks x two row blocks).
__device__ __forceinline__ int record_entries(double gu, double gv, uint32_t plane,
                                              const KeyGeom &k, uint32_t *keys) {
    // invalid coordinates (flagged by the validation) reach no item
    if (!(gu >= 0.0 && gu < (double)k.n_u && gv >= 0.0 && gv < (double)k.n_v) || plane >= (uint32_t)k.n_w)
        return 0;
    int i0, i1, j0, j1;
    if (!tap_range(gu, k.S, 0, k.n_u - 1, &i0, &i1)) return 0;
    if (!tap_range(gv, k.S, k.v_start, k.v_start + k.v_count - 1, &j0, &j1)) return 0;
    const int anchor = (int)floor(gv) - k.S;
    const int ss0 = i0 / kSSCols, ss1 = i1 / kSSCols;
    const int rb0 = (j0 - k.v_start) / kItemRows, rb1 = (j1 - k.v_start) / kItemRows;
    // entries in (row block, column block) order; a record spans at most two of each
    const uint32_t rr0 = (uint32_t)(anchor - (k.v_start + rb0 * kItemRows - 2 * k.S));
    const uint32_t it0 = ((uint32_t)plane * k.n_ss + ss0) * (uint32_t)k.n_rb + rb0;
    const uint32_t key00 = it0 << kRowBits | rr0;
    const uint32_t dss = (uint32_t)k.n_rb << kRowBits;                // next column block
    const uint32_t drb = (1u << kRowBits) - (uint32_t)kItemRows;      // next row block
    const bool two_ss = ss1 > ss0, two_rb = rb1 > rb0;
    keys[0] = key00;
    keys[1] = two_ss ? key00 + dss : key00 + drb;
    keys[2] = key00 + drb;
    keys[3] = key00 + drb + dss;
    return (two_ss ? 2 : 1) * (two_rb ? 2 : 1);
}

__device__ __forceinline__ int check_record(double uu, double vv, double ww, float wt) {
    int e = 0;
    // VisChunk.validate (visdata.py:178-184): u,v in [0,1), w in [0,1], finite weights >= 0
    if (!(uu >= 0.0 && uu < 1.0 && vv >= 0.0 && vv < 1.0)) e |= kErrUV;
    if (!(ww >= 0.0 && ww <= 1.0)) e |= kErrW;
    if (!isfinite(wt) || wt < 0.0f) e |= kErrWeight;
    return e;
}

__device__ __forceinline__ uint32_t plane_of_w(double ww, int n_w) {
    if (n_w <= 1) return 0;
    // floor(w*(n_w-1) + 0.5), two rounded FP64 ops, then clip (comms.py:484-488)
    double k = floor(__dadd_rn(__dmul_rn(ww, (double)(n_w - 1)), 0.5));
    k = fmin(fmax(k, 0.0), (double)(n_w - 1));
    return (uint32_t)(k == k ? k : 0.0);
}

struct KeysArgs {
    // FROM_INPUT: the visibility columns (one channel); else prepared records
    const double *u, *v, *w;
    const float2 *vis;
    const float *wt;
    const uint32_t *tidx;       // nullable: time order check
    double4 *rec;               // FROM_INPUT: written; else read
    uint32_t *plane;            // FROM_INPUT: written if non-null; else read
    int64_t n;
    KeyGeom g;
    uint32_t *keys, *idx;       // entries in record order
    const uint32_t *block_off;  // [n_blocks] first entry of each tile (k_count + scan)
    uint32_t cap;               // entries the key / index buffers hold (more are dropped: re-run)
    int *err;
};

// entries per tile (the compaction offsets of k_keys): taps depend on gu, gv
// only, so the count pass reads 16 of the 36 bytes per record
template <bool FROM_INPUT>
__global__ void __launch_bounds__(kThreads) k_count(const double *__restrict__ u,
                                                    const double *__restrict__ v,
                                                    const double4 *__restrict__ rec, int64_t n,
                                                    KeyGeom g, uint32_t *__restrict__ block_cnt) {
    __shared__ uint32_t wsum[kThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kTile;
    uint32_t mine = 0;
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
        const int64_t i = base + r * kThreads + threadIdx.x;
        if (i >= n) continue;
        double gu, gv;
        if constexpr (FROM_INPUT) {
            gu = __dmul_rn(__ldg(&u[i]), (double)g.n_u);
            gv = __dmul_rn(__ldg(&v[i]), (double)g.n_v);
        } else {
            const double2 c = __ldg(reinterpret_cast<const double2 *>(rec + i));
            gu = c.x;
            gv = c.y;
        }
        uint32_t k4[4];
        mine += record_entries(gu, gv, 0u, g, k4);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t += wsum[w];
        block_cnt[blockIdx.x] = t;
    }
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// 1D bulk copy global -> shared (TMA, completion on an mbarrier)
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

template <bool FROM_INPUT>
struct KeysSmem {
    static constexpr int N = kTile;
    // FROM_INPUT: u, v, w, vis, weight in; rec out. Else: rec, plane in.
    // (bulk-copy destinations: 16-byte aligned)
    alignas(16) double4 rec[FROM_INPUT ? 1 : N];
    alignas(16) double u[FROM_INPUT ? N : 2];
    alignas(16) double v[FROM_INPUT ? N : 2];
    alignas(16) double w[FROM_INPUT ? N : 2];
    alignas(16) float2 vis[FROM_INPUT ? N : 2];
    alignas(16) float wt[FROM_INPUT ? N : 4];
    alignas(16) uint32_t plane[FROM_INPUT ? 4 : N];
    uint64_t bar;
    uint64_t wsum[kThreads / 32];
    uint32_t bid;
    int err;
};

// One pass over a tile of kTile records: TMA bulk loads of the columns (or
// of the prepared records) into shared memory, prepare_chunk fused in, the
// tile's entries compacted in record order at the tile's offset (k_count +
// scan). (A bulk store of the prepared tile measured no faster than each
// thread writing its 4 consecutive records, and cost 32 KB of shared memory.)
template <bool FROM_INPUT>
__global__ void __launch_bounds__(kThreads) k_keys(KeysArgs a) {
    using Sm = KeysSmem<FROM_INPUT>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Sm &sm = *reinterpret_cast<Sm *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        sm.bid = blockIdx.x;
        sm.err = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(&sm.bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const uint32_t bid = sm.bid;
    const int64_t base = (int64_t)bid * kTile;
    const int cnt_tile = (int)min((int64_t)kTile, a.n - base);
    const bool full = cnt_tile == kTile;
    // ---- tile in: bulk copies (full tiles) or plain loads (the last one) ----
    if (full) {
        if (tid == 0) {
            const uint32_t bytes = FROM_INPUT ? kTile * (3 * 8 + 8 + 4) : kTile * (32 + 4);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(&sm.bar)),
                         "r"(bytes)
                         : "memory");
            if constexpr (FROM_INPUT) {
                bulk_load(sm.u, a.u + base, kTile * 8, &sm.bar);
                bulk_load(sm.v, a.v + base, kTile * 8, &sm.bar);
                bulk_load(sm.w, a.w + base, kTile * 8, &sm.bar);
                bulk_load(sm.vis, a.vis + base, kTile * 8, &sm.bar);
                bulk_load(sm.wt, a.wt + base, kTile * 4, &sm.bar);
            } else {
                bulk_load(sm.rec, a.rec + base, kTile * 32, &sm.bar);
                bulk_load(sm.plane, a.plane + base, kTile * 4, &sm.bar);
            }
        }
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
            " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(&sm.bar))
            : "memory");
    } else {
        for (int i = tid; i < cnt_tile; i += kThreads) {
            if constexpr (FROM_INPUT) {
                sm.u[i] = a.u[base + i];
                sm.v[i] = a.v[base + i];
                sm.w[i] = a.w[base + i];
                sm.vis[i] = a.vis[base + i];
                sm.wt[i] = a.wt[base + i];
            } else {
                sm.rec[i] = a.rec[base + i];
                sm.plane[i] = a.plane[base + i];
            }
        }
        __syncthreads();
    }
    // ---- per thread: records tid, tid + 256, ... (conflict-free shared-memory
    // reads; each warp writes 32 consecutive prepared records per round) ----
    uint32_t keys[kPer][4];
    int cnt[kPer];
    int e = 0;
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
        const int li = r * kThreads + tid;
        cnt[r] = 0;
        if (li >= cnt_tile) continue;
        double gu, gv;
        uint32_t pl;
        if constexpr (FROM_INPUT) {
            const int64_t i = base + li;
            const double uu = sm.u[li], vv = sm.v[li], ww = sm.w[li];
            const float wt = sm.wt[li];
            const float2 vs = sm.vis[li];
            e |= check_record(uu, vv, ww, wt);
            if (a.tidx && i + 1 < a.n && __ldg(&a.tidx[i]) > __ldg(&a.tidx[i + 1])) e |= kErrTime;
            gu = __dmul_rn(uu, (double)a.g.n_u);
            gv = __dmul_rn(vv, (double)a.g.n_v);
            pl = plane_of_w(ww, a.g.n_w);
            // value = 0.0 + (-0.0 + vis*weight): NumPy's complex multiply with a
            // zero imaginary weight and its pairwise-sum start, bit-exact
            const double ar = vs.x, ai = vs.y, br = wt;
            const double re = __dadd_rn(0.0, __dadd_rn(-0.0, __dsub_rn(__dmul_rn(ar, br), __dmul_rn(ai, 0.0))));
            const double im = __dadd_rn(0.0, __dadd_rn(-0.0, __dadd_rn(__dmul_rn(ar, 0.0), __dmul_rn(ai, br))));
            a.rec[i] = make_double4(gu, gv, re, im);
            if (a.plane) a.plane[i] = pl;
        } else {
            const double4 rc = sm.rec[li];
            gu = rc.x;
            gv = rc.y;
            pl = sm.plane[li];
        }
        cnt[r] = record_entries(gu, gv, pl, a.g, keys[r]);
    }
    if (FROM_INPUT && e) atomicOr(&sm.err, e);
    // entry positions in record order (r, tid): one block scan of the four
    // per-round counts packed in 16-bit fields
    uint64_t mine = 0;
#pragma unroll
    for (int r = 0; r < kPer; ++r) mine |= (uint64_t)cnt[r] << (16 * r);
    uint64_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sm.wsum[warp] = incl;
    __syncthreads();   // (also: every thread has read its inputs -- the staging below reuses them)
    uint64_t wbase = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const uint64_t s_ = sm.wsum[w];
        if (w < warp) wbase += s_;
        agg += s_;
    }
    if (tid == 0 && FROM_INPUT && sm.err) atomicOr(a.err, sm.err);
    const uint64_t ex = wbase + incl - mine;
    // stage the tile's entries compacted in shared memory, then write them
    // with consecutive threads on consecutive entries
    uint32_t *sk = reinterpret_cast<uint32_t *>(smem_raw);
    uint32_t *si = sk + 4 * kTile;
    uint32_t rbase = 0;
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
        uint32_t q = rbase + (uint32_t)((ex >> (16 * r)) & 0xFFFFu);
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (t < cnt[r]) {
                sk[q] = keys[r][t];
                si[q] = (uint32_t)(base + r * kThreads + tid);
                ++q;
            }
        rbase += (uint32_t)((agg >> (16 * r)) & 0xFFFFu);
    }
    __syncthreads();
    const uint32_t pos0 = a.block_off[bid];
    WSB_DCHECK((int64_t)pos0 + rbase <= 4 * a.n, "tile %u pos %u", bid, pos0);
    for (uint32_t q = tid; q < rbase; q += kThreads) {
        if (pos0 + q < a.cap) {
            a.keys[pos0 + q] = sk[q];
            a.idx[pos0 + q] = si[q];
        }
    }
}

// item offsets from the sorted keys: off[it] = first entry of item it (the
// next non-empty item's first entry for an empty one), off[n_items] = n --
// one binary search per item (Earth-rotation tracks leave long runs of empty
// items between two entries: a fill loop per boundary serialised them)
__global__ void k_item_offsets(const uint32_t *__restrict__ keys, int64_t n, int64_t n_items,
                               uint32_t *__restrict__ off) {
    const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (it > n_items) return;
    int64_t lo = 0, hi = n;
    if (it == n_items) {
        lo = n;
    } else {
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)(__ldg(&keys[mid]) >> kRowBits) < it)
                lo = mid + 1;
            else
                hi = mid;
        }
    }
    off[it] = (uint32_t)lo;
}

}  // namespace

int bucket_items(wsb_ctx *ctx, const wsb_grid *g, int S, int v_start, int v_count,
                 const VisColumns *in, double *rec, uint32_t *plane, int64_t m,
                 ItemBuckets *out) {
    KeyGeom k;
    k.n_u = g->n_u;
    k.n_v = g->n_v;
    k.n_w = g->n_w;
    k.v_start = v_start;
    k.v_count = v_count;
    k.S = S;
    k.n_ss = ceil_div(g->n_u, kSSCols);
    k.n_rb = ceil_div(v_count, kItemRows);
    const int64_t n_items = (int64_t)g->n_w * k.n_ss * k.n_rb;
    k.item_bits = std::max(1, ilog2(n_items));
    // item << kRowBits | rowrel (rowrel < kItemRows + 2S) in 32 bits
    static_assert(kItemRows + 2 * kMaxS <= (1 << kRowBits), "row offset bits");
    if (k.item_bits + kRowBits > 32) return fail(WSB_EUNSUPPORTED, "gridder item space exceeds 32-bit keys");
    // (at most 4 entries per record: the u32 entry count cannot wrap)
    if (m > (int64_t)1 << 30) return fail(WSB_EUNSUPPORTED, "more than 2^30 records per GPU");
    uint32_t *off;
    WSB_TRY(ensure(ctx, kSlotTileOff, sizeof(uint32_t) * (n_items + 1), (void **)&off));
    const int nb = std::max(1, ceil_div(m, kTile));
    // tile entry counts -> offsets (+ total), error flag
    uint32_t *bcnt, *boff;
    WSB_TRY(ensure(ctx, kSlotBlockCounts, sizeof(uint32_t) * (nb + 8), (void **)&bcnt));
    WSB_TRY(ensure(ctx, kSlotBlockOffsets, sizeof(uint32_t) * (nb + 8), (void **)&boff));
    WSB_CUDA_TRY(cudaMemsetAsync(bcnt, 0, sizeof(uint32_t) * (nb + 8), ctx->stream));
    uint32_t *total = boff + nb;       // exclusive scan over nb + 1 counts: the total
    int *err = reinterpret_cast<int *>(bcnt + nb + 4);
    if (m > 0) {
        if (in)
            k_count<true><<<nb, kThreads, 0, ctx->stream>>>(in->u, in->v, nullptr, m, k, bcnt);
        else
            k_count<false><<<nb, kThreads, 0, ctx->stream>>>(nullptr, nullptr, (const double4 *)rec, m,
                                                              k, bcnt);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
    }
    WSB_TRY(exclusive_scan_u32(ctx, bcnt, boff, nb + 1, nullptr));
    // k_keys writes into buffers of the capacity they have (at least 2 entries
    // per record: 1.1-1.4 typical, 4 the worst case); the entry count comes
    // back with the validation flags, and an overflow re-runs k_keys once
    // with exact buffers
    auto cap_of = [&](int slot) { return ctx->bufs[slot].bytes / sizeof(uint32_t); };
    uint32_t *ka, *ia;
    WSB_TRY(ensure(ctx, kSlotKeysA, sizeof(uint32_t) * std::max<int64_t>(1024, 2 * m + 1024), (void **)&ka));
    WSB_TRY(ensure(ctx, kSlotIdxA, sizeof(uint32_t) * std::max<int64_t>(1024, 2 * m + 1024), (void **)&ia));
    KeysArgs a;
    a.u = in ? in->u : nullptr;
    a.v = in ? in->v : nullptr;
    a.w = in ? in->w : nullptr;
    a.vis = in ? (const float2 *)in->vis : nullptr;
    a.wt = in ? in->weight : nullptr;
    a.tidx = in ? in->time_index : nullptr;
    a.rec = (double4 *)rec;
    a.plane = plane;
    a.n = m;
    a.g = k;
    a.block_off = boff;
    a.err = err;
    auto run_keys = [&]() -> int {
        a.keys = ka;
        a.idx = ia;
        a.cap = (uint32_t)std::min<size_t>(std::min(cap_of(kSlotKeysA), cap_of(kSlotIdxA)), 0xFFFFFFFFu);
        if (m > 0) {
            if (in) {
                const int sm = (int)sizeof(KeysSmem<true>);
                WSB_CUDA_TRY(cudaFuncSetAttribute(k_keys<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
                k_keys<true><<<nb, kThreads, sm, ctx->stream>>>(a);
            } else {
                const int sm = (int)sizeof(KeysSmem<false>);
                WSB_CUDA_TRY(cudaFuncSetAttribute(k_keys<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
                k_keys<false><<<nb, kThreads, sm, ctx->stream>>>(a);
            }
            ctx->launches += 1;
            WSB_CUDA_TRY(cudaGetLastError());
        }
        // entry count (and, from the columns, the validation flags) to the host
        WSB_CUDA_TRY(cudaMemcpyAsync(ctx->flag_host, total, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        WSB_CUDA_TRY(cudaMemcpyAsync(ctx->flag_host + kFlagBucketErr, err, sizeof(int), cudaMemcpyDeviceToHost,
                                     ctx->stream));
        WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        return WSB_OK;
    };
    WSB_TRY(run_keys());
    const uint32_t n_entries = m > 0 ? (uint32_t)ctx->flag_host[0] : 0u;
    if (n_entries > a.cap) {   // more than 2 entries per record on average: exact buffers, again
        WSB_TRY(ensure(ctx, kSlotKeysA, sizeof(uint32_t) * (size_t)n_entries, (void **)&ka));
        WSB_TRY(ensure(ctx, kSlotIdxA, sizeof(uint32_t) * (size_t)n_entries, (void **)&ia));
        WSB_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int), ctx->stream));
        WSB_TRY(run_keys());
    }
    ctx->pending_bucket_err = in != nullptr;
    WSB_TRY(bucket_errors(ctx));
    uint32_t *kb, *ib;
    const size_t eb = sizeof(uint32_t) * std::max<size_t>(4, n_entries);
    WSB_TRY(ensure(ctx, kSlotKeysB, eb, (void **)&kb));
    WSB_TRY(ensure(ctx, kSlotIdxB, eb, (void **)&ib));
    uint32_t *ks, *is;
    WSB_TRY(radix_sort_pairs(ctx, ka, kb, ia, ib, n_entries, k.item_bits + kRowBits, &ks, &is));
    k_item_offsets<<<ceil_div(n_items + 1, 256), 256, 0, ctx->stream>>>(ks, n_entries, n_items, off);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    out->keys = ks;
    out->idx = is;
    out->off = off;
    out->n_entries = n_entries;
    out->n_items = n_items;
    out->n_rec = m;
    out->n_ss = k.n_ss;
    out->n_rb = k.n_rb;
    out->item_bits = k.item_bits;
    ctx->last_keys = ks;
    ctx->last_idx = is;
    ctx->last_off = off;
    ctx->last_entries = n_entries;
    ctx->last_tiles = n_items;
    return WSB_OK;
}

int bucket_errors(wsb_ctx *ctx) {
    if (!ctx->pending_bucket_err) return WSB_OK;
    ctx->pending_bucket_err = false;
    const int e = ctx->flag_host[kFlagBucketErr];
    if (e & kErrUV) return fail(WSB_EINVAL, "u and v must lie in [0, 1)");
    if (e & kErrW) return fail(WSB_EINVAL, "w must lie in [0, 1]");
    if (e & kErrWeight) return fail(WSB_EINVAL, "weights must be finite and >= 0");
    // partition_time_ordered (visdata.py:354-355), reached by run_pipeline
    // through _partition_for_ranks (pipeline.py:47-52)
    if (e & kErrTime) return fail(WSB_EINVAL, "records must be sorted by time_index");
    return WSB_OK;
}

}  // namespace wsb
