// Exclusive scan and stable LSD radix sort (8..11-bit digits) for the K1
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

// Single-pass exclusive scan: tiles taken in launch order (atomic ticket);
// each publishes its total, warp 0 then looks back over the 32 preceding
// tiles at a time until one with an inclusive prefix, and publishes its own.
// Status word: (epoch << 2 | flag) << 32 | value; words of earlier scans
// (older epochs) read as unpublished, so the array is never cleared.
constexpr uint32_t kScAgg = 1u, kScInc = 2u;
constexpr int kScanOnePassMaxTiles = 1024;   // (cfg2's scans: <= 210 tiles; cfg3's radix scans: 3900)

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kScanThreads) k_scan_onepass(const uint32_t *__restrict__ in,
                                                               uint32_t *out, int64_t n, int nb,
                                                               uint64_t *status, uint32_t *ticket,
                                                               uint32_t epoch, uint32_t *total) {
    __shared__ uint32_t s_tile, s_excl, s_tot;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = (int64_t)tile * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems], sum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < n ? in[base + i] : 0u;
        sum += v[i];
    }
    uint32_t ex = block_excl_scan(sum, &s_tot);
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const uint32_t tot = s_tot;
        const uint64_t hi = (uint64_t)epoch << 34;
        if (lane == 0) st_relaxed(&status[tile], hi | (uint64_t)(tile == 0 ? kScInc : kScAgg) << 32 | tot);
        uint32_t excl = 0;
        if (tile > 0) {
            for (int64_t j = (int64_t)tile - 1 - lane;; j -= 32) {
                uint64_t st = hi | (uint64_t)kScInc << 32;    // before tile 0: an inclusive 0
                if (j >= 0) {
                    do {
                        st = ld_relaxed(&status[j]);
                    } while ((uint32_t)(st >> 34) != epoch);
                }
                const uint32_t inc = __ballot_sync(0xffffffffu, ((uint32_t)(st >> 32) & 3u) == kScInc);
                const int first = inc ? __ffs(inc) - 1 : 32;   // nearest tile with an inclusive prefix
                uint32_t val = lane <= first ? (uint32_t)st : 0u;
#pragma unroll
                for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                excl += val;
                if (inc) break;
            }
            if (lane == 0) st_relaxed(&status[tile], hi | (uint64_t)kScInc << 32 | (excl + tot));
        }
        if (lane == 0) {
            s_excl = excl;
            if (total && tile == (uint32_t)nb - 1) *total = excl + tot;
        }
    }
    __syncthreads();
    ex += s_excl;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = ex;
        ex += v[i];
    }
}

// ---------------------------------------------------------------------------
// radix sort: B-bit digits (B = 8..9, chosen so the key needs as few passes
// as possible: cfg3's 26-bit keys take 3 passes of 9 bits instead of 4 of 8;
// wider digits scatter too thinly -- 2 passes of 12 bits were measured 1.6x
// slower than 3 of 8 at cfg2)
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
#ifndef WSB_RS_IPT
#define WSB_RS_IPT 8
#endif
constexpr int kRsIpt = WSB_RS_IPT;              // rounds of 32 per warp
constexpr int kRsItems = kRsThreads * kRsIpt;   // 4096 per block
constexpr int kRsPerWarp = 32 * kRsIpt;         // 512

template <int B>
struct RsSmem {
    static constexpr int D = 1 << B;
    uint16_t wc[kRsWarps][D];     // per-warp digit counts, then per-warp starts (<= 4096)
    uint32_t bstart[D], goff[D];  // block-local digit starts, global digit offsets
    uint32_t ks[kRsItems], vs[kRsItems];
    uint32_t wsum[kRsWarps];
};

template <int B>
__global__ void __launch_bounds__(kRsThreads) k_radix_hist(const uint32_t *__restrict__ keys,
                                                           int64_t n, int shift, uint32_t dmask,
                                                           uint32_t *hist, int nb) {
    // one sub-histogram per warp (shared-memory atomics, little contention),
    // all loads of a thread issued up front
    constexpr int D = 1 << B;
    extern __shared__ __align__(16) unsigned char raw[];
    uint32_t(*h)[D] = reinterpret_cast<uint32_t(*)[D]>(raw);
    const int warp = threadIdx.x >> 5;
    for (int e = threadIdx.x; e < kRsWarps * D; e += kRsThreads) (&h[0][0])[e] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRsItems;
    uint32_t d[kRsIpt];
#pragma unroll
    for (int r = 0; r < kRsIpt; ++r) {
        const int64_t i = base + (int64_t)r * kRsThreads + threadIdx.x;
        d[r] = i < n ? (__ldg(&keys[i]) >> shift) & dmask : (uint32_t)D;
    }
#pragma unroll
    for (int r = 0; r < kRsIpt; ++r)
        if (d[r] < (uint32_t)D) atomicAdd(&h[warp][d[r]], 1u);
    __syncthreads();
    for (int dg = threadIdx.x; dg < D; dg += kRsThreads) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) s += h[w][dg];
        hist[(int64_t)dg * nb + blockIdx.x] = s;
    }
}

// LAST: the final pass -- its keys are not needed (the consumers read the
// values and the key histogram only), so each item's global position is
// staged in place of its key and only the values are written
template <int B, bool LAST>
#ifndef WSB_RS_MINB
#define WSB_RS_MINB (16 / kRsIpt * 2)
#endif
__global__ void __launch_bounds__(kRsThreads, WSB_RS_MINB) k_radix_scatter(
    const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint32_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, int shift, uint32_t dmask,
    const uint32_t *__restrict__ offs, int nb) {
    constexpr int D = 1 << B;
    constexpr int DPT = D / kRsThreads;  // digits per thread in the block scan (1..8)
    extern __shared__ __align__(16) unsigned char raw[];
    RsSmem<B> &sm = *reinterpret_cast<RsSmem<B> *>(raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = lane; i < D; i += 32) sm.wc[warp][i] = 0;
    __syncwarp();
    const int64_t base = (int64_t)blockIdx.x * kRsItems + warp * kRsPerWarp;
    uint32_t k[kRsIpt], v[kRsIpt], pm[kRsIpt];   // pm: rank among the warp's items of the digit
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
        const uint32_t d = ok ? (k[r] >> shift) & dmask : (uint32_t)D;
        // peers with the same digit: one ballot per digit bit (and the
        // out-of-range bit B) -- measured 12% faster than MATCH.ANY here
        {
            uint32_t peers = 0xffffffffu;
#pragma unroll
            for (int bit = 0; bit <= B; ++bit) {
                const bool on = (d >> bit) & 1u;
                const uint32_t bb = __ballot_sync(0xffffffffu, on);
                peers &= on ? bb : ~bb;
            }
            // rank of this item among the warp's items of its digit so far
            const uint32_t before = d < (uint32_t)D ? sm.wc[warp][d] : 0u;
            pm[r] = before + __popc(peers & ((1u << lane) - 1u));
            __syncwarp();
            if (d < (uint32_t)D && lane == __ffs(peers) - 1) sm.wc[warp][d] = before + __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    // block-local start of each digit run (exclusive scan over the D digits
    // of the block totals; thread t owns digits [t*DPT, (t+1)*DPT)) and the
    // start of each warp inside it
    {
        uint32_t tot[DPT], sum = 0;
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            const int d = threadIdx.x * DPT + q;
            uint32_t t = 0;
#pragma unroll
            for (int w = 0; w < kRsWarps; ++w) {
                const uint32_t c = sm.wc[w][d];
                sm.wc[w][d] = (uint16_t)t;
                t += c;
            }
            tot[q] = t;
            sum += t;
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) sm.wsum[warp] = incl;
        __syncthreads();
        uint32_t run = incl - sum;
        for (int w = 0; w < warp; ++w) run += sm.wsum[w];
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            const int d = threadIdx.x * DPT + q;
            sm.bstart[d] = run;
            sm.goff[d] = offs[(int64_t)d * nb + blockIdx.x];
            run += tot[q];
        }
    }
    __syncthreads();
    // stable rank inside the block -> shared-memory staging in digit order
#pragma unroll
    for (int r = 0; r < kRsIpt; ++r) {
        int64_t i = base + r * 32 + lane;
        bool ok = i < n;
        uint32_t d = ok ? (k[r] >> shift) & dmask : (uint32_t)D;
        // block start of the digit + this warp's start in it + the item's rank
        const uint32_t pos = ok ? sm.bstart[d] + sm.wc[warp][d] + pm[r] : 0u;
        if (ok) {
            sm.ks[pos] = LAST ? sm.goff[d] + (pos - sm.bstart[d]) : k[r];
            sm.vs[pos] = v[r];
        }
    }
    __syncthreads();
    // consecutive threads write consecutive positions of each digit run
    const int64_t nblk = min((int64_t)kRsItems, n - (int64_t)blockIdx.x * kRsItems);
    if (LAST) {
        for (int p = threadIdx.x; p < nblk; p += kRsThreads) vout[sm.ks[p]] = sm.vs[p];
        return;
    }
    for (int p = threadIdx.x; p < nblk; p += kRsThreads) {
        const uint32_t key = sm.ks[p];
        const uint32_t d = (key >> shift) & dmask;
        const uint32_t gpos = sm.goff[d] + (p - sm.bstart[d]);
        WSB_DCHECK(gpos < n, "radix gpos %u n %lld", gpos, (long long)n);
        kout[gpos] = key;
        vout[gpos] = sm.vs[p];
    }
}

template <int B>
int radix_pass(wsb_ctx *ctx, const uint32_t *ka, const uint32_t *va, uint32_t *kb, uint32_t *vb,
               int64_t n, int shift, int bits, uint32_t *hist, int nb, bool last) {
    constexpr int D = 1 << B;
    // the digit covers key bits [shift, min(shift + B, bits)): key bits above
    // `bits` (the payload the caller keeps in the key) are not sorted on
    const uint32_t dmask = (bits - shift >= B) ? (uint32_t)(D - 1) : ((1u << (bits - shift)) - 1u);
    const size_t hsm = sizeof(uint32_t) * kRsWarps * D, ssm = sizeof(RsSmem<B>);
    auto scatter = last ? k_radix_scatter<B, true> : k_radix_scatter<B, false>;
    WSB_CUDA_TRY(cudaFuncSetAttribute(k_radix_hist<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)hsm));
    WSB_CUDA_TRY(cudaFuncSetAttribute(scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
    k_radix_hist<B><<<nb, kRsThreads, hsm, ctx->stream>>>(ka, n, shift, dmask, hist, nb);
    ctx->launches += 1;
    WSB_TRY(exclusive_scan_u32(ctx, hist, hist, (int64_t)D * nb, nullptr));
    scatter<<<nb, kRsThreads, ssm, ctx->stream>>>(ka, va, kb, vb, n, shift, dmask, hist, nb);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
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
    if (nb > kScanOnePassMaxTiles) {
        // many tiles: reduce / scan of the tile sums / final (the single pass's
        // look-back chains grow with the resident tiles)
        WSB_TRY(ensure(ctx, kSlotScanTmp2, sizeof(uint32_t) * (nb + 1), (void **)&sums));
        k_scan_reduce<<<nb, kScanThreads, 0, ctx->stream>>>(in, n, sums);
        k_scan_sums<<<1, kScanThreads, 0, ctx->stream>>>(sums, nb, sums + nb);
        k_scan_final<<<nb, kScanThreads, 0, ctx->stream>>>(in, out, n, sums);
        ctx->launches += 3;
        WSB_CUDA_TRY(cudaGetLastError());
        sums += nb;
    } else {
        // [nb] status words, then the ticket and the total
        const size_t bytes = sizeof(uint64_t) * ((size_t)nb + 2);
        unsigned char *work;
        const void *before = (int)ctx->bufs.size() > kSlotScanTmp ? ctx->bufs[kSlotScanTmp].ptr : nullptr;
        WSB_TRY(ensure(ctx, kSlotScanTmp, bytes, (void **)&work));
        uint64_t *status = reinterpret_cast<uint64_t *>(work);
        uint32_t *ticket = reinterpret_cast<uint32_t *>(status + nb);
        sums = ticket + 1;   // the total
        uint32_t epoch = ++ctx->scan_epoch;
        if (work != before || epoch >= (1u << 29)) {   // fresh memory (or epochs used up)
            WSB_CUDA_TRY(cudaMemsetAsync(work, 0, bytes, ctx->stream));
            epoch = ctx->scan_epoch = 1;
        }
        WSB_CUDA_TRY(cudaMemsetAsync(ticket, 0, sizeof(uint32_t), ctx->stream));
        k_scan_onepass<<<nb, kScanThreads, 0, ctx->stream>>>(in, out, n, nb, status, ticket, epoch, sums);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
    }
    if (total_host) {
        WSB_CUDA_TRY(cudaMemcpyAsync(ctx->flag_host, sums, sizeof(uint32_t),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        *total_host = (uint32_t)ctx->flag_host[0];
    }
    return WSB_OK;
}

int radix_sort_pairs(wsb_ctx *ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                     uint32_t *vals_alt, int64_t n, int bits, uint32_t **keys_out,
                     uint32_t **vals_out, bool keep_keys) {
    *keys_out = keys;
    *vals_out = vals;
    if (n <= 1 || bits <= 0) return WSB_OK;
    // digits of at most 9 bits (wider digits scatter too thinly: measured
    // slower), as few passes as that allows: 21 or 23 bits -> 3 x 8,
    // 26 -> 3 x 9 (never below 8 bits)
    const int passes = (bits + 8) / 9;
    const int B = std::max(8, (bits + passes - 1) / passes);
    const int nb = ceil_div(n, kRsItems);
    uint32_t *hist;
    WSB_TRY(ensure(ctx, kSlotRadixHist, sizeof(uint32_t) * ((size_t)1 << B) * (size_t)nb,
                   (void **)&hist));
    uint32_t *ka = keys, *kb = keys_alt, *va = vals, *vb = vals_alt;
    for (int shift = 0; shift < bits; shift += B) {
        const bool last = !keep_keys && shift + B >= bits;
        switch (B) {
            case 8: WSB_TRY(radix_pass<8>(ctx, ka, va, kb, vb, n, shift, bits, hist, nb, last)); break;
            case 9: WSB_TRY(radix_pass<9>(ctx, ka, va, kb, vb, n, shift, bits, hist, nb, last)); break;
            case 10: WSB_TRY(radix_pass<10>(ctx, ka, va, kb, vb, n, shift, bits, hist, nb, last)); break;
            case 11: WSB_TRY(radix_pass<11>(ctx, ka, va, kb, vb, n, shift, bits, hist, nb, last)); break;
            default: return fail(WSB_EUNSUPPORTED, "radix digit width");
        }
        uint32_t *t = ka; ka = kb; kb = t;
        t = va; va = vb; vb = t;
    }
    *keys_out = ka;
    *vals_out = va;
    return WSB_OK;
}

}  // namespace wsb
