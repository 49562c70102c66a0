// Slab-transpose push (fft2d_slab's all-to-all, transform.py:152-161) as
// plain NVLink stores: every destination's block of the row-pass output is
// copied from local HBM into that rank's column-pass input, mapped in this
// process through symmetric (peer) memory. 16-byte vector loads and stores,
// fully coalesced (512 contiguous bytes per warp instruction), several
// independent loads in flight per thread. No protocol, no staging: one
// launch moves the blocks of all destinations (blockIdx.y = destination).
#include <cstdlib>

#include "wsb_internal.cuh"

namespace wsb {
namespace {

constexpr int kPushThreads = 512;
constexpr int kPushUnroll = 4;

struct PushArgs {
    const uint4 *src[8];
    uint4 *dst[8];
    int64_t n16[8];   // 16-byte units per destination
};

__global__ void __launch_bounds__(kPushThreads) k_push(PushArgs a) {
    const int d = blockIdx.y;
    const uint4 *__restrict__ s = a.src[d];
    uint4 *__restrict__ t = a.dst[d];
    const int64_t n = a.n16[d];
    const int64_t step = (int64_t)gridDim.x * kPushThreads * kPushUnroll;
    for (int64_t base = (int64_t)blockIdx.x * kPushThreads * kPushUnroll + threadIdx.x; base < n;
         base += step) {
        uint4 v[kPushUnroll];
#pragma unroll
        for (int u = 0; u < kPushUnroll; ++u) {
            const int64_t i = base + (int64_t)u * kPushThreads;
            if (i < n) v[u] = __ldcs(&s[i]);   // streamed: read once
        }
#pragma unroll
        for (int u = 0; u < kPushUnroll; ++u) {
            const int64_t i = base + (int64_t)u * kPushThreads;
            if (i < n) t[i] = v[u];
        }
    }
}

// 4-byte granular variant (blocks of int32 columns at arbitrary offsets)
struct PushArgs4 {
    const uint32_t *src[8];
    uint32_t *dst[8];
    int64_t n4[8];
};

__global__ void __launch_bounds__(kPushThreads) k_push4(PushArgs4 a) {
    const int d = blockIdx.y;
    const uint32_t *__restrict__ s = a.src[d];
    uint32_t *__restrict__ t = a.dst[d];
    const int64_t n = a.n4[d];
    for (int64_t i = (int64_t)blockIdx.x * kPushThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kPushThreads)
        t[i] = __ldcs(&s[i]);
}

}  // namespace

int push_blocks(wsb_ctx *ctx, int n_dest, const void *const *src, void *const *dst,
                const int64_t *bytes) {
    if (n_dest < 1 || n_dest > 8) return fail(WSB_EINVAL, "n_dest must be in [1, 8]");
    PushArgs a;
    int64_t most = 0;
    for (int d = 0; d < 8; ++d) {
        a.src[d] = nullptr;
        a.dst[d] = nullptr;
        a.n16[d] = 0;
    }
    bool wide = true;
    for (int d = 0; d < n_dest; ++d) {
        if (bytes[d] < 0 || bytes[d] % 4) return fail(WSB_EINVAL, "block sizes must be multiples of 4 bytes");
        if (bytes[d] && (!src[d] || !dst[d])) return fail(WSB_EINVAL, "NULL block pointer");
        if (((uintptr_t)src[d] | (uintptr_t)dst[d]) % 4) return fail(WSB_EINVAL, "blocks must be 4-byte aligned");
        if (bytes[d] % 16 || ((uintptr_t)src[d] | (uintptr_t)dst[d]) % 16) wide = false;
    }
    if (!wide) {
        PushArgs4 b;
        int64_t most4 = 0;
        for (int d = 0; d < 8; ++d) {
            b.src[d] = d < n_dest ? (const uint32_t *)src[d] : nullptr;
            b.dst[d] = d < n_dest ? (uint32_t *)dst[d] : nullptr;
            b.n4[d] = d < n_dest ? bytes[d] / 4 : 0;
            most4 = std::max(most4, b.n4[d]);
        }
        if (most4 == 0) return WSB_OK;
        const int per = (int)std::min<int64_t>(64, (most4 + kPushThreads - 1) / kPushThreads);
        k_push4<<<dim3(per, n_dest), kPushThreads, 0, ctx->stream>>>(b);
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
        return WSB_OK;
    }
    for (int d = 0; d < n_dest; ++d) {
        a.src[d] = (const uint4 *)src[d];
        a.dst[d] = (uint4 *)dst[d];
        a.n16[d] = bytes[d] / 16;
        most = std::max(most, a.n16[d]);
    }
    if (most == 0) return WSB_OK;
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->device);
    // about two SMs' worth of CTAs per destination: enough outstanding
    // stores for the link, most SMs stay with the concurrent row pass
    // CTAs per destination: enough outstanding stores for the link; capped
    // (WSB_PUSH_CTAS overrides) so a push overlapping compute leaves it SMs
    int cap = 64;
    if (const char *e = std::getenv("WSB_PUSH_CTAS")) cap = std::max(1, std::atoi(e));
    const int per = (int)std::min<int64_t>(std::min(cap, std::max(2, 2 * dev_sms / (n_dest + 1))),
                                           (most + kPushThreads * kPushUnroll - 1) /
                                               (kPushThreads * kPushUnroll));
    k_push<<<dim3(per, n_dest), kPushThreads, 0, ctx->stream>>>(a);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

}  // namespace wsb

extern "C" int wsb_push_blocks(wsb_ctx *ctx, int32_t n_dest, const void *const *src_ptrs,
                               void *const *dst_ptrs, const int64_t *bytes_host) {
    if (!ctx || !src_ptrs || !dst_ptrs || !bytes_host) return wsb::fail(WSB_EINVAL, "NULL argument");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return wsb::fail(WSB_ECUDA, cudaGetErrorString(e));
    return wsb::push_blocks(ctx, n_dest, src_ptrs, dst_ptrs, bytes_host);
}
