// K2: tile-staged convolutional gridder (gridder.py:160-259, Eq. 3).
//
// One CTA owns one 64x64 tile of one w plane of the slab and accumulates it
// in shared memory (complex128, 64 KiB, XOR-swizzled rows). Each of the 8
// warps owns 8 tile rows; lane (c, q) = (lane & 7, lane >> 3) owns the
// cells whose column is = c (mod 8) and whose row is = q (mod 4) inside its
// warp band, so a record's footprint (<= 8 columns per pass, <= 2 rows per
// lane) is spread over the warp without two lanes touching one cell.
// Records of the tile list are processed in list (= gindex) order, hence
// every cell is accumulated by one lane in the global record order:
// deterministic and independent of tiling and GPU count.
//
// Records are staged 64 (or 32) at a time: 4 (or 8) threads per record
// compute the separable per-axis kernel weights (exp / Cephes I0, FP64)
// once per record. Warps then pick the records that touch their band with
// a ballot and scatter-add. The flush writes the tile once to HBM in the P
// layout with the checkerboard sign (transform.py:180-185) applied:
// coalesced 256-byte runs, no global atomics, no read-modify-write of HBM.
#include "i0_coeffs.h"
#include "wsb_internal.cuh"

namespace wsb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileBytes = kTile * kTile * 16;

__device__ __forceinline__ double chbevl(double x, const double *vals, int n) {
    // numpy _chbevl: b0 = x*b1 - b2 + vals[i] with separate roundings
    double b0 = vals[0], b1 = 0.0, b2 = 0.0;
    for (int i = 1; i < n; ++i) {
        b2 = b1;
        b1 = b0;
        b0 = __dadd_rn(__dsub_rn(__dmul_rn(x, b1), b2), vals[i]);
    }
    return __dmul_rn(0.5, __dsub_rn(b0, b2));
}

// np.i0 (Cephes): exp(x)*chbevl(x/2-2, A) for x <= 8, else
// exp(x)*chbevl(32/x-2, B)/sqrt(x).
__device__ __forceinline__ double bessel_i0(double x) {
    x = fabs(x);
    if (x <= 8.0)
        return __dmul_rn(exp(x), chbevl(__dsub_rn(__ddiv_rn(x, 2.0), 2.0), kI0A, kI0A_N));
    return __ddiv_rn(__dmul_rn(exp(x), chbevl(__dsub_rn(__ddiv_rn(32.0, x), 2.0), kI0B, kI0B_N)),
                     __dsqrt_rn(x));
}

// Per-axis factor of kernel_value (gridder.py:75-98) at offset d (|d| <= S
// already checked). Gaussian: exp(-d^2/(2 sigma^2)) (the 2-D weight is the
// product of the two axes, equal to the reference's exp(-(du^2+dv^2)/s2) to
// a few ulp). Kaiser-Bessel: I0(beta sqrt(1-(d/S)^2)) / I0(beta).
template <int KIND>
__device__ __forceinline__ double axis_weight(double d, double S, double p0, double p1) {
    if (KIND == WSB_KERNEL_GAUSSIAN) {
        return exp(__ddiv_rn(-__dmul_rn(d, d), p0));  // p0 = 2 sigma^2
    } else {
        const double x = __ddiv_rn(d, S);
        const double t = __dsub_rn(1.0, __dmul_rn(x, x));
        return __ddiv_rn(bessel_i0(__dmul_rn(p0, __dsqrt_rn(t))), p1);  // p0 = beta, p1 = I0(beta)
    }
}

struct GridArgs {
    const double4 *rec;
    const uint32_t *sidx;
    const uint32_t *toff;
    double2 *out;               // P layout
    unsigned long long *updates;
    int n_u, v_start, v_count, n_tu, n_tv, n_groups;
    double p0;
    const double *i0beta;       // device scalar, np.i0(beta) for Kaiser-Bessel
};

template <int KIND, int S, int CHUNK>
struct Stage {
    static constexpr int W = 2 * S + 1;
    double2 val[CHUNK];
    double wu[W][CHUNK];
    double wv[W][CHUNK];
    int ib[CHUNK];
    int jb[CHUNK];
    uint32_t um[CHUNK];
    uint32_t vm[CHUNK];
    uint32_t band[CHUNK];
};

template <int KIND, int S, int CHUNK>
__global__ void __launch_bounds__(kThreads) k_grid_tiles(GridArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double2 *tile = reinterpret_cast<double2 *>(smem);
    using St = Stage<KIND, S, CHUNK>;
    St &st = *reinterpret_cast<St *>(smem + kTileBytes);
    constexpr int W = St::W;
    constexpr int PARTS = kThreads / CHUNK;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x;
    const int per_plane = a.n_tv * a.n_tu;
    const int plane = t / per_plane;
    const int rem = t - plane * per_plane;
    const int tv = rem / a.n_tu, tu = rem - tv * a.n_tu;
    const int row0 = tv * kTile, col0 = tu * kTile;               // slab-local row, global col
    const int rows = min(kTile, a.v_count - row0), cols = min(kTile, a.n_u - col0);
    const int grow0 = a.v_start + row0;                           // global row of tile row 0

    // zero this warp's band
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[warp * 8 * kTile + k * 32 + lane] = make_double2(0.0, 0.0);

    const uint32_t beg = a.toff[t], end = a.toff[t + 1];
    const int c = lane & 7, q = lane >> 3;
    const int lr0 = warp * 8 + q, lr1 = lr0 + 4;                  // this lane's two rows
    const int swz = q << 1;                                       // (lr & 3) << 1, same for both
    unsigned cnt = 0;

    for (uint32_t cb = beg; cb < end; cb += CHUNK) {
        // ---- stage: per-record ints, masks and separable weights --------
        {
            const int r = threadIdx.x % CHUNK, part = threadIdx.x / CHUNK;
            const uint32_t e = cb + r;
            const bool valid = e < end;
            double4 R = make_double4(0, 0, 0, 0);
            if (valid) {
                const double2 *p = reinterpret_cast<const double2 *>(a.rec + __ldg(&a.sidx[e]));
                const double2 lo = __ldg(p), hi = __ldg(p + 1);
                R = make_double4(lo.x, lo.y, hi.x, hi.y);
            }
            const double gu = R.x, gv = R.y;
            const int ibg = (int)floor(gu) - S, jbg = (int)floor(gv) - S;
            if (part == 0) {
                uint32_t um = 0, vm = 0;
                if (valid) {
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        const int ci = ibg + k - col0, rj = jbg + k - grow0;
                        const bool iu = fabs(__dsub_rn(gu, (double)(ibg + k))) <= (double)S &&
                                        ci >= 0 && ci < cols;
                        const bool iv = fabs(__dsub_rn(gv, (double)(jbg + k))) <= (double)S &&
                                        rj >= 0 && rj < rows;
                        um |= (uint32_t)iu << k;
                        vm |= (uint32_t)iv << k;
                    }
                }
                uint32_t band = 0;
                if (um && vm) {
                    const int lo = jbg - grow0 + __ffs(vm) - 1;
                    const int hi = jbg - grow0 + 31 - __clz(vm);
                    for (int b = lo >> 3; b <= (hi >> 3); ++b) band |= 1u << b;
                }
                st.val[r] = make_double2(R.z, R.w);
                st.ib[r] = ibg - col0;
                st.jb[r] = jbg - grow0;
                st.um[r] = um;
                st.vm[r] = vm;
                st.band[r] = band;
            }
            // weights: value index vi in [0, 2W): < W -> u axis, else v axis
            for (int vi = part; vi < 2 * W; vi += PARTS) {
                const bool is_u = vi < W;
                const int k = is_u ? vi : vi - W;
                const double g = is_u ? gu : gv;
                const double d = __dsub_rn(g, (double)((is_u ? ibg : jbg) + k));
                double wgt = 0.0;
                if (valid && fabs(d) <= (double)S)
                    wgt = axis_weight<KIND>(d, (double)S, a.p0, KIND ? *a.i0beta : 0.0);
                if (is_u) st.wu[k][r] = wgt; else st.wv[k][r] = wgt;
            }
        }
        __syncthreads();
        // ---- scatter: each warp takes the records touching its band -----
#pragma unroll
        for (int grp = 0; grp < CHUNK / 32; ++grp) {
            uint32_t bits = __ballot_sync(0xffffffffu, (st.band[grp * 32 + lane] >> warp) & 1u);
            while (bits) {
                const int r = grp * 32 + __ffs(bits) - 1;
                bits &= bits - 1;
                const double2 val = st.val[r];
                const int ib = st.ib[r], jb = st.jb[r];
                const uint32_t um = st.um[r], vm = st.vm[r];
                const int b0 = lr0 - jb, b1 = lr1 - jb;
                const bool ok0 = (unsigned)b0 < (unsigned)W && ((vm >> b0) & 1u);
                const bool ok1 = (unsigned)b1 < (unsigned)W && ((vm >> b1) & 1u);
                if (!(ok0 || ok1)) continue;
                const double wv0 = ok0 ? st.wv[b0][r] : 0.0;
                const double wv1 = ok1 ? st.wv[b1][r] : 0.0;
#pragma unroll
                for (int it = 0; it < (W + 7) / 8; ++it) {
                    const int col = ib + ((c - ib) & 7) + 8 * it;
                    const int k = col - ib;
                    if (k < W && ((um >> k) & 1u)) {
                        const double wu = st.wu[k][r];
                        const double tr = __dmul_rn(val.x, wu), ti = __dmul_rn(val.y, wu);
                        const int pc = col ^ swz;
                        if (ok0) {
                            double2 *p = &tile[lr0 * kTile + pc];
                            double2 z = *p;
                            z.x = fma(tr, wv0, z.x);
                            z.y = fma(ti, wv0, z.y);
                            *p = z;
                            ++cnt;
                        }
                        if (ok1) {
                            double2 *p = &tile[lr1 * kTile + pc];
                            double2 z = *p;
                            z.x = fma(tr, wv1, z.x);
                            z.y = fma(ti, wv1, z.y);
                            *p = z;
                            ++cnt;
                        }
                    }
                }
            }
        }
        __syncthreads();
    }

    // ---- flush this warp's band: P layout, checkerboard sign ------------
    // P[plane][group][row][x]; a warp band of one group is 8 rows x 2 = 256 B.
    const int64_t pbase = (int64_t)plane * a.n_groups;
#pragma unroll 4
    for (int it = 0; it < kTile / kG / 2; ++it) {
        const int gl = 2 * it + (lane >> 4);
        const int e = lane & 15;
        const int rr = e >> 1, x = e & 1;
        const int col = gl * kG + x;
        const int lr = warp * 8 + rr;
        if (lr < rows && col < cols) {
            double2 z = tile[lr * kTile + (col ^ ((lr & 3) << 1))];
            const double s = ((col0 + col + grow0 + lr) & 1) ? -1.0 : 1.0;
            z.x *= s;
            z.y *= s;
            const int64_t g = (col0 + col) / kG;
            a.out[((pbase + g) * a.v_count + row0 + lr) * kG + x] = z;
        }
    }

    // ---- update count ----------------------------------------------------
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    __shared__ unsigned long long total;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    if (lane == 0 && cnt) atomicAdd(&total, (unsigned long long)cnt);
    __syncthreads();
    if (threadIdx.x == 0 && total) atomicAdd(a.updates, total);
}

template <int KIND, int S>
int launch_s(wsb_ctx *ctx, const GridArgs &a, int64_t n_tiles) {
    constexpr int CHUNK = S <= 3 ? 64 : 32;
    using St = Stage<KIND, S, CHUNK>;
    const size_t smem = kTileBytes + sizeof(St);
    auto fn = k_grid_tiles<KIND, S, CHUNK>;
    WSB_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<(unsigned)n_tiles, kThreads, smem, ctx->stream>>>(a);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

template <int KIND>
int launch_kind(wsb_ctx *ctx, int S, const GridArgs &a, int64_t n_tiles) {
    switch (S) {
        case 1: return launch_s<KIND, 1>(ctx, a, n_tiles);
        case 2: return launch_s<KIND, 2>(ctx, a, n_tiles);
        case 3: return launch_s<KIND, 3>(ctx, a, n_tiles);
        case 4: return launch_s<KIND, 4>(ctx, a, n_tiles);
        case 5: return launch_s<KIND, 5>(ctx, a, n_tiles);
        case 6: return launch_s<KIND, 6>(ctx, a, n_tiles);
        case 7: return launch_s<KIND, 7>(ctx, a, n_tiles);
        default: return fail(WSB_EUNSUPPORTED, "half_support > 7 not compiled in this build");
    }
}

__global__ void k_i0(double beta, double *out) { *out = bessel_i0(beta); }

}  // namespace

int grid_tiles(wsb_ctx *ctx, const wsb_grid *g, const wsb_kernel *k, int v_start, int v_count,
               const double *rec, const uint32_t *sorted_idx, const uint32_t *tile_off,
               int64_t n_tiles, double *grid_p, unsigned long long *updates_dev) {
    GridArgs a;
    a.rec = (const double4 *)rec;
    a.sidx = sorted_idx;
    a.toff = tile_off;
    a.out = (double2 *)grid_p;
    a.updates = updates_dev;
    a.n_u = g->n_u;
    a.v_start = v_start;
    a.v_count = v_count;
    a.n_tu = ceil_div(g->n_u, kTile);
    a.n_tv = ceil_div(v_count, kTile);
    a.n_groups = g->n_u / kG;
    if (n_tiles <= 0) return WSB_OK;
    if (k->kind == WSB_KERNEL_GAUSSIAN) {
        a.p0 = 2.0 * k->shape_param * k->shape_param;  // gridder.py:85
        a.i0beta = nullptr;
        return launch_kind<WSB_KERNEL_GAUSSIAN>(ctx, k->half_support, a, n_tiles);
    }
    a.p0 = k->shape_param;
    double *i0b;
    WSB_TRY(ensure(ctx, kSlotFlag, 64, (void **)&i0b));
    k_i0<<<1, 1, 0, ctx->stream>>>(k->shape_param, i0b + 4);  // slot bytes 32..39
    ctx->launches += 1;
    a.i0beta = i0b + 4;
    return launch_kind<WSB_KERNEL_KAISER_BESSEL>(ctx, k->half_support, a, n_tiles);
}

}  // namespace wsb
