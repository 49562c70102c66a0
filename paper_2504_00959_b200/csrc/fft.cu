// K3 + K4: per-plane inverse 2-D FFT, w correction and plane stacking.
//
// The reference transforms each plane with an iterative radix-2 loop
// (transform.py:99-127), distributed as row FFT -> block transpose -> row
// FFT -> transpose back (transform.py:130-177), then applies the w phase
// screen (transform.py:192-202) and stacks the planes (transform.py:205-230).
//
// Here a plane makes two passes over HBM:
//   k_fft_rows  : CTA = 4096/N rows of one plane. Radix-16 Stockham autosort
//                 (FP64, twiddles from a sincospi table): the first pass
//                 reads the P layout straight from HBM into registers, the
//                 inner exchanges go through shared memory, the last pass
//                 writes straight back. In place.
//   k_fft_cols  : CTA = 4096/N columns for ALL planes: per plane, column FFT
//                 (radix-8; plane k+1's inputs are loaded into registers
//                 while plane k is transformed; the last pass stays in
//                 registers), the phase screen exp(2 pi i w_k (n-1)) and the
//                 running sum over planes in registers; after the last plane
//                 the 1/(n_u n_v), 1/n_w and n factors, the real part, the
//                 image strip and per-column residual norms. The transpose-back
//                 of the reference is never materialised.
#include <cuda_pipeline_primitives.h>

#include <cstdlib>

#include "wsb_internal.cuh"


namespace wsb {
namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x));
}
// FP32 path (transforms in complex64; coordinates, weights, phases and the
// plane stack stay FP64)
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -(a.y * b.y)), fmaf(a.x, b.y, a.y * b.x));
}
template <class V> __device__ __forceinline__ V cx(double x, double y);
template <> __device__ __forceinline__ double2 cx<double2>(double x, double y) { return make_double2(x, y); }
template <> __device__ __forceinline__ float2 cx<float2>(double x, double y) {
    return make_float2((float)x, (float)y);
}
__device__ __forceinline__ double2 to_d2(double2 z) { return z; }
__device__ __forceinline__ double2 to_d2(float2 z) { return make_double2(z.x, z.y); }

// (cos(pi x), sin(pi x)) for |x| < 2^30: x = t/2 + r with t = rint(2x),
// |r| <= 1/4, then Taylor polynomials of sin(pi r)/r (degree 16) and
// cos(pi r) (degree 16) in r^2, truncation < 1e-18; about a third of the
// instructions of the library sincospi, a few ulp from it.
// FP64 constants live in the constant bank: DFMA takes c[][] operands
// directly, whereas literals are rebuilt with two UMOVs each per use.
__constant__ double kSinPiC[10] = {3.141592653589793, -5.16771278004997, 2.5501640398773455,
                                   -0.5992645293207921, 0.08214588661112823,
                                   -0.0073704309457143504, 0.00046630280576761255,
                                   -2.1915353447830217e-05, 7.952054001475513e-07,
                                   -2.2948428997269873e-08};
__constant__ double kCosPiC[9] = {1.0, -4.934802200544679, 4.0587121264167685,
                                  -1.3352627688545895, 0.2353306303588932, -0.02580689139001406,
                                  0.0019295743094039231, -0.0001046381049248457,
                                  4.303069587032947e-06};

__device__ __forceinline__ double2 cis_pi(double x) {
    const double t = rint(2.0 * x);
    const double r = fma(-0.5, t, x);
    const double r2 = r * r;
    double s = kSinPiC[9];
#pragma unroll
    for (int i = 8; i >= 0; --i) s = fma(s, r2, kSinPiC[i]);
    s *= r;
    double c = kCosPiC[8];
#pragma unroll
    for (int i = 7; i >= 0; --i) c = fma(c, r2, kCosPiC[i]);
    const int q = (int)(long long)t & 3;
    const double cs = (q & 1) ? s : c;
    const double sn = (q & 1) ? c : s;
    return make_double2((q == 1 || q == 2) ? -cs : cs, (q >= 2) ? -sn : sn);
}

// cos/sin(2 pi u / 16), u = 0..7
__constant__ double kRoot16[8][2] = {{1.0, 0.0},
                                     {0.92387953251128673848, 0.38268343236508977173},
                                     {0.70710678118654752440, 0.70710678118654752440},
                                     {0.38268343236508977173, 0.92387953251128673848},
                                     {0.0, 1.0},
                                     {-0.38268343236508977173, 0.92387953251128673848},
                                     {-0.70710678118654752440, 0.70710678118654752440},
                                     {-0.92387953251128673848, 0.38268343236508977173}};

template <class V>
__device__ __forceinline__ V root16(int u) { return cx<V>(kRoot16[u][0], kRoot16[u][1]); }

// a * exp(+2 pi i u/16)
template <class V>
__device__ __forceinline__ V rot16(V a, int u) {
    if (u == 0) return a;
    if (u == 4) { V r; r.x = -a.y; r.y = a.x; return r; }
    return cmul(a, root16<V>(u));
}

constexpr int brev(int i, int R) {
    int r = 0;
    for (int b = 1; b < R; b <<= 1) {
        r <<= 1;
        if (i & b) r |= 1;
    }
    return r;
}

// Everything below is resolved at compile time so the values stay in
// registers (a runtime index would push the array to local memory).
template <int R, int I, class V>
__device__ __forceinline__ void brev_swap(V *y) {
    if constexpr (I < R) {
        constexpr int J = brev(I, R);
        if constexpr (J > I) {
            const V t = y[I];
            y[I] = y[J];
            y[J] = t;
        }
        brev_swap<R, I + 1>(y);
    }
}

template <int R, int LEN, int I, int K, class V>
__device__ __forceinline__ void dit_butterflies(V *y) {
    if constexpr (I < R) {
        if constexpr (K < LEN / 2) {
            const V t = rot16(y[I + K + LEN / 2], K * (16 / LEN));
            const V a = y[I + K];
            y[I + K] = cadd(a, t);
            y[I + K + LEN / 2] = csub(a, t);
            dit_butterflies<R, LEN, I, K + 1>(y);
        } else {
            dit_butterflies<R, LEN, I + LEN, 0>(y);
        }
    }
}

template <int R, int LEN, class V>
__device__ __forceinline__ void dit_stages(V *y) {
    if constexpr (LEN <= R) {
        dit_butterflies<R, LEN, 0, 0>(y);
        dit_stages<R, LEN * 2>(y);
    }
}

// In-register inverse DFT of size R (<= 16), e^{+2 pi i}, natural order out.
template <int R, class V>
__device__ __forceinline__ void dft_inv(V *y) {
    brev_swap<R, 0>(y);
    dit_stages<R, 2>(y);
}

// padded shared-memory index of element idx of a sequence: one pad slot per
// 8 elements keeps the 8 lanes of a 128-byte wavefront on distinct bank
// groups for contiguous runs and for the stride-4/8 and (ns = 4) stores of
// the radix-4/8 passes
__device__ __forceinline__ int pidx(int idx) { return idx + (idx >> 3); }

// padded sequence stride: = 4 (mod 8) in 16-byte units for N >= 64, so the
// two sequences of an interleaved pass (IL = 2) fall on disjoint bank halves
template <int LOGN>
struct Seq {
    static constexpr int N = 1 << LOGN;
    static constexpr int STRIDE = N + (N >> 3) + (N >= 16 ? 4 : 0);
};

// Butterfly b -> (sequence, index j). IL = 1: b / M, b % M. IL = 2: two
// sequences interleaved lane by lane, so a warp touches element j of both
// sequences side by side (the row pass's last stores: rows j0, j0+1 of a
// column are one 32-byte sector of the column-major P layout).
template <int IL, int M>
__device__ __forceinline__ void seq_of(int b, int &seq, int &j) {
    if constexpr (IL == 1) {
        seq = b / M;
        j = b % M;
    } else {
        const int q = b % (M * IL);
        seq = (b / (M * IL)) * IL + q % IL;
        j = q / IL;
    }
}


// ---------------------------------------------------------------------------
// Stockham pass pieces (radix R = 2^RL, N = 2^LOGN, E values per thread, T
// threads; butterfly b of a pass = (sequence b / (N/R), index j = b % (N/R))).
// A pass reads x[j + r N/R], multiplies by the twiddles of its stage,
// applies the radix-R DFT and writes y[(j/ns) ns R + j%ns + r ns].
// ---------------------------------------------------------------------------
template <int LOGN, int RL, int E, int T, int IL = 1, class V, class LD>
__device__ __forceinline__ void pass_load(V (&v)[E], LD ld) {
    constexpr int R = 1 << RL, NB = E / R, M = (1 << LOGN) / R;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        int seq, j;
        seq_of<IL, M>(threadIdx.x + k * T, seq, j);
#pragma unroll
        for (int r = 0; r < R; ++r) v[k * R + r] = ld(seq, j + r * M);
    }
}

// The base twiddle of a pass (span ns, radix R) is stored pass by pass as
// [j % ns] = exp(2 pi i (j % ns) / (ns R)), so the lanes of a warp
// (consecutive j) read consecutive entries: a few sectors per load instead
// of one sector per lane from a strided N-entry table.
constexpr int tw_offset(int logn, int rlmax, int done) {
    int off = 0, d = 0;
    while (d < done) {
        const int first = logn % rlmax;
        const int rl = (d == 0 && first != 0) ? first : rlmax;
        if (d > 0) off += 1 << d;
        d += rl;
    }
    return off;
}

template <int LOGN, int RL, int E, int T, int IL = 1, class V>
__device__ __forceinline__ void pass_compute(int ns, const V *__restrict__ tw, V (&v)[E]) {
    constexpr int N = 1 << LOGN, R = 1 << RL, NB = E / R, M = N / R;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        int seq, j;
        seq_of<IL, M>(threadIdx.x + k * T, seq, j);
        V y[R];
#pragma unroll
        for (int r = 0; r < R; ++r) y[r] = v[k * R + r];
        if (ns > 1) {
            // one table load per butterfly; the other powers by a product
            // tree w^r = w^(r/2) w^(r - r/2) (depth log2 R, a few ulp): the
            // loads, not the FP64 pipe, are what the passes queue on
            V wp[R];
            wp[1] = __ldg(&tw[j % ns]);
#pragma unroll
            for (int r = 2; r < R; ++r) wp[r] = cmul(wp[r / 2], wp[r - r / 2]);
#pragma unroll
            for (int r = 1; r < R; ++r) y[r] = cmul(y[r], wp[r]);
        }
        dft_inv<R>(y);
#pragma unroll
        for (int r = 0; r < R; ++r) v[k * R + r] = y[r];
    }
}

template <int LOGN, int RL, int E, int T, int IL = 1, class V, class ST>
__device__ __forceinline__ void pass_store(int ns, const V (&v)[E], ST st) {
    constexpr int R = 1 << RL, NB = E / R, M = (1 << LOGN) / R;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        int seq, j;
        seq_of<IL, M>(threadIdx.x + k * T, seq, j);
        const int idxd = (j / ns) * ns * R + j % ns;
#pragma unroll
        for (int r = 0; r < R; ++r) st(seq, idxd + r * ns, v[k * R + r]);
    }
}

// Radix plan: the first pass takes LOGN % RLMAX (if non-zero), then RLMAX.
template <int LOGN, int RLMAX, int DONE>
struct Plan {
    static constexpr int FIRST = LOGN % RLMAX;
    static constexpr int RL = (DONE == 0 && FIRST != 0) ? FIRST : RLMAX;
    static constexpr bool LAST = DONE + RL == LOGN;
};

// Passes 1..last-1 in shared memory (in place), then the last pass's loads
// and compute: its results stay in v, at (seq, j + r*N/R) of butterfly b
// (mapped with ILL, the interleave of the last pass).
template <int LOGN, int RLMAX, int E, int T, int DONE, int ILL = 1, class V>
__device__ __forceinline__ void smem_passes(V *s, const V *tw, V (&v)[E]) {
    using P = Plan<LOGN, RLMAX, DONE>;
    constexpr int STRIDE = Seq<LOGN>::STRIDE;
    constexpr int IL = P::LAST ? ILL : 1;
    auto ld = [&](int seq, int idx) { return s[seq * STRIDE + pidx(idx)]; };
    pass_load<LOGN, P::RL, E, T, IL>(v, ld);
    if constexpr (!P::LAST) __syncthreads();
    pass_compute<LOGN, P::RL, E, T, IL>(1 << DONE, tw + tw_offset(LOGN, RLMAX, DONE), v);
    if constexpr (!P::LAST) {
        auto st = [&](int seq, int idx, V z) { s[seq * STRIDE + pidx(idx)] = z; };
        pass_store<LOGN, P::RL, E, T>(1 << DONE, v, st);
        __syncthreads();
        smem_passes<LOGN, RLMAX, E, T, DONE + P::RL, ILL>(s, tw, v);
    }
}

// ---------------------------------------------------------------------------
// row pass: global -> registers -> (shared memory passes) -> global
// ---------------------------------------------------------------------------
// 4096/N rows per CTA (2 at N = 2048, 2 CTAs per SM): independent CTAs keep
// the per-pass barriers of different rows out of phase, so one CTA's HBM
// latency overlaps another's transform (measured: 1 row/128 threads and
// 4 rows/512 threads are both slower at N = 2048)
template <int LOGN>
struct RowCfg {
#ifndef WSB_ROW_MIN_T
#define WSB_ROW_MIN_T 256
#endif
    // N = 4096 takes 2 rows (512 threads) so the interleaved last pass can
    // write whole 32-byte sectors of the column-major P layout
#ifndef WSB_ROW12_DIV
#define WSB_ROW12_DIV 8
#endif
    static constexpr int T = LOGN >= 12 ? (1 << LOGN) / WSB_ROW12_DIV
                             : ((1 << LOGN) / 16 > WSB_ROW_MIN_T) ? (1 << LOGN) / 16 : WSB_ROW_MIN_T;
    static constexpr int MINB = T <= 128 ? 4 : (T <= 256 ? 2 : 1);
};
constexpr int kRowE = 16;
constexpr int kRowRL = 4;

// Column-group partition of the row pass output over the destination ranks.
// Destination d receives column groups [g0[d], g0[d+1]) of every row, laid
// out from ptr[d] as [plane - plane0][g - g0[d]][row][G]. ptr[d] is either a
// block of a local send buffer or -- the fused transpose -- this source's
// block of rank d's column-pass input in peer memory (NVLink stores).
struct RowDest {
    void *ptr[8];
    int plane0;
    int g0[9];   // first group of each destination, g0[n_dest] = n_u/G, unused = INT_MAX
};

// z * exp(2 pi i q / 4), exact
template <class V>
__device__ __forceinline__ V rot_quarter(V z, int q) {
    V r;
    switch (q & 3) {
        case 0: return z;
        case 1: r.x = -z.y; r.y = z.x; return r;
        case 2: r.x = -z.x; r.y = -z.y; return r;
        default: r.x = z.y; r.y = -z.x; return r;
    }
}

// Rows longer than the on-chip limit (N = SP * M, M = 2^LOGN <= 4096):
// CTA residue e computes the outputs X[k SP + e] = FFT_M(u_e)[k] of the
// decimation-in-frequency split
//   u_e[n] = W_N^(n e) * sum_s x[n + s M] W_SP^(s e),   W_K = exp(2 pi i / K),
// so every CTA reads the whole row (SP-fold reads) and runs the on-chip
// M-point transform. twN: exp(2 pi i m / N), m < N.
template <int SPL, class V>
__device__ __forceinline__ V dif_split(const V *x, int stride, int e, int n, int M,
                                       const V *__restrict__ twN) {
    constexpr int SP = 1 << SPL;
    V u = x[0];
#pragma unroll
    for (int s = 1; s < SP; ++s) {
        const V y = rot_quarter(x[(int64_t)s * stride], (4 / SP) * s * e);
        u = cadd(u, y);
    }
    return e ? cmul(u, __ldg(&twN[n * e])) : u;
}

// the same for a loader ld(s) of the s-th column of the split
template <int SPL, class V, class LD>
__device__ __forceinline__ V dif_split_ld(LD ld, int e, int n, const V *__restrict__ twN) {
    constexpr int SP = 1 << SPL;
    V u = ld(0);
#pragma unroll
    for (int s = 1; s < SP; ++s) u = cadd(u, rot_quarter(ld(s), (4 / SP) * s * e));
    return e ? cmul(u, __ldg(&twN[n * e])) : u;
}

// 4096/N rows per CTA. The first pass reads its inputs straight from HBM
// (32-byte sectors, 16 loads in flight per thread) and the last pass writes
// its outputs straight back: shared memory only carries the inner exchanges.
// SPL > 0: rows of N = 2^(LOGN+SPL) points, residue e = blockIdx.z (above).
template <int LOGN, int SPL, class V>
__device__ __forceinline__ void rows_body(const V *__restrict__ in, int n_strips, int v_count,
                                          const V *__restrict__ tw, const V *__restrict__ twN,
                                          const RowDest &dst, const int j0, const int64_t plane,
                                          const int e) {
    constexpr int N = 1 << LOGN;          // on-chip transform length M
    constexpr int SP = 1 << SPL;
    constexpr int RT = RowCfg<LOGN>::T;
    constexpr int NSEQ = RT * kRowE / N;  // rows per CTA
    constexpr int STRIDE = Seq<LOGN>::STRIDE;
    using P0 = Plan<LOGN, kRowRL, 0>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V *s = reinterpret_cast<V *>(smem_raw);
    // in: strip layout [plane][col/WSB_STRIP][row][re | im][col%WSB_STRIP]
    // (a strip row holds its WSB_STRIP real parts, then the imaginary parts)
    constexpr int SW = WSB_STRIP;
    using Sc = decltype(V{}.x);
    const Sc *ins = reinterpret_cast<const Sc *>(in);
    auto gld = [&](int seq, int col) {
        if (j0 + seq >= v_count) return cx<V>(0.0, 0.0);
        const Sc *p = ins + ((plane * n_strips + col / SW) * v_count + j0 + seq) * (2 * SW) + (col % SW);
        if constexpr (SPL == 0) {
            V z;
            z.x = p[0];
            z.y = p[SW];
            return z;
        } else {
            // column col + s*N lies (N/SW) strips further on
            const int64_t stride = (int64_t)(N / SW) * v_count * (2 * SW);
            return dif_split_ld<SPL, V>(
                [&](int s_) {
                    V z;
                    z.x = p[s_ * stride];
                    z.y = p[s_ * stride + SW];
                    return z;
                },
                e, col, twN);
        }
    };
    // out: P[plane][col/G][row][col%G] per destination (RowDest); with a
    // single destination this is the plain P layout
    auto gst = [&](int seq, int k, V z) {
        const int col = k * SP + e;
        if (j0 + seq < v_count) {
            const int g = col / kG;
            int lo = 0, hi = dst.g0[1];
            V *base = reinterpret_cast<V *>(dst.ptr[0]);
#pragma unroll
            for (int d = 1; d < 8; ++d)
                if (g >= dst.g0[d]) {
                    lo = dst.g0[d];
                    hi = dst.g0[d + 1];
                    base = reinterpret_cast<V *>(dst.ptr[d]);
                }
            base[(((plane - dst.plane0) * (hi - lo) + (g - lo)) * v_count + j0 + seq) * kG +
                 (col % kG)] = z;
        }
    };
    V v[kRowE];
    pass_load<LOGN, P0::RL, kRowE, RT>(v, gld);
    pass_compute<LOGN, P0::RL, kRowE, RT>(1, tw, v);
    if constexpr (P0::LAST) {
        pass_store<LOGN, P0::RL, kRowE, RT>(1, v, gst);
    } else {
        auto sst = [&](int seq, int idx, V z) { s[seq * STRIDE + pidx(idx)] = z; };
        pass_store<LOGN, P0::RL, kRowE, RT>(1, v, sst);
        __syncthreads();
        // last pass with the two rows of a CTA interleaved lane by lane: the
        // column-major P layout then receives full 32-byte sectors
        constexpr int ILL = NSEQ >= 2 ? 2 : 1;
        smem_passes<LOGN, kRowRL, kRowE, RT, P0::RL, ILL>(s, tw, v);
        constexpr int RLL = kRowRL;  // the last pass is always a full-radix pass here
        pass_store<LOGN, RLL, kRowE, RT, ILL>(N >> RLL, v, gst);
    }
}

// persist_nbx > 0 (rows of <= 4096 points): CTAs stride over the linear
// (plane, row pair) index (persist_nbx row pairs per plane); l2pf: each
// also prefetches its next pair into L2 (TMA bulk prefetch, one per strip)
// while the current one is transformed (measured slower: off by default)
template <int LOGN, int SPL, class V>
__global__ void __launch_bounds__(RowCfg<LOGN>::T, RowCfg<LOGN>::MINB)
    k_fft_rows(const V *__restrict__ in, int n_strips, int n_groups, int v_count,
               int plane_lo, const V *__restrict__ tw, const V *__restrict__ twN,
               RowDest dst, int persist_nbx, int64_t n_pairs, int l2pf) {
    constexpr int N = 1 << LOGN;
    constexpr int NSEQ = RowCfg<LOGN>::T * kRowE / N;
    if (SPL == 0 && persist_nbx > 0) {
        using Sc = decltype(V{}.x);
        constexpr int SW = WSB_STRIP;
        const Sc *ins = reinterpret_cast<const Sc *>(in);
        for (int64_t L = blockIdx.x; L < n_pairs; L += gridDim.x) {
            const int64_t Ln = L + gridDim.x;
            if (l2pf && Ln < n_pairs) {
                const int jn = (int)(Ln % persist_nbx) * NSEQ;
                const int64_t pn = plane_lo + Ln / persist_nbx;
                const uint32_t bytes = (uint32_t)(min(NSEQ, v_count - jn) * 2 * SW * sizeof(Sc));
                for (int st = threadIdx.x; st < n_strips; st += blockDim.x) {
                    const Sc *q = ins + ((pn * n_strips + st) * v_count + jn) * (2 * SW);
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(q), "r"(bytes) : "memory");
                }
            }
            rows_body<LOGN, SPL, V>(in, n_strips, v_count, tw, twN, dst, (int)(L % persist_nbx) * NSEQ,
                                    plane_lo + L / persist_nbx, 0);
            __syncthreads();   // shared memory is reused by the next pair
        }
        return;
    }
    rows_body<LOGN, SPL, V>(in, n_strips, v_count, tw, twN, dst, blockIdx.x * NSEQ, plane_lo + blockIdx.y,
                            SPL ? (int)blockIdx.z : 0);
}


// ---------------------------------------------------------------------------
// column pass + w correction + stacking
// ---------------------------------------------------------------------------
// one column per CTA at N >= 2048: two 256-thread CTAs per SM at N = 2048
template <int LOGN>
struct ColCfg {
    static constexpr int T = ((1 << LOGN) / 8 > 256) ? (1 << LOGN) / 8 : 256;
    static constexpr int MINB = T <= 256 ? 2 : 1;
};
#ifndef WSB_COLS_ZREG
#define WSB_COLS_ZREG 1
#endif
constexpr int kColE = 8;
constexpr int kColRL = 3;

struct ColArgs {
    const void *tgrid;      // planes [k0, k1) only (complex128, or complex64 on the FP32 path)
    double *strip;          // [n_v][ncols]
    double *partials;       // [ncols][2]
    double2 *run;           // running stack between plane ranges, per thread element
    const void *twN;        // exp(2 pi i m / n_v), m < n_v (split columns only)
    int n_w, n_u, n_v, ncols, g0;
    int k0, k1;             // plane range of this call
    int k_top, k_bottom;    // planes this process stacks: [k_bottom, k_top) (default [0, n_w))
    double2 *pimg;          // non-null: write the partial stack of [k_bottom, k_top) as a
                            // complex128 image [n_v][ncols] instead of finishing
    int n_src;
    int src_start[9];       // row start of each source slab (+ sentinel)
    double cell, inv_nuv, inv_nw, w_min, w_max;
};

// native w of plane k (mesh.py:101-112), the same IEEE operations as the host
__device__ __forceinline__ double plane_w(const ColArgs &a, int k) {
    if (a.n_w == 1) return __dmul_rn(0.5, __dadd_rn(a.w_min, a.w_max));
    const double frac = __ddiv_rn((double)k, (double)(a.n_w - 1));
    return __dadd_rn(a.w_min, __dmul_rn(frac, __dsub_rn(a.w_max, a.w_min)));
}

// CTA = 4096/N columns for all planes. The planes are stacked by Horner's
// rule from the top plane down: with w_k = w_0 + k dw (mesh.py:101-112),
//   sum_k P_k exp(2 pi i w_k (n-1)) = c * sum_k P_k z^k
//       = c * (((P_{K-1} z + P_{K-2}) z + ...) z + P_0),
//   z = exp(2 pi i dw (n-1)),  c = exp(2 pi i w_0 (n-1)),
// so a plane costs one complex multiply-add per pixel instead of a phase
// evaluation (|z| = 1: the rounding grows by about one ulp per plane).
// Plane k-1's first-pass inputs are loaded into registers while plane k is
// transformed; the last pass leaves its outputs in registers.
// SPL > 0 (n_v = SP * 4096): residue CTA e = blockIdx.y transforms output
// rows k SP + e of its columns through the decimation-in-frequency split of
// dif_split (every CTA reads its whole columns).
template <int LOGN, int SPL, class V>
__global__ void __launch_bounds__(ColCfg<LOGN>::T, ColCfg<LOGN>::MINB)
    k_fft_cols(ColArgs a, const V *__restrict__ tw) {
    constexpr int CT = ColCfg<LOGN>::T;
    constexpr int N = 1 << LOGN;                 // n_v
    constexpr int C = CT * kColE / N;   // columns per CTA
    constexpr int STRIDE = Seq<LOGN>::STRIDE;
    constexpr int RLM = LOGN < kColRL ? LOGN : kColRL;
    using P0 = Plan<LOGN, RLM, 0>;
    constexpr int R = 1 << RLM;                  // radix of the last pass
    constexpr int M = N / R;
    constexpr int NB = kColE / R;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *sbuf = reinterpret_cast<double2 *>(smem_raw);  // finish: pixels + squares
    V *sv = reinterpret_cast<V *>(smem_raw);                 // transform exchanges
    double2 *zbuf = sbuf + 2 * C * STRIDE;       // z per pixel, [C][N]
    const V *tg = reinterpret_cast<const V *>(a.tgrid);
    const V *twN = reinterpret_cast<const V *>(a.twN);

    const int c0 = blockIdx.x * C;                 // first local column
    const int nk = a.k1 - a.k0;                    // planes in this call
    constexpr int SP = 1 << SPL;
    const int eres = SPL ? (int)blockIdx.y : 0;
    auto prow = [&](int k) { return k * SP + eres; };   // image row of transform output k
    // Offset of each first-pass input of this thread in plane 0 and its
    // per-plane stride (both the same for every plane): element (row j,
    // local column c0+seq) in the transposed layout
    // [s][plane - k0][g][row - row_start_s][x], where source s holds rows
    // [row_start_s, row_start_{s+1}) -- load-balanced slabs differ in height,
    // so a plane advances each source block by its own ncols * rows_s.
    // off = -1 past the last column.
    int off[kColE], pst[kColE];
    {
        auto offset = [&](int seq, int j) -> double2 {
            const int lc = c0 + seq;
            if (lc >= a.ncols) return make_double2(__hiloint2double(-1, 0), 0.0);
            int r0 = 0, r1 = a.src_start[1];
#pragma unroll
            for (int sidx = 1; sidx < 8; ++sidx)
                if (j >= a.src_start[sidx]) {
                    r0 = a.src_start[sidx];
                    r1 = a.src_start[sidx + 1];
                }
            const int o = nk * a.ncols * r0 + ((lc / kG) * (r1 - r0) + (j - r0)) * kG + (lc % kG);
            return make_double2(__hiloint2double(o, a.ncols * (r1 - r0)), 0.0);
        };
        double2 t[kColE];
        pass_load<LOGN, P0::RL, kColE, CT>(t, offset);
#pragma unroll
        for (int i = 0; i < kColE; ++i) {
            off[i] = __double2hiint(t[i].x);
            pst[i] = __double2loint(t[i].x);
        }
    }
    // The next plane's inputs are prefetched into the otherwise idle second
    // buffer while this plane is transformed: no registers held across it.
    // FP64: TMA bulk copies (cp.async.bulk, one elected thread, completion on
    // an mbarrier) of each column's contiguous runs -- one per source slab --
    // into [column][row]; each thread then reads its first-pass inputs from
    // shared memory. FP32 (8-byte elements, runs not always 16-byte
    // multiples): per-thread asynchronous copies (LDGSTS) into private slots.
    V *pbuf = reinterpret_cast<V *>(sbuf + C * STRIDE);
    constexpr bool BULK = sizeof(V) == 16 && SPL == 0;
    uint64_t *bar = reinterpret_cast<uint64_t *>(zbuf + C * N);
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bar);
    int lidx[kColE];   // BULK: this thread's first-pass inputs at pbuf[lidx[i]]
    if constexpr (BULK) {
        double2 t[kColE];
        pass_load<LOGN, P0::RL, kColE, CT>(
            t, [&](int seq, int j) { return make_double2(__hiloint2double(seq * N + j, 0), 0.0); });
#pragma unroll
        for (int i = 0; i < kColE; ++i) lidx[i] = __double2hiint(t[i].x);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
    }
    uint32_t bar_phase = 0;
    auto prefetch = [&](int k) {
        if constexpr (BULK) {
            if (threadIdx.x == 0) {
                // the buffer was read through the generic proxy: order that
                // before the async-proxy writes
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                uint32_t bytes = 0;
                for (int cc = 0; cc < C && c0 + cc < a.ncols; ++cc)
                    for (int sidx = 0; sidx < a.n_src; ++sidx)
                        bytes += (uint32_t)(a.src_start[sidx + 1] - a.src_start[sidx]) * (uint32_t)sizeof(V);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s), "r"(bytes)
                             : "memory");
                for (int cc = 0; cc < C && c0 + cc < a.ncols; ++cc)
                    for (int sidx = 0; sidx < a.n_src; ++sidx) {
                        const int r0 = a.src_start[sidx], r1 = a.src_start[sidx + 1];
                        const V *src = tg + (int64_t)nk * a.ncols * r0 +
                                       ((int64_t)k * a.ncols + c0 + cc) * (r1 - r0);
                        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(pbuf + cc * N + r0);
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                                dst),
                            "l"(src), "r"((uint32_t)((r1 - r0) * sizeof(V))), "r"(bar_s)
                            : "memory");
                    }
            }
        } else {
#pragma unroll
            for (int i = 0; i < kColE; ++i)
                if (off[i] >= 0)
                    __pipeline_memcpy_async(&pbuf[i * CT + threadIdx.x], &tg[off[i] + k * pst[i]],
                                            sizeof(V));
            __pipeline_commit();
        }
    };
    // split columns: input k of the on-chip transform combines rows k + s N
    auto ld_split = [&](int kpl, int seq, int j) -> V {
        const int lc = c0 + seq;
        if (lc >= a.ncols) return cx<V>(0.0, 0.0);
        V u = cx<V>(0.0, 0.0);
#pragma unroll
        for (int s = 0; s < SP; ++s) {
            const int row = j + s * N;
            int r0 = 0, r1 = a.src_start[1];
#pragma unroll
            for (int sidx = 1; sidx < 8; ++sidx)
                if (row >= a.src_start[sidx]) {
                    r0 = a.src_start[sidx];
                    r1 = a.src_start[sidx + 1];
                }
            const int64_t o = (int64_t)nk * a.ncols * r0 + ((int64_t)kpl * a.ncols + lc) * (r1 - r0) +
                              (row - r0);
            u = cadd(u, rot_quarter(tg[o], (4 / SP) * s * eres));
        }
        return eres ? cmul(u, __ldg(&twN[j * eres])) : u;
    };
    // direction-cosine factor of a pixel (mesh.py:202-208, transform.py:200)
    auto n_of = [&](int cc, int j) {
        const int gi = a.g0 * kG + c0 + cc;
        const double l = (double)(gi - a.n_u / 2) * a.cell;
        const double m = (double)(j - a.n_v / 2) * a.cell;
        return __dsqrt_rn(__dsub_rn(__dsub_rn(1.0, __dmul_rn(l, l)), __dmul_rn(m, m)));
    };

    const double dw = a.n_w > 1 ? (a.w_max - a.w_min) / (double)(a.n_w - 1) : 0.0;
    // z per pixel, staged once; with the TMA prefetch holding no registers the
    // thread's eight z then live in registers for every plane (WSB_COLS_ZREG:
    // cfg3 6.92 -> 6.47 ms; round 1, with register prefetch, they spilled)
    for (int e = threadIdx.x; e < C * N; e += CT)
        zbuf[e] = cis_pi(2.0 * dw * (n_of(e / N, prow(e % N)) - 1.0));

    // the running stack of the planes above this range continues
    double2 *run = a.run + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kColE * CT + threadIdx.x;
    double2 acc[kColE];
#pragma unroll
    for (int i = 0; i < kColE; ++i) acc[i] = a.k1 < a.k_top ? run[i * CT] : make_double2(0.0, 0.0);
    if constexpr (SPL == 0) prefetch(nk - 1);
#if WSB_COLS_ZREG
    // z of this thread's output pixels, in registers for every plane
    __syncthreads();
    double2 zr[kColE];
#pragma unroll
    for (int kb = 0; kb < NB; ++kb) {
        const int b = threadIdx.x + kb * CT;
        const int seq = b / M, j = b % M;
#pragma unroll
        for (int r = 0; r < R; ++r) zr[kb * R + r] = zbuf[seq * N + j + r * M];
    }
#endif

    for (int kl = nk - 1; kl >= 0; --kl) {
        V v[kColE];
        if constexpr (BULK) {
            asm volatile(
                "{\n .reg .pred p;\n WAIT_%=:\n"
                " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                " @!p bra WAIT_%=;\n}\n" ::"r"(bar_s),
                "r"(bar_phase)
                : "memory");
            bar_phase ^= 1;
#if WSB_COLS_ZREG
            pass_load<LOGN, P0::RL, kColE, CT>(
                v, [&](int seq, int j) { return c0 + seq < a.ncols ? pbuf[seq * N + j] : cx<V>(0.0, 0.0); });
#else
#pragma unroll
            for (int i = 0; i < kColE; ++i) v[i] = off[i] >= 0 ? pbuf[lidx[i]] : cx<V>(0.0, 0.0);
#endif
            __syncthreads();   // every thread has its inputs: the buffer takes the next plane
            if (kl > 0) prefetch(kl - 1);
            pass_compute<LOGN, P0::RL, kColE, CT>(1, tw, v);
        } else if constexpr (SPL == 0) {
            __pipeline_wait_prior(0);
#pragma unroll
            for (int i = 0; i < kColE; ++i)
                v[i] = off[i] >= 0 ? pbuf[i * CT + threadIdx.x] : cx<V>(0.0, 0.0);
            pass_compute<LOGN, P0::RL, kColE, CT>(1, tw, v);
            // v has been consumed from the slots: refill them with the next plane
            if (kl > 0) prefetch(kl - 1);
        } else {
            auto ld = [&](int seq, int j) { return ld_split(kl, seq, j); };
            pass_load<LOGN, P0::RL, kColE, CT>(v, ld);
            pass_compute<LOGN, P0::RL, kColE, CT>(1, tw, v);
        }
        if constexpr (!P0::LAST) {
            __syncthreads();  // the previous plane's last pass has read sbuf
            auto sst = [&](int seq, int idx, V z) { sv[seq * STRIDE + pidx(idx)] = z; };
            pass_store<LOGN, P0::RL, kColE, CT>(1, v, sst);
            __syncthreads();
            smem_passes<LOGN, RLM, kColE, CT, P0::RL>(sv, tw, v);
        }
        // v[kb*R + r] is output row j + r*M of sequence (column) seq
#pragma unroll
        for (int kb = 0; kb < NB; ++kb) {
            const int b = threadIdx.x + kb * CT;
            const int seq = b / M, j = b % M;
#pragma unroll
            for (int r = 0; r < R; ++r) {
#if WSB_COLS_ZREG
                const double2 z = zr[kb * R + r];
                (void)seq;
                (void)j;
#else
                const double2 z = zbuf[seq * N + j + r * M];
#endif
                const double2 p = to_d2(v[kb * R + r]);
                double2 &q = acc[kb * R + r];
                const double qx = fma(q.x, z.x, fma(-q.y, z.y, p.x));
                q.y = fma(q.x, z.y, fma(q.y, z.x, p.y));
                q.x = qx;
            }
        }
    }

    if (a.k0 > a.k_bottom) {  // planes below this range to come: park the running stack
#pragma unroll
        for (int i = 0; i < kColE; ++i) run[i * CT] = acc[i];
        return;
    }

    // finish: /(n_u n_v) (exact power of two), /n_w (numpy multiplies by the
    // reciprocal), * n (complex * real). Pixels go through shared memory so
    // the image strip is written row by row and the residual norms are
    // reduced per column in a fixed tree order (identical for any GPU count).
    __syncthreads();  // both plane buffers are free now
    const double w0 = plane_w(a, a.k0);   // k0 = k_bottom: phase of the lowest stacked plane
    if (a.pimg) {
        // partial stack of a plane range (w-plane decomposition): sum_k P_k
        // exp(2 pi i w_k (n-1)) over [k_bottom, k_top); summed over the ranks
        // and finished by k_image_finish
        double2 *pix = sbuf;
#pragma unroll
        for (int kb = 0; kb < NB; ++kb) {
            const int b = threadIdx.x + kb * CT;
            const int seq = b / M, j = b % M;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int row = j + r * M;
                const double n = n_of(seq, prow(row));
                pix[seq * STRIDE + pidx(row)] = cmul(acc[kb * R + r], cis_pi(2.0 * w0 * (n - 1.0)));
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < C * N; e += CT) {
            const int cc = e % C, row = e / C;
            if (c0 + cc < a.ncols)
                a.pimg[(int64_t)prow(row) * a.ncols + c0 + cc] = pix[cc * STRIDE + pidx(row)];
        }
        return;
    }
    double2 *pix = sbuf;                        // (re, im) per pixel, [C][STRIDE]
    double2 *sq = sbuf + C * STRIDE;            // (im^2, re^2) per pixel
#pragma unroll
    for (int kb = 0; kb < NB; ++kb) {
        const int b = threadIdx.x + kb * CT;
        const int seq = b / M, j = b % M;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int row = j + r * M;
            const double n = n_of(seq, prow(row));
            double2 z = cmul(acc[kb * R + r], cis_pi(2.0 * w0 * (n - 1.0)));
            z.x *= a.inv_nuv;
            z.y *= a.inv_nuv;
            z.x = __dmul_rn(z.x, a.inv_nw);
            z.y = __dmul_rn(z.y, a.inv_nw);
            const double re = __dsub_rn(__dmul_rn(z.x, n), __dmul_rn(z.y, 0.0));
            const double im = __dadd_rn(__dmul_rn(z.x, 0.0), __dmul_rn(z.y, n));
            pix[seq * STRIDE + pidx(row)] = make_double2(re, im);
            sq[seq * STRIDE + row] = make_double2(__dmul_rn(im, im), __dmul_rn(re, re));
        }
    }
    __syncthreads();
    // image rows: the C columns of a row are contiguous in the strip
    for (int e = threadIdx.x; e < C * N; e += CT) {
        const int cc = e % C, row = e / C;
        if (c0 + cc < a.ncols)
            a.strip[(int64_t)prow(row) * a.ncols + c0 + cc] = pix[cc * STRIDE + pidx(row)].x;
    }
    // per-column pairwise tree over the N rows
    for (int half = N / 2; half > 0; half >>= 1) {
        for (int e = threadIdx.x; e < C * half; e += CT) {
            const int cc = e / half, i = e % half;
            double2 *p = sq + cc * STRIDE;
            p[i] = make_double2(p[i].x + p[i + half].x, p[i].y + p[i + half].y);
        }
        __syncthreads();
    }
    for (int cc = threadIdx.x; cc < C; cc += CT)
        if (c0 + cc < a.ncols) {   // partials [residue][column][2]
            a.partials[2 * ((int64_t)eres * a.ncols + c0 + cc) + 0] = sq[cc * STRIDE].x;
            a.partials[2 * ((int64_t)eres * a.ncols + c0 + cc) + 1] = sq[cc * STRIDE].y;
        }
}

// Finish of a summed partial-stack image (w-plane decomposition): the same
// per-pixel operations as k_fft_cols' finish -- /(n_u n_v), /n_w, * n, real
// part -- and per-column residual norm partials [residue][column][2], row
// residues e = blockIdx.y summed in row order (fixed association).
__global__ void __launch_bounds__(256) k_image_finish(const double2 *__restrict__ sum, int n_u,
                                                      int n_v, double cell, double inv_nuv,
                                                      double inv_nw, double *__restrict__ image,
                                                      double *__restrict__ partials) {
    __shared__ double2 red[8][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int col = blockIdx.x * 32 + tx;
    const int rs = gridDim.y, e = blockIdx.y;
    const int rows = n_v / rs, r0 = e * rows;
    double2 s = make_double2(0.0, 0.0);
    if (col < n_u) {
        const double l = (double)(col - n_u / 2) * cell;
        for (int row = r0 + ty; row < r0 + rows; row += 8) {
            const double m = (double)(row - n_v / 2) * cell;
            const double n = __dsqrt_rn(__dsub_rn(__dsub_rn(1.0, __dmul_rn(l, l)), __dmul_rn(m, m)));
            double2 z = sum[(int64_t)row * n_u + col];
            z.x *= inv_nuv;
            z.y *= inv_nuv;
            z.x = __dmul_rn(z.x, inv_nw);
            z.y = __dmul_rn(z.y, inv_nw);
            const double re = __dsub_rn(__dmul_rn(z.x, n), __dmul_rn(z.y, 0.0));
            const double im = __dadd_rn(__dmul_rn(z.x, 0.0), __dmul_rn(z.y, n));
            image[(int64_t)row * n_u + col] = re;
            s.x += __dmul_rn(im, im);
            s.y += __dmul_rn(re, re);
        }
    }
    red[ty][tx] = s;
    __syncthreads();
    if (ty == 0 && col < n_u) {
        double2 t = red[0][tx];
        for (int k = 1; k < 8; ++k) t = make_double2(t.x + red[k][tx].x, t.y + red[k][tx].y);
        partials[2 * ((int64_t)e * n_u + col) + 0] = t.x;
        partials[2 * ((int64_t)e * n_u + col) + 1] = t.y;
    }
}

// pass-ordered twiddle table of an N-point plan (see tw_offset): entry [t]
// of the pass with span ns and radix R is exp(2 pi i m / N), m = t N / (ns R)
template <class V>
__global__ void k_twiddles(V *tw, int logn, int rlmax, int size) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= size) return;
    const int n = 1 << logn;
    int off = 0, d = 0, m = rlmax == 0 ? e : 0;
    while (rlmax != 0 && d < logn) {
        const int first = logn % rlmax;
        const int rl = (d == 0 && first != 0) ? first : rlmax;
        if (d > 0) {
            const int ns = 1 << d;
            if (e < off + ns) {
                m = (e - off) * (n >> (d + rl));
                break;
            }
            off += ns;
        }
        d += rl;
    }
    double sn, cs;
    sincospi(2.0 * (double)m / (double)n, &sn, &cs);
    tw[e] = cx<V>(cs, sn);
}

template <int LOGN, class V>
int launch_rows(wsb_ctx *ctx, const V *in, int n_strips, int n_groups, int v_count, int plo,
                int phi, const V *tw, const V *twN, const RowDest &dst, int spl) {
    constexpr int N = 1 << LOGN;
    constexpr int RT = RowCfg<LOGN>::T;
    constexpr int NSEQ = RT * kRowE / N;
    const size_t smem = sizeof(V) * NSEQ * Seq<LOGN>::STRIDE;
    dim3 grd(ceil_div(v_count, NSEQ), phi - plo, 1 << spl);
    if (spl == 0) {
        WSB_CUDA_TRY(cudaFuncSetAttribute(k_fft_rows<LOGN, 0, V>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // persistent CTAs: 16 x the resident count (measured: rows 1.08 ->
        // 0.99 ms at cfg2, 10.8 -> 9.5 ms at cfg3; 1-4 x is slower, and so is
        // an L2 prefetch of the next pair); WSB_ROW_PERSIST=0 launches one
        // CTA per row pair
        static int persist = -1, l2pf = 0;
        if (persist < 0) {
            const char *e = std::getenv("WSB_ROW_PERSIST");
            persist = e ? std::atoi(e) : 16;
            const char *f = std::getenv("WSB_ROW_L2PF");
            l2pf = f ? std::atoi(f) : 0;
        }
        if (persist > 0) {
            int per_sm = 0, dev = 0, n_sm = 0;
            WSB_CUDA_TRY(cudaGetDevice(&dev));
            WSB_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
            WSB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fft_rows<LOGN, 0, V>, RT, smem));
            const int64_t n_pairs = (int64_t)grd.x * grd.y;
            const int ctas = (int)std::min<int64_t>(n_pairs, (int64_t)per_sm * n_sm * persist);
            k_fft_rows<LOGN, 0, V><<<ctas, RT, smem, ctx->stream>>>(in, n_strips, n_groups, v_count, plo, tw,
                                                                     twN, dst, (int)grd.x, n_pairs, l2pf);
        } else {
            k_fft_rows<LOGN, 0, V><<<grd, RT, smem, ctx->stream>>>(in, n_strips, n_groups, v_count, plo,
                                                                   tw, twN, dst, 0, 0, 0);
        }
    } else if constexpr (LOGN == 12) {
        if (spl == 1) {
            WSB_CUDA_TRY(cudaFuncSetAttribute(k_fft_rows<LOGN, 1, V>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_fft_rows<LOGN, 1, V><<<grd, RT, smem, ctx->stream>>>(in, n_strips, n_groups, v_count,
                                                                   plo, tw, twN, dst, 0, 0, 0);
        } else if (spl == 2) {
            WSB_CUDA_TRY(cudaFuncSetAttribute(k_fft_rows<LOGN, 2, V>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_fft_rows<LOGN, 2, V><<<grd, RT, smem, ctx->stream>>>(in, n_strips, n_groups, v_count,
                                                                   plo, tw, twN, dst, 0, 0, 0);
        } else {
            return fail(WSB_EUNSUPPORTED, "row length above 16384");
        }
    } else {
        return fail(WSB_EUNSUPPORTED, "split rows run on the 4096-point transform");
    }
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

template <int LOGN, class V>
int launch_cols(wsb_ctx *ctx, const ColArgs &a, const V *tw, int *nblocks, int spl) {
    static_assert(kG == 1, "the split column loads assume the column-major P layout");
    constexpr int N = 1 << LOGN;
    constexpr int CT = ColCfg<LOGN>::T;
    constexpr int C = CT * kColE / N;
    // the finish stages complex128 pixels whatever the transform precision
    const size_t smem = sizeof(double2) * (2 * C * Seq<LOGN>::STRIDE + C * N) + 16;   // + mbarrier
    *nblocks = ceil_div(a.ncols, C);
    const dim3 grd(*nblocks, 1 << spl);
    if (spl == 0) {
        WSB_CUDA_TRY(cudaFuncSetAttribute(k_fft_cols<LOGN, 0, V>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_fft_cols<LOGN, 0, V><<<grd, CT, smem, ctx->stream>>>(a, tw);
    } else if constexpr (LOGN == 12) {
        if (spl == 1) {
            WSB_CUDA_TRY(cudaFuncSetAttribute(k_fft_cols<LOGN, 1, V>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_fft_cols<LOGN, 1, V><<<grd, CT, smem, ctx->stream>>>(a, tw);
        } else if (spl == 2) {
            WSB_CUDA_TRY(cudaFuncSetAttribute(k_fft_cols<LOGN, 2, V>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_fft_cols<LOGN, 2, V><<<grd, CT, smem, ctx->stream>>>(a, tw);
        } else {
            return fail(WSB_EUNSUPPORTED, "column length above 16384");
        }
    } else {
        return fail(WSB_EUNSUPPORTED, "split columns run on the 4096-point transform");
    }
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

template <class V>
int rows_dispatch(wsb_ctx *ctx, const wsb_grid *g, int v_count, const void *grid_a, int plo,
                  int phi, const RowDest &dst) {
    const int ng = g->n_u / kG, ns = ceil_div(g->n_u, WSB_STRIP);
    const int prec = sizeof(V) == 8 ? 32 : 64;
    // rows above the on-chip 4096 points: SP = n_u / 4096 residue CTAs per row
    const int logn = ilog2(g->n_u), logs = std::min(logn, kMaxOnChipLog), spl = logn - logs;
    const void *tw = nullptr, *twn = nullptr;
    WSB_TRY(twiddles(ctx, 1 << logs, kRowRL, &tw, prec));
    if (spl > 0) WSB_TRY(twiddles(ctx, g->n_u, 0, &twn, prec));
    const V *ga = (const V *)grid_a, *t2 = (const V *)tw, *tn = (const V *)twn;
    switch (logs) {
#define WSB_ROWS(L) \
    case L: return launch_rows<L, V>(ctx, ga, ns, ng, v_count, plo, phi, t2, tn, dst, spl);
        WSB_ROWS(1) WSB_ROWS(2) WSB_ROWS(3) WSB_ROWS(4) WSB_ROWS(5) WSB_ROWS(6)
        WSB_ROWS(7) WSB_ROWS(8) WSB_ROWS(9) WSB_ROWS(10) WSB_ROWS(11) WSB_ROWS(12)
#undef WSB_ROWS
        default: return fail(WSB_EUNSUPPORTED, "transform length not supported");
    }
}

template <class V>
int cols_dispatch(wsb_ctx *ctx, ColArgs &a, int n_v) {
    const int prec = sizeof(V) == 8 ? 32 : 64;
    const int logn = ilog2(n_v), logs = std::min(logn, kMaxOnChipLog), spl = logn - logs;
    const void *tw = nullptr, *twn = nullptr;
    WSB_TRY(twiddles(ctx, 1 << logs, kColRL, &tw, prec));
    if (spl > 0) WSB_TRY(twiddles(ctx, n_v, 0, &twn, prec));
    a.twN = twn;
    const V *t2 = (const V *)tw;
    int nb = 0;
    switch (logs) {
#define WSB_COLS(L) \
    case L: return launch_cols<L, V>(ctx, a, t2, &nb, spl);
        WSB_COLS(1) WSB_COLS(2) WSB_COLS(3) WSB_COLS(4) WSB_COLS(5) WSB_COLS(6)
        WSB_COLS(7) WSB_COLS(8) WSB_COLS(9) WSB_COLS(10) WSB_COLS(11) WSB_COLS(12)
#undef WSB_COLS
        default: return fail(WSB_EUNSUPPORTED, "transform length not supported");
    }
}

}  // namespace

int twiddles(wsb_ctx *ctx, int n, int rlmax, const void **out, int prec) {
    // rlmax 3/4: pass-ordered table of an n-point plan; 0: plain exp(2 pi i m / n);
    // complex128 (prec 64) or complex64 (prec 32) entries
    const int l = ilog2(n);
    if (!(rlmax == 0 || rlmax == 3 || rlmax == 4) || l > 15) return fail(WSB_EINVAL, "twiddle table");
    const int key = l + 16 * (rlmax == 0 ? 2 : rlmax - 3) + (prec == 32 ? 48 : 0);
    if (!ctx->twiddle[key]) {
        const int size = rlmax == 0 ? n : std::max(1, tw_offset(l, rlmax, l));
        if (prec == 32) {
            WSB_CUDA_TRY(cudaMalloc(&ctx->twiddle[key], sizeof(float2) * size));
            k_twiddles<float2><<<ceil_div(size, 256), 256, 0, ctx->stream>>>(
                (float2 *)ctx->twiddle[key], l, rlmax, size);
        } else {
            WSB_CUDA_TRY(cudaMalloc(&ctx->twiddle[key], sizeof(double2) * size));
            k_twiddles<double2><<<ceil_div(size, 256), 256, 0, ctx->stream>>>(
                (double2 *)ctx->twiddle[key], l, rlmax, size);
        }
        ctx->launches += 1;
        WSB_CUDA_TRY(cudaGetLastError());
    }
    *out = ctx->twiddle[key];
    return WSB_OK;
}

int fft_rows(wsb_ctx *ctx, const wsb_grid *g, int v_count, const void *grid_a, void *grid_p,
             int plo, int phi, int n_dest, const int32_t *dest_groups, void *const *dest_ptrs,
             int prec) {
    if (phi <= plo || v_count <= 0) return WSB_OK;
    const int ng = g->n_u / kG;
    const size_t esz = prec == 32 ? sizeof(float2) : sizeof(double2);
    RowDest dst;
    if (n_dest < 1 || n_dest > 8) return fail(WSB_EINVAL, "n_dest must be in [1, 8]");
    dst.g0[0] = 0;
    for (int d = 0; d < n_dest; ++d) dst.g0[d + 1] = dst.g0[d] + (dest_groups ? dest_groups[d] : ng);
    if (dst.g0[n_dest] != ng) return fail(WSB_EINVAL, "destination column groups must sum to n_u/G");
    for (int d = n_dest + 1; d < 9; ++d) dst.g0[d] = 0x7fffffff;
    for (int d = 0; d < 8; ++d) dst.ptr[d] = nullptr;
    if (dest_ptrs) {
        // fused transpose: every destination's block holds all n_w planes
        dst.plane0 = 0;
        for (int d = 0; d < n_dest; ++d) {
            if (!dest_ptrs[d]) return fail(WSB_EINVAL, "NULL destination pointer");
            dst.ptr[d] = dest_ptrs[d];
        }
    } else {
        // local destination-major buffer holding planes [plo, phi) only
        dst.plane0 = plo;
        for (int d = 0; d < n_dest; ++d)
            dst.ptr[d] = (char *)grid_p + esz * (int64_t)(phi - plo) * v_count * kG * dst.g0[d];
    }
    return prec == 32 ? rows_dispatch<float2>(ctx, g, v_count, grid_a, plo, phi, dst)
                      : rows_dispatch<double2>(ctx, g, v_count, grid_a, plo, phi, dst);
}

int fft_cols_stack(wsb_ctx *ctx, const wsb_grid *g, int n_sources, const int32_t *src_rows,
                   int g0, int ng, int plo, int phi, const void *tgrid, double *image_strip,
                   double *norm_partials, int prec, int k_bottom, int k_top, double *partial_img) {
    if (phi <= plo) return WSB_OK;
    if (k_top < 0) k_top = g->n_w;
    if (!(0 <= k_bottom && k_bottom <= plo && phi <= k_top && k_top <= g->n_w))
        return fail(WSB_EINVAL, "plane range outside the stacked planes");
    if (n_sources < 1 || n_sources > 8) return fail(WSB_EINVAL, "n_sources must be in [1, 8]");
    ColArgs a;
    a.tgrid = tgrid;
    a.strip = image_strip;
    a.partials = norm_partials;
    a.n_w = g->n_w;
    a.n_u = g->n_u;
    a.n_v = g->n_v;
    a.ncols = ng * kG;
    a.g0 = g0;
    a.n_src = n_sources;
    a.src_start[0] = 0;
    for (int s = 0; s < n_sources; ++s) a.src_start[s + 1] = a.src_start[s] + src_rows[s];
    for (int s = n_sources + 1; s < 9; ++s) a.src_start[s] = 1 << 30;
    if (a.src_start[n_sources] != g->n_v) return fail(WSB_EINVAL, "source rows must sum to n_v");
    for (int s = 0; s < n_sources; ++s)
        if (src_rows[s] < 1) return fail(WSB_EINVAL, "every source slab needs at least one row");
    a.cell = g->cell_size_lm;
    a.inv_nuv = 1.0 / ((double)g->n_u * (double)g->n_v);
    a.inv_nw = 1.0 / (double)g->n_w;
    a.w_min = g->w_min_native;
    a.w_max = g->w_max_native;
    a.k0 = plo;
    a.k1 = phi;
    a.k_top = k_top;
    a.k_bottom = k_bottom;
    a.pimg = (double2 *)partial_img;
    // columns above the on-chip 4096 points: SP = n_v / 4096 residue CTAs
    const int logn = ilog2(g->n_v), logs = std::min(logn, kMaxOnChipLog), spl = logn - logs;
    // the running stack (complex128): one per thread element of the launch
    {
        const int ct = std::max((1 << logs) / 8, 256), cpb = std::max(1, ct * 8 / (1 << logs));
        const size_t bytes = sizeof(double2) * (size_t)ceil_div(a.ncols, cpb) * ct * 8 << spl;
        WSB_TRY(ensure(ctx, kSlotColRun, bytes, (void **)&a.run));
    }
    return prec == 32 ? cols_dispatch<float2>(ctx, a, g->n_v) : cols_dispatch<double2>(ctx, a, g->n_v);
}

int image_finish(wsb_ctx *ctx, const wsb_grid *g, const double *sum, double *image,
                 double *norm_partials) {
    const int rs = WSB_FINISH_SPLIT(g->n_v);
    k_image_finish<<<dim3(ceil_div(g->n_u, 32), rs), 256, 0, ctx->stream>>>(
        (const double2 *)sum, g->n_u, g->n_v, g->cell_size_lm, 1.0 / ((double)g->n_u * (double)g->n_v),
        1.0 / (double)g->n_w, image, norm_partials);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

}  // namespace wsb
