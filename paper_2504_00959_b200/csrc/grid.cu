// K2: tensor-core window gridder over (plane, 16-column strip, 128-row
// block) work items (gridder.py:160-259, Eq. 3).
//
// CTA = one warp = one item (or one part of a heavy item): the warp owns the
// item's 16 columns (WSB_ITEM_COLS; a build can widen items to 2-4 strips,
// one warp each). Its accumulator is a window of 8-row tiles held as FP64 MMA
// fragments (m8n8k4: lane = row lane/4, columns 2(lane%4), +1 of an 8x8 tile;
// two column halves x Re/Im per tile). The item's records arrive sorted by
// anchor row (K1); four records at a time are applied as rank-4 updates
// D += A B of every tile they reach, A = their v weights on the tile rows
// (row sign folded), B = value x u weight on the columns (column sign folded)
// -- one DMMA instruction per 256 multiply-adds on the FP64 tensor cores.
// When the records move past a tile it is final: the 32 lanes store it (8
// rows x 16 columns, re | im) straight from the fragments, clear it and the
// window moves 8 rows down (a ring of tiles, one code copy per ring phase).
//
// Each cell accumulates in (anchor row, record) order in groups of four --
// deterministic, and the same for any GPU count when slabs start on 128-row
// boundaries (items then hold the same records) -- and is written once: no
// shared-memory tile, no atomics, no read-modify-write of HBM.
//
// One warp per item keeps skewed data cheap: with four strips per CTA the
// strips of an Earth-rotation track item carry very different record counts
// and three warps waited at every chunk barrier (cfg3: 16.0 -> 10.6 ms). The
// price is K1 entries for each 16-column strip a record reaches (1.36 per
// record at cfg2 instead of 1.12 per 64-column block).
//
// Records stream through the warp in chunks of 32 gathered by cp.async one
// chunk ahead (record index prefetched a chunk before its gather). One lane
// stages a record: value x u weight per window column and the v weights of
// its footprint rows (the sweep offsets them by the record's first row in
// its 8-row step) -- no divergent per-axis tails (K2 1.06 -> 0.95 ms at cfg2).
#include <type_traits>

#include "i0_coeffs.h"
#include "wsb_internal.cuh"

namespace wsb {
namespace {

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

// exp(x) for -700 < x < 700: x = k ln2 + r, |r| <= ln2/2 (two-constant
// Cody-Waite), Taylor to r^14 (truncation < 1e-17), 2^k added to the
// exponent field. A few ulp; no special-case paths.
// Constants in the constant bank (DFMA c[][] operands instead of UMOV pairs).
__constant__ double kExpC[18] = {1.4426950408889634, 0.6931471805599453, 2.3190468138462996e-17,
                                 1.1470745597729725e-11, 1.6059043836821613e-10,
                                 2.08767569878681e-09, 2.505210838544172e-08,
                                 2.755731922398589e-07, 2.7557319223985893e-06,
                                 2.48015873015873e-05, 0.0001984126984126984,
                                 0.001388888888888889, 0.008333333333333333,
                                 0.041666666666666664, 0.16666666666666666, 0.5, 1.0, 1.0};

__device__ __forceinline__ double fast_exp(double x) {
    const double k = rint(x * kExpC[0]);
    double r = fma(-k, kExpC[1], x);
    r = fma(-k, kExpC[2], r);
    double p = kExpC[3];
#pragma unroll
    for (int i = 4; i < 18; ++i) p = fma(p, r, kExpC[i]);
    return __hiloint2double(__double2hiint(p) + ((int)k << 20), __double2loint(p));
}

template <int S>
struct KParams {
    static constexpr int W = 2 * S + 1;
    static constexpr int NKB = 12 + 4 * S;   // Kaiser-Bessel series terms (beta up to ~3.5 S)
    double p0;              // Gaussian: 2 sigma^2; Kaiser-Bessel: beta
    double inv_p0;          // 1 / p0
    double cm[W];           // Gaussian: exp(-m^2/s2), m = S-k (factorised path)
    double kb[NKB];         // Kaiser-Bessel: (beta^2/4)^k / (k!)^2 / I0(beta)
    int factorised;         // Gaussian: 1 if the factorised form cannot overflow
    int series;             // Kaiser-Bessel: 1 if the NKB-term series is exact to 1e-17
};

// Weights of one axis for window taps k = 0..W-1 at offsets d_k = g - (i0+k):
// inclusion |d_k| <= S (reference test) and the per-axis kernel factor of
// kernel_value (gridder.py:75-98). The Gaussian product of the two axes
// equals exp(-(du^2+dv^2)/s2) to a few ulp; it is evaluated as
//   exp(-(f+m)^2/s2) = exp(-f^2/s2) * exp(-2f/s2)^m * exp(-m^2/s2),
//   f = d_S = g - floor(g), m = S - k,
// i.e. 2 exps per axis instead of W, when no factor can overflow.
template <int KIND, int S>
__device__ __forceinline__ uint32_t axis_weights(double g, int i0, const KParams<S> &kp,
                                                 double i0beta, double *w) {
    constexpr int W = 2 * S + 1;
    // with i0 = floor(g) - S, d_k = g - (i0 + k) lies in (S - k - 1, S - k]
    // exactly for k >= 1 (Sterbenz): |d_k| <= S holds for k = 1..2S; only the
    // first tap needs the reference's rounded test |g - i| <= S
    uint32_t mask = (2u << (W - 1)) - 2u;
    mask |= (uint32_t)(fabs(__dsub_rn(g, (double)i0)) <= (double)S);
    if (KIND == WSB_KERNEL_GAUSSIAN && kp.factorised) {
        const double f = __dsub_rn(g, (double)(i0 + S));
        // (multiplying by 1/s2 instead of dividing: a few ulp, no FP64 division)
        const double a = fast_exp(-__dmul_rn(f, f) * kp.inv_p0);
        const double b = fast_exp(-2.0 * f * kp.inv_p0);  // m > 0 side
        const double bi = __drcp_rn(b);                         // m < 0 side
        w[S] = a;
        double pb = a, pbi = a;
#pragma unroll
        for (int m = 1; m <= S; ++m) {
            pb *= b;
            pbi *= bi;
            w[S - m] = pb * kp.cm[S - m];   // k = S - m, offset f + m
            w[S + m] = pbi * kp.cm[S + m];  // k = S + m, offset f - m
        }
    } else {
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const double d = __dsub_rn(g, (double)(i0 + k));
            if (KIND == WSB_KERNEL_GAUSSIAN) {
                w[k] = exp(__ddiv_rn(-__dmul_rn(d, d), kp.p0));
            } else {
                // I0(beta sqrt(t)) / I0(beta), t = 1 - (d/S)^2 (gridder.py:92-98),
                // as the power series sum_k (beta^2 t / 4)^k / (k!)^2 / I0(beta):
                // positive terms, no cancellation, no exp/sqrt/division --
                // within a few ulp of np.i0's Chebyshev evaluation
                if (kp.series) {
                    // t = 1 - d^2/S^2 without the FP64 division (a few ulp)
                    constexpr double kInvS2 = 1.0 / (double)(S * S);
                    const double t = fmax(fma(-d, d * kInvS2, 1.0), 0.0);
                    double p = kp.kb[KParams<S>::NKB - 1];
#pragma unroll
                    for (int q = KParams<S>::NKB - 2; q >= 0; --q) p = fma(p, t, kp.kb[q]);
                    w[k] = p;
                } else {  // large beta: np.i0's own Chebyshev evaluation
                    const double x = __ddiv_rn(d, (double)S);
                    const double t = fmax(__dsub_rn(1.0, __dmul_rn(x, x)), 0.0);
                    w[k] = __ddiv_rn(bessel_i0(__dmul_rn(kp.p0, __dsqrt_rn(t))), i0beta);
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < W; ++k)
        if (!((mask >> k) & 1)) w[k] = 0.0;
    return mask;
}


// Calls f(std::integral_constant<int, phase>) for a runtime phase in [0, N).
template <int I, int N, class F>
__device__ __forceinline__ void dispatch_phase(int phase, F &&f) {
    if constexpr (I < N) {
        if (phase == I)
            f(std::integral_constant<int, I>{});
        else
            dispatch_phase<I + 1, N>(phase, f);
    }
}

constexpr int kC = WSB_STRIP;          // columns per warp strip
constexpr int kSS = kSSCols;           // item width (WSB_ITEM_COLS)
constexpr int kWarps = kSS / kC;       // strips (warps) per item
constexpr int kThreads = 32 * kWarps;
// WSB_STAGE_ONE: one lane stages a whole record (both axes; the v weights
// stored compactly, 8-row offset applied when the sweep reads them) instead
// of a lane pair splitting the axes (the warp then runs both axes' tails)
#ifndef WSB_STAGE_ONE
#define WSB_STAGE_ONE 1
#endif
constexpr bool kOne = WSB_STAGE_ONE && kWarps == 1;
constexpr int kLPR = kOne ? 1 : 2;       // lanes per record (gather and staging)
constexpr int kRPR = kThreads / kLPR;    // records per gather / staging round
#ifndef WSB_CHUNK
#define WSB_CHUNK 32
#endif
constexpr int kChunk = WSB_CHUNK;      // records staged per round (<= 255: byte indices)
constexpr int kCM = kChunk / kRPR;     // gather / staging rounds per chunk
static_assert(kChunk % kRPR == 0 && (kWarps == 1 || kChunk % 32 == 0) && kChunk < 256, "chunk");
#ifndef WSB_RAW
#define WSB_RAW 2
#endif
constexpr int kRaw = WSB_RAW;          // gather ring: chunks in flight

struct SweepArgs {
    const double4 *rec;
    const uint32_t *keys;      // sorted entries: item | rowrel << item_bits
    const uint32_t *idx;       // record index per entry
    const uint4 *parts;        // (item, first entry, end entry, slot | ~0 = direct)
    uint2 *part_rows;          // split parts: rows [lo, hi) (relative to the block) they wrote
    void *out;                 // strip layout [n_w][n_u/16][v_count][16]
    double2 *partial;          // [slot][kItemRows][kSS] partial tiles of split items
    unsigned long long *updates;
    const double *i0beta;      // device scalar, np.i0(beta) (Kaiser-Bessel)
    int out_f32;               // 1: complex64 grid (FP32 path; accumulation stays FP64)
    int n_u, v_start, v_count, n_ss, n_rb, item_bits, n_s16;
    int64_t n_parts;           // launched CTAs (the count or an upper bound of it)
    const uint32_t *n_parts_dev, *n_split_dev;   // the actual counts (device)
    int64_t n_rec, out_elems;  // bounds (debug checks)
};

// Window of the tensor-core sweep: a ring of NT tiles of 8 rows; a window
// step is 8 rows. A record anchored at offset d (0..7) in its step's first
// tile covers rows d .. d+2S: NTR = ceil((2S+8)/8) tiles from its step.
// WSB_WIN_EXTRA extra tiles let a group of records span that many steps.
#ifndef WSB_WIN_EXTRA
#define WSB_WIN_EXTRA 0
#endif
template <int S>
struct Win {
    static constexpr int W = 2 * S + 1;
    static constexpr int NTR = (W + 7 + 7) / 8;     // 2 for S <= 4, 3 for S <= 8
    static constexpr int NT = NTR + WSB_WIN_EXTRA;
};

// One staged record: everything a lane reads to apply it, at one base
// address (one IMAD per record).
template <int S>
struct StagedRec {
    static constexpr int W = 2 * S + 1;
    static constexpr int NV = kOne ? (W + 1) & ~1 : 8 * Win<S>::NTR;
    double2 tu[W + 1];     // value * u weight per window column; slot W = 0 (signs folded)
    double wv[NV];         // v weight of row b = d .. d+W-1 of the record's step; 0 elsewhere
                           // (kOne: of footprint row k = 0 .. W-1, signs folded)
    int4 meta;             // (first window column - item col0, window step, row offset d, strip mask)
};

template <int KIND, int S>
struct Shm {
    static constexpr int NROW = kItemRows + 2 * S;   // anchor rows that reach the item
    StagedRec<S> rec[kChunk + 1];   // + a zero sentinel filling the last group
    double4 raw[kRaw][kChunk];      // gathered records (gu, gv, Re, Im)
    uint8_t prec[kWarps][kChunk];   // per strip: the chunk's records touching it, in order
};

template <int KIND, int S>
constexpr int sweep_min_blocks() {
    // measured per kernel: Gaussian S <= 4 21 (80 registers either way, 21
    // schedules better than 24: 0.955 -> 0.911 ms at cfg2); Kaiser-Bessel
    // 2 <= S <= 4 18 (94 registers, no spills: support 7 14.6 -> 13.4 ms);
    // S > 4 14
    return (S > 4 ? 14 : (KIND == WSB_KERNEL_KAISER_BESSEL && S >= 2) ? 18 : 21) / kWarps;
}

// m8n8k4 FP64 MMA, D = A B + D: a(row lane/4, k lane%4), b(k lane%4, col lane/4),
// d(row lane/4, cols 2(lane%4), 2(lane%4)+1)
__device__ __forceinline__ void dmma(double2 &d, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d.x), "+d"(d.y)
                 : "d"(a), "d"(b));
}

template <int KIND, int S>
__global__ void __launch_bounds__(kThreads, sweep_min_blocks<KIND, S>())
    k_grid_items(SweepArgs a, KParams<S> kp) {
    constexpr int W = 2 * S + 1;
    using Sm = Shm<KIND, S>;
    using Rec = StagedRec<S>;
    constexpr int NT = Win<S>::NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Sm &sm = *reinterpret_cast<Sm *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (blockIdx.x >= *a.n_parts_dev) return;   // (grids sized by an upper bound)
    const uint4 pd = a.parts[blockIdx.x];
    const int64_t item = pd.x;
    const int rb = (int)(item % a.n_rb);
    const int64_t pt = item / a.n_rb;
    const int ss = (int)(pt % a.n_ss);
    const int plane = (int)(pt / a.n_ss);
    const int col0 = ss * kSS;
    const int R0 = a.v_start + rb * kItemRows;
    const int R1 = min(R0 + kItemRows, a.v_start + a.v_count);
    const int Bfirst = R0 - 2 * S;      // first anchor row that reaches the block: window base of step 0
    const uint32_t eb = pd.y, n = pd.z - pd.y;
    const bool direct = pd.w == 0xFFFFFFFFu;

    // The part's entries arrive sorted by (anchor row, record) -- the order
    // every cell accumulates in, whatever the slab split. A direct part
    // sweeps (and writes) the whole block; a split part only the rows its
    // records reach, recorded for k_combine.
    const int rr_first = n ? (int)(__ldg(&a.keys[eb]) & 0xFFu) : 0;
    const int rr_last = n ? (int)(__ldg(&a.keys[eb + n - 1]) & 0xFFu) : 0;
    const int step0 = direct ? 0 : rr_first >> 3;
    const int row_end = direct ? R1 : min(R1, Bfirst + rr_last + 2 * S + 1);
    if (!direct && tid == 0)
        a.part_rows[blockIdx.x] = make_uint2((uint32_t)max(Bfirst + 8 * step0 - R0, 0),
                                             (uint32_t)max(row_end - R0, 0));

    // ---- the sweep --------------------------------------------------------
    // Warp w owns columns [16w, 16w+16) of the item. Its window holds
    // rows B .. B + 8 NT - 1 (B = Bfirst + 8 step) as a ring of NT tiles of 8
    // rows: tile (phase + t) % NT holds rows B + 8t .. B + 8t + 7, as four 8x8
    // FP64 MMA accumulators (two 8-column halves x Re/Im; lane holds row
    // lane/4, columns 2(lane%4), +1). The records of a window step (anchor
    // rows B .. B+7) are applied four at a time as one rank-4 update per tile
    // they reach: A = their v weights on the tile's rows, B = value x u weight
    // on its columns (FP64 tensor cores: one MMA instruction per 256
    // multiply-adds). When the records move on to a later step, tile `phase`
    // (rows B .. B+7) is final: the 32 lanes write it (8 rows x 16 columns,
    // re | im, 2 KB), clear it, and the window moves 8 rows down.
    const double i0b = KIND == WSB_KERNEL_KAISER_BESSEL ? *a.i0beta : 0.0;
    const bool f32 = direct && a.out_f32;
    const int g4 = lane >> 2, k4 = lane & 3;       // MMA fragment coordinates
    double2 acc[NT][2][2];                         // [ring tile][column half][Re, Im]
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[t][h][0] = acc[t][h][1] = make_double2(0.0, 0.0);
    int step = step0, phase = step0 % NT;
    unsigned cnt_upd = 0;
    const int64_t strip_base = ((int64_t)plane * a.n_s16 + (col0 / kC + warp)) * a.v_count;
    double2 *const ptile = direct ? nullptr : a.partial + (int64_t)pd.w * kItemRows * kSS;
    // Output strip rows hold 16 real parts, then 16 imaginary parts: a lane's
    // two columns of a half are one 16-byte store straight from its
    // accumulator fragment. Lane row at step s: Bfirst + 8 s + g4.
    const int c_lane = 2 * k4;
    double *const ob = direct ? reinterpret_cast<double *>(a.out) +
                                    (strip_base + ((int64_t)Bfirst + g4 - a.v_start)) * (2 * kC) + c_lane
                              : nullptr;
    float *const ob32 = direct ? reinterpret_cast<float *>(a.out) +
                                     (strip_base + ((int64_t)Bfirst + g4 - a.v_start)) * (2 * kC) + c_lane
                               : nullptr;
    const bool col_ok = col0 + warp * kC + c_lane < a.n_u;

    // tile `P` (rows B .. B+7) final: write, clear, move the window
    auto emit = [&](auto P) {
        constexpr int p = decltype(P)::value;
        const int row = Bfirst + 8 * step + g4;
        if (row >= R0 && row < R1 && col_ok) {
            if (direct) {
                const int64_t o = (int64_t)step * (16 * kC);        // 8 rows x (16 re + 16 im)
                if (f32) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        *reinterpret_cast<float2 *>(ob32 + o + 8 * h) =
                            make_float2((float)acc[p][h][0].x, (float)acc[p][h][0].y);
                        *reinterpret_cast<float2 *>(ob32 + o + kC + 8 * h) =
                            make_float2((float)acc[p][h][1].x, (float)acc[p][h][1].y);
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        *reinterpret_cast<double2 *>(ob + o + 8 * h) = acc[p][h][0];
                        *reinterpret_cast<double2 *>(ob + o + kC + 8 * h) = acc[p][h][1];
                    }
                }
            } else {
                // partial tile [row][re | im][kSS columns] of the item
                double *pt_ = reinterpret_cast<double *>(ptile) + (int64_t)(row - R0) * (2 * kSS) +
                              warp * kC + c_lane;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    *reinterpret_cast<double2 *>(pt_ + 8 * h) = acc[p][h][0];
                    *reinterpret_cast<double2 *>(pt_ + kSS + 8 * h) = acc[p][h][1];
                }
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[p][h][0] = acc[p][h][1] = make_double2(0.0, 0.0);
        ++step;
        phase = (p + 1 == NT) ? 0 : p + 1;
    };

    // gather: thread pair (2r, 2r+1) copies the two 16-byte halves of
    // records r, r + kRPR, ...; an entry's record index is loaded one chunk
    // before its gather
    const int nchunks = (int)((n + kChunk - 1) / kChunk);
    struct Ids { uint32_t v[kCM]; };
    auto index_of = [&](int ch) -> Ids {
        Ids ids;
#pragma unroll
        for (int q = 0; q < kCM; ++q) {
            const uint32_t r = ch * kChunk + q * kRPR + tid / kLPR;
            ids.v[q] = (ch < nchunks && r < n) ? __ldg(&a.idx[eb + r]) : 0u;
        }
        return ids;
    };
    auto fetch = [&](int ch, const Ids &ids) {
        if (ch < nchunks) {
#pragma unroll
            for (int q = 0; q < kCM; ++q) {
                const uint32_t r = ch * kChunk + q * kRPR + tid / kLPR;
                if (r < n) {
                    const uint32_t id = ids.v[q];
                    WSB_DCHECK(id < a.n_rec, "item %lld id %u", (long long)item, id);
#pragma unroll
                    for (int h = (kLPR == 2 ? (tid & 1) : 0); h < 2; h += kLPR) {
                        const double2 *src = reinterpret_cast<const double2 *>(a.rec + id) + h;
                        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(
                            reinterpret_cast<double2 *>(&sm.raw[ch % kRaw][q * kRPR + tid / kLPR]) + h);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
                    }
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
#pragma unroll
    for (int ch = 0; ch < kRaw - 1; ++ch) fetch(ch, index_of(ch));
    Ids nid = index_of(kRaw - 1);

    const unsigned char *const recbase = reinterpret_cast<const unsigned char *>(&sm.rec[0]);
    // the sentinel: zero weights
    for (int e = tid; e < (int)(sizeof(Rec) / 8); e += kThreads)
        reinterpret_cast<double *>(&sm.rec[kChunk])[e] = 0.0;
    const double rs = (Bfirst & 1) ? -1.0 : 1.0;    // (-1)^row of window row 0 (8 step is even)
    for (int ch = 0; ch < nchunks; ++ch) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kRaw - 2) : "memory");
        __syncthreads();   // raw[ch] landed for every thread; the previous sweep is done
        fetch(ch + kRaw - 1, nid);
        nid = index_of(ch + kRaw);
        const int nr = (int)min((uint32_t)kChunk, n - (uint32_t)ch * kChunk);
        // ---- stage: thread pair per record, thread (2r + ax) does axis ax of
        // record r. Both axes run the same weight code (one instruction stream
        // for the warp); only the short tails differ.
        if constexpr (kOne) {
#pragma unroll 1
            for (int q = 0; q < kCM; ++q) {
                const int r = q * kRPR + tid;
                if (r < nr) {
                    const double4 rc = sm.raw[ch % kRaw][r];
                    Rec &st = sm.rec[r];
                    double wgt[W];
                    // u axis: value * weight per window column, column sign folded
                    // (transform.py:180-185; a sign flip commutes with rounding)
                    const int i0 = (int)floor(rc.x) - S;
                    const uint32_t wmu = axis_weights<KIND, S>(rc.x, i0, kp, i0b, wgt);
                    const double cs = (i0 & 1) ? -1.0 : 1.0;
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        const double wk = (k & 1) ? -cs * wgt[k] : cs * wgt[k];
                        st.tu[k] = make_double2(__dmul_rn(rc.z, wk), __dmul_rn(rc.w, wk));
                    }
                    st.tu[W] = make_double2(0.0, 0.0);
                    const int k_lo = max(col0 - i0, 0), k_hi = min(min(col0 + kSS, a.n_u) - i0, W) - 1;
                    const uint32_t uin = k_hi >= k_lo ? wmu & (((2u << k_hi) - 1u) & ~((1u << k_lo) - 1u)) : 0u;
                    // v axis: weight of footprint row k, row sign (-1)^row folded
                    const int j0 = (int)floor(rc.y) - S;
                    const uint32_t wmv = axis_weights<KIND, S>(rc.y, j0, kp, i0b, wgt);
                    const int rel = j0 - Bfirst;
                    WSB_DCHECK(rel >= 0 && rel < Sm::NROW, "item %lld rel %d", (long long)item, rel);
                    const double sj = (rel & 1) ? -rs : rs;
#pragma unroll
                    for (int k = 0; k < W; ++k) st.wv[k] = (k & 1) ? -sj * wgt[k] : sj * wgt[k];
                    st.meta = make_int4(i0 - col0, rel >> 3, rel & 7, uin ? 1 : 0);
                    // cell updates inside this item (grid_sector's count): u taps x v taps
                    const int r_lo = max(R0 - j0, 0), r_hi = min(R1 - j0, W) - 1;
                    cnt_upd += __popc(uin) *
                               __popc(r_hi >= r_lo ? wmv & (((2u << r_hi) - 1u) & ~((1u << r_lo) - 1u)) : 0u);
                }
            }
        } else
#pragma unroll 1
        for (int q = 0; q < kCM; ++q) {
            const int r = q * kRPR + (tid >> 1), ax = tid & 1;
            unsigned mine = 0;      // taps of this axis inside the item
            if (r < nr) {
                const double4 rc = sm.raw[ch % kRaw][r];
                Rec &st = sm.rec[r];
                double wgt[W];
                const double g = ax ? rc.y : rc.x;
                const int i0 = (int)floor(g) - S;
                const uint32_t wm = axis_weights<KIND, S>(g, i0, kp, i0b, wgt);
                if (ax == 0) {
                    // u axis: value * weight per window column, with the column
                    // factor (-1)^i of the checkerboard sign (transform.py:180-185;
                    // a sign flip commutes with rounding)
                    const double cs = (i0 & 1) ? -1.0 : 1.0;
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        const double wk = (k & 1) ? -cs * wgt[k] : cs * wgt[k];
                        st.tu[k] = make_double2(__dmul_rn(rc.z, wk), __dmul_rn(rc.w, wk));
                    }
                    st.tu[W] = make_double2(0.0, 0.0);
                    // tap columns inside the item (and the mesh); the strips they touch
                    const int k_lo = max(col0 - i0, 0), k_hi = min(min(col0 + kSS, a.n_u) - i0, W) - 1;
                    const uint32_t uin = k_hi >= k_lo ? wm & (((2u << k_hi) - 1u) & ~((1u << k_lo) - 1u)) : 0u;
                    int mask = 0;
                    if (uin) {
                        const int w_lo = (i0 + __ffs(uin) - 1 - col0) / kC;
                        const int w_hi = (i0 + 31 - __clz(uin) - col0) / kC;
                        mask = ((2 << w_hi) - 1) & ~((1 << w_lo) - 1);
                    }
                    st.meta.x = i0 - col0;
                    st.meta.w = mask;
                    mine = __popc(uin);
                } else {
                    // v axis: weight of row b of the record's window step; the
                    // footprint starts at row d = anchor - step base, 0..7; with
                    // the row factor (-1)^row
                    const int rel = i0 - Bfirst;
                    WSB_DCHECK(rel >= 0 && rel < Sm::NROW, "item %lld rel %d", (long long)item, rel);
                    const int d = rel & 7;
#pragma unroll
                    for (int b = 0; b < Rec::NV; b += 2)
                        *reinterpret_cast<double2 *>(&st.wv[b]) = make_double2(0.0, 0.0);
                    const double sd = (d & 1) ? -rs : rs;
                    double *const wr = st.wv + d;
#pragma unroll
                    for (int k = 0; k < W; ++k) wr[k] = (k & 1) ? -sd * wgt[k] : sd * wgt[k];
                    st.meta.y = rel >> 3;
                    st.meta.z = d;
                    const int r_lo = max(R0 - i0, 0), r_hi = min(R1 - i0, W) - 1;
                    mine = __popc(r_hi >= r_lo ? wm & (((2u << r_hi) - 1u) & ~((1u << r_lo) - 1u)) : 0u);
                }
            }
            // cell updates inside this item (grid_sector's count): u taps x v taps
            const unsigned other = __shfl_xor_sync(0xffffffffu, mine, 1);
            if (ax == 0) cnt_upd += mine * other;
        }
        __syncthreads();   // stage complete
        // ---- sweep: this warp's strip ---------------------------------------
        {
            // The chunk's records touching the strip, in order, taken four at a
            // time: lane (g4, k4) holds record k4 of the group. A record is
            // applied once the window's first tile is its step's (or, with
            // WSB_WIN_EXTRA, up to that many steps earlier); a group whose
            // records lie further apart is applied in several passes, the
            // window moving on in between.
            const uint32_t lt = (1u << lane) - 1u;
            int tot;
            if constexpr (kWarps == 1) {
                tot = nr;   // (K1 gives a one-strip item only records whose taps reach it)
            } else {
                tot = 0;
#pragma unroll
                for (int q = 0; q < kChunk / 32; ++q) {
                    const int r = 32 * q + lane;
                    const bool t = r < nr && ((sm.rec[r].meta.w >> warp) & 1);
                    const uint32_t m = __ballot_sync(0xffffffffu, t);
                    if (t) sm.prec[warp][tot + __popc(m & lt)] = (uint8_t)r;
                    tot += __popc(m);
                }
                __syncwarp();
            }
            constexpr int NTR = Win<S>::NTR;
            const int wc8 = warp * kC + g4;        // this lane's B column (half 0) in the item
            int pos = k4;                          // this lane's record position in the list
            bool pend;                             // its record still to apply
            int srec, span;                        // its window step; tiles it reaches from there
            int dl;                                // its first footprint row in the step (0..7)
            double2 b0, b1;                        // B: value x u weight at the lane's columns
            const double *wvp;                     // A: v weights of its rows
            auto load = [&]() {
                pend = pos < tot;
                const int slot = kWarps == 1 ? pos : (int)sm.prec[warp][pos];
                const unsigned char *rp = recbase + (pend ? slot : kChunk) * (int)sizeof(Rec);
                const int4 m = *reinterpret_cast<const int4 *>(rp + offsetof(Rec, meta));
                const int c0 = wc8 - m.x;
                const int i0 = (unsigned)c0 < (unsigned)W ? c0 : W;
                const int i1 = (unsigned)(c0 + 8) < (unsigned)W ? c0 + 8 : W;
                b0 = *reinterpret_cast<const double2 *>(rp + 16 * i0);
                b1 = *reinterpret_cast<const double2 *>(rp + 16 * i1);
                wvp = reinterpret_cast<const double *>(rp + offsetof(Rec, wv)) + (kOne ? 0 : g4);
                dl = m.z;
                srec = m.y;
                span = (m.z + W + 7) >> 3;
            };
            load();
            // phase P: apply groups while their first pending record is in the
            // current step, then emit tile P. false: chunk done
            auto run = [&](auto P) -> bool {
                constexpr int p = decltype(P)::value;
                for (;;) {
                    if (!__any_sync(0xffffffffu, pend)) return false;   // (the list is used up)
                    const int smin = __reduce_min_sync(0xffffffffu, pend ? srec : 0x7FFFFFFF);
                    if (smin != step) break;
                    const int delta = srec - step;
                    const bool act = pend && delta <= NT - NTR;
                    const int ntile = __reduce_max_sync(0xffffffffu, act ? delta + span : 0);
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        if (t < ntile) {   // (uniform) tiles the pass reaches
                            // A: v weight of the records on tile row g4 (window row 8t + g4)
                            const int tt = t - delta;
                            double av;
                            if constexpr (kOne) {   // footprint row of tile row g4
                                const int kr = 8 * tt + g4 - dl;
                                av = (act && (unsigned)kr < (unsigned)W) ? wvp[kr] : 0.0;
                            } else {
                                av = (act && (unsigned)tt < (unsigned)NTR) ? wvp[8 * tt] : 0.0;
                            }
                            const int tr = (p + t) % NT;          // ring tile holding window tile t (folds)
                            dmma(acc[tr][0][0], av, b0.x);
                            dmma(acc[tr][0][1], av, b0.y);
                            dmma(acc[tr][1][0], av, b1.x);
                            dmma(acc[tr][1][1], av, b1.y);
                        }
                    }
                    pend = pend && !act;
                    if (!__any_sync(0xffffffffu, pend)) {
                        pos += 4;
                        load();
                    }
                }
                emit(P);   // rows above the next pending record's step are final
                return true;
            };
            for (;;) {
                bool more = true;
                switch (phase) {
#define WSB_PHASE(q)                                                        \
    case q:                                                                 \
        if constexpr (q < NT) {                                             \
            if (!(more = run(std::integral_constant<int, q>{}))) break;     \
        }                                                                   \
        [[fallthrough]];
                    WSB_PHASE(0) WSB_PHASE(1) WSB_PHASE(2) WSB_PHASE(3)
#undef WSB_PHASE
                    default: break;
                }
                if (!more) break;
            }
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    // flush the rest of the block (split parts: of their rows)
    while (Bfirst + 8 * step < row_end) dispatch_phase<0, NT>(phase, emit);

#pragma unroll
    for (int o = 16; o; o >>= 1) cnt_upd += __shfl_xor_sync(0xffffffffu, cnt_upd, o);
    if (lane == 0 && cnt_upd) atomicAdd(a.updates, (unsigned long long)cnt_upd);
}

__global__ void k_i0(double beta, double *out) { *out = bessel_i0(beta); }

template <int KIND, int S>
int launch_s(wsb_ctx *ctx, const SweepArgs &a, double p0) {
    constexpr int W = 2 * S + 1;
    KParams<S> kp;
    kp.p0 = p0;
    kp.factorised = 0;
    kp.series = 0;
    kp.inv_p0 = 1.0 / p0;
    for (int k = 0; k < W; ++k) kp.cm[k] = 0.0;
    for (int q = 0; q < KParams<S>::NKB; ++q) kp.kb[q] = 0.0;
    if (KIND == WSB_KERNEL_KAISER_BESSEL) {
        // series of I0(beta sqrt(t)) in t, normalised by I0(beta) = its value at t = 1
        const double h = p0 * p0 / 4.0;
        double term = 1.0, i0b = 0.0;
        for (int q = 0; q < 400; ++q) {
            if (q > 0) term *= h / ((double)q * (double)q);
            i0b += term;
            if (q >= KParams<S>::NKB && term < 1e-18 * i0b) break;
        }
        term = 1.0;
        for (int q = 0; q < KParams<S>::NKB; ++q) {
            if (q > 0) term *= h / ((double)q * (double)q);
            kp.kb[q] = term / i0b;
        }
        // the truncated tail must be negligible (|t| <= 1): else shape_param
        // is beyond what this half_support's series length covers
        double tail = term, tsum = 0.0;
        for (int q = KParams<S>::NKB; q < 400 && tail > 1e-30 * i0b; ++q) {
            tail *= h / ((double)q * (double)q);
            tsum += tail;
        }
        kp.series = tsum <= 1e-17 * i0b ? 1 : 0;
    }
    if (KIND == WSB_KERNEL_GAUSSIAN) {
        // exp(+2f/s2)^S must stay far from overflow, exp(-m^2/s2) from underflow
        kp.factorised = (2.0 * S / p0 < 600.0 && (double)S * S / p0 < 600.0) ? 1 : 0;
        for (int k = 0; k < W; ++k) {
            const double m = (double)(S - k);
            kp.cm[k] = std::exp(-(m * m) / p0);
        }
    }
    const size_t smem = sizeof(Shm<KIND, S>);
    auto kern = k_grid_items<KIND, S>;
    WSB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)a.n_parts, kThreads, smem, ctx->stream>>>(a, kp);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

template <int KIND>
int launch_kind(wsb_ctx *ctx, int S, const SweepArgs &a, double p0) {
    switch (S) {
        case 1: return launch_s<KIND, 1>(ctx, a, p0);
        case 2: return launch_s<KIND, 2>(ctx, a, p0);
        case 3: return launch_s<KIND, 3>(ctx, a, p0);
        case 4: return launch_s<KIND, 4>(ctx, a, p0);
        case 5: return launch_s<KIND, 5>(ctx, a, p0);
        case 6: return launch_s<KIND, 6>(ctx, a, p0);
        case 7: return launch_s<KIND, 7>(ctx, a, p0);
        default: return fail(WSB_EUNSUPPORTED, "half_support > 7 not compiled in this build");
    }
}

// ---------------------------------------------------------------------------
// Work parts. An item holding more than kPartCap entries (Earth-rotation
// tracks pile millions of records into a few central items) is split into
// equal consecutive ranges of its entry list (record order); each part
// sweeps the item into its own partial tile, and k_combine adds the tiles in
// part order: a fixed association, the same for any GPU count when slabs
// start on item boundaries (the item then holds the same entries).
// ---------------------------------------------------------------------------
__global__ void k_item_parts(const uint32_t *off, int64_t n_items, uint32_t *nparts,
                             uint32_t *nslots, uint32_t *split) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= n_items) return;
    const uint32_t cnt = off[item + 1] - off[item];
    const uint32_t np = cnt > kPartCap ? (cnt + kPartCap - 1) / kPartCap : 1;
    nparts[item] = np;
    nslots[item] = np > 1 ? np : 0;
    split[item] = np > 1 ? 1 : 0;
}

__global__ void k_split_count(const uint32_t *pre, int64_t seg, uint32_t *n_split) {
    if (threadIdx.x == 0) *n_split = pre[3 * seg] - pre[2 * seg];
}

// slot_off / split_off: segments of one concatenated scan, minus their bases
__global__ void k_build_parts(const uint32_t *off, int64_t n_items, const uint32_t *part_off,
                              const uint32_t *slot_off, const uint32_t *slot_base_p, const uint32_t *split_off,
                              const uint32_t *split_base_p, uint4 *parts, uint2 *split_items) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= n_items) return;
    const uint32_t slot_base = *slot_base_p, split_base = *split_base_p;
    const uint32_t b = off[item], e = off[item + 1];
    const uint32_t np = part_off[item + 1] - part_off[item];
    if (np == 1) {
        parts[part_off[item]] = make_uint4((uint32_t)item, b, e, 0xFFFFFFFFu);
        return;
    }
    const uint32_t chunk = (e - b + np - 1) / np;
    const uint32_t slot = slot_off[item] - slot_base;
    for (uint32_t p = 0; p < np; ++p) {
        const uint32_t pb = min(e, b + p * chunk), pe = min(e, pb + chunk);
        parts[part_off[item] + p] = make_uint4((uint32_t)item, pb, pe, slot + p);
    }
    split_items[split_off[item] - split_base] = make_uint2((uint32_t)item, slot);
}

// one thread per (row, column) of a split item: its parts' partial tiles
// (signed, [row][re | im][kSS]) summed in part order, written to the strip
// layout
__device__ __forceinline__ void combine_item(const SweepArgs &a, uint2 si, const uint32_t *part_off) {
    const int64_t item = si.x;
    const int np = (int)(part_off[item + 1] - part_off[item]);
    const int rb = (int)(item % a.n_rb);
    const int64_t pt = item / a.n_rb;
    const int ss = (int)(pt % a.n_ss), plane = (int)(pt / a.n_ss);
    const int R0 = a.v_start + rb * kItemRows;
    const int R1 = min(R0 + kItemRows, a.v_start + a.v_count);
    constexpr int RPI = 128 / kSS;                     // rows per iteration of the block
    const int wc = threadIdx.x % kSS;                  // column inside the item
    const int col = ss * kSS + wc;
    const uint2 *pr = a.part_rows + part_off[item];
    for (int r = blockIdx.y * RPI + threadIdx.x / kSS; r < kItemRows; r += gridDim.y * RPI) {
        const int row = R0 + r;
        if (row >= R1) break;
        double re = 0.0, im = 0.0;
        const double *src = reinterpret_cast<const double *>(a.partial) +
                            ((int64_t)si.y * kItemRows + r) * (2 * kSS) + wc;
        for (int p = 0; p < np; ++p) {          // parts in order; rows ascend with p
            const uint2 span = pr[p];
            if ((uint32_t)r < span.x) break;
            if ((uint32_t)r >= span.y) continue;
            const double *z = src + (int64_t)p * kItemRows * (2 * kSS);
            re += z[0];
            im += z[kSS];
        }
        if (col < a.n_u) {
            const int64_t o = (((int64_t)plane * a.n_s16 + col / kC) * a.v_count + (row - a.v_start)) * (2 * kC) +
                              col % kC;
            if (a.out_f32) {
                ((float *)a.out)[o] = (float)re;
                ((float *)a.out)[o + kC] = (float)im;
            } else {
                ((double *)a.out)[o] = re;
                ((double *)a.out)[o + kC] = im;
            }
        }
    }
}

__global__ void __launch_bounds__(128) k_combine(SweepArgs a, const uint2 *split_items,
                                                  const uint32_t *part_off) {
    // (the grid is sized by a bound: blocks stride over the device count)
    const uint32_t n_split = *a.n_split_dev;
    for (uint32_t sidx = blockIdx.x; sidx < n_split; sidx += gridDim.x)
        combine_item(a, split_items[sidx], part_off);
}

}  // namespace

int grid_items(wsb_ctx *ctx, const wsb_grid *g, const wsb_kernel *k, int v_start, int v_count,
               const double *rec, const ItemBuckets &bk, void *grid_s,
               unsigned long long *updates_dev, int prec) {
    SweepArgs a;
    a.rec = (const double4 *)rec;
    a.keys = bk.keys;
    a.idx = bk.idx;
    a.out = grid_s;
    a.out_f32 = prec == 32 ? 1 : 0;
    a.updates = updates_dev;
    a.i0beta = nullptr;
    a.n_u = g->n_u;
    a.v_start = v_start;
    a.v_count = v_count;
    a.n_ss = bk.n_ss;
    a.n_rb = bk.n_rb;
    a.item_bits = bk.item_bits;
    a.n_s16 = ceil_div(g->n_u, kC);
    const int64_t ni = bk.n_items;
    if (ni <= 0) {
        WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        return bucket_errors(ctx);
    }
    const int S = k->half_support;
    // ---- work parts (split heavy items) ------------------------------------
    // per item: parts, partial-tile slots, split flag -- three count arrays
    // scanned as one concatenation (one scan, one host round trip)
    const int64_t seg = ni + 1, len = 3 * seg + 1;
    uint32_t *cnt, *pre;
    WSB_TRY(ensure(ctx, kSlotPartCnt, sizeof(uint32_t) * len, (void **)&cnt));
    WSB_TRY(ensure(ctx, kSlotPartOff, sizeof(uint32_t) * len, (void **)&pre));
    WSB_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * len, ctx->stream));
    k_item_parts<<<ceil_div(ni, 256), 256, 0, ctx->stream>>>(bk.off, ni, cnt, cnt + seg, cnt + 2 * seg);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    WSB_TRY(exclusive_scan_u32(ctx, cnt, pre, len, nullptr));
    // The launch sizes need the part / slot / split counts. Without a host
    // round trip they are bounded from the entry count: parts <= items +
    // entries / cap, slots <= 2 entries / cap, split items <= entries / (cap+1);
    // CTAs beyond the device counts exit at once. Above 1 GiB of bounded
    // partial tiles the exact counts are read back instead.
    const uint64_t ne = (uint64_t)bk.n_entries;
    uint64_t n_parts = (uint64_t)ni + ne / kPartCap + 1, n_slots = 2 * (ne / kPartCap) + 2,
             n_split = ne / (kPartCap + 1) + 1;
    if (sizeof(double2) * n_slots * kItemRows * kSS > ((size_t)1 << 30)) {
        for (int q = 0; q < 3; ++q)
            WSB_CUDA_TRY(cudaMemcpyAsync(ctx->flag_host + q, pre + (q + 1) * seg, sizeof(uint32_t),
                                         cudaMemcpyDeviceToHost, ctx->stream));
        WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        WSB_TRY(bucket_errors(ctx));
        const uint32_t b1 = (uint32_t)ctx->flag_host[0], b2 = (uint32_t)ctx->flag_host[1],
                       b3 = (uint32_t)ctx->flag_host[2];
        n_parts = b1;
        n_slots = b2 - b1;
        n_split = b3 - b2;
    }
    const uint32_t *np_off = pre;
    // device counts: parts = pre[seg]; splits = pre[3 seg] - pre[2 seg] (one word)
    uint32_t *n_split_dev;
    WSB_TRY(ensure(ctx, kSlotFlag, 64, (void **)&n_split_dev));
    uint4 *parts;
    uint2 *split_items, *part_rows;
    double2 *partial = nullptr;
    WSB_TRY(ensure(ctx, kSlotParts, sizeof(uint4) * n_parts + sizeof(uint2) * (n_split + 1 + n_parts),
                   (void **)&parts));
    split_items = reinterpret_cast<uint2 *>(parts + n_parts);
    part_rows = split_items + n_split + 1;
    if (n_slots)
        WSB_TRY(ensure(ctx, kSlotPartial, sizeof(double2) * (size_t)n_slots * kItemRows * kSS,
                       (void **)&partial));
    k_build_parts<<<ceil_div(ni, 256), 256, 0, ctx->stream>>>(bk.off, ni, np_off, pre + seg, pre + seg,
                                                              pre + 2 * seg, pre + 2 * seg, parts, split_items);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    k_split_count<<<1, 32, 0, ctx->stream>>>(pre, seg, n_split_dev + 12);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    a.n_parts_dev = pre + seg;
    a.n_split_dev = n_split_dev + 12;
    a.parts = parts;
    a.part_rows = part_rows;
    a.partial = partial;
    a.n_parts = n_parts;
    a.n_rec = bk.n_rec;
    a.out_elems = (int64_t)g->n_w * a.n_s16 * kC * v_count;
    // ---- sweep ---------------------------------------------------------------
    int rc;
    if (k->kind == WSB_KERNEL_GAUSSIAN) {  // s2 = 2 sigma^2 (gridder.py:85)
        rc = launch_kind<WSB_KERNEL_GAUSSIAN>(ctx, S, a, 2.0 * k->shape_param * k->shape_param);
    } else {
        double *i0b;
        WSB_TRY(ensure(ctx, kSlotFlag, 64, (void **)&i0b));
        k_i0<<<1, 1, 0, ctx->stream>>>(k->shape_param, i0b + 4);  // slot bytes 32..39
        ctx->launches += 1;
        a.i0beta = i0b + 4;
        rc = launch_kind<WSB_KERNEL_KAISER_BESSEL>(ctx, S, a, k->shape_param);
    }
    if (rc != WSB_OK || n_split == 0) return rc;
    k_combine<<<dim3((unsigned)std::min<uint64_t>(n_split, 1184), kItemRows / 2 / 8), 128, 0, ctx->stream>>>(
        a, split_items, np_off);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

}  // namespace wsb

