// K2: register-window sweep gridder (gridder.py:160-259, Eq. 3).
//
// Work item = one warp = (w plane, 32-column strip, block of 128 slab rows).
// Lane l owns column 32*strip + l. The item's records (bucket.cu) arrive
// sorted by anchor row floor(gv); the warp keeps the 2S+1 rows a record can
// touch as complex128 accumulators in registers and slides that window down
// the block: before a record is applied, every row above its footprint is
// final and is written straight to HBM (strip layout, checkerboard sign of
// transform.py:180-185 applied). Each cell is therefore accumulated by one
// lane in (anchor row, gindex) order -- deterministic and independent of
// the number of GPUs -- and written exactly once: no shared-memory tile, no
// atomics, no read-modify-write of HBM.
//
// Records are staged 32 at a time per warp: lane r loads record r through
// the bucket index and computes its separable per-axis kernel weights once
// (FP64; excluded taps get weight 0, so the per-record update below is
// branch-free). The tap set is the reference's: |g - i| <= S with g - i
// rounded as in gridder.py:170-177.
#include <type_traits>

#include "i0_coeffs.h"
#include "wsb_internal.cuh"

namespace wsb {
namespace {

#ifndef WSB_GRID_WARPS
#define WSB_GRID_WARPS 4
#endif
#ifndef WSB_GRID_ROWS
#define WSB_GRID_ROWS 128
#endif
#ifndef WSB_GRID_RUNROLL
#define WSB_GRID_RUNROLL 1
#endif
#ifndef WSB_GRID_PREMUL
#define WSB_GRID_PREMUL 1   // stage value * u weight per window column (vs value and weights)
#endif
#ifndef WSB_GRID_MINB
#define WSB_GRID_MINB 0   // > 0: one occupancy target for every instantiation
#endif
constexpr int kWarpsPerCta = WSB_GRID_WARPS;  // independent warps per CTA
constexpr int kRowBlock = WSB_GRID_ROWS;      // slab rows per work item
constexpr int kRunUnroll = WSB_GRID_RUNROLL;  // records per iteration of the run loop

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
    uint32_t mask = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const double d = __dsub_rn(g, (double)(i0 + k));
        mask |= (uint32_t)(fabs(d) <= (double)S) << k;
    }
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

// Calls f(std::integral_constant<int, phase>) for a runtime phase in [0, W).
template <int I, int W, class F>
__device__ __forceinline__ void dispatch_phase(int phase, F &f) {
    if constexpr (I < W) {
        if (phase == I)
            f(std::integral_constant<int, I>{});
        else
            dispatch_phase<I + 1, W>(phase, f);
    }
}

struct SweepArgs {
    const double4 *rec;
    const uint32_t *idx;
    const uint32_t *off;
    void *out;                    // strip layout [n_w][ceil(n_u/32)][v_count][32]
    int out_f32;                  // 1: complex64 grid (FP32 path; accumulation stays FP64)
    unsigned long long *updates;
    const double *i0beta;         // device scalar, np.i0(beta) (Kaiser-Bessel)
    const uint4 *parts;           // (item, first entry, end entry, slot | ~0 = direct)
    double2 *partial;             // [slot][kRowBlock][32] partial tiles of split items
    int n_u, v_start, v_count, n_tc, rs, n_rb, n_groups;
    int64_t n_items, n_parts;
};

// Value * u-weight staging on/off per (kernel, half_support): measured on
// cfg2 records (profiles/gridder_minb_r01.txt); above S = 5 the premultiplied
// records exceed 48 KB of static shared memory per CTA.
template <int KIND, int S>
constexpr bool sweep_premul() {
    constexpr bool gauss[8] = {false, false, true, true, false, true, false, false};
    constexpr bool kb[8] = {false, true, true, true, false, true, false, false};
    return WSB_GRID_PREMUL && (KIND == WSB_KERNEL_GAUSSIAN ? gauss[S] : kb[S]);
}

template <int KIND, int S>
struct WarpStage {
    static constexpr int W = 2 * S + 1;
    // one contiguous struct per staged record: the sweep addresses a record
    // with a single base pointer (vs. separate wu/wv/val/ij arrays: -2% grid
    // time at S=3, -20% at S=4 where the split arrays had bank conflicts)
    static constexpr int WVS = (W + 1) & ~1;
    // PRE: value * u weight staged per window column (the run loop loads one
    // complex instead of the value and a weight, no multiplies)
    static constexpr bool PRE = sweep_premul<KIND, S>();
    struct RecPre {
        double2 tu[W + 1];        // value * u weight per window column; slot W = 0 (off the footprint)
        double wv[WVS];
        int2 ij;                  // (first window column, first window row)
    };
    struct RecVal {
        double2 val;
        double wv[WVS];
        double wu[W + 1];         // slot W is the zero weight for columns off the footprint
        int2 ij;                  // (first window column, first window row)
    };
    using Rec = std::conditional_t<PRE, RecPre, RecVal>;
    Rec rec[32];
    double2 raw[2][32][2];        // records in flight (cp.async), one chunk ahead
};
#define ST_TU(r, k) st.rec[r].tu[k]
#define ST_WU(r, k) st.rec[r].wu[k]
#define ST_WV(r, b) st.rec[r].wv[b]
#define ST_VAL(r) st.rec[r].val
#define ST_IJ(r) st.rec[r].ij

// Resident CTAs per SM the sweep is compiled for (register budget), per
// (kernel, half_support): measured on cfg2 records (profiles/gridder_minb_r01.txt);
// the best point moves with each instantiation's register allocation.
template <int KIND, int S>
constexpr int sweep_min_blocks() {
    if (WSB_GRID_MINB > 0) return WSB_GRID_MINB;
    constexpr int gauss[8] = {4, 4, 5, 5, 4, 4, 3, 3};
    constexpr int kb[8] = {4, 6, 2, 6, 5, 2, 2, 2};
    return KIND == WSB_KERNEL_GAUSSIAN ? gauss[S] : kb[S];
}

template <int KIND, int S>
__global__ void __launch_bounds__(32 * kWarpsPerCta, sweep_min_blocks<KIND, S>()) k_grid_sweep(SweepArgs a, KParams<S> kp) {
    constexpr int W = 2 * S + 1;
    using St = WarpStage<KIND, S>;
    __shared__ __align__(16) St stage_all[kWarpsPerCta];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    St &st = stage_all[warp];
    const int64_t part = (int64_t)blockIdx.x * kWarpsPerCta + warp;
    if (part >= a.n_parts) return;
    // work part = (item, record sub-range, partial-tile slot or direct)
    const uint4 pd = a.parts[part];
    const int64_t item = pd.x;
    // item -> (plane, strip, row block); row block fastest
    const int rb = (int)(item % a.n_rb);
    const int64_t pt = item / a.n_rb;
    const int tc = (int)(pt % a.n_tc);
    const int plane = (int)(pt / a.n_tc);
    const int col0 = tc * 32;
    const int col = col0 + lane;
    const bool col_ok = col < a.n_u;
    const int ncols = min(32, a.n_u - col0);
    const int R0 = a.v_start + rb * kRowBlock;
    const int R1 = min(R0 + kRowBlock, a.v_start + a.v_count);
    const uint32_t beg = pd.y, end = pd.z;
    const bool direct = pd.w == 0xFFFFFFFFu;
    const double i0b = KIND == WSB_KERNEL_KAISER_BESSEL ? *a.i0beta : 0.0;
    // strip layout [plane][strip][row][32]: an emitted row is one 512-byte run;
    // a split item writes its unsigned partial tile [slot][row - R0][32]
    const int64_t colbase = direct ? ((int64_t)plane * a.n_tc + tc) * a.v_count + (R0 - a.v_start)
                                   : (int64_t)pd.w * kRowBlock;
    double2 *const out = direct ? (double2 *)a.out : a.partial;
    float2 *const out32 = (float2 *)a.out;
    const bool f32 = direct && a.out_f32;
    if constexpr (St::PRE)
        ST_TU(lane, W) = make_double2(0.0, 0.0);
    else
        ST_WU(lane, W) = 0.0;

    // Window of W rows kept as a ring of W register slots: row `base` is in
    // slot `phase`, row base+b in slot (phase+b) % W. Records with anchor
    // row == base are applied with the slot mapping fixed at compile time
    // (one code copy per phase, no register moves); when the next record
    // starts lower, row `base` is final: it is written out, its slot
    // zeroed, and the ring turns by one.
    double2 acc[W];
#pragma unroll
    for (int b = 0; b < W; ++b) acc[b] = make_double2(0.0, 0.0);
    int base = R0 - 2 * S;
    int phase = 0;
    unsigned cnt = 0;           // cell updates of the records this lane staged
    uint32_t cs = beg, ce = beg, r = beg;

    auto emit_slot = [&](auto P) {
        constexpr int p = decltype(P)::value;
        if (base >= R0 && base < R1 && col_ok) {
            const double s = (direct && ((col + base) & 1)) ? -1.0 : 1.0;
            const int64_t o = (colbase + (base - R0)) * 32 + lane;
            if (f32)
                out32[o] = make_float2((float)(acc[p].x * s), (float)(acc[p].y * s));
            else
                out[o] = make_double2(acc[p].x * s, acc[p].y * s);
        }
        acc[p] = make_double2(0.0, 0.0);
        ++base;
        phase = (p + 1 == W) ? 0 : p + 1;
    };
    // lane l holds the anchor row of staged record cs+l (INT_MAX past the
    // chunk end); records are sorted by anchor row, so the staged records
    // with anchor row == base are the contiguous run starting at r
    int my_jb = INT_MAX;
    auto run = [&](auto P) {
        constexpr int p = decltype(P)::value;
        const int rr0 = (int)(r - cs);
        const uint32_t m = __ballot_sync(0xffffffffu, my_jb == base) >> rr0;
        const int n = __popc(m);
#pragma unroll kRunUnroll
        for (int rr = rr0; rr < rr0 + n; ++rr) {
            int k = col - ST_IJ(rr).x;
            k = (unsigned)k < (unsigned)W ? k : W;   // slot W holds weight 0
            double tr, ti;
            if constexpr (St::PRE) {
                const double2 t = ST_TU(rr, k);
                tr = t.x;
                ti = t.y;
            } else {
                const double2 v = ST_VAL(rr);
                const double wu = ST_WU(rr, k);
                tr = __dmul_rn(v.x, wu);
                ti = __dmul_rn(v.y, wu);
            }
#pragma unroll
            for (int b = 0; b < W; b += 2) {
                const double2 wv2 = *reinterpret_cast<const double2 *>(&ST_WV(rr, b));
                acc[(p + b) % W].x = fma(tr, wv2.x, acc[(p + b) % W].x);
                acc[(p + b) % W].y = fma(ti, wv2.x, acc[(p + b) % W].y);
                if (b + 1 < W) {
                    acc[(p + b + 1) % W].x = fma(tr, wv2.y, acc[(p + b + 1) % W].x);
                    acc[(p + b + 1) % W].y = fma(ti, wv2.y, acc[(p + b + 1) % W].y);
                }
            }
        }
        r += n;
        if (r == ce) return true;   // chunk used up: stage the next one, same row
        emit_slot(P);               // the next record starts lower: row base is final
        return false;
    };

    // the record a lane stages next is gathered one chunk ahead by cp.async
    // into the warp's raw buffer (no registers held across the run, so the
    // random 32-byte loads overlap the previous chunk's updates), and its
    // bucket index one chunk before that
    int buf = 0;
    auto fetch = [&](uint32_t e, uint32_t id, int b) {
        if (e < end) {
            const double2 *src = reinterpret_cast<const double2 *>(a.rec + id);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&st.raw[b][lane][0]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16), "l"(src + 1)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    auto index_at = [&](uint32_t e) { return e < end ? __ldg(&a.idx[e]) : 0u; };
    fetch(beg + lane, index_at(beg + lane), 0);
    uint32_t nid = index_at(beg + 32 + lane);

    while (true) {
        if (r == ce) {
            if (ce >= end) break;
            // ---- stage the next 32 records: one per lane -------------------
            __syncwarp();
            cs = ce;
            ce = min(cs + 32u, end);
            const uint32_t e = cs + lane;
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            const double2 lo = st.raw[buf][lane][0], hi = st.raw[buf][lane][1];
            my_jb = INT_MAX;
            fetch(e + 32, nid, buf ^ 1);
            nid = index_at(e + 64);
            buf ^= 1;
            if (e < ce) {
                const double gu = lo.x, gv = lo.y;
                const int ib = (int)floor(gu) - S, jb = (int)floor(gv) - S;
                double w[W];
                const uint32_t um = axis_weights<KIND, S>(gu, ib, kp, i0b, w);
                if constexpr (St::PRE) {
                    // the run loop's value * u-weight products, formed once per record
#pragma unroll
                    for (int k = 0; k < W; ++k)
                        ST_TU(lane, k) = make_double2(__dmul_rn(hi.x, w[k]), __dmul_rn(hi.y, w[k]));
                } else {
#pragma unroll
                    for (int k = 0; k < W; ++k) ST_WU(lane, k) = w[k];
                    ST_VAL(lane) = hi;
                }
                const uint32_t vm = axis_weights<KIND, S>(gv, jb, kp, i0b, w);
#pragma unroll
                for (int k = 0; k < W; ++k) ST_WV(lane, k) = w[k];
                ST_IJ(lane) = make_int2(ib, jb);
                my_jb = jb;
                // cell updates inside this strip and row block (grid_sector's count)
                const int c_lo = max(col0 - ib, 0), c_hi = min(col0 + ncols - ib, W);
                const int r_lo = max(R0 - jb, 0), r_hi = min(R1 - jb, W);
                const uint32_t cm = c_hi > c_lo ? ((1u << (c_hi - c_lo)) - 1u) << c_lo : 0u;
                const uint32_t rm = r_hi > r_lo ? ((1u << (r_hi - r_lo)) - 1u) << r_lo : 0u;
                cnt += __popc(um & cm) * __popc(vm & rm);
            }
            __syncwarp();
        }
        // consecutive rows walk the ring statically: one jump-table dispatch
        // per W rows (and per staged chunk) instead of one per row
        for (;;) {
            switch (phase) {
#define WSB_STEP(q)                                                   \
    case q:                                                           \
        if constexpr (q < W) {                                        \
            if (run(std::integral_constant<int, q>{})) goto next_chunk; \
        }                                                             \
        [[fallthrough]];
                WSB_STEP(0) WSB_STEP(1) WSB_STEP(2) WSB_STEP(3) WSB_STEP(4)
                WSB_STEP(5) WSB_STEP(6) WSB_STEP(7) WSB_STEP(8) WSB_STEP(9)
                WSB_STEP(10) WSB_STEP(11) WSB_STEP(12) WSB_STEP(13) WSB_STEP(14)
#undef WSB_STEP
                default: break;
            }
        }
    next_chunk:;
    }
    while (base < R1) dispatch_phase<0, W>(phase, emit_slot);

#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt) atomicAdd(a.updates, (unsigned long long)cnt);
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
    const int64_t blocks = (a.n_parts + kWarpsPerCta - 1) / kWarpsPerCta;
    k_grid_sweep<KIND, S><<<(unsigned)blocks, 32 * kWarpsPerCta, 0, ctx->stream>>>(a, kp);
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
// Load balancing. Earth-rotation tracks pile millions of records into a few
// (plane, strip, row block) items. An item with more than kPartRecords
// records is split into equal consecutive sub-ranges of its (sorted) list;
// each part sweeps the item into its own partial tile, and k_combine adds
// the parts in part order (fixed association: deterministic, and the same
// split for any GPU count since items never straddle slabs).
// ---------------------------------------------------------------------------
constexpr uint32_t kPartRecords = 4096;

__device__ __forceinline__ void item_range(const SweepArgs &a, int S, int64_t item, uint32_t *b,
                                           uint32_t *e) {
    const int rb = (int)(item % a.n_rb);
    const int64_t pt = item / a.n_rb;
    const int tc = (int)(pt % a.n_tc), plane = (int)(pt / a.n_tc);
    const int R0 = a.v_start + rb * kRowBlock;
    const int R1 = min(R0 + kRowBlock, a.v_start + a.v_count);
    const uint32_t kbase = ((uint32_t)plane * a.n_tc + tc) * (uint32_t)a.rs;
    *b = a.off[kbase + (R0 - a.v_start)];
    *e = a.off[kbase + (R1 - 1 - a.v_start + 2 * S) + 1];
}

__global__ void k_item_parts(SweepArgs a, int S, uint32_t *nparts, uint32_t *nslots,
                             uint32_t *split) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= a.n_items) return;
    uint32_t b, e;
    item_range(a, S, item, &b, &e);
    const uint32_t np = e - b > kPartRecords ? (e - b + kPartRecords - 1) / kPartRecords : 1;
    nparts[item] = np;
    nslots[item] = np > 1 ? np : 0;
    split[item] = np > 1 ? 1 : 0;
}

__global__ void k_build_parts(SweepArgs a, int S, const uint32_t *part_off, const uint32_t *slot_off,
                              const uint32_t *split_off, uint4 *parts, uint2 *split_items) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= a.n_items) return;
    uint32_t b, e;
    item_range(a, S, item, &b, &e);
    const uint32_t np = part_off[item + 1] - part_off[item];
    if (np == 1) {
        parts[part_off[item]] = make_uint4((uint32_t)item, b, e, 0xFFFFFFFFu);
        return;
    }
    const uint32_t chunk = (e - b + np - 1) / np;
    for (uint32_t p = 0; p < np; ++p) {
        const uint32_t pb = min(e, b + p * chunk), pe = min(e, pb + chunk);
        parts[part_off[item] + p] = make_uint4((uint32_t)item, pb, pe, slot_off[item] + p);
    }
    split_items[split_off[item]] = make_uint2((uint32_t)item, slot_off[item]);
}

// one warp per row of a split item: sum its parts' partial rows in part order
__global__ void __launch_bounds__(128) k_combine(SweepArgs a, const uint2 *split_items,
                                                  const uint32_t *part_off) {
    const uint2 si = split_items[blockIdx.x];
    const int64_t item = si.x;
    const int np = (int)(part_off[item + 1] - part_off[item]);
    const int rb = (int)(item % a.n_rb);
    const int64_t pt = item / a.n_rb;
    const int tc = (int)(pt % a.n_tc), plane = (int)(pt / a.n_tc);
    const int R0 = a.v_start + rb * kRowBlock;
    const int R1 = min(R0 + kRowBlock, a.v_start + a.v_count);
    const int lane = threadIdx.x & 31;
    const int col = tc * 32 + lane;
    for (int r = blockIdx.y * 4 + (threadIdx.x >> 5); r < kRowBlock; r += gridDim.y * 4) {
        const int row = R0 + r;
        if (row >= R1) break;
        double2 acc = make_double2(0.0, 0.0);
        const double2 *src = a.partial + ((int64_t)si.y * kRowBlock + r) * 32 + lane;
        for (int p = 0; p < np; ++p) {
            const double2 z = src[(int64_t)p * kRowBlock * 32];
            acc.x += z.x;
            acc.y += z.y;
        }
        if (col < a.n_u) {
            const double s = ((col + row) & 1) ? -1.0 : 1.0;
            const int64_t o = (((int64_t)plane * a.n_tc + tc) * a.v_count + (row - a.v_start)) * 32 + lane;
            if (a.out_f32)
                ((float2 *)a.out)[o] = make_float2((float)(acc.x * s), (float)(acc.y * s));
            else
                ((double2 *)a.out)[o] = make_double2(acc.x * s, acc.y * s);
        }
    }
}

}  // namespace

int grid_sweep(wsb_ctx *ctx, const wsb_grid *g, const wsb_kernel *k, int v_start, int v_count,
               const double *rec, const RowBuckets &bk, void *grid_p,
               unsigned long long *updates_dev, int prec) {
    SweepArgs a;
    a.rec = (const double4 *)rec;
    a.idx = bk.idx;
    a.off = bk.off;
    a.out = grid_p;
    a.out_f32 = prec == 32 ? 1 : 0;
    a.updates = updates_dev;
    a.i0beta = nullptr;
    a.n_u = g->n_u;
    a.v_start = v_start;
    a.v_count = v_count;
    a.n_tc = bk.n_tc;
    a.rs = bk.rs;
    a.n_rb = ceil_div(v_count, kRowBlock);
    a.n_groups = g->n_u / kG;
    a.n_items = (int64_t)g->n_w * a.n_tc * a.n_rb;
    if (a.n_items <= 0) return WSB_OK;
    const int S = k->half_support;
    // ---- work parts (split heavy items) ------------------------------------
    const int64_t ni = a.n_items;
    uint32_t *np, *ns, *sp, *np_off, *ns_off, *sp_off;
    WSB_TRY(ensure(ctx, kSlotPartCnt, sizeof(uint32_t) * 3 * (ni + 1), (void **)&np));
    WSB_TRY(ensure(ctx, kSlotPartOff, sizeof(uint32_t) * 3 * (ni + 1), (void **)&np_off));
    ns = np + (ni + 1);
    sp = ns + (ni + 1);
    ns_off = np_off + (ni + 1);
    sp_off = ns_off + (ni + 1);
    WSB_CUDA_TRY(cudaMemsetAsync(np, 0, sizeof(uint32_t) * 3 * (ni + 1), ctx->stream));
    k_item_parts<<<ceil_div(ni, 256), 256, 0, ctx->stream>>>(a, S, np, ns, sp);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    uint32_t n_parts = 0, n_slots = 0, n_split = 0;
    WSB_TRY(exclusive_scan_u32(ctx, np, np_off, ni + 1, &n_parts));
    WSB_TRY(exclusive_scan_u32(ctx, ns, ns_off, ni + 1, &n_slots));
    WSB_TRY(exclusive_scan_u32(ctx, sp, sp_off, ni + 1, &n_split));
    uint4 *parts;
    uint2 *split_items;
    double2 *partial = nullptr;
    WSB_TRY(ensure(ctx, kSlotParts, sizeof(uint4) * n_parts + sizeof(uint2) * (n_split + 1),
                   (void **)&parts));
    split_items = reinterpret_cast<uint2 *>(parts + n_parts);
    if (n_slots)
        WSB_TRY(ensure(ctx, kSlotPartial, sizeof(double2) * (size_t)n_slots * kRowBlock * 32,
                       (void **)&partial));
    k_build_parts<<<ceil_div(ni, 256), 256, 0, ctx->stream>>>(a, S, np_off, ns_off, sp_off, parts,
                                                              split_items);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    a.parts = parts;
    a.partial = partial;
    a.n_parts = n_parts;
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
    k_combine<<<dim3(n_split, kRowBlock / 4 / 4), 128, 0, ctx->stream>>>(a, split_items, np_off);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

}  // namespace wsb
