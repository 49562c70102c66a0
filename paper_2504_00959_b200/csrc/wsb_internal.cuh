// Internal declarations shared by the libwsb.so translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/wsb.h"

// Device-side bounds checks of the debug build (python -m
// paper_2504_00959_b200.build --debug: libwsb_dbg.so, loaded with
// WSB_LIB=.../libwsb_dbg.so): a failed check prints and traps.
#ifdef WSB_DEBUG_CHECKS
#define WSB_DCHECK(cond, ...)                                                   \
    do {                                                                        \
        if (!(cond)) {                                                          \
            printf("WSB_DCHECK %s:%d: %s | ", __FILE__, __LINE__, #cond);       \
            printf(__VA_ARGS__);                                                \
            printf("\n");                                                       \
            __trap();                                                           \
        }                                                                       \
    } while (0)
#else
#define WSB_DCHECK(cond, ...) \
    do {                      \
    } while (0)
#endif

namespace wsb {

constexpr int kG = WSB_P_GROUP;    // P-layout column group
constexpr int kMaxS = 7;           // largest half support compiled (window 15)
constexpr int kMaxOnChipLog = 12;  // longest on-chip transform (4096); longer ones split

// thread-local error detail
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

#define WSB_CUDA_TRY(expr)                                                        \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess)                                                    \
            return ::wsb::fail(_e == cudaErrorMemoryAllocation ? WSB_ENOMEM       \
                                                               : WSB_ECUDA,       \
                               std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define WSB_TRY(expr)               \
    do {                            \
        int _rc = (expr);           \
        if (_rc != WSB_OK) return _rc; \
    } while (0)

// Grow-only device workspace slot.
struct Buf {
    void *ptr = nullptr;
    size_t bytes = 0;
};

struct Timing {
    cudaEvent_t ev[8];
    bool created = false;
};

}  // namespace wsb

struct wsb_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::vector<wsb::Buf> bufs;       // indexed by slot id
    int *flag_host = nullptr;         // pinned scratch for small readbacks
    unsigned long long *u64_host = nullptr;
    wsb::Timing timing;
    // twiddle tables keyed by log2(n) + 16 * {0: radix-8 plan, 1: radix-16 plan, 2: plain}
    double *twiddle[96] = {nullptr};   // + 48: complex64 copies
    // last bucketing (for wsb_tiles_debug)
    int64_t last_entries = 0, last_tiles = 0;
    uint32_t *last_keys = nullptr, *last_idx = nullptr, *last_off = nullptr;
    int launches = 0;
    bool pending_bucket_err = false;
    uint32_t scan_epoch = 0;          // single-pass scan: status words of earlier scans are stale   // bucket_items' validation flags await a host round trip
    // route_count -> route_pack hand-over: the pack reuses the counts of the
    // immediately preceding count on the same records and slabs
    struct {
        const double *rec = nullptr;
        const uint32_t *plane = nullptr;
        int by_plane = -1;
        int64_t n = -1;
        int S = -1, R = -1, n_v = -1, nb = 0;
        int starts[9] = {0};
        bool valid = false;
    } route;
    int precision = 64;               // wsb_ctx_set_precision: 64 or 32 (complex64 grids)
    int energy = 0;                   // wsb_ctx_set_energy: NVML/RAPL counters around calls
    double last_ms[6] = {0, 0, 0, 0, 0, 0};
};

namespace wsb {

enum Slot {
    kSlotFlag = 0,
    kSlotBlockCounts,
    kSlotBlockOffsets,
    kSlotScanTmp,
    kSlotScanTmp2,
    kSlotKeysA,
    kSlotKeysB,
    kSlotIdxA,
    kSlotIdxB,
    kSlotTileCount,
    kSlotTileOff,
    kSlotRadixHist,
    kSlotU64,
    kSlotRec,
    kSlotPlane,
    kSlotGrid,
    kSlotGridP,
    kSlotStrip,
    kSlotColRun,
    kSlotHostIn,
    kSlotPartCnt,
    kSlotPartOff,
    kSlotParts,
    kSlotPartial,
    kSlotRadixTmpA,
    kSlotRadixTmpB,
    kSlotRadixTmpC,
    kSlotRouteCnt,
    kSlotRouteOff,
    kSlotCount
};

int ensure(wsb_ctx *ctx, int slot, size_t bytes, void **out);
int twiddles(wsb_ctx *ctx, int n, int rlmax, const void **out, int prec = 64);

// scan.cu
int exclusive_scan_u32(wsb_ctx *ctx, const uint32_t *in, uint32_t *out, int64_t n,
                       uint32_t *total_host);

// sort.cu: stable LSD radix sort of (key, val) pairs by the low `bits` of key.
// Returns the buffers holding the result in *keys_out/*vals_out; the final
// pass writes the values only (*keys_out then holds a previous pass's keys).
// Report bucket_items' validation flags (call after a stream synchronisation).
int bucket_errors(wsb_ctx *ctx);

int radix_sort_pairs(wsb_ctx *ctx, uint32_t *keys, uint32_t *keys_alt, uint32_t *vals,
                     uint32_t *vals_alt, int64_t n, int bits, uint32_t **keys_out,
                     uint32_t **vals_out, bool keep_keys = true);

// prepare.cu
int prepare(wsb_ctx *ctx, const wsb_grid *g, const double *u, const double *v,
            const double *w, const float *vis, const float *weight, int64_t n,
            int32_t n_chan, double *rec, uint32_t *plane, const uint32_t *time_index = nullptr);
// by_plane = 0: v-slabs with the +-S halo; 1: w-plane ranges (plane is read,
// packed planes are rebased to the destination's first plane)
int route_count(wsb_ctx *ctx, const wsb_grid *g, int S, int R, const int32_t *starts,
                const double *rec, int64_t n, int64_t *counts_host, uint32_t **offs_out,
                int *nb_out, const uint32_t *plane = nullptr, int by_plane = 0);
int route_pack(wsb_ctx *ctx, const wsb_grid *g, int S, int R, const int32_t *starts,
               const double *rec, const uint32_t *plane, int64_t n, double *send_rec,
               uint32_t *send_plane, int64_t *src_index, int by_plane = 0);
int row_histogram(wsb_ctx *ctx, const wsb_grid *g, const double *rec, int64_t n, uint32_t *hist);
int plane_histogram(wsb_ctx *ctx, const wsb_grid *g, const uint32_t *plane, int64_t n,
                    uint32_t *hist);

// Gridder work items (bucket.cu, grid.cu): (w plane, kSSCols-column block,
// kItemRows-row block of the slab); one CTA per item, one warp per
// WSB_STRIP-column strip of it.
constexpr int kItemRows = 128;
constexpr int kSSCols = WSB_ITEM_COLS;
static_assert(kSSCols % WSB_STRIP == 0 && kSSCols <= 4 * WSB_STRIP, "item columns");
constexpr int kPartCap = 2048;     // entries per work part (split heavy items)
constexpr int kFlagBucketErr = 8;  // flag_host slot of bucket_items' validation flags
constexpr int kRowBits = 8;        // entry key = item << kRowBits | row offset

// the visibility columns of one channel (fused prepare + bucketing)
struct VisColumns {
    const double *u, *v, *w;
    const float *vis, *weight;
    const uint32_t *time_index;   // nullable
};

struct ItemBuckets {
    uint32_t *keys = nullptr;  // item << kRowBits | rowrel, sorted: (item, row, record) order
    uint32_t *idx = nullptr;   // record index per entry
    uint32_t *off = nullptr;   // [n_items + 1] exclusive offsets
    int64_t n_entries = 0, n_items = 0, n_rec = 0;
    int n_ss = 0, n_rb = 0, item_bits = 0;
};
// in != nullptr: records are prepared from the columns on the fly (rec
// written, plane written if non-null; one channel); else rec/plane are read.
// Synchronises once (entry count, validation flags).
int bucket_items(wsb_ctx *ctx, const wsb_grid *g, int S, int v_start, int v_count,
                 const VisColumns *in, double *rec, uint32_t *plane, int64_t m,
                 ItemBuckets *out);

// grid.cu
int grid_items(wsb_ctx *ctx, const wsb_grid *g, const wsb_kernel *k, int v_start, int v_count,
               const double *rec, const ItemBuckets &bk, void *grid_s,
               unsigned long long *updates_dev, int prec = 64);

// peer.cu: copy n_dest contiguous blocks src[d] -> dst[d] (bytes[d] each; dst
// may be peer memory) with one launch on the context stream
int push_blocks(wsb_ctx *ctx, int n_dest, const void *const *src, void *const *dst,
                const int64_t *bytes);

// fft.cu
// prec 64: complex128 grids; 32: complex64 grids (FP32 path)
int fft_rows(wsb_ctx *ctx, const wsb_grid *g, int v_count, const void *grid_a, void *grid_p,
             int plane_lo, int plane_hi, int n_dest, const int32_t *dest_groups,
             void *const *dest_ptrs = nullptr, int prec = 64);
int fft_cols_stack(wsb_ctx *ctx, const wsb_grid *g, int n_sources, const int32_t *src_rows,
                   int g0, int ng, int plane_lo, int plane_hi, const void *tgrid,
                   double *image_strip, double *norm_partials, int prec = 64,
                   int k_bottom = 0, int k_top = -1, double *partial_img = nullptr);
int image_finish(wsb_ctx *ctx, const wsb_grid *g, const double *sum, double *image,
                 double *norm_partials);
int strip_to_image(wsb_ctx *ctx, const wsb_grid *g, const double *strip, double *image);

// NVML (GPU) + RAPL (host) energy over a window of host time (api.cu)
struct EnergyWindow {
    int device = 0;
    double gpu0 = -1.0;
    bool host_ok = false;
    std::vector<std::pair<double, double>> host0;
    void start(int dev);
    void stop(double *gpu_j, double *host_j);
};

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
inline int ilog2(int64_t n) {
    int l = 0;
    while ((int64_t(1) << l) < n) ++l;
    return l;
}

}  // namespace wsb
