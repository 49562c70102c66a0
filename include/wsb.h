/*
 * wsb.h — C ABI of the B200 w-stacking imager (libwsb.so, sm_100a).
 *
 * The reference (`wstack`, pure Python/NumPy) has no FFI; its drop-in
 * boundary is the Python call `pipeline.run_pipeline` phases 2-5
 * (/root/reference/pkg/src/wstack/pipeline.py:95-152) plus the finer hooks
 * `gridder.grid_sector` (gridder.py:186-259) and `gridder.grid_all`
 * (gridder.py:262-294). Each entry point below names the reference function
 * it replaces. The Python host package `paper_2504_00959_b200` binds this
 * ABI with ctypes and mirrors the reference API on top.
 *
 * Conventions
 *   - Plain C types only. Inputs are caller-owned and read-only; nothing is
 *     retained after a call returns. Device pointers are CUDA global-memory
 *     pointers on the context's device; host pointers are ordinary memory
 *     (pinned memory is faster but not required).
 *   - Every function returns 0 or a negative WSB_E* code. The Python layer
 *     maps WSB_EINVAL -> ValueError (mesh.py:79-95, gridder.py:56-62,
 *     visdata.py:178-184), WSB_ECUDA/WSB_ENCCL -> RuntimeError,
 *     WSB_ENOMEM -> MemoryError, WSB_EUNSUPPORTED -> NotImplementedError.
 *     wsb_last_error() returns a thread-local detail string.
 *   - Stage functions enqueue on the context's stream and return without
 *     synchronising unless they must read a device value back
 *     (validation flags, counts); they say so.
 *   - No CPU fallback: every compute entry point runs CUDA kernels.
 */
#ifndef WSB_H
#define WSB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WSB_VERSION 100

#define WSB_OK            0
#define WSB_EINVAL       -1
#define WSB_ECUDA        -2
#define WSB_ENCCL        -3
#define WSB_ENOMEM       -4
#define WSB_EUNSUPPORTED -5

#define WSB_KERNEL_GAUSSIAN       0
#define WSB_KERNEL_KAISER_BESSEL  1

/* Column-group width of the internal "P layout" grid (row-pass output,
 * column-pass input):
 *   P[plane][col / WSB_P_GROUP][row][col % WSB_P_GROUP]  (complex128)
 * i.e. column-major: every column of a plane is one contiguous run, read
 * by the column pass with full 32-byte sectors. The sign (-1)^(i+j) of
 * transform.py:180-185 is already applied. */
#define WSB_P_GROUP 1

/* Column width of the gridder's output "strip layout":
 *   grid_s[plane][col / WSB_STRIP][row][re | im][col % WSB_STRIP]
 * (each strip row stores its WSB_STRIP real parts, then its imaginary parts,
 * f64 -- f32 on the FP32 path; every two rows of a strip are one 512-byte
 * run); the checkerboard sign of transform.py:180-185 is applied. */
#define WSB_STRIP 16
/* Columns of one gridder work item (one K2 CTA): a multiple of WSB_STRIP. */
#ifndef WSB_ITEM_COLS
#define WSB_ITEM_COLS 16
#endif

/* Longest transform handled on chip (one CTA) and longest transform
 * supported: rows/columns of SP = N / WSB_ONCHIP_FFT_N > 1 blocks are split
 * by decimation in frequency into SP on-chip transforms (one CTA per output
 * residue class, each reading the whole row/column). */
#define WSB_ONCHIP_FFT_N 4096
#define WSB_MAX_FFT_N 16384
/* Residue classes of the column pass: norm partials are laid out
 * [WSB_COL_SPLIT(n_v)][columns][2]. */
#define WSB_COL_SPLIT(n_v) ((n_v) > WSB_ONCHIP_FFT_N ? (n_v) / WSB_ONCHIP_FFT_N : 1)

/* GridSpec (mesh.py:59-112). w_min/w_max normalised are fixed to [0, 1]. */
typedef struct {
    int32_t n_u, n_v, n_w, reserved;
    double cell_size_lm, w_min_native, w_max_native;
} wsb_grid;

/* KernelSpec (gridder.py:47-72). shape_param = Gaussian sigma or KB beta. */
typedef struct {
    int32_t kind, half_support;
    double shape_param;
} wsb_kernel;

typedef struct {
    int32_t device;        /* CUDA ordinal */
    int32_t precision;     /* 64 (FP64 path) or 32 (FP32 path, see wsb_ctx_set_precision) */
    int32_t deterministic; /* accepted for API parity; results are always deterministic */
    int32_t flags;         /* WSB_EXEC_* bits */
} wsb_exec;

/* wsb_exec.flags / wsb_ctx_set_energy: read the NVML (GPU) and RAPL (host)
 * energy counters around the call into wsb_diag.gpu_joules / host_joules.
 * Off by default: an NVML energy query costs milliseconds. */
#define WSB_EXEC_ENERGY 1

/* Diagnostics: FinalImage norms (transform.py:72-83, 233-241) and the ops /
 * phase-time surrogates of run_pipeline (pipeline.py:178-186). */
typedef struct {
    double imag_residual_norm, real_norm;
    int64_t grid_updates;     /* == ops["grid_updates"] */
    int64_t records;          /* == ops["records"] */
    int64_t tile_entries;     /* (record, gridder work item) pairs bucketed */
    double phase_ms[7];       /* read, gridding, reduce, fft, wcorrect, write, total (exclusive) */
    int64_t exchanged_records;/* records sent to another GPU (ops["exchange_bytes"] / 36); 0 on one GPU */
    double gpu_joules;        /* NVML energy of the call's GPU over the call; -1 if not measured
                                 (WSB_EXEC_ENERGY off) or unreadable */
    double host_joules;       /* RAPL package energy of the host over the call; -1 likewise */
} wsb_diag;

typedef struct wsb_ctx wsb_ctx;

const char *wsb_strerror(int code);
const char *wsb_last_error(void);
int wsb_version(void);

int wsb_ctx_create(int32_t device, wsb_ctx **out);
int wsb_ctx_destroy(wsb_ctx *ctx);
/* Use `stream` (a cudaStream_t; NULL = legacy default) for later calls. */
int wsb_ctx_set_stream(wsb_ctx *ctx, void *stream);
/* Grid precision of wsb_image_device on this context: 64 (complex128, the
 * default) or 32 (the FP32 path: complex64 grid and transforms; prepare,
 * weights, accumulation, phase screen and plane stack stay FP64; within 1e-5
 * relative L2 of the reference image). wsb_image takes it from exec. */
int wsb_ctx_set_precision(wsb_ctx *ctx, int32_t precision);
/* Energy counters around wsb_image_device calls on this context (see
 * WSB_EXEC_ENERGY): on != 0 to enable. */
int wsb_ctx_set_energy(wsb_ctx *ctx, int32_t on);
/* Release cached device workspace. */
int wsb_ctx_trim(wsb_ctx *ctx);

/* ---- whole hot path ---------------------------------------------------- */

/* Replaces run_pipeline phases 2-5 (pipeline.py:95-152) for one GPU, HOST
 * buffers in and out: uvw f64[n], time_index u32[n] (nullable; when given
 * it must be non-decreasing, else WSB_EINVAL "records must be sorted by
 * time_index" as partition_time_ordered raises, visdata.py:354-355, on the
 * run_pipeline path, pipeline.py:47-52; records are processed in array
 * order = the (time_index, gindex) order of comms.py:534), vis = interleaved (re, im) f32
 * [n][n_chan][2], weight f32[n][n_chan]; image_out f64[n_v][n_u].
 * Copies in and out are part of the call. Synchronous. Page-locked buffers
 * (cudaHostAlloc / cudaHostRegister) move at DMA speed; pageable ones work
 * but the driver stages them (~10x slower for the image copy-out). */
int wsb_image(const wsb_grid *grid, const wsb_kernel *kern, const wsb_exec *exec,
              const double *u, const double *v, const double *w,
              const uint32_t *time_index, const float *vis, const float *weight,
              int64_t n, int32_t n_chan, double *image_out, wsb_diag *diag);

/* Same on DEVICE buffers, enqueued on the context stream. image_out is a
 * device f64[n_v][n_u]. Synchronises once (validation flag) and at the end
 * (diagnostics) when diag != NULL. */
int wsb_image_device(wsb_ctx *ctx, const wsb_grid *grid, const wsb_kernel *kern,
                     const double *u, const double *v, const double *w,
                     const float *vis, const float *weight, int64_t n, int32_t n_chan,
                     double *image_out, wsb_diag *diag);

/* ---- stages (device pointers; used by the multi-GPU host driver) ------- */

/* prepare_chunk (comms.py:477-492) + VisChunk.validate (visdata.py:178-184):
 * rec[i] = {gu, gv, Re value, Im value} f64x4, plane[i] u32.
 * Synchronises to read the validation flag; WSB_EINVAL on bad input. */
int wsb_prepare(wsb_ctx *ctx, const wsb_grid *grid,
                const double *u, const double *v, const double *w,
                const float *vis, const float *weight, int64_t n, int32_t n_chan,
                double *rec, uint32_t *plane);

/* Destination slabs of the time->space exchange (comms.py:516-523): counts
 * of records per destination slab with the +-half_support halo predicate.
 * Slabs are partition_1d(n_v, n_ranks) (mesh.py:34-45) when
 * slab_starts_host is NULL, else rows [starts[d], starts[d+1]) with
 * starts[0] = 0 < ... < starts[n_ranks] = n_v (load-balanced slabs; the
 * image does not depend on the slab rows). counts_host: int64[n_ranks].
 * Synchronous. */
int wsb_route_count(wsb_ctx *ctx, const wsb_grid *grid, int32_t half_support, int32_t n_ranks,
                    const int32_t *slab_starts_host, const double *rec, int64_t n,
                    int64_t *counts_host);

/* Pack the exchange send buffers: records for slab d land at
 * [displ_d, displ_d + count_d) in array (gindex) order; optional src_index
 * receives the local index of each packed record (nullable). Directly
 * after wsb_route_count on the same records and slabs (no wsb_prepare in
 * between) the counts of that call are reused instead of recounted. */
int wsb_route_pack(wsb_ctx *ctx, const wsb_grid *grid, int32_t half_support, int32_t n_ranks,
                   const int32_t *slab_starts_host, const double *rec, const uint32_t *plane,
                   int64_t n, double *send_rec, uint32_t *send_plane, int64_t *src_index);

/* w-plane decomposition (the alternative to the v-slabs above): rank d
 * owns the planes [plane_starts[d], plane_starts[d+1]) (plane_starts[0] = 0
 * < ... < plane_starts[n_ranks] = n_w) and grids, transforms and stacks
 * them on its own; the ranks' partial images are summed afterwards
 * (wsb_fft_cols_partial, wsb_image_finish). Each record goes to exactly one
 * rank (no halo). Counts per destination, as wsb_route_count. Synchronous. */
/* Records per w plane of prepared records: hist u32[n_w] (device); feeds the
 * load balancing of the plane ranges. Enqueued, no synchronisation. */
int wsb_plane_histogram(wsb_ctx *ctx, const wsb_grid *grid, const uint32_t *plane, int64_t n,
                        uint32_t *hist);

int wsb_route_planes_count(wsb_ctx *ctx, const wsb_grid *grid, int32_t n_ranks,
                           const int32_t *plane_starts_host, const double *rec,
                           const uint32_t *plane, int64_t n, int64_t *counts_host);

/* Pack for the plane decomposition, as wsb_route_pack; send_plane holds the
 * plane index relative to the destination's first plane. */
int wsb_route_planes_pack(wsb_ctx *ctx, const wsb_grid *grid, int32_t n_ranks,
                          const int32_t *plane_starts_host, const double *rec,
                          const uint32_t *plane, int64_t n, double *send_rec,
                          uint32_t *send_plane, int64_t *src_index);

/* Records per anchor row floor(gv) of prepared records: hist u32[n_v]
 * (device). Feeds the load balancing of the slab rows (the
 * v-slabs of partition_1d are unbalanced for centrally concentrated uv
 * coverage). Enqueued, no synchronisation. */
int wsb_row_histogram(wsb_ctx *ctx, const wsb_grid *grid, const double *rec, int64_t n,
                      uint32_t *hist);

/* grid_sector (gridder.py:186-259) for the slab rows [v_start, v_start+v_count):
 * buckets the m records into work items (w plane, WSB_ITEM_COLS-column
 * block, 128-row block; stable radix sort, (anchor row, record) order inside
 * an item), grids them with the convolution kernel as rank-4 FP64 tensor-core
 * updates of a register window of 8-row tiles and writes the slab
 * in the strip layout (grid_s: complex128[n_w][ceil(n_u/WSB_STRIP)][v_count]
 * [WSB_STRIP], sign applied). grid_updates (host, nullable) receives the
 * number of cell updates. Synchronises (entry count). Slabs that start on a
 * multiple of 128 rows grid every cell bit-identically to a whole-mesh call. */
int wsb_grid_slab(wsb_ctx *ctx, const wsb_grid *grid, const wsb_kernel *kern,
                  int32_t v_start, int32_t v_count,
                  const double *rec, const uint32_t *plane, int64_t m,
                  double *grid_s, int64_t *grid_updates);

/* Row pass of the inverse 2D FFT (transform.py:151 / fft1d inverse) on planes
 * [plane_lo, plane_hi): strip-layout slab in, P-layout slab out (out of
 * place). With n_dest > 1 the column pairs are split over destination ranks
 * (dest_pairs_host[d] pairs each, in order) and the output is destination
 * major, [d][plane - plane_lo][pair - first_pair_d][row][G], so ONE
 * all-to-all moves the slab transpose of the range (fft2d_slab's send loop,
 * transform.py:152-161). grid_p holds planes [plane_lo, plane_hi) only, so a
 * plane range can be sent while the next one is transformed.
 * dest_pairs_host NULL = one destination = plain P layout. Unnormalised. */
int wsb_fft_rows(wsb_ctx *ctx, const wsb_grid *grid, int32_t v_count,
                 const double *grid_s, double *grid_p, int32_t plane_lo, int32_t plane_hi,
                 int32_t n_dest, const int32_t *dest_pairs_host);

/* Row pass fused with the slab transpose (fft2d_slab's send loop,
 * transform.py:152-161, without a separate all-to-all): the results for
 * destination rank d (dest_cols_host[d] column groups, in order) are stored
 * straight into d's column-pass input through dest_ptrs_host[d], a device
 * pointer valid on this GPU (peer memory over NVLink, e.g. a symmetric
 * allocation; or local memory for d = this rank), pointing at this source
 * slab's block: element (plane k, column group g, row j) of this slab goes
 * to dest_ptrs_host[d][(k * dest_cols_host[d] + g - first_d) * v_count + j]
 * (x G), k absolute in [0, n_w). The caller orders the writes of all ranks
 * before the column pass reads them (a barrier after this call). */
int wsb_fft_rows_peer(wsb_ctx *ctx, const wsb_grid *grid, int32_t v_count,
                      const double *grid_s, int32_t plane_lo, int32_t plane_hi, int32_t n_dest,
                      const int32_t *dest_cols_host, void *const *dest_ptrs_host);

/* Slab-transpose / record-exchange push: copies n_dest contiguous device
 * blocks src_ptrs[d] -> dst_ptrs[d] (bytes_host[d] each, multiples of 4,
 * 4-byte aligned; 16-byte vector stores when all are 16-byte multiples) in
 * ONE launch on the context stream; dst may be peer memory
 * (NVLink stores). Used to move each plane range of the wsb_fft_rows
 * destination-major output into the other ranks' column-pass inputs while
 * the next range is transformed. Enqueued, no synchronisation. */
int wsb_push_blocks(wsb_ctx *ctx, int32_t n_dest, const void *const *src_ptrs,
                    void *const *dst_ptrs, const int64_t *bytes_host);

/* Column pass + w correction + stacking (transform.py:162-175, 192-230) of
 * planes [plane_lo, plane_hi): input tgrid holds this rank's column pairs
 * [g0, g0+ng) of those planes for all n_v rows, concatenated by source slab s
 * (src_rows[s] >= 1 rows each; slabs may differ in height) as
 *   [s][plane - plane_lo][g - g0][row - row_start_s][G]   (the all-to-all
 * output of wsb_fft_rows with destinations; one source = the P layout).
 * The planes are stacked from the top plane down (Horner's rule in the w
 * phase step), so plane ranges are passed in DESCENDING order: the first call
 * ends at n_w, each next call ends where the previous one began, with the
 * same (grid, g0, ng); the context carries the running sum between calls and
 * the result equals that of a single call over [0, n_w). The call whose range
 * starts at plane 0 writes image_strip
 * f64[n_v][ng*G] (row-major) and norm_partials
 * f64[WSB_COL_SPLIT(n_v)][ng*G][2] = (sum Im^2, sum Re^2) per image column
 * (and row residue class mod WSB_COL_SPLIT(n_v); fixed pairwise tree over
 * the rows); the caller sums residue-major, columns in order, which makes
 * the norms independent of the GPU count. Earlier calls leave both
 * untouched. */
int wsb_fft_cols_stack(wsb_ctx *ctx, const wsb_grid *grid, int32_t n_sources,
                       const int32_t *src_rows_host, int32_t g0, int32_t ng,
                       int32_t plane_lo, int32_t plane_hi, const double *tgrid,
                       double *image_strip, double *norm_partials);

/* Column pass + stack for the w-plane decomposition: this rank stacks the
 * planes [rank_plane_lo, rank_plane_hi) over all n_v rows and n_u columns;
 * tgrid holds planes [plane_lo, plane_hi) in the P layout (the output of
 * wsb_fft_rows of the rank's full-height grid, one destination). Ranges in
 * DESCENDING order as for wsb_fft_cols_stack, the first ending at
 * rank_plane_hi. The call whose range starts at rank_plane_lo writes
 * partial_image c128[n_v][n_u] = sum_k P_k exp(2 pi i w_k (n-1)) over the
 * rank's planes (unscaled); earlier calls leave it untouched. The sum of
 * the ranks' partial images goes through wsb_image_finish. */
int wsb_fft_cols_partial(wsb_ctx *ctx, const wsb_grid *grid, int32_t plane_lo, int32_t plane_hi,
                         int32_t rank_plane_lo, int32_t rank_plane_hi, const double *tgrid,
                         double *partial_image);

/* Number of row residues of wsb_image_finish's norm partials. */
#define WSB_FINISH_SPLIT(n_v) ((n_v) >= 4096 ? 16 : ((n_v) >= 256 ? (n_v) / 256 : 1))

/* Finish of a summed partial-stack image (w-plane decomposition): image
 * f64[n_v][n_u] = Re(sum / (n_u n_v) / n_w * n) (transform.py:192-230, the
 * same operations as the column pass' finish) and norm_partials
 * f64[WSB_FINISH_SPLIT(n_v)][n_u][2] = (sum Im^2, sum Re^2) per column and
 * row block (rows in order); the caller sums them residue-major, columns in
 * order. Enqueued. */
int wsb_image_finish(wsb_ctx *ctx, const wsb_grid *grid, const double *image_sum, double *image,
                     double *norm_partials);

/* Debug / parity: strip-layout slab -> natural (plane, row, col) complex128
 * with the checkerboard sign removed (the grid_all output layout,
 * mesh.py:131-146). */
int wsb_grid_unpack(wsb_ctx *ctx, const wsb_grid *grid, int32_t v_start, int32_t v_count,
                    const double *grid_s, double *grid_out);
/* Same for the slab rows [row_lo, row_hi) only: grid_out is
 * (n_w, row_hi - row_lo, n_u) complex128 (the slab-restricted parity check
 * of large meshes). */
int wsb_grid_unpack_rows(wsb_ctx *ctx, const wsb_grid *grid, int32_t v_start, int32_t v_count,
                         int32_t row_lo, int32_t row_hi, const double *grid_s, double *grid_out);

/* Debug / parity: the bucketing of the last wsb_grid_slab / wsb_image_device
 * call: record indices in item order (record order inside an item) and the
 * n_items+1 item offsets, item = (plane * ceil(n_u/WSB_ITEM_COLS) + column
 * block) * ceil(v_count/128) + row block. Sizes via wsb_tiles_debug(ctx, NULL, NULL,
 * &n, &nb). */
int wsb_tiles_debug(wsb_ctx *ctx, uint32_t *idx_host, uint32_t *off_host,
                    int64_t *n_entries, int64_t *n_buckets);

/* Debug / parity: the gridder's bucketing (K1) of m prepared records for
 * the slab rows [v_start, v_start+v_count): entries (record, work item)
 * with key = item << 8 | rowrel (item = (plane * ceil(n_u/WSB_ITEM_COLS) +
 * column block) * ceil(v_count/128) + row block, rowrel = floor(gv) - S - (first row of the
 * block - 2S)), sorted by key, record order for equal keys.
 * Host buffers (nullable): keys/idx u32[n_entries] (at most 4 m), off
 * u32[n_items + 1]. Sizes returned in *n_entries / *n_items / *item_bits.
 * Synchronous. */
int wsb_bucket_items(wsb_ctx *ctx, const wsb_grid *grid, int32_t half_support, int32_t v_start,
                     int32_t v_count, const double *rec, const uint32_t *plane, int64_t m,
                     uint32_t *keys_host, uint32_t *idx_host, uint32_t *off_host,
                     int64_t *n_entries, int64_t *n_items, int32_t *item_bits);

/* Timing of the kernels launched by the last wsb_image_device call, in ms,
 * measured with CUDA events on the context stream:
 * [0] prepare, [1] bucket+sort, [2] grid, [3] fft rows, [4] fft cols+stack,
 * [5] finish.  Returns the number of kernel launches in *launches. */
int wsb_last_timings(wsb_ctx *ctx, double *ms6, int32_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* WSB_H */
