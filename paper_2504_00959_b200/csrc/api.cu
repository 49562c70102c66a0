// C ABI of libwsb.so (include/wsb.h): contexts, workspace, validation and
// the whole-hot-path entry points that replace run_pipeline phases 2-5
// (pipeline.py:95-152).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "wsb_internal.cuh"

namespace wsb {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

int ensure(wsb_ctx *ctx, int slot, size_t bytes, void **out) {
    if ((int)ctx->bufs.size() <= slot) ctx->bufs.resize(kSlotCount > slot + 1 ? kSlotCount : slot + 1);
    Buf &b = ctx->bufs[slot];
    if (b.bytes < bytes) {
        if (b.ptr) {
            // a pending kernel may still read the old buffer
            WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
            WSB_CUDA_TRY(cudaFree(b.ptr));
            b.ptr = nullptr;
            b.bytes = 0;
        }
        size_t want = std::max<size_t>(bytes, 256);
        cudaError_t e = cudaMalloc(&b.ptr, want);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(WSB_ENOMEM, "device allocation of " + std::to_string(want) + " bytes failed");
        }
        b.bytes = want;
    }
    *out = b.ptr;
    return WSB_OK;
}

// GridSpec (mesh.py:79-95) + KernelSpec (gridder.py:56-62) rules.
static int validate_grid(const wsb_grid *g) {
    if (!g) return fail(WSB_EINVAL, "grid is NULL");
    auto pow2 = [](int n) { return n >= 1 && (n & (n - 1)) == 0; };
    if (g->n_u < 2 || !pow2(g->n_u)) return fail(WSB_EINVAL, "n_u must be a power of two >= 2");
    if (g->n_v < 2 || !pow2(g->n_v)) return fail(WSB_EINVAL, "n_v must be a power of two >= 2");
    if (g->n_w < 1) return fail(WSB_EINVAL, "n_w must be >= 1");
    if (!(g->cell_size_lm > 0.0)) return fail(WSB_EINVAL, "cell_size_lm must be positive");
    const double hl = g->n_u * g->cell_size_lm / 2.0, hm = g->n_v * g->cell_size_lm / 2.0;
    if (hl >= 1.0 || hm >= 1.0 || hl * hl + hm * hm >= 1.0)
        return fail(WSB_EINVAL, "field of view too wide: corner pixels leave the unit disc");
    if (g->w_min_native > g->w_max_native) return fail(WSB_EINVAL, "w_min_native must be <= w_max_native");
    if (g->n_u > WSB_MAX_FFT_N || g->n_v > WSB_MAX_FFT_N)
        return fail(WSB_EUNSUPPORTED, "grids above 16384 per axis are not supported in this build");
    return WSB_OK;
}

static int validate_kernel(const wsb_kernel *k) {
    if (!k) return fail(WSB_EINVAL, "kernel is NULL");
    if (k->kind != WSB_KERNEL_GAUSSIAN && k->kind != WSB_KERNEL_KAISER_BESSEL)
        return fail(WSB_EINVAL, "kernel kind must be gaussian or kaiser_bessel");
    if (k->half_support < 1) return fail(WSB_EINVAL, "half_support must be >= 1");
    if (!(k->shape_param > 0.0)) return fail(WSB_EINVAL, "shape_param must be positive");
    if (k->half_support > kMaxS) return fail(WSB_EUNSUPPORTED, "half_support > 7 not compiled in this build");
    return WSB_OK;
}

static int set_device(wsb_ctx *ctx) {
    WSB_CUDA_TRY(cudaSetDevice(ctx->device));
    return WSB_OK;
}

// Device-side final sum of the per-column norm partials in a fixed
// two-level association: chunks of kNormChunk consecutive partials summed left
// to right (one thread per chunk), then the chunk sums left to right -- the
// association the multi-GPU root applies to the gathered partials
// (distributed.norm_sum), so the norms do not depend on the GPU count.
constexpr int kNormChunk = 64;
__global__ void __launch_bounds__(256) k_sum_partials(const double *p, int nb, double *out) {
    __shared__ double2 cs[1024];
    const int nc = (nb + kNormChunk - 1) / kNormChunk;
    double si = 0.0, sr = 0.0;
    for (int base = 0; base < nc; base += 1024) {
        const int n = min(1024, nc - base);
        for (int c = threadIdx.x; c < n; c += blockDim.x) {
            const int lo = (base + c) * kNormChunk, hi = min(lo + kNormChunk, nb);
            double a = 0.0, b = 0.0;
#pragma unroll 8
            for (int i = lo; i < hi; ++i) {
                const double2 x = *reinterpret_cast<const double2 *>(p + 2 * i);
                a += x.x;
                b += x.y;
            }
            cs[c] = make_double2(a, b);
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int c = 0; c < n; ++c) {
                si += cs[c].x;
                sr += cs[c].y;
            }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = si;
        out[1] = sr;
    }
}

// Strip layout -> (plane, row, col) complex128 with the checkerboard sign
// removed, for slab rows [r0, r0 + nr) (relative to v_start).
__global__ void k_unpack(const double2 *p, double2 *out, int n_w, int n_u, int v_start, int v_count,
                         int r0, int nr) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)n_w * nr * n_u;
    if (e >= total) return;
    const int i = e % n_u;
    const int64_t t = e / n_u;
    const int j = (int)(t % nr) + r0;
    const int k = (int)(t / nr);
    // strip layout [plane][col/WSB_STRIP][row][re | im][col%WSB_STRIP]
    constexpr int SW = WSB_STRIP;
    const double *q = reinterpret_cast<const double *>(p) +
                      (((int64_t)k * ((n_u + SW - 1) / SW) + i / SW) * v_count + j) * (2 * SW) + i % SW;
    double2 z = make_double2(q[0], q[SW]);
    const double s = ((i + v_start + j) & 1) ? -1.0 : 1.0;
    out[e] = make_double2(z.x * s, z.y * s);
}

// ---------------------------------------------------------------------------
// Energy over a call (SURVEY 8b wsb_diag.gpu_joules / host_joules): NVML's
// total-energy counter of the call's GPU (mJ; libnvidia-ml is opened at run
// time, no link dependency) and the RAPL package counters of the host
// (/sys/class/powercap/intel-rapl:N/energy_uj, wrap-around corrected).
// -1 when a counter is unreadable. The counters update every few ms, so a
// single short call reads coarse values; metered runs loop many calls.
// ---------------------------------------------------------------------------
namespace {

struct Nvml {
    void *so = nullptr;
    int (*get_handle)(const char *, void **) = nullptr;
    int (*energy)(void *, unsigned long long *) = nullptr;
    bool ok = false;
    Nvml() {
        so = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
        if (!so) return;
        auto init = (int (*)())dlsym(so, "nvmlInit_v2");
        get_handle = (int (*)(const char *, void **))dlsym(so, "nvmlDeviceGetHandleByPciBusId_v2");
        energy = (int (*)(void *, unsigned long long *))dlsym(so, "nvmlDeviceGetTotalEnergyConsumption");
        ok = init && get_handle && energy && init() == 0;
    }
    // millijoules of the CUDA device `dev` (matched by PCI bus id), or -1
    double mj(int dev) {
        if (!ok) return -1.0;
        char bus[32];
        if (cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess) {
            cudaGetLastError();
            return -1.0;
        }
        void *h = nullptr;
        unsigned long long e = 0;
        if (get_handle(bus, &h) != 0 || energy(h, &e) != 0) return -1.0;
        return (double)e;
    }
};

Nvml &nvml() {
    static Nvml n;
    return n;
}

// sum over package domains of (energy_uj, max_energy_range_uj); false if none readable
bool rapl_read(std::vector<std::pair<double, double>> *out) {
    out->clear();
    for (int i = 0; i < 16; ++i) {
        const std::string base = "/sys/class/powercap/intel-rapl:" + std::to_string(i);
        FILE *f = std::fopen((base + "/energy_uj").c_str(), "r");
        if (!f) continue;
        double e = -1, r = 0;
        if (std::fscanf(f, "%lf", &e) != 1) e = -1;
        std::fclose(f);
        if ((f = std::fopen((base + "/max_energy_range_uj").c_str(), "r"))) {
            if (std::fscanf(f, "%lf", &r) != 1) r = 0;
            std::fclose(f);
        }
        if (e >= 0) out->push_back({e, r});
    }
    return !out->empty();
}

}  // namespace

void EnergyWindow::start(int dev) {
    device = dev;
    gpu0 = nvml().mj(dev);
    host_ok = rapl_read(&host0);
}

void EnergyWindow::stop(double *gpu_j, double *host_j) {
    const double g1 = nvml().mj(device);
    *gpu_j = (gpu0 >= 0 && g1 >= 0) ? (g1 - gpu0) / 1e3 : -1.0;
    std::vector<std::pair<double, double>> h1;
    if (host_ok && rapl_read(&h1) && h1.size() == host0.size()) {
        double uj = 0;
        for (size_t i = 0; i < h1.size(); ++i) {
            double d = h1[i].first - host0[i].first;
            if (d < 0) d += host0[i].second;   // counter wrapped
            uj += d;
        }
        *host_j = uj / 1e6;
    } else {
        *host_j = -1.0;
    }
}

}  // namespace wsb

using namespace wsb;

extern "C" {

const char *wsb_strerror(int code) {
    switch (code) {
        case WSB_OK: return "ok";
        case WSB_EINVAL: return "invalid argument";
        case WSB_ECUDA: return "CUDA error";
        case WSB_ENCCL: return "NCCL error";
        case WSB_ENOMEM: return "out of device memory";
        case WSB_EUNSUPPORTED: return "unsupported configuration";
        default: return "unknown error";
    }
}

const char *wsb_last_error(void) { return g_last_error.c_str(); }

int wsb_version(void) { return WSB_VERSION; }

int wsb_ctx_create(int32_t device, wsb_ctx **out) {
    if (!out) return fail(WSB_EINVAL, "out is NULL");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(WSB_ECUDA, "no CUDA device available");
    }
    if (device < 0 || device >= n) return fail(WSB_EINVAL, "device ordinal out of range");
    wsb_ctx *c = new wsb_ctx();
    c->device = device;
    c->bufs.resize(kSlotCount);
    int rc = set_device(c);
    if (rc == WSB_OK) {
        // The gridder gathers 32-byte records at random; larger L2 fetches
        // only waste HBM bandwidth (streaming kernels read whole lines anyway).
        if (cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32) != cudaSuccess) cudaGetLastError();
        cudaError_t a = cudaMallocHost(&c->flag_host, 64);
        if (a != cudaSuccess) rc = fail(WSB_ENOMEM, "pinned allocation failed");
    }
    if (rc == WSB_OK) {
        for (int i = 0; i < 8; ++i) cudaEventCreate(&c->timing.ev[i]);
        c->timing.created = true;
    }
    if (rc != WSB_OK) {
        delete c;
        return rc;
    }
    *out = c;
    return WSB_OK;
}

int wsb_ctx_trim(wsb_ctx *ctx) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(set_device(ctx));
    WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    for (auto &b : ctx->bufs) {
        if (b.ptr) cudaFree(b.ptr);
        b.ptr = nullptr;
        b.bytes = 0;
    }
    return WSB_OK;
}

int wsb_ctx_destroy(wsb_ctx *ctx) {
    if (!ctx) return WSB_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto &b : ctx->bufs)
        if (b.ptr) cudaFree(b.ptr);
    for (int i = 0; i < 96; ++i)
        if (ctx->twiddle[i]) cudaFree(ctx->twiddle[i]);
    if (ctx->timing.created)
        for (int i = 0; i < 8; ++i) cudaEventDestroy(ctx->timing.ev[i]);
    if (ctx->flag_host) cudaFreeHost(ctx->flag_host);
    delete ctx;
    return WSB_OK;
}

int wsb_ctx_set_precision(wsb_ctx *ctx, int32_t precision) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    if (precision != 64 && precision != 32) return fail(WSB_EINVAL, "precision must be 64 or 32");
    ctx->precision = precision;
    return WSB_OK;
}

int wsb_ctx_set_energy(wsb_ctx *ctx, int32_t on) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    ctx->energy = on ? 1 : 0;
    return WSB_OK;
}

int wsb_ctx_set_stream(wsb_ctx *ctx, void *stream) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    ctx->stream = (cudaStream_t)stream;
    return WSB_OK;
}

int wsb_prepare(wsb_ctx *ctx, const wsb_grid *grid, const double *u, const double *v,
                const double *w, const float *vis, const float *weight, int64_t n, int32_t n_chan,
                double *rec, uint32_t *plane) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(validate_grid(grid));
    if (n < 0 || n_chan < 1) return fail(WSB_EINVAL, "n must be >= 0 and n_chan >= 1");
    if (n > 0xFFFFFFFFll) return fail(WSB_EUNSUPPORTED, "more than 2^32 records per GPU");
    WSB_TRY(set_device(ctx));
    return prepare(ctx, grid, u, v, w, vis, weight, n, n_chan, rec, plane);
}

int wsb_route_count(wsb_ctx *ctx, const wsb_grid *grid, int32_t half_support, int32_t n_ranks,
                    const int32_t *slab_starts_host, const double *rec, int64_t n,
                    int64_t *counts_host) {
    if (!ctx || !counts_host) return fail(WSB_EINVAL, "NULL argument");
    WSB_TRY(validate_grid(grid));
    if (half_support < 0) return fail(WSB_EINVAL, "halo_rows must be >= 0");
    WSB_TRY(set_device(ctx));
    return wsb::route_count(ctx, grid, half_support, n_ranks, slab_starts_host, rec, n, counts_host,
                            nullptr, nullptr);
}

int wsb_route_pack(wsb_ctx *ctx, const wsb_grid *grid, int32_t half_support, int32_t n_ranks,
                   const int32_t *slab_starts_host, const double *rec, const uint32_t *plane,
                   int64_t n, double *send_rec, uint32_t *send_plane, int64_t *src_index) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(validate_grid(grid));
    if (half_support < 0) return fail(WSB_EINVAL, "halo_rows must be >= 0");
    WSB_TRY(set_device(ctx));
    return wsb::route_pack(ctx, grid, half_support, n_ranks, slab_starts_host, rec, plane, n,
                           send_rec, send_plane, src_index);
}

int wsb_plane_histogram(wsb_ctx *ctx, const wsb_grid *grid, const uint32_t *plane, int64_t n,
                        uint32_t *hist) {
    if (!ctx || !hist) return fail(WSB_EINVAL, "NULL argument");
    WSB_TRY(validate_grid(grid));
    WSB_TRY(set_device(ctx));
    return plane_histogram(ctx, grid, plane, n, hist);
}

int wsb_route_planes_count(wsb_ctx *ctx, const wsb_grid *grid, int32_t n_ranks,
                           const int32_t *plane_starts_host, const double *rec,
                           const uint32_t *plane, int64_t n, int64_t *counts_host) {
    if (!ctx || !counts_host) return fail(WSB_EINVAL, "NULL argument");
    WSB_TRY(validate_grid(grid));
    WSB_TRY(set_device(ctx));
    return wsb::route_count(ctx, grid, 0, n_ranks, plane_starts_host, rec, n, counts_host, nullptr,
                            nullptr, plane, 1);
}

int wsb_route_planes_pack(wsb_ctx *ctx, const wsb_grid *grid, int32_t n_ranks,
                          const int32_t *plane_starts_host, const double *rec,
                          const uint32_t *plane, int64_t n, double *send_rec,
                          uint32_t *send_plane, int64_t *src_index) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(validate_grid(grid));
    WSB_TRY(set_device(ctx));
    return wsb::route_pack(ctx, grid, 0, n_ranks, plane_starts_host, rec, plane, n, send_rec,
                           send_plane, src_index, 1);
}

int wsb_row_histogram(wsb_ctx *ctx, const wsb_grid *grid, const double *rec, int64_t n,
                      uint32_t *hist) {
    if (!ctx || !hist) return fail(WSB_EINVAL, "NULL argument");
    WSB_TRY(validate_grid(grid));
    WSB_TRY(set_device(ctx));
    return wsb::row_histogram(ctx, grid, rec, n, hist);
}

static int grid_slab_impl(wsb_ctx *ctx, const wsb_grid *grid, const wsb_kernel *kern,
                          int32_t v_start, int32_t v_count, const double *rec,
                          const uint32_t *plane, int64_t m, double *grid_p,
                          unsigned long long *updates_dev, int64_t *n_entries_out,
                          const cudaEvent_t *mid = nullptr) {
    ItemBuckets bk;
    WSB_TRY(bucket_items(ctx, grid, kern->half_support, v_start, v_count, nullptr,
                         const_cast<double *>(rec), const_cast<uint32_t *>(plane), m, &bk));
    if (n_entries_out) *n_entries_out = bk.n_entries;
    if (mid) WSB_CUDA_TRY(cudaEventRecord(*mid, ctx->stream));
    return grid_items(ctx, grid, kern, v_start, v_count, rec, bk, grid_p, updates_dev);
}

int wsb_grid_slab(wsb_ctx *ctx, const wsb_grid *grid, const wsb_kernel *kern, int32_t v_start,
                  int32_t v_count, const double *rec, const uint32_t *plane, int64_t m,
                  double *grid_p, int64_t *grid_updates) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(validate_grid(grid));
    WSB_TRY(validate_kernel(kern));
    if (v_start < 0 || v_count < 1 || v_start + v_count > grid->n_v)
        return fail(WSB_EINVAL, "slab rows outside the mesh");
    if (m < 0 || m > 0xFFFFFFFFll) return fail(WSB_EINVAL, "record count out of range");
    WSB_TRY(set_device(ctx));
    unsigned long long *upd;
    WSB_TRY(ensure(ctx, kSlotU64, 64, (void **)&upd));
    WSB_CUDA_TRY(cudaMemsetAsync(upd, 0, sizeof(unsigned long long), ctx->stream));
    // bucket / sweep times of this call go to wsb_last_timings slots 1 and 2
    // (read when the call synchronises anyway, i.e. grid_updates requested)
    cudaEvent_t *ev = ctx->timing.ev;
    WSB_CUDA_TRY(cudaEventRecord(ev[0], ctx->stream));
    WSB_TRY(grid_slab_impl(ctx, grid, kern, v_start, v_count, rec, plane, m, grid_p, upd, nullptr,
                           &ev[1]));
    WSB_CUDA_TRY(cudaEventRecord(ev[2], ctx->stream));
    if (grid_updates) {
        unsigned long long h;
        WSB_CUDA_TRY(cudaMemcpyAsync(ctx->flag_host, upd, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        std::memcpy(&h, ctx->flag_host, sizeof(h));
        *grid_updates = (int64_t)h;
        float a = 0.f, b = 0.f;
        WSB_CUDA_TRY(cudaEventElapsedTime(&a, ev[0], ev[1]));
        WSB_CUDA_TRY(cudaEventElapsedTime(&b, ev[1], ev[2]));
        for (int i = 0; i < 6; ++i) ctx->last_ms[i] = 0.0;
        ctx->last_ms[1] = a;
        ctx->last_ms[2] = b;
    }
    return WSB_OK;
}

int wsb_fft_rows(wsb_ctx *ctx, const wsb_grid *grid, int32_t v_count, const double *grid_s,
                 double *grid_p, int32_t plane_lo, int32_t plane_hi, int32_t n_dest,
                 const int32_t *dest_pairs_host) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(validate_grid(grid));
    if (plane_lo < 0 || plane_hi > grid->n_w || plane_lo > plane_hi)
        return fail(WSB_EINVAL, "plane range outside [0, n_w]");
    if (grid_s == grid_p) return fail(WSB_EINVAL, "the row pass is out of place");
    WSB_TRY(set_device(ctx));
    return fft_rows(ctx, grid, v_count, grid_s, grid_p, plane_lo, plane_hi,
                    dest_pairs_host ? n_dest : 1, dest_pairs_host);
}

int wsb_fft_rows_peer(wsb_ctx *ctx, const wsb_grid *grid, int32_t v_count, const double *grid_s,
                      int32_t plane_lo, int32_t plane_hi, int32_t n_dest,
                      const int32_t *dest_cols_host, void *const *dest_ptrs_host) {
    if (!ctx || !dest_cols_host || !dest_ptrs_host) return fail(WSB_EINVAL, "NULL argument");
    WSB_TRY(validate_grid(grid));
    if (plane_lo < 0 || plane_hi > grid->n_w || plane_lo > plane_hi)
        return fail(WSB_EINVAL, "plane range outside [0, n_w]");
    WSB_TRY(set_device(ctx));
    return fft_rows(ctx, grid, v_count, grid_s, nullptr, plane_lo, plane_hi, n_dest,
                    dest_cols_host, dest_ptrs_host);
}

int wsb_fft_cols_stack(wsb_ctx *ctx, const wsb_grid *grid, int32_t n_sources,
                       const int32_t *src_rows_host, int32_t g0, int32_t ng, int32_t plane_lo,
                       int32_t plane_hi, const double *tgrid, double *image_strip,
                       double *norm_partials) {
    if (!ctx || !src_rows_host) return fail(WSB_EINVAL, "NULL argument");
    WSB_TRY(validate_grid(grid));
    if (plane_lo < 0 || plane_hi > grid->n_w || plane_lo > plane_hi)
        return fail(WSB_EINVAL, "plane range outside [0, n_w]");
    if (g0 < 0 || ng < 1 || (g0 + ng) * kG > grid->n_u) return fail(WSB_EINVAL, "column groups outside the mesh");
    WSB_TRY(set_device(ctx));
    return fft_cols_stack(ctx, grid, n_sources, src_rows_host, g0, ng, plane_lo, plane_hi, tgrid,
                          image_strip, norm_partials);
}

int wsb_fft_cols_partial(wsb_ctx *ctx, const wsb_grid *grid, int32_t plane_lo, int32_t plane_hi,
                         int32_t rank_plane_lo, int32_t rank_plane_hi, const double *tgrid,
                         double *partial_image) {
    if (!ctx || !tgrid || !partial_image) return fail(WSB_EINVAL, "NULL argument");
    WSB_TRY(validate_grid(grid));
    if (!(0 <= rank_plane_lo && rank_plane_lo <= plane_lo && plane_lo < plane_hi &&
          plane_hi <= rank_plane_hi && rank_plane_hi <= grid->n_w))
        return fail(WSB_EINVAL, "plane range outside the rank's planes");
    WSB_TRY(set_device(ctx));
    const int32_t rows[1] = {grid->n_v};
    return fft_cols_stack(ctx, grid, 1, rows, 0, grid->n_u / kG, plane_lo, plane_hi, tgrid, nullptr,
                          nullptr, 64, rank_plane_lo, rank_plane_hi, partial_image);
}

int wsb_image_finish(wsb_ctx *ctx, const wsb_grid *grid, const double *image_sum, double *image,
                     double *norm_partials) {
    if (!ctx || !image_sum || !image || !norm_partials) return fail(WSB_EINVAL, "NULL argument");
    WSB_TRY(validate_grid(grid));
    WSB_TRY(set_device(ctx));
    return image_finish(ctx, grid, image_sum, image, norm_partials);
}

int wsb_grid_unpack_rows(wsb_ctx *ctx, const wsb_grid *grid, int32_t v_start, int32_t v_count,
                         int32_t row_lo, int32_t row_hi, const double *grid_p, double *grid_out) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(validate_grid(grid));
    if (v_start < 0 || v_count < 1 || v_start + v_count > grid->n_v)
        return fail(WSB_EINVAL, "slab rows outside the mesh");
    if (row_lo < v_start || row_hi > v_start + v_count || row_lo > row_hi)
        return fail(WSB_EINVAL, "rows outside the slab");
    WSB_TRY(set_device(ctx));
    const int nr = row_hi - row_lo;
    const int64_t total = (int64_t)grid->n_w * nr * grid->n_u;
    if (total == 0) return WSB_OK;
    k_unpack<<<ceil_div(total, 256), 256, 0, ctx->stream>>>((const double2 *)grid_p,
                                                            (double2 *)grid_out, grid->n_w,
                                                            grid->n_u, v_start, v_count,
                                                            row_lo - v_start, nr);
    WSB_CUDA_TRY(cudaGetLastError());
    return WSB_OK;
}

int wsb_grid_unpack(wsb_ctx *ctx, const wsb_grid *grid, int32_t v_start, int32_t v_count,
                    const double *grid_p, double *grid_out) {
    return wsb_grid_unpack_rows(ctx, grid, v_start, v_count, v_start, v_start + v_count, grid_p,
                                grid_out);
}

int wsb_tiles_debug(wsb_ctx *ctx, uint32_t *idx_host, uint32_t *off_host, int64_t *n_entries,
                    int64_t *n_buckets) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(set_device(ctx));
    if (n_entries) *n_entries = ctx->last_entries;
    if (n_buckets) *n_buckets = ctx->last_tiles;
    WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (idx_host && ctx->last_entries)
        WSB_CUDA_TRY(cudaMemcpy(idx_host, ctx->last_idx, 4 * ctx->last_entries, cudaMemcpyDeviceToHost));
    if (off_host && ctx->last_tiles)
        WSB_CUDA_TRY(cudaMemcpy(off_host, ctx->last_off, 4 * (ctx->last_tiles + 1), cudaMemcpyDeviceToHost));
    return WSB_OK;
}

int wsb_bucket_items(wsb_ctx *ctx, const wsb_grid *grid, int32_t half_support, int32_t v_start,
                     int32_t v_count, const double *rec, const uint32_t *plane, int64_t m,
                     uint32_t *keys_host, uint32_t *idx_host, uint32_t *off_host,
                     int64_t *n_entries, int64_t *n_items, int32_t *item_bits) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(validate_grid(grid));
    if (half_support < 1 || half_support > kMaxS) return fail(WSB_EINVAL, "half_support out of range");
    if (v_start < 0 || v_count < 1 || v_start + v_count > grid->n_v)
        return fail(WSB_EINVAL, "slab rows outside the mesh");
    WSB_TRY(set_device(ctx));
    ItemBuckets bk;
    WSB_TRY(bucket_items(ctx, grid, half_support, v_start, v_count, nullptr, const_cast<double *>(rec),
                         const_cast<uint32_t *>(plane), m, &bk));
    if (n_entries) *n_entries = bk.n_entries;
    if (n_items) *n_items = bk.n_items;
    if (item_bits) *item_bits = bk.item_bits;
    WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    WSB_TRY(bucket_errors(ctx));
    if (keys_host && bk.n_entries)
        WSB_CUDA_TRY(cudaMemcpy(keys_host, bk.keys, 4 * bk.n_entries, cudaMemcpyDeviceToHost));
    if (idx_host && bk.n_entries)
        WSB_CUDA_TRY(cudaMemcpy(idx_host, bk.idx, 4 * bk.n_entries, cudaMemcpyDeviceToHost));
    if (off_host)
        WSB_CUDA_TRY(cudaMemcpy(off_host, bk.off, 4 * (bk.n_items + 1), cudaMemcpyDeviceToHost));
    return WSB_OK;
}

int wsb_last_timings(wsb_ctx *ctx, double *ms6, int32_t *launches) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    if (ms6)
        for (int i = 0; i < 6; ++i) ms6[i] = ctx->last_ms[i];
    if (launches) *launches = ctx->launches;
    return WSB_OK;
}

static int image_device_impl(wsb_ctx *ctx, const wsb_grid *grid, const wsb_kernel *kern,
                             const double *u, const double *v, const double *w, const float *vis,
                             const float *weight, const uint32_t *time_index, int64_t n,
                             int32_t n_chan, double *image_out, wsb_diag *diag) {
    if (!ctx) return fail(WSB_EINVAL, "ctx is NULL");
    WSB_TRY(validate_grid(grid));
    WSB_TRY(validate_kernel(kern));
    if (n < 0 || n_chan < 1) return fail(WSB_EINVAL, "n must be >= 0 and n_chan >= 1");
    if (n > 0xFFFFFFFFll) return fail(WSB_EUNSUPPORTED, "more than 2^32 records per GPU");
    WSB_TRY(set_device(ctx));
    ctx->launches = 0;
    cudaEvent_t *ev = ctx->timing.ev;
    const int n_u = grid->n_u, n_v = grid->n_v, n_w = grid->n_w;
    double *rec, *partials;
    void *gs, *gp;
    const int prec = ctx->precision;
    const size_t esz = prec == 32 ? 8 : 16;   // complex64 / complex128 grid cells
    uint32_t *plane;
    unsigned long long *upd;
    const int64_t nn = std::max<int64_t>(n, 1);
    WSB_TRY(ensure(ctx, kSlotRec, 32 * (size_t)nn, (void **)&rec));
    WSB_TRY(ensure(ctx, kSlotPlane, 4 * (size_t)nn, (void **)&plane));
    // strip layout (gridder output) and P layout (row-pass output)
    WSB_TRY(ensure(ctx, kSlotGrid, esz * n_w * ceil_div(n_u, WSB_STRIP) * WSB_STRIP * n_v, &gs));
    WSB_TRY(ensure(ctx, kSlotGridP, esz * n_w * n_u * n_v, &gp));
    // norm partials [residue][column][2] (residues: columns longer than 4096 are split)
    const int sp = std::max(1, n_v >> kMaxOnChipLog);
    WSB_TRY(ensure(ctx, kSlotStrip, sizeof(double) * (2 * (size_t)n_u * sp + 4), (void **)&partials));
    WSB_TRY(ensure(ctx, kSlotU64, 64, (void **)&upd));
    const void *tw;   // tables built outside the timed region
    WSB_TRY(twiddles(ctx, std::min(n_u, 1 << kMaxOnChipLog), 4, &tw, prec));   // rows (radix 16)
    WSB_TRY(twiddles(ctx, std::min(n_v, 1 << kMaxOnChipLog), 3, &tw, prec));   // columns (radix 8)
    if (n_u > (1 << kMaxOnChipLog)) WSB_TRY(twiddles(ctx, n_u, 0, &tw, prec));
    if (n_v > (1 << kMaxOnChipLog)) WSB_TRY(twiddles(ctx, n_v, 0, &tw, prec));

    WSB_CUDA_TRY(cudaEventRecord(ev[0], ctx->stream));
    WSB_CUDA_TRY(cudaMemsetAsync(upd, 0, sizeof(unsigned long long), ctx->stream));
    ItemBuckets bk;
    if (n_chan == 1) {
        // prepare_chunk fused into the bucketing pass (one read of the columns)
        WSB_CUDA_TRY(cudaEventRecord(ev[1], ctx->stream));
        const VisColumns cols{u, v, w, vis, weight, time_index};
        WSB_TRY(bucket_items(ctx, grid, kern->half_support, 0, n_v, &cols, rec, nullptr, n, &bk));
    } else {
        WSB_TRY(prepare(ctx, grid, u, v, w, vis, weight, n, n_chan, rec, plane, time_index));
        WSB_CUDA_TRY(cudaEventRecord(ev[1], ctx->stream));
        WSB_TRY(bucket_items(ctx, grid, kern->half_support, 0, n_v, nullptr, rec, plane, n, &bk));
    }
    const int64_t n_entries = bk.n_entries;
    WSB_CUDA_TRY(cudaEventRecord(ev[2], ctx->stream));
    WSB_TRY(grid_items(ctx, grid, kern, 0, n_v, rec, bk, gs, upd, prec));
    WSB_CUDA_TRY(cudaEventRecord(ev[3], ctx->stream));
    WSB_TRY(fft_rows(ctx, grid, n_v, gs, gp, 0, n_w, 1, nullptr, nullptr, prec));
    WSB_CUDA_TRY(cudaEventRecord(ev[4], ctx->stream));
    const int32_t rows[1] = {n_v};
    WSB_TRY(fft_cols_stack(ctx, grid, 1, rows, 0, n_u / kG, 0, n_w, gp, image_out, partials, prec));
    WSB_CUDA_TRY(cudaEventRecord(ev[5], ctx->stream));
    const int nb = n_u * sp;  // one norm partial per image column (and residue)
    k_sum_partials<<<1, 256, 0, ctx->stream>>>(partials, nb, partials + 2 * (size_t)nb);
    ctx->launches += 1;
    WSB_CUDA_TRY(cudaGetLastError());
    WSB_CUDA_TRY(cudaEventRecord(ev[6], ctx->stream));
    if (diag) {
        double norms[2];
        unsigned long long h;
        WSB_CUDA_TRY(cudaMemcpyAsync(norms, partials + 2 * (size_t)nb, sizeof(norms),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        WSB_CUDA_TRY(cudaMemcpyAsync(&h, upd, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        WSB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        diag->imag_residual_norm = std::sqrt(norms[0]);
        diag->real_norm = std::sqrt(norms[1]);
        diag->grid_updates = (int64_t)h;
        diag->records = n;
        diag->tile_entries = n_entries;
        float ms[6];
        for (int i = 0; i < 6; ++i) {
            cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]);
            ctx->last_ms[i] = ms[i];
        }
        for (int i = 0; i < 7; ++i) diag->phase_ms[i] = 0.0;
        diag->phase_ms[1] = ms[0] + ms[1] + ms[2];      // gridding: prepare + bucket + grid
        diag->phase_ms[3] = ms[3] + ms[4];              // fft (column pass carries w correction)
        diag->phase_ms[4] = ms[5];                      // wcorrect: final reduction
        diag->phase_ms[6] = ms[0] + ms[1] + ms[2] + ms[3] + ms[4] + ms[5];
        diag->exchanged_records = 0;   // one GPU: no record leaves the device
    }
    return WSB_OK;
}

int wsb_image_device(wsb_ctx *ctx, const wsb_grid *grid, const wsb_kernel *kern, const double *u,
                     const double *v, const double *w, const float *vis, const float *weight,
                     int64_t n, int32_t n_chan, double *image_out, wsb_diag *diag) {
    EnergyWindow en;
    const bool metered = diag && ctx && ctx->energy;
    if (metered) en.start(ctx->device);
    int rc = image_device_impl(ctx, grid, kern, u, v, w, vis, weight, nullptr, n, n_chan, image_out,
                               diag);
    if (rc == WSB_OK && diag) {
        diag->gpu_joules = diag->host_joules = -1.0;
        if (metered) en.stop(&diag->gpu_joules, &diag->host_joules);
    }
    return rc;
}

static std::mutex g_host_mu;
static wsb_ctx *g_host_ctx[64] = {nullptr};

int wsb_image(const wsb_grid *grid, const wsb_kernel *kern, const wsb_exec *exec, const double *u,
              const double *v, const double *w, const uint32_t *time_index, const float *vis,
              const float *weight, int64_t n, int32_t n_chan, double *image_out, wsb_diag *diag) {
    WSB_TRY(validate_grid(grid));
    WSB_TRY(validate_kernel(kern));
    if (n < 0 || n_chan < 1) return fail(WSB_EINVAL, "n must be >= 0 and n_chan >= 1");
    if ((n > 0 && (!u || !v || !w || !vis || !weight)) || !image_out)
        return fail(WSB_EINVAL, "NULL buffer");
    const int dev = exec ? exec->device : 0;
    const int prec = exec ? exec->precision : 64;
    if (prec != 64 && prec != 32) return fail(WSB_EINVAL, "precision must be 64 or 32");
    if (dev < 0 || dev >= 64) return fail(WSB_EINVAL, "device ordinal out of range");
    std::lock_guard<std::mutex> lock(g_host_mu);
    if (!g_host_ctx[dev]) WSB_TRY(wsb_ctx_create(dev, &g_host_ctx[dev]));
    wsb_ctx *ctx = g_host_ctx[dev];
    ctx->precision = prec;
    WSB_TRY(set_device(ctx));
    const int64_t nn = std::max<int64_t>(n, 1);
    auto rnd = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t b_uvw = rnd(8 * (size_t)nn), b_vis = rnd(8 * (size_t)nn * n_chan),
                 b_wt = rnd(4 * (size_t)nn * n_chan);
    const size_t b_img = 8 * (size_t)grid->n_u * grid->n_v;
    const size_t b_t = time_index ? rnd(4 * (size_t)nn) : 0;
    unsigned char *in;
    WSB_TRY(ensure(ctx, kSlotHostIn, 3 * b_uvw + b_vis + b_wt + b_img + b_t, (void **)&in));
    uint32_t *dt = time_index ? (uint32_t *)(in + 3 * b_uvw + b_vis + b_wt + b_img) : nullptr;
    EnergyWindow en;
    const bool metered = diag && exec && (exec->flags & WSB_EXEC_ENERGY);
    if (metered) en.start(dev);
    double *du = (double *)in, *dv = (double *)(in + b_uvw), *dw = (double *)(in + 2 * b_uvw);
    float *dvis = (float *)(in + 3 * b_uvw), *dwt = (float *)(in + 3 * b_uvw + b_vis);
    double *dimg = (double *)(in + 3 * b_uvw + b_vis + b_wt);
    cudaEvent_t a0, a1, a2, a3;
    cudaEventCreate(&a0);
    cudaEventCreate(&a1);
    cudaEventCreate(&a2);
    cudaEventCreate(&a3);
    cudaEventRecord(a0, ctx->stream);
    if (n > 0) {
        WSB_CUDA_TRY(cudaMemcpyAsync(du, u, 8 * n, cudaMemcpyHostToDevice, ctx->stream));
        WSB_CUDA_TRY(cudaMemcpyAsync(dv, v, 8 * n, cudaMemcpyHostToDevice, ctx->stream));
        WSB_CUDA_TRY(cudaMemcpyAsync(dw, w, 8 * n, cudaMemcpyHostToDevice, ctx->stream));
        WSB_CUDA_TRY(cudaMemcpyAsync(dvis, vis, 8 * (size_t)n * n_chan, cudaMemcpyHostToDevice, ctx->stream));
        WSB_CUDA_TRY(cudaMemcpyAsync(dwt, weight, 4 * (size_t)n * n_chan, cudaMemcpyHostToDevice, ctx->stream));
        if (dt) WSB_CUDA_TRY(cudaMemcpyAsync(dt, time_index, 4 * (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
    }
    cudaEventRecord(a1, ctx->stream);
    wsb_diag local;
    int rc = image_device_impl(ctx, grid, kern, du, dv, dw, dvis, dwt, dt, n, n_chan, dimg, &local);
    if (rc == WSB_OK) {
        cudaEventRecord(a2, ctx->stream);
        cudaError_t e = cudaMemcpyAsync(image_out, dimg, b_img, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaEventRecord(a3, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) rc = fail(WSB_ECUDA, std::string("copy-out: ") + cudaGetErrorString(e));
    }
    if (rc == WSB_OK && diag) {
        float r, wr, tot;
        cudaEventElapsedTime(&r, a0, a1);
        cudaEventElapsedTime(&wr, a2, a3);
        cudaEventElapsedTime(&tot, a0, a3);
        *diag = local;
        diag->phase_ms[0] = r;
        diag->phase_ms[5] = wr;
        diag->phase_ms[6] = tot;
        diag->gpu_joules = diag->host_joules = -1.0;
        if (metered) en.stop(&diag->gpu_joules, &diag->host_joules);
    }
    cudaEventDestroy(a0);
    cudaEventDestroy(a1);
    cudaEventDestroy(a2);
    cudaEventDestroy(a3);
    return rc;
}

}  // extern "C"
