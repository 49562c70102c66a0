// HBM efficiency of the access patterns the FFT layouts produce:
// every warp reads (and writes back) SEG-byte runs spaced STRIDE bytes apart.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_seg(const double2 *__restrict__ in, double2 *__restrict__ out, long n_elem,
                      int seg_elems, long stride_elems, long n_segs_per_col) {
    // element e -> segment s = e / seg_elems, within w = e % seg_elems
    // segments laid out column-major: seg s -> column s % n_cols, row s / n_cols
    const long n_cols = n_elem / seg_elems / n_segs_per_col;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n_elem;
         e += (long)gridDim.x * blockDim.x) {
        const long s = e / seg_elems, w = e % seg_elems;
        const long col = s % n_segs_per_col, row = s / n_segs_per_col;
        const long addr = col * stride_elems + row * seg_elems + w;
        out[addr] = in[addr];
    }
    (void)n_cols;
}

int main() {
    const long bytes = 2l << 30;  // 2 GiB
    const long n = bytes / 16;
    double2 *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int segs[] = {1, 2, 4, 8, 16, 32, 64};
    for (int si = 0; si < 7; ++si) {
        const int seg = segs[si];
        // n_segs_per_col "columns" each a contiguous region of (n / n_segs_per_col) elements
        for (long nsc : {1l, 1024l, 65536l}) {
            const long stride = n / nsc;
            if (stride < seg) continue;
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                cudaEventRecord(e0);
                k_seg<<<148 * 16, 256>>>(a, b, n, seg, stride, nsc);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("seg %4d B  interleave %6ld  : %7.1f GB/s (r+w)\n", seg * 16, nsc,
                   2.0 * bytes / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
