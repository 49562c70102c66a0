// Throughput of FP64 warp MMA (mma.sync m8n8k4 f64) vs DFMA on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_bench dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_dmma(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
    if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void k_dfma(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) c[i] = fma(a, b, c[i]);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += c[i];
    if (s == 1234.5) out[0] = s;
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {4, 8, 16}) {
        dim3 g(sms * 4), b(32 * warps / 4 * 1);
        b = dim3(32 * warps);
        g = dim3(sms);
        k_dmma<8><<<g, b>>>(out, 100);
        cudaEventRecord(e0);
        k_dmma<8><<<g, b>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 256 * 8 * (double)iters * warps * sms;   // 256 FMA per mma
        printf("DMMA m8n8k4 warps/SM %2d: %.2f TFLOPS (%.3f ms)\n", warps, fl / ms / 1e9, ms);
        k_dfma<16><<<g, b>>>(out, 100);
        cudaEventRecord(e0);
        k_dfma<16><<<g, b>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 32 * 16 * (double)iters * warps * sms;
        printf("DFMA          warps/SM %2d: %.2f TFLOPS (%.3f ms)\n", warps, fl / ms / 1e9, ms);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
