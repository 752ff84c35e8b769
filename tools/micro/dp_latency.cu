// Microbenchmark: fp64 DADD/DMUL dependent latency and issue throughput on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false dp_latency.cu -o dp_latency
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_add(double* out, long long* cyc, int iters) {
    double x = out[0] + threadIdx.x, y = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = x + y;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
    if (x == 123.0) out[1] = x;
}
__global__ void lat_mul(double* out, long long* cyc, int iters) {
    double x = out[0] + threadIdx.x, y = 1.0000000001;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = x * y;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
    if (x == 123.0) out[1] = x;
}
// independent chains: K chains per thread, W warps per block (one block on one SM)
template <int K>
__global__ void thr(double* out, long long* cyc, int iters) {
    double x[K];
    for (int k = 0; k < K; ++k) x[k] = out[0] + threadIdx.x + k;
    const double y = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = x[k] + y;
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
    double s = 0; for (int k = 0; k < K; ++k) s += x[k];
    if (s == 123.0) out[1] = s;
}
__global__ void shfl_lat(double* out, long long* cyc, int iters) {
    double x = out[0] + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = __shfl_xor_sync(0xffffffffu, x, 1);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
    if (x == 123.0) out[1] = x;
}
__global__ void div_lat(double* out, long long* cyc, int iters) {
    double x = out[0] + threadIdx.x + 1.5, y = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) x = x / y;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
    if (x == 123.0) out[1] = x;
}
int main() {
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 16); cudaMemset(out, 0, 16); cudaMalloc(&cyc, 8);
    const int it = 10000;
    lat_add<<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", (double)h / (16.0 * it));
    lat_mul<<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMUL dependent latency: %.2f cycles\n", (double)h / (16.0 * it));
    shfl_lat<<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("SHFL(f64) dependent latency: %.2f cycles\n", (double)h / (16.0 * it));
    div_lat<<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("f64 divide dependent latency: %.2f cycles\n", (double)h / (4.0 * it));
    for (int w : {1, 2, 4, 8, 16}) {
        thr<8><<<1, 32 * w>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        double ops = 8.0 * it * 32 * w;
        printf("DADD throughput, %2d warps x 8 chains: %.1f ops/cycle/SM\n", w, ops / h);
    }
    for (int w : {4, 8, 16}) {
        thr<16><<<1, 32 * w>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        double ops = 16.0 * it * 32 * w;
        printf("DADD throughput, %2d warps x 16 chains: %.1f ops/cycle/SM\n", w, ops / h);
    }
    return 0;
}
