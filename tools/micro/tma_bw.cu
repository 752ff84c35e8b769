// Microbenchmark: aggregate L2->SMEM bandwidth of 1-D TMA bulk copies when
// every SM streams 32 KB "pivot stages" out of a small L2-resident buffer
// (the cascade's access pattern), for 1 or 2 CTAs per SM and 2..6 stages.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
__global__ void tma_stream(const double* src, long long nbuf, int iters, int bytes, long long* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    unsigned char* buf = sm + 128;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(full + s)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long nchunks = nbuf * 8 / bytes;
    double acc = 0;
    for (int i = 0; i < iters + S; ++i) {
        if (threadIdx.x == 0 && i < iters) {
            int s = i % S;
            if (i >= S) {  // wait until consumed (we consume immediately below)
            }
            long long chunk = (blockIdx.x * 7 + i) % nchunks;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(buf + (size_t)s * bytes)), "l"(src + chunk * (bytes / 8)), "r"(bytes), "r"(sa(full + s)) : "memory");
        }
        int j = i - S + 1;
        if (j >= 0 && j < iters) {
            int s = j % S;
            uint32_t par = (j / S) & 1;
            asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(full + s)), "r"(par) : "memory");
            acc += reinterpret_cast<double*>(buf + (size_t)s * bytes)[threadIdx.x];
            __syncthreads();
        }
    }
    if (acc == 1.2345) sink[0] = 1;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long nbuf = 1 << 19;  // 4 MB of doubles: L2-resident
    double* src; cudaMalloc(&src, nbuf * 8); cudaMemset(src, 0, nbuf * 8);
    long long* sink; cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2000;
    for (int bytes : {16000, 32000}) for (int ctas : {1, 2}) {
        auto k = tma_stream<4>;
        size_t smem = 128 + 4 * (size_t)bytes;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<sms * ctas, 256, smem>>>(src, nbuf, iters, bytes, sink);
        cudaEventRecord(e0);
        k<<<sms * ctas, 256, smem>>>(src, nbuf, iters, bytes, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double tb = (double)sms * ctas * iters * bytes / (ms * 1e-3) / 1e12;
        printf("TMA stream: %5d B stages, %d CTA/SM, 4 stages: %.2f TB/s aggregate (%s)\n", bytes, ctas, tb,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
