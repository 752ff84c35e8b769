// Does programmatic dependent launch (PDL) survive stream operations between
// the two kernels?  K1: 148*3 CTAs of ~spin time, last wave partial; K2 records
// its first CTA's start.  Prints K2 start relative to K1's last CTA end.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long g_t[4];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void k1(int spin_us) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    unsigned long long t0 = gtime();
    while (gtime() - t0 < (unsigned long long)spin_us * 1000) {}
    if (threadIdx.x == 0) atomicMax(&g_t[0], gtime());
}
__global__ void k2() {
    if (threadIdx.x == 0) atomicMin(&g_t[1], gtime());
}
int main() {
    cudaStream_t s, s2;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e, e2;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
    cudaEventRecord(e2, s2);
    const char* names[4] = {"plain", "pdl", "pdl+record", "pdl+record+wait"};
    for (int mode = 0; mode < 4; ++mode) {
        unsigned long long init[4] = {0, ~0ull, 0, 0};
        cudaMemcpyToSymbol(g_t, init, sizeof(init));
        cudaDeviceSynchronize();
        k1<<<148 * 2 + 20, 1024, 0, s>>>(200);
        if (mode >= 2) cudaEventRecord(e, s);
        if (mode >= 3) cudaStreamWaitEvent(s, e2, 0);
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(148);
        lc.blockDim = dim3(128);
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = mode > 0;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaLaunchKernelEx(&lc, k2);
        cudaDeviceSynchronize();
        unsigned long long t[4];
        cudaMemcpyFromSymbol(t, g_t, sizeof(t));
        printf("%-18s K2 first start - K1 last end = %+.1f us  (%s)\n", names[mode],
               ((double)t[1] - (double)t[0]) / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
