// PDL across an event wait on work that is still RUNNING on another stream
// (the cascade's U(b-1) -> [wait panel(b)] -> U(b) pattern): does the
// dependent kernel start before the primary's last wave ends?
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
__global__ void kpanel(int spin_us) {
    unsigned long long t0 = gtime();
    while (gtime() - t0 < (unsigned long long)spin_us * 1000) {}
    if (threadIdx.x == 0) atomicMax(&g_t[2], gtime());
}
__global__ void k2() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) atomicMin(&g_t[1], gtime());
}
int main() {
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t s, ps;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithPriority(&ps, cudaStreamNonBlocking, hi);
    cudaEvent_t eP, eU;
    cudaEventCreateWithFlags(&eP, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&eU, cudaEventDisableTiming);
    const char* names[3] = {"no event wait", "wait panel (done early)", "wait panel (done late)"};
    k1<<<148, 1024, 0, s>>>(1);  // warm up (lazy module loading)
    kpanel<<<1, 32, 0, ps>>>(1);
    k2<<<1, 32, 0, s>>>();
    cudaDeviceSynchronize();
    for (int mode = 0; mode < 3; ++mode) {
        unsigned long long init[4] = {0, ~0ull, 0, 0};
        cudaMemcpyToSymbol(g_t, init, sizeof(init));
        cudaDeviceSynchronize();
        cudaEventRecord(eU, s);  // main stream before K1 (the cascade's eU = up to U(b-1))
        k1<<<148 * 2 + 20, 1024, 0, s>>>(300);  // 2 waves of 2 CTAs/SM, the last one 20 CTAs
        if (mode > 0) {
            cudaStreamWaitEvent(ps, eU, 0);
            kpanel<<<32, 256, 0, ps>>>(mode == 1 ? 50 : 700);
            cudaEventRecord(eP, ps);
            cudaStreamWaitEvent(s, eP, 0);
        }
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(148);
        lc.blockDim = dim3(128);
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaLaunchKernelEx(&lc, k2);
        cudaDeviceSynchronize();
        unsigned long long t[4];
        cudaMemcpyFromSymbol(t, g_t, sizeof(t));
        printf("%-26s K2 first start - K1 last end = %+.1f us; panel end - K1 end = %+.1f us (%s)\n",
               names[mode], ((double)t[1] - (double)t[0]) / 1e3,
               mode ? ((double)t[2] - (double)t[0]) / 1e3 : 0.0, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
