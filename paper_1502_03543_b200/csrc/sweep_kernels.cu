// sweep_kernels.cu -- the reference's single-step API (rank_one_step /
// parallel_sweep, normal.py:127-160; parallel.py:94-166): build_v,
// sweep_phase1, sweep_phase2 as separate kernels.  The production cascade
// (cascade.cu) fuses these; these exist for API parity and tests.
#include "common.cuh"
#include "pdas_internal.h"

namespace pdas {

__global__ void k_build_v(const double* __restrict__ a, idx_t m, idx_t l0, double dl,
                          double* __restrict__ v) {
    const double f = dl - 1.0;
    for (idx_t i = (idx_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (idx_t)gridDim.x * blockDim.x)
        v[i] = a[l0 * m + i] * f;
}

template <int R>
__global__ void __launch_bounds__(256) k_sweep_phase1(const double* __restrict__ cols, idx_t m,
                                                      const double* __restrict__ v,
                                                      double* __restrict__ inner, idx_t k0,
                                                      idx_t k1) {
    const int lane = threadIdx.x & 31;
    idx_t k = k0 + (idx_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (k >= k1) return;
    double t = warp_tree_dot<R>(v, cols + k * m, m, lane);
    if (lane == 0) inner[k] = t;
}

__global__ void k_sweep_phase2(double* __restrict__ cols, idx_t m, idx_t l0,
                               const double* __restrict__ inner, double denom, idx_t k0,
                               idx_t k1) {
    const double* __restrict__ piv = cols + l0 * m;
    for (idx_t k = k0 + blockIdx.y; k < k1; k += gridDim.y) {
        const double g = inner[k] / denom;
        for (idx_t i = (idx_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
             i += (idx_t)gridDim.x * blockDim.x) {
            double prod = g * piv[i];
            cols[k * m + i] = cols[k * m + i] - prod;
        }
    }
}

int launch_build_v(const double* a, idx_t m, idx_t l0, double dl, double* v, cudaStream_t st) {
    unsigned g = (unsigned)((m + 255) / 256);
    k_build_v<<<g, 256, 0, st>>>(a, m, l0, dl, v);
    return PDAS_OK;
}

int launch_sweep_phase1(const double* cols, idx_t m, const double* v, double* inner, idx_t k0,
                        idx_t k1, cudaStream_t st) {
    if (k1 <= k0) return PDAS_OK;
    int R = warp_R(m);
    if (R > 256) return PDAS_ERR_UNSUPPORTED;
    unsigned g = (unsigned)((k1 - k0 + 7) / 8);
    PDAS_DISPATCH_R(R, 256, k_sweep_phase1<R_><<<g, 256, 0, st>>>(cols, m, v, inner, k0, k1));
    return PDAS_OK;
}

int launch_sweep_phase2(double* cols, idx_t m, idx_t l0, const double* inner, double denom,
                        idx_t k0, idx_t k1, cudaStream_t st) {
    if (k1 <= k0) return PDAS_OK;
    unsigned gx = (unsigned)((m + 255) / 256);
    idx_t gy = k1 - k0;
    if (gy > 4096) gy = 4096;
    k_sweep_phase2<<<dim3(gx, (unsigned)gy), 256, 0, st>>>(cols, m, l0, inner, denom, k0, k1);
    return PDAS_OK;
}

}  // namespace pdas
