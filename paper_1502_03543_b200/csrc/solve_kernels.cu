// solve_kernels.cu -- (L L^T) x = b for ONE right-hand side, scheduled for
// latency.  This is init_workspace's x0 = (A A^T)^{-1} (A x) (normal.py:123,
// via linalg.cholesky_solve -> _kernels.pyx:174-193 with k = 1), on the
// critical path of every PDAS iteration.
//
// Forward  x[i] = (x[i] - sum_{j<i} L[i,j] x[j]) / L[i,i], j ascending: a
//   right-looking sweep gives every row its subtractions in the same order;
//   one CTA of 1024 threads, rows in registers, L columns prefetched two
//   steps ahead, one barrier per step.
// Backward x[i] = (x[i] - sum_{j>i} L[j,i] x[j]) / L[i,i], j ascending: an
//   inherently serial chain (x[i]'s first term needs x[i+1]).  One thread
//   runs the chain out of shared memory while 31 helper warps compute the
//   NEXT row's products L[j,i-1] x[j] (j > i) -- exactly the rounded
//   products of the reference -- so the chain costs one dependent
//   subtraction per term.
#include "common.cuh"
#include "pdas_internal.h"

namespace pdas {

template <int Q>
__global__ void __launch_bounds__(1024) k_fwd_one(const double* __restrict__ L, int m,
                                                  double* __restrict__ x) {
    __shared__ double xb[2];
    const int t = threadIdx.x;
    double xr[Q], l0[Q], l1[Q], l2[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int i = t + 1024 * q;
        xr[q] = i < m ? x[i] : 0.0;
        l0[q] = i < m ? __ldg(L + i) : 0.0;
        l1[q] = (i < m && m > 1) ? __ldg(L + (size_t)m + i) : 0.0;
    }
    for (int j = 0; j < m; ++j) {
        const int owner = j & 1023, slot = j >> 10;
        if (t == owner) {
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (q == slot) {
                    xr[q] = xr[q] / l0[q];
                    xb[j & 1] = xr[q];
                }
        }
        const int j2 = j + 2;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int i = t + 1024 * q;
            l2[q] = (j2 < m && i < m) ? __ldg(L + (size_t)j2 * m + i) : 0.0;
        }
        __syncthreads();
        const double xj = xb[j & 1];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int i = t + 1024 * q;
            if (i > j && i < m) {
                double p = l0[q] * xj;
                xr[q] = xr[q] - p;
            }
            l0[q] = l1[q];
            l1[q] = l2[q];
        }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int i = t + 1024 * q;
        if (i < m) x[i] = xr[q];
    }
}

// dynamic smem: xs[m] | qa[m] | qb[m]
__global__ void __launch_bounds__(1024) k_bwd_one(const double* __restrict__ L, int m,
                                                  double* __restrict__ x) {
    extern __shared__ double sm[];
    double* xs = sm;
    double* qa = sm + m;
    double* qb = sm + 2 * m;
    const int t = threadIdx.x;
    const bool chain = t == 0;
    const int helper = t - 32;  // >= 0 for warps 1..31
    double xnext = 0.0;         // x_{r+1} (chain thread)
    double y_r = 0.0, l_off = 0.0, l_diag = 0.0;
    if (chain) {
        y_r = x[m - 1];
        l_diag = L[(size_t)(m - 1) * m + (m - 1)];
    }
    for (int r = m - 1; r >= 0; --r) {
        double* qcur = ((m - 1 - r) & 1) ? qb : qa;  // products for row r
        double* qnext = ((m - 1 - r) & 1) ? qa : qb;  // products for row r-1
        if (chain) {
            double s = y_r;
            if (r + 1 < m) {
                double p = l_off * xnext;
                s = s - p;
            }
            // prefetch next round's scalars while the chain runs
            double y_n = 0.0, lo_n = 0.0, ld_n = 0.0;
            if (r >= 1) {
                y_n = x[r - 1];
                lo_n = L[(size_t)(r - 1) * m + r];
                ld_n = L[(size_t)(r - 1) * m + (r - 1)];
            }
            int j = r + 2;
            for (; j + 8 <= m; j += 8) {
                double q[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) q[u] = qcur[j + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) s = s - q[u];
            }
            for (; j < m; ++j) s = s - qcur[j];
            xnext = s / l_diag;
            xs[r] = xnext;
            y_r = y_n;
            l_off = lo_n;
            l_diag = ld_n;
        } else if (helper >= 0 && r >= 1) {
            const double* lc = L + (size_t)(r - 1) * m;
            for (int j = r + 1 + helper; j < m; j += 992) {
                double p = __ldg(lc + j) * xs[j];
                qnext[j] = p;
            }
        }
        __syncthreads();
    }
    for (int i = t; i < m; i += 1024) x[i] = xs[i];
}

idx_t solve_one_work_doubles(idx_t) { return 0; }

int launch_solve_one(const double* low, idx_t m, double* x, double* work, cudaStream_t st) {
    (void)work;
    if (m < 1) return PDAS_ERR_ARG;
    const int Q = (int)((m + 1023) / 1024);
    const int mi = (int)m;
    switch (Q <= 1 ? 1 : Q <= 2 ? 2 : Q <= 4 ? 4 : Q <= 8 ? 8 : Q <= 16 ? 16 : 0) {
        case 1: k_fwd_one<1><<<1, 1024, 0, st>>>(low, mi, x); break;
        case 2: k_fwd_one<2><<<1, 1024, 0, st>>>(low, mi, x); break;
        case 4: k_fwd_one<4><<<1, 1024, 0, st>>>(low, mi, x); break;
        case 8: k_fwd_one<8><<<1, 1024, 0, st>>>(low, mi, x); break;
        case 16: k_fwd_one<16><<<1, 1024, 0, st>>>(low, mi, x); break;
        default: return PDAS_ERR_UNSUPPORTED;
    }
    const size_t smem = (size_t)3 * m * sizeof(double);
    if (smem > 200 * 1024) return PDAS_ERR_UNSUPPORTED;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_bwd_one, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bwd_one<<<1, 1024, smem, st>>>(low, mi, x);
    return PDAS_OK;
}

}  // namespace pdas
