// factor_kernels.cu -- gram / scaled_gram, Cholesky and the triangular
// solves, reproducing the compiled core's sequential orders exactly.
//
//   gram / scaled_gram    _kernels.pyx:108-141   k-outer accumulation per (i,j)
//   cholesky_factor       _kernels.pyx:144-171   left-looking; restated here in
//                                                right-looking form (same per-
//                                                element subtraction sequence)
//   cholesky_solve_many   _kernels.pyx:174-193   forward right-looking (same
//                                                order), backward per-RHS chain
#include <cooperative_groups.h>

#include "common.cuh"
#include "pdas_internal.h"

namespace cg = cooperative_groups;

namespace pdas {

// ---------------------------------------------------------------- gram
// One CTA per upper tile pair (I <= J) of 64x64; 256 threads x 4x4 elements.
// Every element accumulates g = g + a[i,k]*w[j,k] for k = 0..n-1 in order,
// starting from +0.0, with w = a[j,k] (gram) or a[j,k]*d[k] rounded first
// (scaled_gram).  The k loop is staged through shared memory 16 columns at a
// time (each staged column slice is 64 contiguous doubles).
constexpr int GT = 64, GK = 16;

template <bool SCALED>
__global__ void __launch_bounds__(256) k_gram(const double* __restrict__ a, idx_t m, idx_t n,
                                              const double* __restrict__ d,
                                              const int2* __restrict__ tiles,
                                              double* __restrict__ g) {
    __shared__ double sa[2][GK][GT];
    __shared__ double sb[2][GK][GT];
    const int2 tile = tiles[blockIdx.x];
    const idx_t i0 = (idx_t)tile.x * GT, j0 = (idx_t)tile.y * GT;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;

    // loader mapping: 256 threads x 4 = 1024 = GK*GT values per operand
    const int lr = threadIdx.x & 63, lk = threadIdx.x >> 6;  // row in tile, k offset 0..3
    double ra[4], rb[4];
    auto load = [&](idx_t k0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            idx_t k = k0 + lk + 4 * u;
            idx_t ia = i0 + lr, jb = j0 + lr;
            double va = 0.0, vb = 0.0;
            if (k < n) {
                if (ia < m) va = a[k * m + ia];
                if (jb < m) {
                    vb = a[k * m + jb];
                    if (SCALED) vb = vb * d[k];
                }
            }
            ra[u] = va;
            rb[u] = vb;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            sa[buf][lk + 4 * u][lr] = ra[u];
            sb[buf][lk + 4 * u][lr] = rb[u];
        }
    };
    load(0);
    store(0);
    __syncthreads();
    int buf = 0;
    for (idx_t k0 = 0; k0 < n; k0 += GK) {
        const bool more = k0 + GK < n;
        if (more) load(k0 + GK);
        const idx_t kend = (n - k0) < GK ? (n - k0) : GK;
        for (int kk = 0; kk < kend; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) av[p] = sa[buf][kk][tx + 16 * p];
#pragma unroll
            for (int q = 0; q < 4; ++q) bv[q] = sb[buf][kk][ty + 16 * q];
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    double prod = av[p] * bv[q];
                    acc[p][q] = acc[p][q] + prod;
                }
        }
        if (more) {
            store(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            idx_t i = i0 + tx + 16 * p, j = j0 + ty + 16 * q;
            if (i < m && j < m && i <= j) {
                g[j * m + i] = acc[p][q];
                g[i * m + j] = acc[p][q];  // mirror (_kernels.pyx:120-122)
            }
        }
}

int launch_gram(const double* a, idx_t m, idx_t n, const double* d, double* g, cudaStream_t st) {
    if (m < 1 || n < 0) return PDAS_ERR_ARG;
    if (n == 0) {
        cudaMemsetAsync(g, 0, (size_t)(m * m) * sizeof(double), st);
        return PDAS_OK;
    }
    const int nt = (int)((m + GT - 1) / GT);
    const int ntiles = nt * (nt + 1) / 2;
    int2* tiles = nullptr;
    if (cudaMallocAsync(&tiles, sizeof(int2) * ntiles, st) != cudaSuccess) return PDAS_ERR_NOMEM;
    int2* h = new int2[ntiles];
    int c = 0;
    for (int J = 0; J < nt; ++J)
        for (int I = 0; I <= J; ++I) h[c++] = make_int2(I, J);
    cudaMemcpyAsync(tiles, h, sizeof(int2) * ntiles, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);  // h must outlive the copy
    delete[] h;
    if (d)
        k_gram<true><<<ntiles, 256, 0, st>>>(a, m, n, d, tiles, g);
    else
        k_gram<false><<<ntiles, 256, 0, st>>>(a, m, n, d, tiles, g);
    cudaFreeAsync(tiles, st);
    return PDAS_OK;
}

// ---------------------------------------------------------------- Cholesky
// Right-looking restatement of the left-looking column Cholesky: element
// (i,c) of the work matrix S receives  S -= L[i,j]*L[c,j]  for j = 0,1,..
// in ascending order -- the same rounding sequence as the reference's
// `s -= low[i,k]*low[j,k]` loop.  One grid-wide barrier per column: while
// updating step j the warp that owns column j+1 finishes it (pivot, fail
// test, scaling) so step j+1 can start right after the barrier.
__device__ __forceinline__ void chol_finish_column(double* __restrict__ S, double* __restrict__ L,
                                                   idx_t nn, idx_t c, double eps, int lane,
                                                   volatile int64_t* fail) {
    double s = S[c * nn + c];
    if (!isfinite(s) || s <= eps) {
        if (lane == 0) *fail = c;
        return;
    }
    double piv = sqrt(s);
    if (lane == 0) L[c * nn + c] = piv;
    for (idx_t i = c + 1 + lane; i < nn; i += 32) L[c * nn + i] = S[c * nn + i] / piv;
}

__global__ void __launch_bounds__(256) k_cholesky(double* __restrict__ S, double* __restrict__ L,
                                                  idx_t nn, double eps_rel, int64_t* fail_out,
                                                  int64_t* fail_work, double* dmax_work) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const idx_t gw = ((idx_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const idx_t nwarps = ((idx_t)gridDim.x * blockDim.x) >> 5;
    volatile int64_t* fail = fail_work;
    // dmax: max(0, diag) ignoring NaN (`if g[j,j] > dmax`), order-free
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        double dm = 0.0;
        for (idx_t j = lane; j < nn; j += 32) {
            double gj = S[j * nn + j];
            if (gj > dm) dm = gj;
        }
        for (int k = 16; k >= 1; k >>= 1) {
            double o = __shfl_xor_sync(0xffffffffu, dm, k);
            if (o > dm) dm = o;
        }
        if (lane == 0) {
            *dmax_work = dm;
            *fail = -1;
        }
    }
    grid.sync();
    const double eps = eps_rel * *dmax_work;
    if (gw == 0) chol_finish_column(S, L, nn, 0, eps, lane, fail);
    grid.sync();
    for (idx_t j = 0; j < nn; ++j) {
        if (*fail >= 0) break;
        // trailing update with column j: columns c in (j, nn), rows i >= c
        for (idx_t c = j + 1 + gw; c < nn; c += nwarps) {
            const double lcj = L[j * nn + c];
            for (idx_t i = c + lane; i < nn; i += 32) {
                double prod = L[j * nn + i] * lcj;
                S[c * nn + i] = S[c * nn + i] - prod;
            }
            if (c == j + 1) {
                __syncwarp();
                chol_finish_column(S, L, nn, c, eps, lane, fail);
            }
        }
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *fail_out = *fail;
}

__global__ void k_zero_upper_copy(const double* __restrict__ g, double* __restrict__ S,
                                  double* __restrict__ L, idx_t total) {
    for (idx_t t = (idx_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (idx_t)gridDim.x * blockDim.x) {
        S[t] = g[t];
        L[t] = 0.0;
    }
}

idx_t cholesky_work_doubles(idx_t nn) { return nn * nn + 2; }

int launch_cholesky(const double* g, idx_t nn, double eps_rel, double* low, int64_t* fail_dev,
                    double* work, cudaStream_t st) {
    if (nn < 1) return PDAS_ERR_ARG;
    double* S = work;
    double* dmax = work + nn * nn;
    int64_t* failw = (int64_t*)(work + nn * nn + 1);
    idx_t total = nn * nn;
    unsigned g1 = (unsigned)((total + 255) / 256);
    if (g1 > 4096) g1 = 4096;
    k_zero_upper_copy<<<g1, 256, 0, st>>>(g, S, low, total);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cholesky, 256, 0);
    if (per < 1) return PDAS_ERR_CUDA;
    int blocks = sms * (per < 2 ? per : 2);
    idx_t need = (nn + 7) / 8;  // one warp per column is plenty
    if (need < blocks) blocks = (int)(need < 1 ? 1 : need);
    void* args[] = {(void*)&S, (void*)&low, (void*)&nn, (void*)&eps_rel, (void*)&fail_dev,
                    (void*)&failw, (void*)&dmax};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_cholesky, dim3(blocks), dim3(256), args,
                                                0, st);
    return e == cudaSuccess ? PDAS_OK : PDAS_ERR_CUDA;
}

// ---------------------------------------------------------------- solves
// Forward substitution, warp per right-hand side, x staged in shared memory.
// Right-looking: after x[j] /= L[j,j] every later row subtracts L[i,j]*x[j],
// so row i sees its subtractions in ascending j exactly as the reference's
// `s -= low[i,j]*x[j]` loop; the result goes to xt (row-major m x k).
__global__ void __launch_bounds__(128) k_forward(const double* __restrict__ L, idx_t m,
                                                 const double* __restrict__ x, idx_t k,
                                                 double* __restrict__ xt) {
    extern __shared__ double smx[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const idx_t c = (idx_t)blockIdx.x * (blockDim.x >> 5) + warp;
    double* xs = smx + (idx_t)warp * m;
    if (c >= k) return;
    for (idx_t i = lane; i < m; i += 32) xs[i] = x[c * m + i];
    __syncwarp();
    for (idx_t j = 0; j < m; ++j) {
        const double xj = xs[j] / L[j * m + j];
        __syncwarp();
        if (lane == 0) xs[j] = xj;
        for (idx_t i = j + 1 + lane; i < m; i += 32) {
            double prod = L[j * m + i] * xj;
            xs[i] = xs[i] - prod;
        }
        __syncwarp();
    }
    for (idx_t i = lane; i < m; i += 32) xt[i * k + c] = xs[i];
}

// Backward substitution, thread per right-hand side (xt row-major: the 32
// threads of a warp read one 256-byte row segment per step).  Each x[i] is a
// sequential chain  s = x[i]; s -= L[j,i]*x[j] (j = i+1 .. m-1); x[i] = s/L[i,i]
// -- inherently serial, exactly the reference order.
__global__ void __launch_bounds__(128) k_backward(const double* __restrict__ L, idx_t m,
                                                  double* __restrict__ xt, idx_t k) {
    const idx_t c = (idx_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k) return;
    for (idx_t i = m - 1; i >= 0; --i) {
        const double* __restrict__ lc = L + i * m;  // column i of L: L[j,i] at i*m + j
        double s = xt[i * k + c];
        idx_t j = i + 1;
        // 16 independent loads in flight per batch; the subtraction chain
        // itself stays strictly in ascending j.
        for (; j + 16 <= m; j += 16) {
            double p[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) p[u] = lc[j + u] * xt[(j + u) * k + c];
#pragma unroll
            for (int u = 0; u < 16; ++u) s = s - p[u];
        }
        for (; j < m; ++j) {
            double p = lc[j] * xt[j * k + c];
            s = s - p;
        }
        xt[i * k + c] = s / lc[i];
    }
}

// Backward substitution with each right-hand side resident in shared memory
// (no m-fold re-read of x from global memory): warp 0, lane c, runs the serial
// chain of right-hand side c0 + c -- for i = m-1 .. 0:
//   s = x[i]; s -= L[j,i]*x[j] (j = i+1 .. m-1, ascending); x[i] = s / L[i,i]
// (_kernels.pyx:186-192, the reference's exact order) -- reading x[j] from
// shared memory (layout [row][NR], lane-contiguous) and L's column i from a
// shared double buffer that warp 1 fills with column i-1 meanwhile.  The
// result goes straight to column-major x (no transpose pass).
__global__ void __launch_bounds__(64) k_backward_s(const double* __restrict__ L, idx_t m,
                                                   const double* __restrict__ xt, idx_t k,
                                                   double* __restrict__ x, int NR) {
    extern __shared__ double smx[];
    double* xs = smx;            // [m][NR]
    double* lb = smx + m * NR;   // [2][m]: columns i (parity i & 1)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const idx_t c0 = (idx_t)blockIdx.x * NR;
    const int nr = (int)(k - c0 < NR ? k - c0 : NR);
    for (idx_t e = threadIdx.x; e < m * nr; e += blockDim.x) {
        const idx_t i = e / nr, c = e % nr;
        xs[i * NR + c] = xt[i * k + c0 + c];
    }
    for (idx_t j = threadIdx.x; j < m; j += blockDim.x)
        lb[((m - 1) & 1) * m + j] = __ldg(L + (m - 1) * m + j);
    __syncthreads();
    for (idx_t i = m - 1; i >= 0; --i) {
        const double* lc = lb + (i & 1) * m;
        if (warp == 1) {
            if (i > 0) {
                double* nb = lb + ((i - 1) & 1) * m;
                for (idx_t j = i - 1 + lane; j < m; j += 32) nb[j] = __ldg(L + (i - 1) * m + j);
            }
        } else if (lane < nr) {
            double s = xs[i * NR + lane];
            idx_t j = i + 1;
            for (; j + 16 <= m; j += 16) {
                double p[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) p[u] = lc[j + u] * xs[(j + u) * NR + lane];
#pragma unroll
                for (int u = 0; u < 16; ++u) s = s - p[u];
            }
            for (; j < m; ++j) {
                const double p = lc[j] * xs[j * NR + lane];
                s = s - p;
            }
            xs[i * NR + lane] = s / lc[i];
        }
        __syncthreads();  // row i final, column i-1 staged
    }
    for (int c = 0; c < nr; ++c)
        for (idx_t i = threadIdx.x; i < m; i += blockDim.x) x[(c0 + c) * m + i] = xs[i * NR + c];
}

// xt (m x k row-major) -> x (m x k column-major), 32x32 tiles.
__global__ void k_transpose_back(const double* __restrict__ xt, idx_t m, idx_t k,
                                 double* __restrict__ x) {
    __shared__ double t[32][33];
    idx_t i0 = (idx_t)blockIdx.y * 32, c0 = (idx_t)blockIdx.x * 32;
    int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        idx_t i = i0 + r, c = c0 + tx;
        if (i < m && c < k) t[r][tx] = xt[i * k + c];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        idx_t c = c0 + r, i = i0 + tx;
        if (i < m && c < k) x[c * m + i] = t[tx][r];
    }
}

idx_t solve_many_work_doubles(idx_t m, idx_t k) { return m * k; }

int launch_solve_many(const double* low, idx_t m, double* x, idx_t k, double* work,
                      cudaStream_t st) {
    if (m < 1 || k < 0) return PDAS_ERR_ARG;
    if (k == 0) return PDAS_OK;
    if (k == 1 && 3 * m * (idx_t)sizeof(double) <= 200 * 1024)
        return launch_solve_one(low, m, x, work, st);
    // forward: one warp per right-hand side with its x in shared memory, as many
    // warps per CTA as fit (1 at m up to 25600)
    constexpr size_t kSmem = 200 * 1024;
    const size_t per = (size_t)m * sizeof(double);
    if (per > kSmem) return PDAS_ERR_UNSUPPORTED;
    const int wpc = (int)(kSmem / per < 4 ? kSmem / per : 4);
    const size_t smem = (size_t)wpc * per;
    cudaFuncSetAttribute(k_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_forward<<<(unsigned)((k + wpc - 1) / wpc), 32 * wpc, smem, st>>>(low, m, x, k, work);
    // backward: NR right-hand sides per CTA resident in shared memory next to
    // a double-buffered column of L; falls back to the streaming kernel when
    // not even one fits
    const idx_t nr = (idx_t)(kSmem / per) - 2;
    if (nr >= 1) {
        const int NR = (int)(nr < 32 ? nr : 32);
        const size_t sb = ((size_t)m * NR + 2 * (size_t)m) * sizeof(double);
        cudaFuncSetAttribute(k_backward_s, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
        k_backward_s<<<(unsigned)((k + NR - 1) / NR), 64, sb, st>>>(low, m, work, k, x, NR);
        return PDAS_OK;
    }
    k_backward<<<(unsigned)((k + 127) / 128), 128, 0, st>>>(low, m, work, k);
    dim3 grid((unsigned)((k + 31) / 32), (unsigned)((m + 31) / 32));
    k_transpose_back<<<grid, dim3(32, 8), 0, st>>>(work, m, k, x);
    return PDAS_OK;
}

}  // namespace pdas
