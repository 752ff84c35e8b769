// cascade.cu -- the Egidi-Maponi rank-one cascade (the north-star kernel).
//
// Reference: _kernels.pyx:234-291 (_cascade / solve_sweeps), per step l:
//   skip if d[l] == 1.0
//   v      = A[:,l] * (d[l] - 1)                      (build_v, :196-202)
//   inner  = tree(v, col_k)       k = l .. n          (phase 1, :247-253)
//   denom  = 1 + inner[l]; |denom| <= 1e-12 (1 + |inner[l]|) -> return l+1
//   col_k -= (inner[k]/denom) * col_l   k = l+1 .. n  (phase 2, :257-266)
//
// Column k's trajectory depends only on its own values and on the final
// pivot columns P_l = col_l (l < k), their v_l and denom_l.  Any schedule that
// applies pivots to a column in ascending l therefore reproduces the
// reference bit for bit.  B200 schedule:
//
//   * the columns of [Y | x] are cut into tiles of C columns held in
//     REGISTERS by one CTA (thread t owns tree s-indices t + T r, i.e. rows
//     t + T r and t + T r + H of every tile column);
//   * pivots are grouped in blocks of B.  For each block: a panel kernel
//     finalises the block's own columns (intra-block triangle), then an
//     update kernel streams every trailing tile through registers once and
//     applies all B pivots to it (pivot columns + A columns come from L2).
//   HBM traffic per element-step drops from 16 B (one streaming pass per
//   step) to 16/B B; L2 traffic is 16/C B per element-step; the arithmetic
//   (4 non-fused fp64 ops per element-step) becomes the bound.
#include "common.cuh"
#include "pdas_internal.h"
#include "tma.cuh"

namespace pdas {

// ------------------------------------------------------------ reference-API
// single-step kernels (rank_one_step / parallel_sweep, normal.py:127-160)
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

// ------------------------------------------------------------ tile engine
template <int T, int R, int C>
struct Tile {
    static constexpr int NW = T / 32;
    double xl[R][C];  // rows t + T r
    double xh[R][C];  // rows t + T r + H
    idx_t m, H;
    bool m1;  // m == 1: the tree is a bare product (no +0.0, _kernels.pyx:39-40)
    int t;

    __device__ __forceinline__ idx_t row(int r) const { return (idx_t)t + (idx_t)T * r; }
    __device__ __forceinline__ bool vlo(int r) const {
        idx_t hs = H > 0 ? H : 1;
        return row(r) < hs;
    }
    __device__ __forceinline__ bool vhi(int r) const { return !m1 && row(r) + H < m; }

    __device__ __forceinline__ void load(const double* __restrict__ cols, idx_t col0, idx_t ncols) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const idx_t col = col0 + c;
            const bool on = col < ncols;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                xl[r][c] = (on && vlo(r)) ? __ldcg(cols + col * m + row(r)) : 0.0;
                xh[r][c] = (on && vhi(r)) ? __ldcg(cols + col * m + row(r) + H) : 0.0;
            }
        }
    }

    __device__ __forceinline__ void store(double* __restrict__ cols, idx_t col0, idx_t ncols) const {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const idx_t col = col0 + c;
            if (col >= ncols) continue;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (vlo(r)) cols[col * m + row(r)] = xl[r][c];
                if (vhi(r)) cols[col * m + row(r) + H] = xh[r][c];
            }
        }
    }

    // level-0 value of s-index row(r) for column c against v = (vl, vh)
    __device__ __forceinline__ double lvl0(const double (&vl)[R], const double (&vh)[R], int r,
                                           int c) const {
        double lo = vlo(r) ? vl[r] * xl[r][c] : 0.0;
        if (m1) return lo;
        double hi = vhi(r) ? vh[r] * xh[r][c] : 0.0;
        return lo + hi;
    }

    // Per-thread partial (levels >= T) of tree(v, column c).
    __device__ __forceinline__ void partials(const double (&vl)[R], const double (&vh)[R],
                                             double (&part)[C]) const {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double s[R];
#pragma unroll
            for (int r = 0; r < R; ++r) s[r] = lvl0(vl, vh, r, c);
            part[c] = lane_tree<R>(s);
        }
    }

    // Cross-thread levels T/2 .. 1.  DIV: out[c] = inner[c] / denom, else inner[c].
    // Every thread returns all C values.  red: C*T doubles, bc: C doubles.
    template <bool DIV>
    __device__ __forceinline__ void reduce(double (&part)[C], double denom, double (&out)[C],
                                           double* red, double* bc) const {
        const int lane = t & 31;
        if (T == 32) {
            const int w = H >= 32 ? 32 : (H > 0 ? (int)H : 1);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                double v = warp_butterfly(part[c], w);
                if (H < 32) v = __shfl_sync(0xffffffffu, v, 0);
                out[c] = DIV ? v / denom : v;
            }
        } else {
#pragma unroll
            for (int c = 0; c < C; ++c) red[c * T + t] = part[c];
            __syncthreads();
            const int warp = t >> 5;
            for (int c = warp; c < C; c += NW) {
                double q[NW];
#pragma unroll
                for (int k = 0; k < NW; ++k) q[k] = red[c * T + lane + 32 * k];
                double v = warp_butterfly32(lane_tree<NW>(q));
                if (lane == 0) bc[c] = DIV ? v / denom : v;
            }
            __syncthreads();
#pragma unroll
            for (int c = 0; c < C; ++c) out[c] = bc[c];
        }
    }

    __device__ __forceinline__ void axpy(const double (&g)[C], const double (&pl)[R],
                                         const double (&ph)[R]) {
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double p0 = g[c] * pl[r];
                xl[r][c] = xl[r][c] - p0;
                double p1 = g[c] * ph[r];
                xh[r][c] = xh[r][c] - p1;
            }
    }
};

// Shared-memory pipeline of pivot data: stage s holds [P_l | A_l] (2 x mp
// doubles) delivered by two 1-D TMA bulk copies completing on mbar[s].
struct Pipe {
    double* buf;     // S stages of 2*mp doubles
    uint64_t* mbar;  // S barriers
    int S;
    idx_t mp;        // column stride inside a stage (m rounded up to even)
    uint32_t phase;  // bit s: parity expected at the next wait on stage s
};

__device__ __forceinline__ void pipe_issue(Pipe& p, int s, const double* __restrict__ cols,
                                           const double* __restrict__ a, idx_t l, idx_t m) {
    const uint32_t bytes = (uint32_t)(m * sizeof(double));
    double* dst = p.buf + (idx_t)s * 2 * p.mp;
    mbar_arrive_expect_tx(p.mbar + s, 2 * bytes);
    tma_load_1d(dst, cols + l * m, bytes, p.mbar + s);
    tma_load_1d(dst + p.mp, a + l * m, bytes, p.mbar + s);
}

// Apply the pivots [l0, l1) stored in global memory (final columns of cols,
// A, d, denoms) to the register tile, in ascending order.  TMA: pivot data is
// streamed through the shared-memory pipeline S stages ahead; otherwise it is
// read straight from L2.
template <bool TMA, int T, int R, int C>
__device__ __forceinline__ void apply_global_pivots(Tile<T, R, C>& tl,
                                                    const double* __restrict__ cols,
                                                    const double* __restrict__ a,
                                                    const double* __restrict__ d,
                                                    const double* __restrict__ denoms, idx_t l0,
                                                    idx_t l1, double* red, double* bc, Pipe& pp) {
    if (l0 >= l1) return;
    const idx_t m = tl.m;
    if (TMA) {
        __syncthreads();  // earlier readers of every stage are done
        if (tl.t == 0)
            for (int s = 0; s < pp.S && l0 + s < l1; ++s) pipe_issue(pp, s, cols, a, l0 + s, m);
    }
    for (idx_t l = l0; l < l1; ++l) {
        const idx_t k = l - l0;
        const int s = (int)(k % pp.S);
        if (TMA && k > 0) {
            __syncthreads();  // iteration k-1 has consumed its stage
            const idx_t lr = l - 1 + pp.S;
            if (tl.t == 0 && lr < l1) pipe_issue(pp, (int)((k - 1) % pp.S), cols, a, lr, m);
        }
        const double dl = __ldg(d + l);
        const double* pc;
        const double* ac;
        if (TMA) {
            mbar_wait(pp.mbar + s, (pp.phase >> s) & 1u);
            pp.phase ^= 1u << s;
            pc = pp.buf + (idx_t)s * 2 * pp.mp;
            ac = pc + pp.mp;
        } else {
            pc = cols + l * m;
            ac = a + l * m;
        }
        if (dl == 1.0) continue;
        const double f = dl - 1.0;
        const double denom = __ldcg(denoms + l);
        double vl[R], vh[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const idx_t i = tl.row(r);
            double al = 0.0, ah = 0.0;
            if (tl.vlo(r)) al = TMA ? ac[i] : __ldcg(ac + i);
            if (tl.vhi(r)) ah = TMA ? ac[i + tl.H] : __ldcg(ac + i + tl.H);
            vl[r] = al * f;
            vh[r] = ah * f;
        }
        double part[C], g[C];
        tl.partials(vl, vh, part);
        tl.template reduce<true>(part, denom, g, red, bc);
        double pl[R], ph[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const idx_t i = tl.row(r);
            pl[r] = 0.0;
            ph[r] = 0.0;
            if (tl.vlo(r)) pl[r] = TMA ? pc[i] : __ldcg(pc + i);
            if (tl.vhi(r)) ph[r] = TMA ? pc[i + tl.H] : __ldcg(pc + i + tl.H);
        }
        tl.axpy(g, pl, ph);
    }
}

template <int T, int R, int C>
__device__ __forceinline__ void tile_init(Tile<T, R, C>& tl, idx_t m) {
    tl.m = m;
    tl.H = m > 1 ? pow2_ceil(m) >> 1 : 0;
    tl.m1 = m == 1;
    tl.t = threadIdx.x;
}

// dynamic shared memory: red[C*T] | bc[C] | mbar[S] | stages[S][2*mp]
template <int T, int C>
__device__ __forceinline__ void carve(double*& red, double*& bc, Pipe& pp, int S, idx_t m) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    red = reinterpret_cast<double*>(smem_raw);
    bc = red + C * T;
    pp.mbar = reinterpret_cast<uint64_t*>(bc + C);
    size_t off = (size_t)(C * T + C + S) * sizeof(double);
    off = (off + 127) & ~(size_t)127;
    pp.buf = reinterpret_cast<double*>(smem_raw + off);
    pp.S = S > 0 ? S : 1;
    pp.mp = (m + 1) & ~(idx_t)1;
    pp.phase = 0;
    if (S > 0) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < S; ++s) mbar_init(pp.mbar + s, 1);
            mbar_fence_init();
        }
        __syncthreads();
    }
}

template <int T, int C>
static size_t casc_smem_bytes(int S, idx_t m) {
    size_t off = (size_t)(C * T + C + S) * sizeof(double);
    off = (off + 127) & ~(size_t)127;
    idx_t mp = (m + 1) & ~(idx_t)1;
    return off + (size_t)S * 2 * mp * sizeof(double);
}

// Trailing update: tile (tile0 + blockIdx.x) receives pivots [p0, p1).
template <bool TMA, int T, int R, int C>
__global__ void __launch_bounds__(T, 1)
    k_casc_update(double* __restrict__ cols, const double* __restrict__ a,
                  const double* __restrict__ d, const double* __restrict__ denoms, idx_t m,
                  idx_t n, idx_t p0, idx_t p1, idx_t tile0, int S,
                  const int32_t* __restrict__ fail) {
    if (*(volatile const int32_t*)fail) return;
    double *red, *bc;
    Pipe pp;
    carve<T, C>(red, bc, pp, TMA ? S : 0, m);
    Tile<T, R, C> tl;
    tile_init(tl, m);
    const idx_t col0 = (tile0 + blockIdx.x) * C;
    tl.load(cols, col0, n + 1);
    apply_global_pivots<TMA>(tl, cols, a, d, denoms, p0, p1, red, bc, pp);
    tl.store(cols, col0, n + 1);
}

// Panel: one CTA finalises the block's columns [p0, p1) tile by tile
// (pivots of earlier tiles from global memory, then the in-register
// triangle), writing denom_l and detecting breakdown in step order.
template <bool TMA, int T, int R, int C>
__global__ void __launch_bounds__(T, 1)
    k_casc_panel(double* __restrict__ cols, const double* __restrict__ a,
                 const double* __restrict__ d, double* __restrict__ denoms, idx_t m, idx_t n,
                 idx_t p0, idx_t p1, int S, int32_t* __restrict__ fail) {
    if (*(volatile int32_t*)fail) return;
    double *red, *bc;
    Pipe pp;
    carve<T, C>(red, bc, pp, TMA ? S : 0, m);
    Tile<T, R, C> tl;
    tile_init(tl, m);
    const idx_t tiles_end = (p1 + C - 1) / C;
    for (idx_t tile = p0 / C; tile < tiles_end; ++tile) {
        const idx_t col0 = tile * C;
        tl.load(cols, col0, n + 1);
        apply_global_pivots<TMA>(tl, cols, a, d, denoms, p0, col0, red, bc, pp);
        // in-register triangle over this tile's own pivot columns
#pragma unroll
        for (int cl = 0; cl < C; ++cl) {
            const idx_t l = col0 + cl;
            if (l >= p1) break;
            const double dl = __ldg(d + l);
            if (dl == 1.0) continue;
            const double f = dl - 1.0;
            double vl[R], vh[R], pl[R], ph[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                vl[r] = tl.vlo(r) ? __ldg(a + l * m + tl.row(r)) * f : 0.0;
                vh[r] = tl.vhi(r) ? __ldg(a + l * m + tl.row(r) + tl.H) * f : 0.0;
                pl[r] = tl.xl[r][cl];
                ph[r] = tl.xh[r][cl];
            }
            double part[C], inner[C];
            tl.partials(vl, vh, part);
            tl.template reduce<false>(part, 0.0, inner, red, bc);
            const double denom = 1.0 + inner[cl];
            if (fabs(denom) <= kDenomEpsRel * (1.0 + fabs(inner[cl]))) {
                if (threadIdx.x == 0) *fail = (int32_t)(l + 1);
                return;
            }
            if (threadIdx.x == 0) denoms[l] = denom;
            double g[C];
#pragma unroll
            for (int c = 0; c < C; ++c) g[c] = c > cl ? inner[c] / denom : 0.0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (c <= cl) continue;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    double q0 = g[c] * pl[r];
                    tl.xl[r][c] = tl.xl[r][c] - q0;
                    double q1 = g[c] * ph[r];
                    tl.xh[r][c] = tl.xh[r][c] - q1;
                }
            }
        }
        tl.store(cols, col0, n + 1);
        __syncthreads();  // stores visible to the next tile's pivot loads
    }
}

// ------------------------------------------------------------ dispatch
struct CascCfg {
    int T, R, C;
};

static CascCfg cascade_cfg(idx_t m) {
    idx_t H = m > 1 ? pow2_ceil(m) >> 1 : 0;
    if (H <= 32) return {32, 1, 8};
    if (H == 64) return {64, 1, 8};
    if (H == 128) return {128, 1, 8};
    if (H == 256) return {256, 1, 8};
    if (H == 512) return {256, 2, 8};
    if (H == 1024) return {256, 4, 8};
    if (H == 2048) return {256, 8, 4};
    if (H == 4096) return {256, 16, 2};
    if (H == 8192) return {256, 32, 1};
    return {0, 0, 0};
}

idx_t cascade_supported_m() { return 16384; }

template <bool TMA, int T, int R, int C>
static int run_cascade_impl(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                            double* denoms, int32_t* fail, int B, int S, cudaStream_t st) {
    B = (B + C - 1) / C * C;
    const size_t smem = casc_smem_bytes<T, C>(TMA ? S : 0, m);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(k_casc_panel<TMA, T, R, C>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_casc_update<TMA, T, R, C>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    const idx_t ntiles = (n + 1 + C - 1) / C;
    for (idx_t p0 = 0; p0 < n; p0 += B) {
        const idx_t p1 = p0 + B < n ? p0 + B : n;
        k_casc_panel<TMA, T, R, C><<<1, T, smem, st>>>(cols, a, d, denoms, m, n, p0, p1, S, fail);
        const idx_t t0 = (p1 + C - 1) / C;
        if (t0 < ntiles)
            k_casc_update<TMA, T, R, C><<<(unsigned)(ntiles - t0), T, smem, st>>>(
                cols, a, d, denoms, m, n, p0, p1, t0, S, fail);
    }
    return cudaGetLastError() == cudaSuccess ? PDAS_OK : PDAS_ERR_CUDA;
}

template <int T, int R, int C>
static int run_cascade(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                       double* denoms, int32_t* fail, int B, cudaStream_t st) {
    // TMA needs 16-byte aligned columns: m even and 16-byte aligned bases.
    const bool aligned = (m % 2 == 0) && (((uintptr_t)cols | (uintptr_t)a) % 16 == 0);
    const size_t budget = 200 * 1024;
    int S = 4;
    while (S > 1 && casc_smem_bytes<T, C>(S, m) > budget) --S;
    if (aligned && casc_smem_bytes<T, C>(S, m) <= budget && m * sizeof(double) < (1u << 20))
        return run_cascade_impl<true, T, R, C>(cols, a, d, m, n, denoms, fail, B, S, st);
    return run_cascade_impl<false, T, R, C>(cols, a, d, m, n, denoms, fail, B, 1, st);
}

int launch_cascade(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                   double* denoms, int32_t* fail_dev, int block_pivots, cudaStream_t st) {
    if (m < 1 || n < 0) return PDAS_ERR_ARG;
    cudaMemsetAsync(fail_dev, 0, sizeof(int32_t), st);
    if (n == 0) return PDAS_OK;
    CascCfg cfg = cascade_cfg(m);
    const int B = block_pivots > 0 ? block_pivots : 64;
#define PDAS_CASC(T_, R_, C_)                                                        \
    if (cfg.T == T_ && cfg.R == R_ && cfg.C == C_)                                   \
        return run_cascade<T_, R_, C_>(cols, a, d, m, n, denoms, fail_dev, B, st);
    PDAS_CASC(32, 1, 8)
    PDAS_CASC(64, 1, 8)
    PDAS_CASC(128, 1, 8)
    PDAS_CASC(256, 1, 8)
    PDAS_CASC(256, 2, 8)
    PDAS_CASC(256, 4, 8)
    PDAS_CASC(256, 8, 4)
    PDAS_CASC(256, 16, 2)
    PDAS_CASC(256, 32, 1)
#undef PDAS_CASC
    return PDAS_ERR_UNSUPPORTED;
}

}  // namespace pdas
