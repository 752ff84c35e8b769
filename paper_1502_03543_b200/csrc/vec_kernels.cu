// vec_kernels.cu -- tree-ordered dots / GEMVs and the fused per-iteration
// vector kernels of the PDAS driver, all bitwise-faithful to the reference.
//
//   dot_tree   _kernels.pyx:55-71        one CTA, thread-strided tree
//   mat_t_vec  _kernels.pyx:91-105       warp per column (contiguous)
//   mat_vec    _kernels.pyx:74-88        row trees: k-split partials + finish
//   iteration  solver.py:142-194, 257-260 (scaling, directions, residuals,
//              ratio test, x/y/s update, gap and objectives)
#include "common.cuh"
#include "pdas_internal.h"

namespace pdas {

// ---------------------------------------------------------------- dot_tree
// One CTA of 1024 threads; thread t owns s-indices t + 1024 r.
template <int R>
__global__ void __launch_bounds__(1024) k_dot_tree(const double* __restrict__ u, idx_t su,
                                                   const double* __restrict__ v, idx_t sv,
                                                   idx_t L, double* out) {
    __shared__ double sm[1024];
    if (L == 1) {
        if (threadIdx.x == 0) *out = u[0] * v[0];
        return;
    }
    const idx_t H = pow2_ceil(L) >> 1;
    const int t = threadIdx.x;
    int nv;
    if (H >= 1024) {
        sm[t] = stream_tree<R>([&](int r) {
            idx_t i = t + 1024 * (idx_t)r, j = i + H;
            double hi = 0.0;
            if (j < L) hi = u[j * su] * v[j * sv];
            double lo = u[i * su] * v[i * sv];
            return lo + hi;
        });
        nv = 1024;
    } else {
        if (t < H) {
            idx_t j = t + H;
            double hi = 0.0;
            if (j < L) hi = u[j * su] * v[j * sv];
            double lo = u[t * su] * v[t * sv];
            sm[t] = lo + hi;
        }
        nv = (int)H;
    }
    double r = block_tree_finish(sm, nv);
    if (t == 0) *out = r;
}

int launch_dot_tree(const double* u, idx_t su, const double* v, idx_t sv, idx_t L, double* out,
                    cudaStream_t st) {
    if (L < 1) return PDAS_ERR_ARG;
    idx_t H = pow2_ceil(L) >> 1;
    int R = H >= 1024 ? (int)(H / 1024) : 1;
    if (R > 256) return PDAS_ERR_UNSUPPORTED;
    PDAS_DISPATCH_R(R, 256, k_dot_tree<R_><<<1, 1024, 0, st>>>(u, su, v, sv, L, out));
    return PDAS_OK;
}

// Three tree dots in one launch (gap, primal and dual objective):
// blockIdx.x selects the pair.  Lengths can differ (n, n, m).
struct DotJob {
    const double* u;
    const double* v;
    idx_t L;
    double* out;
};
struct DotJobs {
    DotJob j[3];
};

template <int R>
__device__ void dot_block(const DotJob& jb, double* sm) {
    const idx_t L = jb.L;
    const double* __restrict__ u = jb.u;
    const double* __restrict__ v = jb.v;
    const int t = threadIdx.x;
    if (L == 1) {
        if (t == 0) *jb.out = u[0] * v[0];
        return;
    }
    const idx_t H = pow2_ceil(L) >> 1;
    int nv;
    if (H >= 1024) {
        sm[t] = stream_tree<R>([&](int r) {
            idx_t i = t + 1024 * (idx_t)r, j = i + H;
            double hi = 0.0;
            if (j < L) hi = u[j] * v[j];
            double lo = u[i] * v[i];
            return lo + hi;
        });
        nv = 1024;
    } else {
        if (t < H) {
            idx_t j = t + H;
            double hi = 0.0;
            if (j < L) hi = u[j] * v[j];
            double lo = u[t] * v[t];
            sm[t] = lo + hi;
        }
        nv = (int)H;
    }
    double r = block_tree_finish(sm, nv);
    if (t == 0) *jb.out = r;
}

__global__ void __launch_bounds__(1024) k_dot3(DotJobs jobs) {
    __shared__ double sm[1024];
    const DotJob& jb = jobs.j[blockIdx.x];
    if (jb.L < 1) return;
    idx_t H = pow2_ceil(jb.L) >> 1;
    int R = H >= 1024 ? (int)(H / 1024) : 1;
    PDAS_DISPATCH_R(R, 256, dot_block<R_>(jb, sm));
}

// ---------------------------------------------------------------- mat_t_vec
template <int R>
__global__ void __launch_bounds__(256) k_mat_t_vec(const double* __restrict__ a, idx_t m, idx_t n,
                                                   const double* __restrict__ y,
                                                   double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    idx_t col = (idx_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (col >= n) return;
    double t = warp_tree_dot<R>(a + col * m, y, m, lane);
    if (lane == 0) out[col] = t;
}

int launch_mat_t_vec(const double* a, idx_t m, idx_t n, const double* y, double* out,
                     cudaStream_t st) {
    if (m < 1 || n < 0) return PDAS_ERR_ARG;
    if (n == 0) return PDAS_OK;
    int R = warp_R(m);
    if (R > 256) return PDAS_ERR_UNSUPPORTED;
    unsigned grid = (unsigned)((n + 7) / 8);
    PDAS_DISPATCH_R(R, 256, k_mat_t_vec<R_><<<grid, 256, 0, st>>>(a, m, n, y, out));
    return PDAS_OK;
}

// ---------------------------------------------------------------- mat_vec
// Row i's tree runs over k = 0..n-1 with stride m in memory.  KT "k-threads"
// each own s-indices w + KT r; lanes of a warp own 32 consecutive rows so
// every load is a 256-byte coalesced segment.  part[i*KT + w] then holds the
// level-KT value; k_mat_vec_finish performs levels KT/2 .. 1.
template <int RK>
__global__ void __launch_bounds__(256) k_mat_vec_part(const double* __restrict__ a, idx_t m,
                                                      idx_t n, const double* __restrict__ x,
                                                      idx_t H, int KT, double* __restrict__ part,
                                                      double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const idx_t i = (idx_t)blockIdx.x * 32 + lane;
    const int w = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (i >= m || w >= KT) return;
    if (n == 1) {
        out[i] = a[i] * x[0];
        return;
    }
    double s = stream_tree<RK>([&](int r) {
        idx_t k = w + (idx_t)KT * r, k2 = k + H;
        double hi = 0.0;
        if (k2 < n) hi = a[k2 * m + i] * x[k2];
        double lo = a[k * m + i] * x[k];
        return lo + hi;
    });
    if (KT == 1)
        out[i] = s;
    else
        part[i * KT + w] = s;
}

template <int Q>
__global__ void __launch_bounds__(256) k_mat_vec_finish(const double* __restrict__ part, idx_t m,
                                                        int KT, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    idx_t i = (idx_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= m) return;
    const double* p = part + i * KT;
    double t;
    if (KT >= 32) {
        double s[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) s[q] = p[lane + 32 * q];
        t = warp_butterfly32(lane_tree<Q>(s));
    } else {
        t = lane < KT ? p[lane] : 0.0;
        t = warp_butterfly(t, KT);
    }
    if (lane == 0) out[i] = t;
}

idx_t mat_vec_scratch(idx_t m, idx_t n) {
    idx_t H = pow2_ceil(n) >> 1;
    idx_t KT = H / 16;
    if (KT < 1) KT = 1;
    if (KT > 4096) KT = 4096;
    return KT > 1 ? m * KT : 0;
}

int launch_mat_vec(const double* a, idx_t m, idx_t n, const double* x, double* out,
                   double* scratch, cudaStream_t st) {
    if (m < 0 || n < 1) return PDAS_ERR_ARG;
    if (m == 0) return PDAS_OK;
    idx_t H = pow2_ceil(n) >> 1;
    idx_t KT = H / 16;
    if (KT < 1) KT = 1;
    if (KT > 4096) KT = 4096;
    idx_t RK = n == 1 ? 1 : H / KT;
    if (RK > 256) return PDAS_ERR_UNSUPPORTED;
    if (KT > 1 && scratch == nullptr) return PDAS_ERR_ARG;
    dim3 grid((unsigned)((m + 31) / 32), (unsigned)((KT + 7) / 8));
    PDAS_DISPATCH_R((int)RK, 256,
                    k_mat_vec_part<R_><<<grid, 256, 0, st>>>(a, m, n, x, H, (int)KT, scratch, out));
    if (KT > 1) {
        int Q = KT >= 32 ? (int)(KT / 32) : 1;
        unsigned g2 = (unsigned)((m + 7) / 8);
        PDAS_DISPATCH_R(Q, 128, if (R_ <= 128) k_mat_vec_finish<R_><<<g2, 256, 0, st>>>(scratch, m, (int)KT, out));
    }
    return PDAS_OK;
}

// ---------------------------------------------------------------- iteration
// d = x/s and the interior test of model.py:116-119 (np.min semantics: a NaN
// anywhere makes the min NaN, and NaN <= 0 is false).
__global__ void k_scaling(const double* __restrict__ x, const double* __restrict__ s, idx_t n,
                          double* __restrict__ d, unsigned* __restrict__ flags) {
    unsigned f = 0;
    for (idx_t j = (idx_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (idx_t)gridDim.x * blockDim.x) {
        double xj = x[j], sj = s[j];
        d[j] = xj / sj;
        if (xj != xj) f |= IT_X_NAN;
        if (xj <= 0.0) f |= IT_X_LE0;
        if (sj != sj) f |= IT_S_NAN;
        if (sj <= 0.0) f |= IT_S_LE0;
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

// Per-block partial of the direction epilogue.
struct DirPartial {
    double max_rdual, max_rcomp, min_ratio;
    long long argmin;
    unsigned nonfinite;
    unsigned pad;
};

__device__ __forceinline__ double nanmax(double a, double b) {
    // np.max semantics: NaN propagates.
    if (a != a) return a;
    if (b != b) return b;
    return a > b ? a : b;
}

// t = A^T dy (warp per column), then solver.py:166-171 elementwise:
//   ds = -t ; dx = d*t - x ; |ds + t| ; |s*dx + x*ds + x*s| ;
// and the ratio test candidates of solver.py:181-186.
template <int R>
__global__ void __launch_bounds__(256) k_directions(const double* __restrict__ a, idx_t m, idx_t n,
                                                    const double* __restrict__ dy,
                                                    const double* __restrict__ d,
                                                    const double* __restrict__ x,
                                                    const double* __restrict__ s,
                                                    double* __restrict__ dx, double* __restrict__ ds,
                                                    DirPartial* __restrict__ partials) {
    __shared__ DirPartial sp[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    idx_t col = (idx_t)blockIdx.x * 8 + warp;
    DirPartial p;
    p.max_rdual = 0.0;
    p.max_rcomp = 0.0;
    p.min_ratio = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    p.argmin = -1;
    p.nonfinite = 0;
    p.pad = 0;
    if (col < n) {
        double t = warp_tree_dot<R>(a + col * m, dy, m, lane);
        if (lane == 0) {
            double xj = x[col], sj = s[col];
            double dsj = -t;
            double dxj = d[col] * t - xj;
            dx[col] = dxj;
            ds[col] = dsj;
            p.max_rdual = fabs(dsj + t);
            double c1 = sj * dxj, c2 = xj * dsj, c3 = xj * sj;
            p.max_rcomp = fabs(c1 + c2 + c3);
            if (!isfinite(dxj) || !isfinite(dsj)) p.nonfinite = 1;
            if (dxj < 0.0) {
                double r = -xj / dxj;
                p.min_ratio = r;
                p.argmin = col;
            }
            if (dsj < 0.0) {
                double r = -sj / dsj;
                if (p.argmin < 0 || r < p.min_ratio) {
                    p.min_ratio = r;
                    p.argmin = n + col;
                }
            }
        }
    }
    if (lane == 0) sp[warp] = p;
    __syncthreads();
    if (threadIdx.x == 0) {
        DirPartial q = sp[0];
        for (int w = 1; w < 8; ++w) {
            const DirPartial& o = sp[w];
            q.max_rdual = nanmax(q.max_rdual, o.max_rdual);
            q.max_rcomp = nanmax(q.max_rcomp, o.max_rcomp);
            q.nonfinite |= o.nonfinite;
            if (o.argmin >= 0 &&
                (q.argmin < 0 || o.min_ratio < q.min_ratio ||
                 (o.min_ratio == q.min_ratio && o.argmin < q.argmin))) {
                q.min_ratio = o.min_ratio;
                q.argmin = o.argmin;
            }
        }
        partials[blockIdx.x] = q;
    }
}

// Single CTA: fold partials, r_primal = max|A dx|, finiteness of dy, alpha.
// solver.py:169 (r_primal), :229-235 (finite), :175-189 (alpha), :237 (cap).
__global__ void __launch_bounds__(1024) k_dir_finish(const DirPartial* __restrict__ partials, int np_,
                                                     const double* __restrict__ adx, idx_t m,
                                                     const double* __restrict__ dy, double rho,
                                                     IterState* st) {
    __shared__ DirPartial sp[32];
    __shared__ double sr[32];
    __shared__ unsigned snf[32];
    DirPartial q;
    q.max_rdual = 0.0;
    q.max_rcomp = 0.0;
    q.min_ratio = __longlong_as_double(0x7ff0000000000000LL);
    q.argmin = -1;
    q.nonfinite = 0;
    q.pad = 0;
    for (int b = threadIdx.x; b < np_; b += blockDim.x) {
        const DirPartial& o = partials[b];
        q.max_rdual = nanmax(q.max_rdual, o.max_rdual);
        q.max_rcomp = nanmax(q.max_rcomp, o.max_rcomp);
        q.nonfinite |= o.nonfinite;
        if (o.argmin >= 0 && (q.argmin < 0 || o.min_ratio < q.min_ratio ||
                              (o.min_ratio == q.min_ratio && o.argmin < q.argmin))) {
            q.min_ratio = o.min_ratio;
            q.argmin = o.argmin;
        }
    }
    double rp = 0.0;
    unsigned nf = 0;
    for (idx_t i = threadIdx.x; i < m; i += blockDim.x) {
        rp = nanmax(rp, fabs(adx[i]));
        if (!isfinite(dy[i])) nf = 1;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = 16; k >= 1; k >>= 1) {
        DirPartial o;
        o.max_rdual = __shfl_xor_sync(0xffffffffu, q.max_rdual, k);
        o.max_rcomp = __shfl_xor_sync(0xffffffffu, q.max_rcomp, k);
        o.min_ratio = __shfl_xor_sync(0xffffffffu, q.min_ratio, k);
        o.argmin = __shfl_xor_sync(0xffffffffu, q.argmin, k);
        o.nonfinite = __shfl_xor_sync(0xffffffffu, q.nonfinite, k);
        q.max_rdual = nanmax(q.max_rdual, o.max_rdual);
        q.max_rcomp = nanmax(q.max_rcomp, o.max_rcomp);
        q.nonfinite |= o.nonfinite;
        if (o.argmin >= 0 && (q.argmin < 0 || o.min_ratio < q.min_ratio ||
                              (o.min_ratio == q.min_ratio && o.argmin < q.argmin))) {
            q.min_ratio = o.min_ratio;
            q.argmin = o.argmin;
        }
        rp = nanmax(rp, __shfl_xor_sync(0xffffffffu, rp, k));
        nf |= __shfl_xor_sync(0xffffffffu, nf, k);
    }
    if (lane == 0) {
        sp[warp] = q;
        sr[warp] = rp;
        snf[warp] = nf;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int nw = (blockDim.x + 31) / 32;
        q = sp[0];
        rp = sr[0];
        nf = snf[0];
        for (int w = 1; w < nw; ++w) {
            const DirPartial& o = sp[w];
            q.max_rdual = nanmax(q.max_rdual, o.max_rdual);
            q.max_rcomp = nanmax(q.max_rcomp, o.max_rcomp);
            q.nonfinite |= o.nonfinite;
            if (o.argmin >= 0 && (q.argmin < 0 || o.min_ratio < q.min_ratio ||
                                  (o.min_ratio == q.min_ratio && o.argmin < q.argmin))) {
                q.min_ratio = o.min_ratio;
                q.argmin = o.argmin;
            }
            rp = nanmax(rp, sr[w]);
            nf |= snf[w];
        }
        st->r_primal = rp;
        st->r_dual = q.max_rdual;
        st->r_comp = q.max_rcomp;
        st->nonfinite = (int)(q.nonfinite | nf);
        st->blocking = q.argmin;
        st->min_ratio = q.min_ratio;
        double alpha = q.argmin < 0 ? kCapAlpha : rho * q.min_ratio;
        st->alpha = alpha;
        int ok = st->cascade_fail == 0 && st->chol_fail < 0 && st->nonfinite == 0 &&
                 !not_interior(st->interior_flags);
        // step only when it is taken by solver.py:236-259 (not the cap/unbounded exit)
        st->stepped = (ok && alpha < kCapAlpha) ? 1 : 0;
    }
}

// x += alpha*dx ; y += alpha*dy ; s += alpha*ds  (solver.py:257-259), gated.
__global__ void k_update(double* __restrict__ x, double* __restrict__ y, double* __restrict__ s,
                         const double* __restrict__ dx, const double* __restrict__ dy,
                         const double* __restrict__ ds, idx_t n, idx_t m,
                         const IterState* __restrict__ st) {
    if (!st->stepped) return;
    const double alpha = st->alpha;
    for (idx_t j = (idx_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (idx_t)gridDim.x * blockDim.x) {
        double px = alpha * dx[j];
        x[j] = x[j] + px;
        double ps = alpha * ds[j];
        s[j] = s[j] + ps;
        if (j < m) {
            double py = alpha * dy[j];
            y[j] = y[j] + py;
        }
    }
}

// The ratio test alone on given directions (the public step_length,
// solver.py:175-189): per-block partial of min(-x/dx | dx<0) and
// min(-s/ds | ds<0) with the first-occurrence index; k_dir_finish folds them.
__global__ void __launch_bounds__(256) k_ratio_part(const double* __restrict__ x,
                                                    const double* __restrict__ s,
                                                    const double* __restrict__ dx,
                                                    const double* __restrict__ ds, idx_t n,
                                                    DirPartial* __restrict__ partials) {
    __shared__ DirPartial sp[8];
    DirPartial p;
    p.max_rdual = 0.0;
    p.max_rcomp = 0.0;
    p.min_ratio = __longlong_as_double(0x7ff0000000000000LL);
    p.argmin = -1;
    p.nonfinite = 0;
    p.pad = 0;
    auto take = [&](double r, long long idx) {
        if (p.argmin < 0 || r < p.min_ratio || (r == p.min_ratio && idx < p.argmin)) {
            p.min_ratio = r;
            p.argmin = idx;
        }
    };
    for (idx_t j = (idx_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (idx_t)gridDim.x * blockDim.x) {
        const double dxj = dx[j], dsj = ds[j];
        if (dxj < 0.0) take(-x[j] / dxj, j);
        if (dsj < 0.0) take(-s[j] / dsj, n + j);
    }
    for (int k = 16; k >= 1; k >>= 1) {
        const double r = __shfl_xor_sync(0xffffffffu, p.min_ratio, k);
        const long long i = __shfl_xor_sync(0xffffffffu, p.argmin, k);
        if (i >= 0) take(r, i);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sp[warp] = p;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w)
            if (sp[w].argmin >= 0) take(sp[w].min_ratio, sp[w].argmin);
        partials[blockIdx.x] = p;
    }
}

// ----------------------------------------------------------- host launchers
int launch_scaling(const double* x, const double* s, idx_t n, double* d, unsigned* flags,
                   cudaStream_t st) {
    if (n < 1) return PDAS_ERR_ARG;
    unsigned grid = (unsigned)((n + 255) / 256);
    if (grid > 1184) grid = 1184;
    k_scaling<<<grid, 256, 0, st>>>(x, s, n, d, flags);
    return PDAS_OK;
}

int launch_directions(const double* a, idx_t m, idx_t n, const double* dy, const double* d,
                      const double* x, const double* s, double* dx, double* ds, void* partials,
                      cudaStream_t st) {
    int R = warp_R(m);
    if (R > 256) return PDAS_ERR_UNSUPPORTED;
    unsigned grid = (unsigned)((n + 7) / 8);
    PDAS_DISPATCH_R(R, 256,
                    k_directions<R_><<<grid, 256, 0, st>>>(a, m, n, dy, d, x, s, dx, ds,
                                                           (DirPartial*)partials));
    return PDAS_OK;
}

idx_t directions_partials_bytes(idx_t n) { return ((n + 7) / 8) * (idx_t)sizeof(DirPartial); }

int launch_dir_finish(const void* partials, idx_t n, const double* adx, idx_t m, const double* dy,
                      double rho, IterState* state, cudaStream_t st) {
    int np_ = (int)((n + 7) / 8);
    k_dir_finish<<<1, 1024, 0, st>>>((const DirPartial*)partials, np_, adx, m, dy, rho, state);
    return PDAS_OK;
}

idx_t ratio_partials_count(idx_t n) {
    const idx_t g = (n + 255) / 256;
    return g < 1184 ? (g > 0 ? g : 1) : 1184;
}

int launch_ratio_test(const double* x, const double* s, const double* dx, const double* ds,
                      idx_t n, double rho, void* partials, IterState* state, cudaStream_t st) {
    const idx_t g = ratio_partials_count(n);
    k_ratio_part<<<(unsigned)g, 256, 0, st>>>(x, s, dx, ds, n, (DirPartial*)partials);
    k_dir_finish<<<1, 1024, 0, st>>>((const DirPartial*)partials, (int)g, nullptr, 0, nullptr, rho,
                                     state);
    return PDAS_OK;
}

idx_t ratio_partials_bytes(idx_t n) { return ratio_partials_count(n) * (idx_t)sizeof(DirPartial); }

int launch_update(double* x, double* y, double* s, const double* dx, const double* dy,
                  const double* ds, idx_t n, idx_t m, const IterState* state, cudaStream_t st) {
    idx_t len = n > m ? n : m;
    unsigned grid = (unsigned)((len + 255) / 256);
    if (grid > 1184) grid = 1184;
    k_update<<<grid, 256, 0, st>>>(x, y, s, dx, dy, ds, n, m, state);
    return PDAS_OK;
}

int launch_dot3(const double* u0, const double* v0, idx_t l0, double* o0, const double* u1,
                const double* v1, idx_t l1, double* o1, const double* u2, const double* v2,
                idx_t l2, double* o2, cudaStream_t st) {
    DotJobs jobs;
    jobs.j[0] = {u0, v0, l0, o0};
    jobs.j[1] = {u1, v1, l1, o1};
    jobs.j[2] = {u2, v2, l2, o2};
    for (int k = 0; k < 3; ++k) {
        idx_t H = pow2_ceil(jobs.j[k].L) >> 1;
        if (H / 1024 > 256) return PDAS_ERR_UNSUPPORTED;
    }
    k_dot3<<<3, 1024, 0, st>>>(jobs);
    return PDAS_OK;
}

}  // namespace pdas

// ---------------------------------------------------------------- fp64 probe
// Diagnostic: sustained rate of separately-rounded DMUL + DADD (the cascade's
// instruction mix: no fused multiply-add).  8 independent chains per thread.
namespace pdas {
__global__ void __launch_bounds__(256) k_fp64_probe(double* sink, long long iters) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
    const double a = 0.999999999, b = 1e-9;
    for (long long i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            double p = x[c] * a;
            x[c] = p + b;
        }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s = s + x[c];
    if (s == 12345.678) sink[0] = s;  // never true; keeps the chains alive
}

int launch_fp64_probe(double* sink, idx_t iters, idx_t* ops, cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8;
    k_fp64_probe<<<blocks, 256, 0, st>>>(sink, (long long)iters);
    *ops = (idx_t)blocks * 256 * iters * 16;
    return PDAS_OK;
}

// div_by (hoisted-reciprocal division, common.cuh) against the plain IEEE
// division on the same operands: out_fast[i] = div_by(a, b, div_recip(b)),
// out_ref[i] = a / b.
__global__ void k_div_selftest(const double* __restrict__ a, const double* __restrict__ b,
                               idx_t n, double* __restrict__ fast, double* __restrict__ ref) {
    for (idx_t i = blockIdx.x * (idx_t)blockDim.x + threadIdx.x; i < n;
         i += (idx_t)gridDim.x * blockDim.x) {
        const double x = a[i], y = b[i];
        fast[i] = div_by(x, y, div_recip(y));
        ref[i] = x / y;
    }
}

int launch_div_selftest(const double* a, const double* b, idx_t n, double* fast, double* ref,
                        cudaStream_t st) {
    if (n <= 0) return PDAS_OK;
    const idx_t blocks = (n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16;
    k_div_selftest<<<(unsigned)blocks, 256, 0, st>>>(a, b, n, fast, ref);
    return PDAS_OK;
}
}  // namespace pdas
