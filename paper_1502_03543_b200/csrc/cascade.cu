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
// applies pivots to a column in ascending l reproduces the reference bit for
// bit.  B200 schedule:
//
//   * [Y | x] is cut into tiles of CT columns.  A CTA holds a tile in
//     REGISTERS: thread t of a T-thread group owns tree s-indices t + T r,
//     i.e. rows t + T r and t + T r + H of each of its columns, so the tree's
//     levels h >= T are register adds and the rest is one shared-memory hop
//     plus a shuffle butterfly.
//   * pivots come in blocks of B.  Pivot data (P_l and A[:,l]) is streamed
//     through a shared-memory ring by 1-D TMA bulk copies (mbarrier full/
//     empty protocol), read once per CTA and reused across its columns.
//   * block b+1 is finalised by a PANEL kernel (one CTA per tile, chained by
//     release/acquire flags): it applies block b, then the block's earlier
//     tiles, then its own triangle.  Meanwhile the UPDATE kernel applies block
//     b to every tile beyond block b+1 (two independent column groups per
//     CTA so one group's reduction latency hides behind the other's math).
//     Panels run on a high-priority side stream one block ahead (lookahead).
//   HBM traffic per element-step drops from 16 B (streaming) to ~16/B B; L2
//   traffic is 16/CT B; the fp64 pipe (4 separately rounded ops per
//   element-step) becomes the bound.
#include <climits>

#include "common.cuh"
#include "pdas_internal.h"
#include "tma.cuh"

namespace pdas {

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------ tile engine
// GEN: general row validity (only for T == 32 configurations, m <= 64).
// Otherwise H >= T, every "lo" row exists, and an absent "hi" row is kept
// exactly +0.0 in x and in v, so its level-0 term is +0.0 -- the reference's
// own padding (`hi = 0.0`, _kernels.pyx:46) -- with no per-element select.
template <int T, int R, int C, bool GEN>
struct Tile {
    double xl[R][C];
    double xh[R][C];
    int t, m, H;
    unsigned hv, lv;
    bool m1;
    int bar;
    double* red;
    double* bc;

    __device__ __forceinline__ int row(int r) const { return t + T * r; }
    __device__ __forceinline__ bool vlo(int r) const { return GEN ? ((lv >> r) & 1u) : true; }
    __device__ __forceinline__ bool vhi(int r) const { return (hv >> r) & 1u; }

    __device__ __forceinline__ void init(int t_, int m_, int bar_, double* red_, double* bc_) {
        t = t_;
        m = m_;
        H = m_ > 1 ? (int)(pow2_ceil(m_) >> 1) : 0;
        m1 = m_ == 1;
        const int hs = H > 0 ? H : 1;
        hv = 0;
        lv = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (row(r) < hs) lv |= 1u << r;
            if (!m1 && row(r) + H < m) hv |= 1u << r;
        }
        bar = bar_;
        red = red_;
        bc = bc_;
    }

    __device__ __forceinline__ void sync() const {
        if (T > 32)
            named_bar(bar, T);
        else
            __syncwarp();
    }

    __device__ __forceinline__ void load(const double* __restrict__ cols, idx_t col0, idx_t ncols) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const idx_t col = col0 + c;
            const bool on = col < ncols;
            const double* p = cols + col * m;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                xl[r][c] = (on && vlo(r)) ? __ldcg(p + row(r)) : 0.0;
                xh[r][c] = (on && vhi(r)) ? __ldcg(p + row(r) + H) : 0.0;
            }
        }
    }

    __device__ __forceinline__ void store(double* __restrict__ cols, idx_t col0, idx_t ncols) const {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const idx_t col = col0 + c;
            if (col >= ncols) continue;
            double* p = cols + col * m;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (vlo(r)) p[row(r)] = xl[r][c];
                if (vhi(r)) p[row(r) + H] = xh[r][c];
            }
        }
    }

    // v = A[:,l] * f for this thread's rows, from a column base pointer
    // (shared-memory stage or global).  Absent rows get exactly +0.0.
    template <bool GLOBAL>
    __device__ __forceinline__ void make_v(const double* ac, double f, double (&vl)[R],
                                           double (&vh)[R]) const {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double al = 0.0, ah = 0.0;
            if (vlo(r)) al = GLOBAL ? __ldcg(ac + row(r)) : ac[row(r)];
            if (vhi(r)) ah = GLOBAL ? __ldcg(ac + row(r) + H) : ac[row(r) + H];
            vl[r] = vlo(r) ? al * f : 0.0;
            vh[r] = vhi(r) ? ah * f : 0.0;
        }
    }

    template <bool GLOBAL>
    __device__ __forceinline__ void load_p(const double* pc, double (&pl)[R], double (&ph)[R]) const {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            pl[r] = 0.0;
            ph[r] = 0.0;
            if (vlo(r)) pl[r] = GLOBAL ? __ldcg(pc + row(r)) : pc[row(r)];
            if (vhi(r)) ph[r] = GLOBAL ? __ldcg(pc + row(r) + H) : pc[row(r) + H];
        }
    }

    // Per-thread partial (tree levels >= T) of tree(v, column c), all c.
    __device__ __forceinline__ void partials(const double (&vl)[R], const double (&vh)[R],
                                             double (&part)[C]) const {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double s[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (GEN) {
                    double lo = vlo(r) ? vl[r] * xl[r][c] : 0.0;
                    double hi = vhi(r) ? vh[r] * xh[r][c] : 0.0;
                    s[r] = m1 ? lo : lo + hi;
                } else {
                    double lo = vl[r] * xl[r][c];
                    double hi = vh[r] * xh[r][c];
                    s[r] = lo + hi;
                }
            }
            part[c] = lane_tree<R>(s);
        }
    }

    // First half of the cross-thread reduction: publish partials (T > 32).
    __device__ __forceinline__ void publish(const double (&part)[C]) const {
        if (T > 32) {
#pragma unroll
            for (int c = 0; c < C; ++c) red[c * T + t] = part[c];
        }
    }

    // Second half (after the group barrier that follows publish()): levels
    // T/2 .. 1.  DIV: out[c] = inner[c] / denom (one lane per column
    // divides), else out[c] = inner[c].  Ends with the group barrier when
    // T > 32; every thread returns all C values.
    template <bool DIV>
    __device__ __forceinline__ void finish(const double (&part)[C], double denom,
                                           double (&out)[C]) const {
        const int lane = t & 31;
        if (T == 32) {
            const int w = H >= 32 ? 32 : (H > 0 ? H : 1);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                double v = warp_butterfly(part[c], w);
                if (GEN && H < 32) v = __shfl_sync(0xffffffffu, v, 0);
                out[c] = DIV ? v / denom : v;
            }
        } else {
            constexpr int NW = T / 32;
            const int warp = t >> 5;
            for (int c = warp; c < C; c += NW) {
                double q[NW];
#pragma unroll
                for (int k = 0; k < NW; ++k) q[k] = red[c * T + lane + 32 * k];
                double v = warp_butterfly32(lane_tree<NW>(q));
                if (lane == 0) bc[c] = DIV ? v / denom : v;
            }
            sync();
#pragma unroll
            for (int c = 0; c < C; ++c) out[c] = bc[c];
        }
    }

    __device__ __forceinline__ void axpy(const double (&g)[C], const double (&pl)[R],
                                         const double (&ph)[R]) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool lo = vlo(r), hi = vhi(r);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (lo) {
                    double q0 = g[c] * pl[r];
                    xl[r][c] = xl[r][c] - q0;
                }
                if (hi) {
                    double q1 = g[c] * ph[r];
                    xh[r][c] = xh[r][c] - q1;
                }
            }
        }
    }
};

// ------------------------------------------------------------ TMA pipeline
// Stage s = [P_l | A[:,l]] (2 x mp doubles).  full[s]: producer arrive +
// TMA bytes.  empty[s]: one arrival per consumer group once it is done.
// `k` counts stage uses (identical in every thread of the CTA).
struct Pipe {
    double* buf;
    uint64_t* full;
    uint64_t* empty;
    int S, mp;
    unsigned k;
};

__device__ __forceinline__ void pipe_issue(Pipe& p, unsigned use, const double* pcol,
                                           const double* acol, int m) {
    const int s = (int)(use % p.S);
    if (use >= (unsigned)p.S) mbar_wait(p.empty + s, ((use / p.S) - 1u) & 1u);
    const uint32_t bytes = (uint32_t)m * (uint32_t)sizeof(double);
    double* dst = p.buf + (size_t)s * 2 * p.mp;
    if (pcol) {
        mbar_arrive_expect_tx(p.full + s, 2 * bytes);
        tma_load_1d(dst, pcol, bytes, p.full + s);
    } else {
        mbar_arrive_expect_tx(p.full + s, bytes);
    }
    tma_load_1d(dst + p.mp, acol, bytes, p.full + s);
}

// dynamic smem: red[G][C*T] | bc[G][C] | full[S] | empty[S] | stages
template <int T, int C, int G>
__host__ __device__ constexpr size_t casc_head_bytes(int S) {
    return (((size_t)G * C * T + (size_t)G * C + 2 * (size_t)S) * sizeof(double) + 127) & ~(size_t)127;
}

template <int T, int C, int G>
__host__ __device__ inline size_t casc_smem_bytes(int S, int m) {
    const size_t mp = (size_t)((m + 1) & ~1);
    return casc_head_bytes<T, C, G>(S) + (size_t)S * 2 * mp * sizeof(double);
}

template <int T, int C, int G>
__device__ __forceinline__ void carve(double*& red, double*& bc, Pipe& pp, int S, int m) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    red = reinterpret_cast<double*>(smem_raw);
    bc = red + G * C * T;
    pp.full = reinterpret_cast<uint64_t*>(bc + G * C);
    pp.empty = pp.full + (S > 0 ? S : 0);
    pp.buf = reinterpret_cast<double*>(smem_raw + casc_head_bytes<T, C, G>(S > 0 ? S : 0));
    pp.S = S > 0 ? S : 1;
    pp.mp = (m + 1) & ~1;
    pp.k = 0;
    if (S > 0) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < S; ++s) {
                mbar_init(pp.full + s, 1);
                mbar_init(pp.empty + s, G);
            }
            mbar_fence_init();
        }
        __syncthreads();
    }
}

// Apply pivots [l0, l1) whose final columns live in global memory to the
// register tile, in ascending order.  `producer` is the CTA's thread 0.
template <bool TMA, int T, int R, int C, bool GEN>
__device__ __forceinline__ void apply_global(Tile<T, R, C, GEN>& tl, Pipe& pp,
                                             const double* __restrict__ cols,
                                             const double* __restrict__ a,
                                             const double* __restrict__ d,
                                             const double* __restrict__ denoms, idx_t l0,
                                             idx_t l1, bool producer) {
    const int cnt = (int)(l1 - l0);
    if (cnt <= 0) return;
    const int m = tl.m;
    const unsigned k0 = pp.k;
    if (TMA && producer) {
        const int pre = cnt < pp.S ? cnt : pp.S;
        for (int i = 0; i < pre; ++i)
            pipe_issue(pp, k0 + i, cols + (l0 + i) * m, a + (l0 + i) * m, m);
    }
    for (int j = 0; j < cnt; ++j) {
        const idx_t l = l0 + j;
        const unsigned use = k0 + j;
        const int s = (int)(use % pp.S);
        const double* pc;
        const double* ac;
        if (TMA) {
            mbar_wait(pp.full + s, (use / pp.S) & 1u);
            pc = pp.buf + (size_t)s * 2 * pp.mp;
            ac = pc + pp.mp;
        } else {
            pc = cols + l * m;
            ac = a + l * m;
        }
        const double dl = __ldg(d + l);
        const bool active = dl != 1.0;
        double part[C];
        if (active) {
            double vl[R], vh[R];
            tl.template make_v<!TMA>(ac, dl - 1.0, vl, vh);
            tl.partials(vl, vh, part);
            tl.publish(part);
        }
        tl.sync();  // B1: partials published; stage of use-1 fully consumed
        if (TMA && j > 0) {
            if (tl.t == 0) mbar_arrive(pp.empty + (int)((use - 1) % pp.S));
            if (producer && j - 1 + pp.S < cnt)
                pipe_issue(pp, use - 1 + pp.S, cols + (l - 1 + pp.S) * m, a + (l - 1 + pp.S) * m,
                           m);
        }
        if (active) {
            const double denom = __ldcg(denoms + l);
            double g[C];
            tl.template finish<true>(part, denom, g);
            double pl[R], ph[R];
            tl.template load_p<!TMA>(pc, pl, ph);
            tl.axpy(g, pl, ph);
        }
    }
    if (TMA) {
        tl.sync();
        if (tl.t == 0) mbar_arrive(pp.empty + (int)((k0 + cnt - 1) % pp.S));
        pp.k = k0 + cnt;
    }
}

// ------------------------------------------------------------ update kernel
// Tile (tile0 + blockIdx.x) of CT = G*C columns receives pivots [p0, p1);
// group g (T threads) owns columns [tile*CT + g*C, +C).
template <bool TMA, int T, int R, int C, int G, bool GEN>
__global__ void __launch_bounds__(T* G, 1)
    k_casc_update(double* __restrict__ cols, const double* __restrict__ a,
                  const double* __restrict__ d, const double* __restrict__ denoms, int m, idx_t n,
                  idx_t p0, idx_t p1, idx_t tile0, int S, const int32_t* __restrict__ fail) {
    if (*(volatile const int32_t*)fail) return;
    double *red, *bc;
    Pipe pp;
    carve<T, C, G>(red, bc, pp, TMA ? S : 0, m);
    const int grp = threadIdx.x / T;
    Tile<T, R, C, GEN> tl;
    tl.init(threadIdx.x % T, m, 1 + grp, red + grp * C * T, bc + grp * C);
    const idx_t col0 = (tile0 + blockIdx.x) * (C * G) + grp * C;
    tl.load(cols, col0, n + 1);
    apply_global<TMA>(tl, pp, cols, a, d, denoms, p0, p1, threadIdx.x == 0);
    tl.store(cols, col0, n + 1);
}

// ------------------------------------------------------------ panel kernel
// One CTA per tile of block [p0, p1): apply the previous block [q0, q1),
// then the pivots of this block's earlier tiles as their CTAs publish them
// (flags[tile] == epoch), then the in-register triangle; publish.  Breakdown
// is detected here, in step order, and reported as the 1-based step.
template <bool TMA, int T, int R, int C, bool GEN>
__global__ void __launch_bounds__(T, 1)
    k_casc_panel(double* __restrict__ cols, const double* __restrict__ a,
                 const double* __restrict__ d, double* __restrict__ denoms, int m, idx_t n,
                 idx_t q0, idx_t q1, idx_t p0, idx_t p1, int S, int32_t* __restrict__ fail,
                 int* __restrict__ flags, int epoch) {
    if (*(volatile int32_t*)fail) return;
    double *red, *bc;
    Pipe pp;
    carve<T, C, 1>(red, bc, pp, TMA ? S : 0, m);
    Tile<T, R, C, GEN> tl;
    tl.init(threadIdx.x, m, 1, red, bc);
    const bool producer = threadIdx.x == 0;
    const idx_t tile = p0 / C + blockIdx.x;
    const idx_t col0 = tile * C;
    tl.load(cols, col0, n + 1);
    apply_global<TMA>(tl, pp, cols, a, d, denoms, q0, q1, producer);
    bool dead = false;
    for (idx_t tp = p0 / C; tp < tile; ++tp) {
        if (producer)
            while (ld_acquire(flags + tp) != epoch) __nanosleep(64);
        __syncthreads();
        if (*(volatile int32_t*)fail) {
            dead = true;
            break;
        }
        fence_proxy_async_global();  // peer CTA's generic stores -> our TMA reads
        const idx_t e = tp * C + C < p1 ? tp * C + C : p1;
        apply_global<TMA>(tl, pp, cols, a, d, denoms, tp * C, e, producer);
    }
    if (!dead) {
        // triangle over this tile's own pivot columns, A columns via the pipe
        const int cnt = (int)((col0 + C < p1 ? col0 + C : p1) - col0);
        const unsigned k0 = pp.k;
        if (TMA && producer) {
            const int pre = cnt < pp.S ? cnt : pp.S;
            for (int i = 0; i < pre; ++i) pipe_issue(pp, k0 + i, nullptr, a + (col0 + i) * m, m);
        }
        bool broken = false;
#pragma unroll
        for (int cl = 0; cl < C; ++cl) {
            if (cl < cnt) {
                const idx_t l = col0 + cl;
                const unsigned use = k0 + cl;
                const int s = (int)(use % pp.S);
                const double* ac = a + l * m;
                if (TMA) {
                    mbar_wait(pp.full + s, (use / pp.S) & 1u);
                    ac = pp.buf + (size_t)s * 2 * pp.mp + pp.mp;
                }
                const double dl = __ldg(d + l);
                const bool active = dl != 1.0 && !broken;
                double part[C];
                if (active) {
                    double vl[R], vh[R];
                    tl.template make_v<!TMA>(ac, dl - 1.0, vl, vh);
                    tl.partials(vl, vh, part);
                    tl.publish(part);
                }
                tl.sync();
                if (TMA && cl > 0) {
                    if (producer) mbar_arrive(pp.empty + (int)((use - 1) % pp.S));
                    if (producer && cl - 1 + pp.S < cnt)
                        pipe_issue(pp, use - 1 + pp.S, nullptr, a + (l - 1 + pp.S) * m, m);
                }
                if (active) {
                    double inner[C];
                    tl.template finish<false>(part, 0.0, inner);
                    const double denom = 1.0 + inner[cl];
                    if (fabs(denom) <= kDenomEpsRel * (1.0 + fabs(inner[cl]))) {
                        if (producer) *fail = (int32_t)(l + 1);
                        broken = true;
                    } else {
                        if (producer) denoms[l] = denom;
                        double pl[R], ph[R];
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            pl[r] = tl.xl[r][cl];
                            ph[r] = tl.xh[r][cl];
                        }
#pragma unroll
                        for (int c = cl + 1; c < C; ++c) {
                            const double g = inner[c] / denom;
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                if (tl.vlo(r)) {
                                    double q0v = g * pl[r];
                                    tl.xl[r][c] = tl.xl[r][c] - q0v;
                                }
                                if (tl.vhi(r)) {
                                    double q1v = g * ph[r];
                                    tl.xh[r][c] = tl.xh[r][c] - q1v;
                                }
                            }
                        }
                    }
                }
            }
        }
        if (TMA) {
            tl.sync();
            if (producer) mbar_arrive(pp.empty + (int)((k0 + cnt - 1) % pp.S));
            pp.k = k0 + cnt;
        }
        if (!broken) tl.store(cols, col0, n + 1);
    }
    __threadfence();
    __syncthreads();
    if (producer) st_release(flags + tile, epoch);
}

// ------------------------------------------------------------ host side
struct CascCfg {
    int T, R, Cu, G, CT;
};

static CascCfg cascade_cfg(idx_t m) {
    const idx_t H = m > 1 ? pow2_ceil(m) >> 1 : 0;
    if (H <= 32) return {32, 1, 8, 1, 8};
    if (H == 64) return {64, 1, 8, 1, 8};
    if (H == 128) return {128, 1, 8, 1, 8};
    if (H == 256) return {256, 1, 8, 2, 16};
    if (H == 512) return {256, 2, 8, 2, 16};
    if (H == 1024) return {256, 4, 4, 2, 8};
    if (H == 2048) return {256, 8, 2, 2, 4};
    if (H == 4096) return {256, 16, 1, 2, 2};
    if (H == 8192) return {256, 32, 1, 1, 1};
    return {0, 0, 0, 0, 0};
}

idx_t cascade_supported_m() { return 16384; }

// Side stream (high priority) + two events for the panel lookahead, per device.
struct SideStream {
    cudaStream_t ps = nullptr;
    cudaEvent_t e0 = nullptr, eP = nullptr, eU = nullptr;
};

static SideStream& side_stream() {
    static thread_local SideStream ss[16];
    int dev = 0;
    cudaGetDevice(&dev);
    SideStream& s = ss[dev & 15];
    if (!s.ps) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        cudaStreamCreateWithPriority(&s.ps, cudaStreamNonBlocking, hi);
        cudaEventCreateWithFlags(&s.e0, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&s.eP, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&s.eU, cudaEventDisableTiming);
    }
    return s;
}

template <bool TMA, int T, int R, int Cu, int G, int CT>
static int run_cascade_impl(double* cols, const double* a, const double* d, int m, idx_t n,
                            double* denoms, int32_t* fail, int* flags, int epoch, int B, int S,
                            cudaStream_t st) {
    constexpr bool GEN = (T == 32);
    static_assert(Cu * G == CT, "tile width");
    B = (B + CT - 1) / CT * CT;
    const size_t smem_u = casc_smem_bytes<T, Cu, G>(TMA ? S : 0, m);
    const size_t smem_p = casc_smem_bytes<T, CT, 1>(TMA ? S : 0, m);
    auto ku = k_casc_update<TMA, T, R, Cu, G, GEN>;
    auto kp = k_casc_panel<TMA, T, R, CT, GEN>;
    cudaFuncSetAttribute(ku, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_u);
    cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
    const idx_t ntiles = (n + 1 + CT - 1) / CT;
    const idx_t nb = (n + B - 1) / B;
    auto blk_end = [&](idx_t b) { return (b + 1) * B < n ? (b + 1) * B : n; };
    auto tiles_of = [&](idx_t b) { return (blk_end(b) - b * B + CT - 1) / CT; };
    SideStream& ss = side_stream();
    cudaEventRecord(ss.e0, st);
    cudaStreamWaitEvent(ss.ps, ss.e0, 0);
    cudaEventRecord(ss.eU, st);  // "U_rest(-1)" = nothing beyond the start
    kp<<<(unsigned)tiles_of(0), T, smem_p, ss.ps>>>(cols, a, d, denoms, m, n, 0, 0, 0, blk_end(0),
                                                    S, fail, flags, epoch);
    cudaEventRecord(ss.eP, ss.ps);
    for (idx_t b = 0; b < nb; ++b) {
        cudaStreamWaitEvent(st, ss.eP, 0);  // panel(b): block b is final
        if (b + 1 < nb) {
            // panel(b+1) needs block b (stream order on ps) and U_rest(b-1)
            cudaStreamWaitEvent(ss.ps, ss.eU, 0);
            kp<<<(unsigned)tiles_of(b + 1), T, smem_p, ss.ps>>>(
                cols, a, d, denoms, m, n, b * B, blk_end(b), (b + 1) * B, blk_end(b + 1), S, fail,
                flags, epoch);
            cudaEventRecord(ss.eP, ss.ps);
        }
        // U_rest(b): every tile beyond block b+1 (or beyond block b at the end)
        const idx_t last = b + 1 < nb ? blk_end(b + 1) : blk_end(b);
        const idx_t t0 = (last + CT - 1) / CT;
        if (t0 < ntiles)
            ku<<<(unsigned)(ntiles - t0), T * G, smem_u, st>>>(cols, a, d, denoms, m, n, b * B,
                                                               blk_end(b), t0, S, fail);
        cudaEventRecord(ss.eU, st);
    }
    return cudaGetLastError() == cudaSuccess ? PDAS_OK : PDAS_ERR_CUDA;
}

template <int T, int R, int Cu, int G, int CT>
static int run_cascade(double* cols, const double* a, const double* d, int m, idx_t n,
                       double* denoms, int32_t* fail, int* flags, int epoch, int B,
                       cudaStream_t st) {
    const bool aligned = (m % 2 == 0) && (((uintptr_t)cols | (uintptr_t)a) % 16 == 0);
    const size_t budget = 200 * 1024;
    int S = 4;
    while (S > 2 && casc_smem_bytes<T, CT, 1>(S, m) > budget) --S;
    if (aligned && casc_smem_bytes<T, CT, 1>(S, m) <= budget &&
        casc_smem_bytes<T, Cu, G>(S, m) <= budget)
        return run_cascade_impl<true, T, R, Cu, G, CT>(cols, a, d, m, n, denoms, fail, flags,
                                                       epoch, B, S, st);
    return run_cascade_impl<false, T, R, Cu, G, CT>(cols, a, d, m, n, denoms, fail, flags, epoch,
                                                    B, 1, st);
}

idx_t cascade_flags_count(idx_t m, idx_t n) {
    CascCfg c = cascade_cfg(m);
    return c.CT > 0 ? (n + 1 + c.CT - 1) / c.CT + 1 : 1;
}

int launch_cascade(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                   double* denoms, int32_t* fail_dev, int* flags, int epoch, int block_pivots,
                   cudaStream_t st) {
    if (m < 1 || n < 0 || m > INT_MAX / 4) return PDAS_ERR_ARG;
    cudaMemsetAsync(fail_dev, 0, sizeof(int32_t), st);
    if (n == 0) return PDAS_OK;
    const CascCfg cfg = cascade_cfg(m);
    const int B = block_pivots > 0 ? block_pivots : 64;
#define PDAS_CASC(T_, R_, C_, G_, CT_)                                                       \
    if (cfg.T == T_ && cfg.R == R_ && cfg.Cu == C_ && cfg.G == G_)                           \
        return run_cascade<T_, R_, C_, G_, CT_>(cols, a, d, (int)m, n, denoms, fail_dev, flags, \
                                                epoch, B, st);
    PDAS_CASC(32, 1, 8, 1, 8)
    PDAS_CASC(64, 1, 8, 1, 8)
    PDAS_CASC(128, 1, 8, 1, 8)
    PDAS_CASC(256, 1, 8, 2, 16)
    PDAS_CASC(256, 2, 8, 2, 16)
    PDAS_CASC(256, 4, 4, 2, 8)
    PDAS_CASC(256, 8, 2, 2, 4)
    PDAS_CASC(256, 16, 1, 2, 2)
    PDAS_CASC(256, 32, 1, 1, 1)
#undef PDAS_CASC
    return PDAS_ERR_UNSUPPORTED;
}

}  // namespace pdas
