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
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "pdas_internal.h"
#include "tma.cuh"


namespace pdas {

#ifndef PDAS_PANEL_TRACE
#define PDAS_PANEL_TRACE 0
#endif
// Diagnostic build only (-DPDAS_HOP_TRACE=1): globaltimer marks of one panel
// hop (tile 15 -> tile 16 of pivot block 5), read back with pdas_debug_hop_trace.
#ifndef PDAS_HOP_TRACE
#define PDAS_HOP_TRACE 0
#endif
#if PDAS_HOP_TRACE
__device__ unsigned long long g_hop_trace[32];
#define HOP_MARK(cond, k)                                                          \
    do {                                                                           \
        if ((cond) && threadIdx.x == 0) {                                          \
            unsigned long long t_;                                                 \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
            g_hop_trace[k] = t_;                                                   \
        }                                                                          \
    } while (0)
#define PW_MARK(cond, k)                                                           \
    do {                                                                           \
        if (cond) {                                                                \
            unsigned long long t_;                                                 \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
            g_hop_trace[k] = t_;                                                   \
        }                                                                          \
    } while (0)
#else
#define HOP_MARK(cond, k) \
    do {                  \
    } while (0)
#define PW_MARK(cond, k) \
    do {                 \
    } while (0)
#endif
#if PDAS_PANEL_TRACE
__device__ long long g_panel_trace[8];
#endif

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

__device__ __forceinline__ int ld_acquire_(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed(int* p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release_sys(int* p, int v) {
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
    int v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

int panel_flag_chunks(int ct);

// Dependencies of an update CTA that may start before the previous update
// kernel has finished (programmatic dependent launch, run_cascade_impl):
//   * the block's panel is complete: its last tile's last chunk flag (pflag)
//     carries this cascade's epoch;
//   * this tile has received the previous block: tile_done[tile] >= need.
// One thread spins; the caller's barrier hands the result to the CTA.
__device__ __forceinline__ void update_deps(const int* pflag, int epoch, const int* tile_done,
                                            idx_t tile, int need, const int32_t* fail) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x != 0) return;
    if (pflag)
        while (*(volatile const int32_t*)fail == 0 && ld_acquire_(pflag) != epoch) __nanosleep(64);
    if (tile_done && need > 0)
        while (*(volatile const int32_t*)fail == 0 && ld_acquire_(tile_done + tile) < need)
            __nanosleep(64);
}

// a value the compiler must keep in a register (it cannot rematerialise it)
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
    asm volatile("" : "+r"(v));
    return v;
}

__device__ __forceinline__ void st_shared_f64(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v));
}

__device__ __forceinline__ double ld_shared_f64(uint32_t a) {
    double x;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a));
    return x;
}

__device__ __forceinline__ void ld_shared_v2_f64(uint32_t a, double& x, double& y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
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

    __device__ __forceinline__ void store(double* __restrict__ cols, idx_t col0, idx_t ncols,
                                          int c_lo = 0, int c_hi = C) const {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const idx_t col = col0 + c;
            if (c < c_lo || c >= c_hi || col >= ncols) continue;
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
    // FULL (warp-uniform): every row this thread owns exists -- no selects.
    __device__ __forceinline__ bool full() const {
        return !GEN && hv == (R >= 32 ? 0xffffffffu : (1u << (R & 31)) - 1u);
    }

    template <bool GLOBAL, bool FULL>
    __device__ __forceinline__ void make_v(const double* ac, double f, double (&vl)[R],
                                           double (&vh)[R]) const {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (FULL) {
                const double al = GLOBAL ? __ldcg(ac + row(r)) : ac[row(r)];
                const double ah = GLOBAL ? __ldcg(ac + row(r) + H) : ac[row(r) + H];
                vl[r] = al * f;
                vh[r] = ah * f;
            } else {
                double al = 0.0, ah = 0.0;
                if (vlo(r)) al = GLOBAL ? __ldcg(ac + row(r)) : ac[row(r)];
                if (vhi(r)) ah = GLOBAL ? __ldcg(ac + row(r) + H) : ac[row(r) + H];
                vl[r] = vlo(r) ? al * f : 0.0;
                vh[r] = vhi(r) ? ah * f : 0.0;
            }
        }
    }

    template <bool GLOBAL, bool FULL>
    __device__ __forceinline__ void load_p(const double* pc, double (&pl)[R], double (&ph)[R]) const {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (FULL) {
                pl[r] = GLOBAL ? __ldcg(pc + row(r)) : pc[row(r)];
                ph[r] = GLOBAL ? __ldcg(pc + row(r) + H) : pc[row(r) + H];
            } else {
                pl[r] = 0.0;
                ph[r] = 0.0;
                if (vlo(r)) pl[r] = GLOBAL ? __ldcg(pc + row(r)) : pc[row(r)];
                if (vhi(r)) ph[r] = GLOBAL ? __ldcg(pc + row(r) + H) : pc[row(r) + H];
            }
        }
    }

    // Per-thread partial (tree levels >= T) of tree(v, column c), all c.
    __device__ __forceinline__ void partials(const double (&vl)[R], const double (&vh)[R],
                                             double (&part)[C], int c0 = 0) const {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (c < c0) continue;
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
    __device__ __forceinline__ void publish(const double (&part)[C], int c0 = 0) const {
        if (T > 32) {
#pragma unroll
            for (int c = 0; c < C; ++c)
                if (c >= c0) red[c * T + t] = part[c];
        }
    }

    // Second half (after the group barrier that follows publish()): levels
    // T/2 .. 1.  DIV: out[c] = inner[c] / denom (one lane per column
    // divides), else out[c] = inner[c].  Ends with the group barrier when
    // T > 32; every thread returns all C values.
    // c0: only columns >= c0 are reduced (the panel triangle's live columns).
    template <bool DIV>
    __device__ __forceinline__ void finish(const double (&part)[C], double denom, double y,
                                           double (&out)[C], int c0 = 0) const {
        const int lane = t & 31;
        if (T == 32) {
            const int w = H >= 32 ? 32 : (H > 0 ? H : 1);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (c < c0) continue;
                double v = warp_butterfly(part[c], w);
                if (GEN && H < 32) v = __shfl_sync(0xffffffffu, v, 0);
                out[c] = DIV ? div_by(v, denom, y) : v;
            }
        } else {
            constexpr int NW = T / 32;
            constexpr int PER = (C + NW - 1) / NW;
            const int warp = t >> 5;
            // a warp's columns (warp, warp+NW, ...) as independent chains
            double v[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int c = warp + NW * k;
                if (c >= c0 && c < C) {
                    double q[NW];
#pragma unroll
                    for (int i = 0; i < NW; ++i) q[i] = red[c * T + lane + 32 * i];
                    v[k] = lane_tree<NW>(q);
                }
            }
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int c = warp + NW * k;
                if (c >= c0 && c < C) {
                    const double u = warp_butterfly32(v[k]);
                    if (lane == 0)
                        bc[c] = DIV ? div_by(u, denom, y) : u;
                }
            }
            sync();
#pragma unroll
            for (int c = 0; c < C; ++c)
                if (c >= c0) out[c] = bc[c];
        }
    }

    // x -= g*P.  Absent rows are never touched (they stay exactly +0.0 even
    // when g is not finite), so the !FULL path predicates them off.
    template <bool FULL>
    __device__ __forceinline__ void axpy(const double (&g)[C], const double (&pl)[R],
                                         const double (&ph)[R]) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool lo = FULL || vlo(r), hi = FULL || vhi(r);
            if (lo) {
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    double q0 = g[c] * pl[r];
                    xl[r][c] = xl[r][c] - q0;
                }
            }
            if (hi) {
#pragma unroll
                for (int c = 0; c < C; ++c) {
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
// `k` counts stage uses (identical in every thread of the CTA).  S (stage
// count) is a compile-time constant so stage arithmetic is shifts/masks.
// a panel tile publishes its final columns in this many chunks (flags per chunk)
constexpr int kPanelChunks = 2;

// Peers of a column-sharded cascade (dist.py): device addresses, valid in
// this process (NVLink peer mappings), of every other rank's [Y|x], cascade
// denominators, fail word and panel flags.  count = 0: single GPU.
struct PeerSet {
    int count;
    double* cols[kMaxPeers];
    double* denoms[kMaxPeers];
    int32_t* fail[kMaxPeers];
    int* flags[kMaxPeers];
};

// Publish a breakdown to the peers (before their flag), then release the
// tile's flag on every peer (system scope: the stores went over NVLink).
__device__ __forceinline__ void peer_signal(const PeerSet& peers, const int32_t* fail,
                                            const int* flags, idx_t flag_idx, int epoch) {
    (void)flags;
    const int32_t f = *(volatile const int32_t*)fail;
    if (f)
        for (int q = 0; q < peers.count; ++q) *(volatile int32_t*)peers.fail[q] = f;
    __threadfence_system();
    for (int q = 0; q < peers.count; ++q) st_release_sys(peers.flags[q] + flag_idx, epoch);
}

template <int S>
struct Pipe {
    double* buf;
    uint64_t* full;
    uint64_t* empty;
    uint32_t full_a, empty_a, buf_a;  // shared-window addresses (no cvta in the loop)
    int mp;
    unsigned k;
    double* sd;    // d[l - base] for the kernel's pivot window (shared memory)
    double* sden;  // denom[l - base]
    double* sy;    // div_recip(denom[l - base]) (common.cuh)
};

__device__ __forceinline__ void mbar_wait_a(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITA_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITA_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_a(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

template <int S>
__device__ __forceinline__ void pipe_issue(Pipe<S>& p, unsigned use, const double* pcol,
                                           const double* acol, int m, bool wait_empty = true) {
    const uint32_t s = use % S;
    const uint32_t fb = p.full_a + 8 * s;
    if (wait_empty && use >= (unsigned)S) mbar_wait_a(p.empty_a + 8 * s, ((use / S) - 1u) & 1u);
    const uint32_t bytes = (uint32_t)m * (uint32_t)sizeof(double);
    const uint32_t dst = p.buf_a + s * 2u * (uint32_t)p.mp * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                 "r"(pcol ? 2 * bytes : bytes)
                 : "memory");
    if (pcol)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(dst),
            "l"(pcol), "r"(bytes), "r"(fb)
            : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(dst + (uint32_t)p.mp * 8u),
        "l"(acol), "r"(bytes), "r"(fb)
        : "memory");
}

// dynamic smem: red[G][C*T] | bc[G][C] | sd[2*kMaxBlock] | sden[2*kMaxBlock]
//               | sy[2*kMaxBlock] | full[S] | empty[S] | stages
template <int T, int C, int G>
__host__ __device__ constexpr size_t casc_head_bytes(int S) {
    return (((size_t)G * C * T + 2 * (size_t)G * C + 6 * kMaxBlock + 2 * (size_t)S) * sizeof(double) +
            127) & ~(size_t)127;
}

template <int T, int C, int G>
__host__ __device__ inline size_t casc_smem_bytes(int S, int m) {
    const size_t mp = (size_t)((m + 1) & ~1);
    return casc_head_bytes<T, C, G>(S) + (size_t)S * 2 * mp * sizeof(double);
}

template <int T, int C, int G, int S>
__device__ __forceinline__ void carve(double*& red, double*& bc, Pipe<S>& pp, bool tma, int m) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    red = reinterpret_cast<double*>(smem_raw);
    bc = red + G * C * T;  // bc[G*C] (+ G*C scratch: the panel triangle's quotients)
    pp.sd = bc + 2 * G * C;
    pp.sden = pp.sd + 2 * kMaxBlock;
    pp.sy = pp.sden + 2 * kMaxBlock;
    pp.full = reinterpret_cast<uint64_t*>(pp.sy + 2 * kMaxBlock);
    pp.empty = pp.full + S;
    pp.buf = reinterpret_cast<double*>(smem_raw + casc_head_bytes<T, C, G>(S));
    pp.full_a = smem_addr(pp.full);
    pp.empty_a = smem_addr(pp.empty);
    pp.buf_a = smem_addr(pp.buf);
    pp.mp = (m + 1) & ~1;
    pp.k = 0;
    if (tma && threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(pp.full + s, 1);
            mbar_init(pp.empty + s, G);
        }
        mbar_fence_init();
    }
}

// Stage the pivot scalars of [lo, hi) (relative to `base`) into shared memory.
template <int S>
__device__ __forceinline__ void stage_scalars(Pipe<S>& pp, const double* __restrict__ d,
                                              const double* __restrict__ denoms, idx_t base,
                                              idx_t lo, idx_t hi, bool with_d) {
    for (idx_t l = lo + threadIdx.x; l < hi; l += blockDim.x) {
        if (with_d) pp.sd[l - base] = __ldg(d + l);
        const double den = __ldcg(denoms + l);
        pp.sden[l - base] = den;
        pp.sy[l - base] = div_recip(den);
    }
}

// Apply pivots [l0, l1) whose final columns live in global memory to the
// register tile, in ascending order.  d and denom come from the shared
// window (index l - base).  `producer` is the CTA's thread 0.
template <bool TMA, bool FULL, int S, int T, int R, int C, bool GEN>
__device__ __forceinline__ void apply_impl(Tile<T, R, C, GEN>& tl, Pipe<S>& pp,
                                           const double* __restrict__ cols,
                                           const double* __restrict__ a, idx_t base, idx_t l0,
                                           int cnt, bool producer) {
    const int m = tl.m;
    const unsigned k0 = pp.k;
    const double* sd = pp.sd + (l0 - base);
    const double* sden = pp.sden + (l0 - base);
    const double* sy = pp.sy + (l0 - base);
    const double* ga = a + l0 * m;      // global A column of pivot l0 + j: ga + j*m
    const double* gc = cols + l0 * m;   // global P column
    const int stage = 2 * pp.mp;
#if PDAS_PANEL_TRACE
    const bool trace = gridDim.x == 32 && blockIdx.x == 31 && threadIdx.x == 0 && T == 256;
    long long tm = clock64();
#define APPLY_LAP(k)                                    \
    do {                                                \
        if (trace) {                                    \
            const long long tn = clock64();             \
            g_panel_trace[k] += tn - tm;                \
            tm = tn;                                    \
        }                                               \
    } while (0)
#else
#define APPLY_LAP(k) \
    do {             \
    } while (0)
#endif
    for (int j = 0; j < cnt; ++j) {
        const unsigned use = k0 + j;
        const double* pc;
        const double* ac;
        if (TMA) {
            const uint32_t s = use % S;
            mbar_wait_a(pp.full_a + 8 * s, (use / S) & 1u);
            pc = pp.buf + s * stage;
            ac = pc + pp.mp;
        } else {
            pc = gc + (size_t)j * m;
            ac = ga + (size_t)j * m;
        }
        APPLY_LAP(4);  // stage wait
        const double dl = sd[j];
        const bool active = dl != 1.0;
        double part[C];
        if (active) {
            double vl[R], vh[R];
            tl.template make_v<!TMA, FULL>(ac, dl - 1.0, vl, vh);
            tl.partials(vl, vh, part);
            tl.publish(part);
        }
        tl.sync();  // B1: partials published; stage of use-1 fully consumed
        APPLY_LAP(5);  // partials + B1
        if (TMA && j > 0) {
            if (tl.t == 0) mbar_arrive_a(pp.empty_a + 8 * ((use - 1) % S));
            if (producer && j - 1 + S < cnt)
                pipe_issue(pp, use - 1 + S, gc + (size_t)(j - 1 + S) * m,
                           ga + (size_t)(j - 1 + S) * m, m);
        }
        double g[C];
        if (active) tl.template finish<true>(part, sden[j], sy[j], g);
        if (active) {
            APPLY_LAP(6);  // refill + reduction + B2
            double pl[R], ph[R];
            tl.template load_p<!TMA, FULL>(pc, pl, ph);
            tl.template axpy<FULL>(g, pl, ph);
            APPLY_LAP(7);  // axpy
        }
    }
    if (TMA) {
        tl.sync();
        if (tl.t == 0) mbar_arrive_a(pp.empty_a + 8 * ((k0 + cnt - 1) % S));
        pp.k = k0 + cnt;
    }
}

__device__ __forceinline__ void named_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// The first min(cnt, S) stages of pivots [l0, l0 + cnt) (producer thread).
template <int S>
__device__ __forceinline__ void apply_prologue(Pipe<S>& pp, const double* __restrict__ cols,
                                               const double* __restrict__ a, idx_t l0, int cnt,
                                               int m) {
    const int pre = cnt < S ? cnt : S;
    for (int i = 0; i < pre; ++i) pipe_issue(pp, pp.k + i, cols + (l0 + i) * m, a + (l0 + i) * m, m);
}

// issued: the caller's producer already ran apply_prologue for [l0, l1).
template <bool TMA, int S, int T, int R, int C, bool GEN>
__device__ __forceinline__ void apply_global(Tile<T, R, C, GEN>& tl, Pipe<S>& pp,
                                             const double* __restrict__ cols,
                                             const double* __restrict__ a, idx_t base, idx_t l0,
                                             idx_t l1, bool producer, bool issued = false) {
    const int cnt = (int)(l1 - l0);
    if (cnt <= 0) return;
    const int m = tl.m;
    if (TMA && producer && !issued) apply_prologue(pp, cols, a, l0, cnt, m);
    // warp-uniform choice of the select-free path (every row of every lane exists)
    if (!GEN && __all_sync(0xffffffffu, tl.full()))
        apply_impl<TMA, true>(tl, pp, cols, a, base, l0, cnt, producer);
    else
        apply_impl<TMA, false>(tl, pp, cols, a, base, l0, cnt, producer);
}

// ------------------------------------------------------------ warp-specialized update
// CTA = 2 compute warpgroups (256 threads: the register tile, T = 256) + 1
// reducer warpgroup (128 threads: cross-thread reductions, divisions, TMA
// producer, stage bookkeeping).  The tile's C columns are two halves A/B
// skewed by half a pivot, so the compute warps always have fp64 work while
// the reducer finishes the other half's serial chain:
//   compute C1(j): axpy B(j-1), partials B(j)        -> arrive PB
//   compute C2(j): axpy A(j),   partials A(j+1)      -> arrive PA
//   reducer R1(j): reduce A(j) -> gA, stage j+1 ready -> arrive GA
//   reducer R2(j): reduce B(j) -> gB                 -> arrive GB
// v_j and P_j are carried in registers between the two uses; stage j is
// recycled by the producer once PA(j+1) shows its last reader finished.
// Named barriers (384 threads): 1 = PA, 2 = PB, 3 = GA, 4 = GB.
constexpr int kWsT = 256;       // compute threads
// compute 224 / reducer 56 (c3 -0.9% vs 232 / 40: the reducer keeps its pivot scalars and
// addresses in registers; the compute tile still fits without spills)
constexpr int kWsRegsCompute = 224, kWsRegsReducer = 56;

// Diagnostic build only (make variant VDEFS=-DPDAS_WS_TRACE=1): clock64 marks
// of compute thread 0 / reducer thread 0 of one CTA per pivot, read back with
// pdas_debug_ws_trace (tools/ws_trace.py).
#ifndef PDAS_WS_TRACE
#define PDAS_WS_TRACE 0
#endif
#if PDAS_WS_TRACE
__device__ long long g_ws_trace[2][kMaxBlock][6];
#define WS_MARK(who, j, k)                                                                   \
    do {                                                                                     \
        if (gridDim.x >= 300 && blockIdx.x == 150 && (threadIdx.x == 0 || threadIdx.x == kWsT) && \
            (j) < kMaxBlock)                                                                 \
            g_ws_trace[who][j][k] = clock64();                                               \
    } while (0)
#else
#define WS_MARK(who, j, k) \
    do {                   \
    } while (0)
#endif

template <int S, int R, int C, bool FULL, int TC = kWsT>
__device__ __forceinline__ void ws_compute(Tile<TC, R, C, false>& tl, const double* buf, int mp,
                                           const double* sd, int cnt, double* redA, double* redB,
                                           const double* bcA, const double* bcB) {
    constexpr int HC = C / 2, NT = TC + 128;
    const int stage = 2 * mp;
    double vl[R], vh[R], pl[R], ph[R];
    auto sptr = [&](int j) -> const double* { return buf + (j % S) * stage; };
    auto act = [&](int j) { return sd[j] != 1.0; };
    auto partials = [&](int h0, double* red) {
#pragma unroll
        for (int c = 0; c < HC; ++c) {
            double s[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double lo = vl[r] * tl.xl[r][h0 + c];
                double hi = vh[r] * tl.xh[r][h0 + c];
                s[r] = lo + hi;
            }
            red[c * TC + tl.t] = lane_tree<R>(s);
        }
    };
    auto axpy = [&](int h0, const double* bc) {
        double g[HC];
#pragma unroll
        for (int c = 0; c < HC; ++c) g[c] = bc[c];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool hi = FULL || tl.vhi(r);
#pragma unroll
            for (int c = 0; c < HC; ++c) {
                double q0 = g[c] * pl[r];
                tl.xl[r][h0 + c] = tl.xl[r][h0 + c] - q0;
            }
            if (hi) {
#pragma unroll
                for (int c = 0; c < HC; ++c) {
                    double q1 = g[c] * ph[r];
                    tl.xh[r][h0 + c] = tl.xh[r][h0 + c] - q1;
                }
            }
        }
    };
    // GA(-1): stage 0 is ready
    named_bar(3, NT);
    bool a_prev = false, a_cur = act(0);
    if (a_cur) {
        tl.template make_v<false, FULL>(sptr(0) + mp, sd[0] - 1.0, vl, vh);
        partials(0, redA);
    }
    named_arrive(1, NT);
    // stage pointers of pivots j and j+1, advanced incrementally (no j % S)
    const double* const ring_end = buf + S * stage;
    const double* st_cur = buf;
    const double* st_nxt = S > 1 ? buf + stage : buf;
    for (int j = 0; j < cnt; ++j) {
        // d of pivot j+1, read before the barriers it would otherwise follow
        const double dn = sd[j + 1 < cnt ? j + 1 : j];
        const bool a_next = j + 1 < cnt && dn != 1.0;
        // ---- C1(j)
        WS_MARK(0, j, 0);
        if (j > 0) {
            named_bar(4, NT);
            WS_MARK(0, j, 1);
            if (a_prev) axpy(HC, bcB);
        }
        if (a_cur) partials(HC, redB);
        named_arrive(2, NT);
        WS_MARK(0, j, 2);
        // ---- C2(j)
        named_bar(3, NT);  // gA(j) ready, stage j+1 ready
        WS_MARK(0, j, 3);
        if (a_cur) {
            tl.template load_p<false, FULL>(st_cur, pl, ph);
            axpy(0, bcA);
        }
        if (a_next) {
            tl.template make_v<false, FULL>(st_nxt + mp, dn - 1.0, vl, vh);
            partials(0, redA);
        }
        named_arrive(1, NT);
        WS_MARK(0, j, 4);
        a_prev = a_cur;
        a_cur = a_next;
        st_cur = st_nxt;
        st_nxt = st_nxt + stage == ring_end ? buf : st_nxt + stage;
    }
    named_bar(4, NT);
    if (a_prev) axpy(HC, bcB);
}

// Direct-load variant: P_l and A[:,l] go L2 -> registers (ld.global.cg), one
// pivot ahead, instead of through a TMA ring in shared memory.  Shared-memory
// traffic per pivot drops from ~100 KB (TMA writes + stage reads +
// reductions) to the 32 KB of the reductions; the reducer warpgroup only
// reduces.  Same arithmetic, same order.
template <int R, int C, bool FULL, int TC = kWsT>
__device__ __forceinline__ void ws_compute_ldg(Tile<TC, R, C, false>& tl,
                                               const double* __restrict__ pcol,
                                               const double* __restrict__ acol, int m,
                                               const double* sd, int cnt, double* redA,
                                               double* redB, const double* bcA,
                                               const double* bcB) {
    constexpr int HC = C / 2, NT = TC + 128;
    double vl[R], vh[R], pl[R], ph[R];
    double npl[R], nph[R], nal[R], nah[R];  // P_{j+1}, raw A_{j+2} in flight
    // 32-bit shared addresses computed once and made opaque, so the loop
    // does not rebuild the shared window base (S2UR/ULEA) and the thread
    // index (S2R) for every reduction store and multiplier load
    const uint32_t sa_red[2] = {opaque_u32(smem_addr(redA + tl.t)),
                                opaque_u32(smem_addr(redB + tl.t))};
    const uint32_t sa_bc[2] = {opaque_u32(smem_addr(bcA)), opaque_u32(smem_addr(bcB))};
    auto partials = [&](int h0, double* red) {
#pragma unroll
        for (int c = 0; c < HC; ++c) {
            double s[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double lo = vl[r] * tl.xl[r][h0 + c];
                double hi = vh[r] * tl.xh[r][h0 + c];
                s[r] = lo + hi;
            }
            st_shared_f64(sa_red[h0 ? 1 : 0] + 8u * (uint32_t)(c * TC), lane_tree<R>(s));
        }
    };
    auto axpy = [&](int h0, const double* bc) {
        double g[HC];
        if constexpr (HC % 2 == 0) {
#pragma unroll
            for (int c = 0; c < HC; c += 2)
                ld_shared_v2_f64(sa_bc[h0 ? 1 : 0] + 8u * c, g[c], g[c + 1]);
        } else {
#pragma unroll
            for (int c = 0; c < HC; ++c) g[c] = bc[c];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool hi = FULL || tl.vhi(r);
#pragma unroll
            for (int c = 0; c < HC; ++c) {
                double q0 = g[c] * pl[r];
                tl.xl[r][h0 + c] = tl.xl[r][h0 + c] - q0;
            }
            if (hi) {
#pragma unroll
                for (int c = 0; c < HC; ++c) {
                    double q1 = g[c] * ph[r];
                    tl.xh[r][h0 + c] = tl.xh[r][h0 + c] - q1;
                }
            }
        }
    };
    auto scale = [&](double f) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            vl[r] = nal[r] * f;
            vh[r] = (FULL || tl.vhi(r)) ? nah[r] * f : 0.0;
        }
    };
    // loop-carried per-thread column pointers (this thread's first row folded
    // in): the loads need no per-pivot address rebuild (S2R/LDC chains the
    // compiler otherwise rematerialises under register pressure)
    const int H = tl.H;
    auto ldp = [&](const double* p, double (&lo)[R], double (&hi)[R]) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            lo[r] = __ldcg(p + TC * r);
            hi[r] = (FULL || tl.vhi(r)) ? __ldcg(p + H + TC * r) : 0.0;
        }
    };
    const double* pnext = pcol + m + tl.t;
    const double* anext = acol + 2 * (size_t)m + tl.t;
    // prologue: v_0, P_0 and A_1 in registers / in flight
    tl.template load_p<true, FULL>(acol, nal, nah);
    tl.template load_p<true, FULL>(pcol, npl, nph);
    bool a_prev = false, a_cur = sd[0] != 1.0;
    scale(sd[0] - 1.0);
    if (cnt > 1) tl.template load_p<true, FULL>(acol + m, nal, nah);
    if (a_cur) partials(0, redA);
    named_arrive(1, NT);
#pragma unroll 2
    for (int j = 0; j < cnt; ++j) {
        const double dn = sd[j + 1 < cnt ? j + 1 : j];
        const bool a_next = j + 1 < cnt && dn != 1.0;
        // ---- C1(j)
        WS_MARK(0, j, 0);
        if (j > 0) {
            named_bar(4, NT);
            WS_MARK(0, j, 1);
            if (a_prev) axpy(HC, bcB);
        }
        if (a_cur) partials(HC, redB);
        named_arrive(2, NT);
        WS_MARK(0, j, 2);
        // ---- C2(j)
        named_bar(3, NT);  // gA(j) ready
        WS_MARK(0, j, 3);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            pl[r] = npl[r];
            ph[r] = nph[r];
        }
        if (j + 1 < cnt) ldp(pnext, npl, nph);
        pnext += m;
        if (a_cur) axpy(0, bcA);
        scale(dn - 1.0);
        if (j + 2 < cnt) ldp(anext, nal, nah);
        anext += m;
        if (a_next) partials(0, redA);
        named_arrive(1, NT);
        WS_MARK(0, j, 4);
        a_prev = a_cur;
        a_cur = a_next;
    }
    named_bar(4, NT);
    if (a_prev) axpy(HC, bcB);
}

template <int R, int C, int TC = kWsT>
__device__ __forceinline__ void ws_reducer_ldg(const double* sd, const double* sden,
                                               const double* sy, int cnt, const double* redA,
                                               const double* redB, double* bcA, double* bcB) {
    constexpr int HC = C / 2, NT = TC + 128, NW = TC / 32;
    const int rt = threadIdx.x - TC;  // 0..127
    const int w = rt >> 5, lane = rt & 31;
    // a warp's columns (w, w+4, ...) as independent chains (HC = 8 at m <= 1024)
    auto reduce = [&](const double* red, double* bc, double denom, double y) {
        constexpr int PER = (HC + 3) / 4;
        double v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int c = w + 4 * k;
            if (c < HC) {
                double q[NW];
#pragma unroll
                for (int i = 0; i < NW; ++i) q[i] = red[c * TC + lane + 32 * i];
                v[k] = lane_tree<NW>(q);
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int c = w + 4 * k;
            if (c < HC) {
                const double u = warp_butterfly32(v[k]);
                const double g = u / denom;
                if (lane == 0) bc[c] = g;
            }
        }
    };
    if constexpr (HC <= 4 && !PDAS_WS_TRACE) {
        // one column per warp: its reduction rows, its multiplier slot and the
        // pivot scalars as pinned 32-bit shared addresses (no per-pivot
        // shared-window rebuild, as in ws_compute_ldg)
        const bool mine = w < HC;
        const uint32_t ra[2] = {opaque_u32(smem_addr(redA + w * TC + lane)),
                                opaque_u32(smem_addr(redB + w * TC + lane))};
        const uint32_t ba[2] = {opaque_u32(smem_addr(bcA + w)), opaque_u32(smem_addr(bcB + w))};
        const uint32_t sda = opaque_u32(smem_addr(sd)), sna = opaque_u32(smem_addr(sden));
        auto reduce1 = [&](int h, double denom) {
            if (mine) {
                double q[NW];
#pragma unroll
                for (int i = 0; i < NW; ++i) q[i] = ld_shared_f64(ra[h] + 256u * i);
                const double u = warp_butterfly32(lane_tree<NW>(q));
                const double g = u / denom;
                if (lane == 0) st_shared_f64(ba[h], g);
            }
        };
        bool act = ld_shared_f64(sda) != 1.0;
        double den = ld_shared_f64(sna);
        for (int j = 0; j < cnt; ++j) {
            const uint32_t jn = (uint32_t)(j + 1 < cnt ? j + 1 : j);
            const bool act_n = ld_shared_f64(sda + 8u * jn) != 1.0;
            const double den_n = ld_shared_f64(sna + 8u * jn);
            named_bar(1, NT);  // partials A(j) published
            if (act) reduce1(0, den);
            named_arrive(3, NT);
            named_bar(2, NT);  // partials B(j) published
            if (act) reduce1(1, den);
            named_arrive(4, NT);
            act = act_n;
            den = den_n;
        }
        named_bar(1, NT);  // the compute warps' final PA arrival
        return;
    }
    bool act = sd[0] != 1.0;
    double den = sden[0], y = sy[0];
    for (int j = 0; j < cnt; ++j) {
        const int jn = j + 1 < cnt ? j + 1 : j;
        const bool act_n = sd[jn] != 1.0;
        const double den_n = sden[jn], y_n = sy[jn];
        WS_MARK(1, j, 0);
        named_bar(1, NT);  // partials A(j) published
        WS_MARK(1, j, 1);
        if (act) reduce(redA, bcA, den, y);
        WS_MARK(1, j, 2);
        named_arrive(3, NT);
        WS_MARK(1, j, 3);
        named_bar(2, NT);  // partials B(j) published
        WS_MARK(1, j, 4);
        if (act) reduce(redB, bcB, den, y);
        named_arrive(4, NT);
        WS_MARK(1, j, 5);
        act = act_n;
        den = den_n;
        y = y_n;
    }
    named_bar(1, NT);  // the compute warps' final PA arrival
}

template <int S, int R, int C, int TC = kWsT>
__device__ __forceinline__ void ws_reducer(Pipe<S>& pp, const double* __restrict__ cols,
                                           const double* __restrict__ a, idx_t p0, int cnt, int m,
                                           const double* redA, const double* redB, double* bcA,
                                           double* bcB) {
    constexpr int HC = C / 2, NT = TC + 128, NW = TC / 32;
    constexpr bool kLateIssue = S >= 3;
    const int rt = threadIdx.x - TC;  // 0..127
    const int w = rt >> 5, lane = rt & 31;
    const bool producer = rt == 0;
    const double* sd = pp.sd;
    const double* sden = pp.sden;
    const double* sy = pp.sy;
    auto wait_stage = [&](int j) {
        if (producer) mbar_wait_a(pp.full_a + 8 * (j % S), (j / S) & 1u);
    };
    // a warp's columns (w, w+4, ...) as independent chains (HC = 8 at m <= 1024)
    auto reduce = [&](const double* red, double* bc, double denom, double y) {
        constexpr int PER = (HC + 3) / 4;
        double v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int c = w + 4 * k;
            if (c < HC) {
                double q[NW];
#pragma unroll
                for (int i = 0; i < NW; ++i) q[i] = red[c * TC + lane + 32 * i];
                v[k] = lane_tree<NW>(q);
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int c = w + 4 * k;
            if (c < HC) {
                const double u = warp_butterfly32(v[k]);
                const double g = u / denom;
                if (lane == 0) bc[c] = g;
            }
        }
    };
    // prologue: stages 0 .. S-1 in flight; release the compute warps once
    // stage 0 has landed (GA(-1))
    if (producer)
        for (int i = 0; i < (cnt < S ? cnt : S); ++i)
            pipe_issue(pp, i, cols + (p0 + i) * m, a + (p0 + i) * m, m, false);
    wait_stage(0);
    named_arrive(3, NT);
    uint32_t w_slot = 1u % S, w_par = (1u / S) & 1u;  // stage/parity of pivot j+1
    // pivot scalars are read one step ahead, off the barrier -> reduce chain
    bool act = sd[0] != 1.0;
    double den = sden[0], y = sy[0];
    for (int j = 0; j < cnt; ++j) {
        const int jn = j + 1 < cnt ? j + 1 : j;
        const bool act_n = sd[jn] != 1.0;
        const double den_n = sden[jn], y_n = sy[jn];
        // ---- R1(j)
        WS_MARK(1, j, 0);
        named_bar(1, NT);  // partials A(j) published (C2(j-1) done: stage j-1 free)
        WS_MARK(1, j, 1);
        // S = 2: stage j+1 is the one C2(j-1) just released -- refill it now,
        // before waiting on it below (the late refill would deadlock)
        if (!kLateIssue && j >= 1 && producer && j - 1 + S < cnt)
            pipe_issue(pp, j - 1 + S, cols + (p0 + j - 1 + S) * m, a + (p0 + j - 1 + S) * m, m,
                       false);
        if (act) reduce(redA, bcA, den, y);
        WS_MARK(1, j, 2);
        if (j + 1 < cnt && producer) mbar_wait_a(pp.full_a + 8 * w_slot, w_par);
        if (++w_slot == (uint32_t)S) {
            w_slot = 0;
            w_par ^= 1u;
        }
        named_arrive(3, NT);
        WS_MARK(1, j, 3);
        // refill the stage C2(j-1) released, after gA(j) is out
        if (kLateIssue && j >= 1 && producer && j - 1 + S < cnt)
            pipe_issue(pp, j - 1 + S, cols + (p0 + j - 1 + S) * m, a + (p0 + j - 1 + S) * m, m,
                       false);
        // ---- R2(j)
        named_bar(2, NT);  // partials B(j) published
        WS_MARK(1, j, 4);
        if (act) reduce(redB, bcB, den, y);
        named_arrive(4, NT);
        WS_MARK(1, j, 5);
        act = act_n;
        den = den_n;
        y = y_n;
    }
    named_bar(1, NT);  // the compute warps' final PA arrival
}

// pipe_issue without the empty-barrier protocol (single producer that knows
// from the named barriers when a stage is free): plain full-barrier refill.
// TC = 256: one CTA per SM (compute 232 / reducer 40 registers).  TC = 128
// (m <= 1024: the same 64-double tile per thread with twice the rows): two
// CTAs per SM, 256 threads each (compute 208 / reducer 48), so the SM
// interleaves two independent barrier/reduction pipelines.
template <int S, int R, int C, int TC = kWsT>
__global__ void __launch_bounds__(TC + 128, TC == 128 ? 2 : 1)
    k_casc_update_ws(double* __restrict__ cols, const double* __restrict__ a,
                     const double* __restrict__ d, const double* __restrict__ denoms, int m,
                     idx_t n, idx_t p0, idx_t p1, idx_t tile0, const int32_t* __restrict__ fail,
                     const int64_t* __restrict__ tiles, int* __restrict__ uflag, int utag,
                     int need, const int* __restrict__ pflag, int epoch) {
    static_assert(TC == 256 || TC == 128, "compute threads");
    constexpr bool kLdg = R <= 4;
    // TC = 128 direct-load: 224/32 (208/48 spilled ~170 B in the pivot loop;
    // c4 cascade 2103 -> 1929 ms, c5 32.4 -> 31.3 ms)
    constexpr int kRegC = TC == 256 ? kWsRegsCompute : (kLdg ? 224 : 216);
    constexpr int kRegR = TC == 256 ? kWsRegsReducer : (kLdg ? 32 : 40);
    double *red, *bc;
    Pipe<S> pp;
    carve<TC, C, 1, S>(red, bc, pp, false, m);
    if (!kLdg && threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(pp.full + s, 1);
        mbar_fence_init();
    }
    const idx_t tile = tiles ? tiles[blockIdx.x] : tile0 + blockIdx.x;
    update_deps(pflag, epoch, uflag, tile, need, fail);
    __syncthreads();
    // TC = 256 (168 registers at launch hold the 64-double tile): the compute
    // threads' tile loads go out first and the reducer warpgroup stages the
    // pivot scalars while they are in flight.  TC = 128 (128 at launch) loads
    // the tile after setmaxnreg.
    constexpr bool kEarly = TC == 256;
    Tile<TC, R, C, false> tl;
    const idx_t col0 = tile * C;
    if (kEarly && threadIdx.x < TC) {
        tl.init(threadIdx.x, m, 0, red, bc);
        tl.load(cols, col0, n + 1);
    } else if (kEarly) {
        for (idx_t l = p0 + (threadIdx.x - TC); l < p1; l += blockDim.x - TC) {
            pp.sd[l - p0] = __ldg(d + l);
            const double den = __ldcg(denoms + l);
            pp.sden[l - p0] = den;
            pp.sy[l - p0] = div_recip(den);
        }
    } else {
        stage_scalars(pp, d, denoms, p0, p0, p1, true);
    }
    // a breakdown found by a concurrent panel: one thread reads the fail word and
    // the whole CTA leaves together (before setmaxnreg and the barrier protocol)
    if (__syncthreads_or(threadIdx.x == 0 && *(volatile const int32_t*)fail != 0)) return;
    const int cnt = (int)(p1 - p0);
    constexpr int HC = C / 2;
    double* redA = red;
    double* redB = red + HC * TC;
    double* bcA = bc;
    double* bcB = bc + HC;
    if (threadIdx.x >= TC) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegR));
        if constexpr (kLdg)
            ws_reducer_ldg<R, C, TC>(pp.sd, pp.sden, pp.sy, cnt, redA, redB, bcA, bcB);
        else
            ws_reducer<S, R, C, TC>(pp, cols, a, p0, cnt, m, redA, redB, bcA, bcB);
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegC));
    if (!kEarly) {
        tl.init(threadIdx.x, m, 0, red, bc);
        tl.load(cols, col0, n + 1);
    }
    const bool full = __all_sync(0xffffffffu, tl.full());
    if constexpr (kLdg) {
        const double* pc = cols + p0 * m;
        const double* ac = a + p0 * m;
        if (full)
            ws_compute_ldg<R, C, true, TC>(tl, pc, ac, m, pp.sd, cnt, redA, redB, bcA, bcB);
        else
            ws_compute_ldg<R, C, false, TC>(tl, pc, ac, m, pp.sd, cnt, redA, redB, bcA, bcB);
    } else {
        if (full)
            ws_compute<S, R, C, true, TC>(tl, pp.buf, pp.mp, pp.sd, cnt, redA, redB, bcA, bcB);
        else
            ws_compute<S, R, C, false, TC>(tl, pp.buf, pp.mp, pp.sd, cnt, redA, redB, bcA, bcB);
    }
    tl.store(cols, col0, n + 1);
    if (uflag) {  // tile done: the next panel and the next update may take it
        // stores -> barrier -> one cumulative gpu-scope release (as the panel)
        named_bar(5, TC);
        if (threadIdx.x == 0) st_release(uflag + col0 / C, utag);
    }
}

// ------------------------------------------------------------ update kernel
// Tile (tile0 + blockIdx.x) of CT = G*C columns receives pivots [p0, p1);
// group g (T threads) owns columns [tile*CT + g*C, +C).
template <bool TMA, int S, int T, int R, int C, int G, bool GEN>
__global__ void __launch_bounds__(T* G, 1)
    k_casc_update(double* __restrict__ cols, const double* __restrict__ a,
                  const double* __restrict__ d, const double* __restrict__ denoms, int m, idx_t n,
                  idx_t p0, idx_t p1, idx_t tile0, const int32_t* __restrict__ fail,
                  const int64_t* __restrict__ tiles, int* __restrict__ uflag, int utag,
                  int need, const int* __restrict__ pflag, int epoch) {
    double *red, *bc;
    Pipe<S> pp;
    carve<T, C, G, S>(red, bc, pp, TMA, m);
    const idx_t tile = tiles ? tiles[blockIdx.x] : tile0 + blockIdx.x;
    update_deps(pflag, epoch, uflag, tile, need, fail);
    __syncthreads();
    stage_scalars(pp, d, denoms, p0, p0, p1, true);
    if (__syncthreads_or(threadIdx.x == 0 && *(volatile const int32_t*)fail != 0)) return;
    const int grp = threadIdx.x / T;
    Tile<T, R, C, GEN> tl;
    tl.init(threadIdx.x % T, m, 1 + grp, red + grp * C * T, bc + grp * C);
    const idx_t col0 = tile * (C * G) + grp * C;
    tl.load(cols, col0, n + 1);
    apply_global<TMA>(tl, pp, cols, a, p0, p0, p1, threadIdx.x == 0);
    tl.store(cols, col0, n + 1);
    if (uflag) {
        __syncthreads();
        if (threadIdx.x == 0) st_release(uflag + tile, utag);
    }
}

// ------------------------------------------------------------ panel triangle
// The panel's in-register triangle over its own pivot columns [col0, min(col0+C, p1)):
// for each pivot in order, the live columns' inner products, the breakdown
// test (first failing step -> *fail = l + 1), the denominator, and the
// rank-one update of the later columns.  pp.sd is indexed l - q0.  Returns
// true on breakdown (the tile must then not be stored).
template <bool TMA, int S, int T, int R, int C, bool GEN>
__device__ __forceinline__ bool panel_triangle(Tile<T, R, C, GEN>& tl, Pipe<S>& pp,
                                               const double* __restrict__ a,
                                               double* __restrict__ denoms, int m, idx_t col0,
                                               idx_t p1, idx_t q0, int32_t* __restrict__ fail,
                                               double* bc, bool producer,
                                               double* __restrict__ cols = nullptr, idx_t n = 0,
                                               int* __restrict__ cflags = nullptr, int epoch = 0,
                                               bool trace = false, int* s_pub = nullptr) {
    (void)trace;
#if PDAS_HOP_TRACE
    long long tq = clock64();
#define TRI_LAP(k)                                         \
    do {                                                   \
        if (trace && threadIdx.x == 0) {                   \
            const long long tn = clock64();                \
            g_hop_trace[8 + (k)] += (unsigned long long)(tn - tq); \
            tq = tn;                                       \
        }                                                  \
    } while (0)
#else
#define TRI_LAP(k) \
    do {           \
    } while (0)
#endif
    // triangle over this tile's own pivot columns, A columns via the pipe
    const int cnt = (int)((col0 + C < p1 ? col0 + C : p1) - col0);
    const unsigned k0 = pp.k;
    if (TMA && producer) {
        const int pre = cnt < S ? cnt : S;
        for (int i = 0; i < pre; ++i) pipe_issue(pp, k0 + i, nullptr, a + (col0 + i) * m, m);
    }
    bool broken = false;
#pragma unroll
    for (int cl = 0; cl < C; ++cl) {
        if (cl < cnt) {
            const idx_t l = col0 + cl;
            const unsigned use = k0 + cl;
            const double* ac = a + l * m;
            TRI_LAP(5);  // chunk publication / loop overhead
            if (TMA) {
                const int s = (int)(use % S);
                mbar_wait(pp.full + s, (use / S) & 1u);
                ac = pp.buf + (size_t)s * 2 * pp.mp + pp.mp;
            }
            TRI_LAP(0);  // stage wait
            const double dl = pp.sd[l - q0];
            const bool active = dl != 1.0 && !broken;
            double part[C];
            if (active) {
                double vl[R], vh[R];
                tl.template make_v<!TMA, false>(ac, dl - 1.0, vl, vh);
                tl.partials(vl, vh, part, cl);  // columns < cl are final
                tl.publish(part, cl);
            }
            tl.sync();
            TRI_LAP(1);  // make_v + partials + B1
            if (TMA && cl > 0) {
                if (producer) mbar_arrive(pp.empty + (int)((use - 1) % S));
                if (producer && cl - 1 + S < cnt)
                    pipe_issue(pp, use - 1 + S, nullptr, a + (l - 1 + S) * m, m);
            }
            if (active) {
                double inner[C];
                tl.template finish<false>(part, 0.0, 0.0, inner, cl);
                TRI_LAP(2);  // reduction + B2
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
                    // T > 32: one thread per live column divides, all read the
                    // quotients back (instead of every thread dividing them all)
                    if (T > 32 && cl + 1 < C) {
                        if (threadIdx.x > cl && threadIdx.x < C) bc[C + threadIdx.x] = bc[threadIdx.x] / denom;
                        tl.sync();
                    }
                    TRI_LAP(3);  // denominator, divisions, B3
#pragma unroll
                    for (int c = cl + 1; c < C; ++c) {
                        const double g = T > 32 ? bc[C + c]
                                         : inner[c] / denom;
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
            TRI_LAP(4);  // axpy of the later columns
            // end of a chunk: its columns are final -- store and publish them so
            // the next tile's CTA starts on them while this triangle goes on
            constexpr int CH = C / kPanelChunks > 0 ? C / kPanelChunks : 1;
            if (s_pub && cflags && (cl + 1) % CH == 0 && cl + 1 < C && cl + 1 < cnt) {
                // publisher warp: the compute threads store and arrive (no wait);
                // the publisher warp's barrier.sync orders their stores before its
                // cumulative release, so no compute thread ever waits on a fence
                if (!broken) tl.store(cols, col0, n + 1, cl + 1 - CH, cl + 1);
                if (producer) *s_pub = broken ? 0 : 1;
                named_arrive(2, T + 32);
            } else if (cflags && (cl + 1) % CH == 0 && cl + 1 < C && cl + 1 < cnt && !broken) {
                // stores -> CTA barrier -> one gpu-scope release by the producer:
                // the barrier orders every thread's stores before the release,
                // which is cumulative (the cooperative-groups grid-sync pattern)
                // (deferring the release by one step: c3 unchanged, 164.2 ms)
                tl.store(cols, col0, n + 1, cl + 1 - CH, cl + 1);
                tl.sync();
                if (producer) st_release(cflags + (cl + 1) / CH - 1, epoch);
            }
        }
    }
    if (TMA) {
        tl.sync();
        if (producer) mbar_arrive(pp.empty + (int)((k0 + cnt - 1) % S));
        pp.k = k0 + cnt;
    }
    return broken;
}

// ------------------------------------------------------------ panel kernel
// One CTA per tile of block [p0, p1): apply the previous block [q0, p0),
// then the pivots of this block's earlier tiles as their CTAs publish them
// (flags[tile] == epoch), then the in-register triangle; publish.  Breakdown
// is detected here, in step order, and reported as the 1-based step.
// PW = 32: one extra publisher warp that issues the mid-triangle chunk
// releases (fence + flag) so the compute threads never stall on them
// (~3.7 us per publication at c2, profiles/r02_hop_trace.txt).
template <bool TMA, int S, int T, int R, int C, bool GEN, int PW = 0>
__global__ void __launch_bounds__(T + PW, 1)
    k_casc_panel(double* __restrict__ cols, const double* __restrict__ a,
                 const double* __restrict__ d, double* __restrict__ denoms, int m, idx_t n,
                 idx_t q0, idx_t p0, idx_t p1, int32_t* __restrict__ fail, int* __restrict__ flags,
                 int epoch, const int* __restrict__ uflag, int utag, const PeerSet peers) {
    // tiles of the block: CTA j takes j, j + G, ... (G = gridDim.x < tiles when
    // the host gives a CTA two tiles: the second one's catch-up fits in the
    // chain's slack, and the panel holds half the SMs)
    const idx_t tile_beg = p0 / C, tile_end = (p1 + C - 1) / C;
    // a tile's final columns are published in NCH chunks of CH (flags[tile*NCH + ch])
    constexpr int CH = C / kPanelChunks > 0 ? C / kPanelChunks : 1;
    constexpr int NCH = C / CH;
    // block-uniform: thread 0 reads the fail word for the whole CTA
    if (__syncthreads_or(threadIdx.x == 0 && *(volatile int32_t*)fail != 0)) {
        // still publish: later tiles may be waiting
        if (threadIdx.x == 0)
            for (idx_t tile = tile_beg + blockIdx.x; tile < tile_end; tile += gridDim.x) {
                for (int ch = 0; ch < NCH; ++ch) st_release(flags + tile * NCH + ch, epoch);
                peer_signal(peers, fail, flags, tile * NCH + NCH - 1, epoch);
            }
        return;
    }
    double *red, *bc;
    Pipe<S> pp;
    carve<T, C, 1, S>(red, bc, pp, TMA, m);
    // d for [q0, p1) and the previous block's denominators, window base q0
    stage_scalars(pp, d, denoms, q0, q0, p0, true);
    for (idx_t l = p0 + threadIdx.x; l < p1; l += blockDim.x) pp.sd[l - q0] = __ldg(d + l);
    __syncthreads();
    const bool pubw = PW > 0 && (int)threadIdx.x >= T;  // the publisher warp
    __shared__ int s_pub;
    for (idx_t tile = tile_beg + blockIdx.x; tile < tile_end; tile += gridDim.x) {
    Tile<T, R, C, GEN> tl;
    tl.init(pubw ? 0 : (int)threadIdx.x, m, 1, red, bc);
    const bool producer = threadIdx.x == 0;
    const idx_t col0 = tile * C;
    bool dead = false;
    const bool hop_pub = gridDim.x == 32 && blockIdx.x == 15 && p0 == 5 * (p1 - p0);
    const bool hop_con = gridDim.x == 32 && blockIdx.x == 16 && p0 == 5 * (p1 - p0);
    (void)hop_pub;
    (void)hop_con;
    if (uflag) {
        // this tile's last update (the update kernel of the previous block,
        // running concurrently) must have landed before the tile is read
        if (producer)
            while (ld_acquire(uflag + tile) != utag) {
                if (*(volatile int32_t*)fail) break;
                __nanosleep(64);
            }
        dead = __syncthreads_or(producer && *(volatile int32_t*)fail != 0);
    }
    if (!dead && !pubw) {
        tl.load(cols, col0, n + 1);
        apply_global<TMA>(tl, pp, cols, a, q0, q0, p0, producer);
    }
#if PDAS_PANEL_TRACE
    // last CTA of a full panel: cycles spent waiting for predecessors (flag
    // acquire) vs applying their pivots vs the triangle
    const bool trace = PDAS_PANEL_TRACE && gridDim.x == 32 && blockIdx.x == 31 && threadIdx.x == 0;
    long long t_wait = 0, t_apply = 0, t_mark = clock64();
#define PANEL_LAP(acc)                      \
    do {                                    \
        const long long t_now = clock64(); \
        acc += t_now - t_mark;              \
        t_mark = t_now;                     \
    } while (0)
#else
#define PANEL_LAP(acc) \
    do {               \
    } while (0)
#endif
    for (idx_t tp = p0 / C; tp < tile && !dead; ++tp) {
        // the previous tile chunk by chunk (its triangle is still running);
        // older tiles are complete: one wait on their last chunk
        const bool prev = tp == tile - 1;
        for (int ch = prev ? 0 : NCH - 1; ch < NCH; ++ch) {
            const idx_t pa = tp * C + (prev ? ch * CH : 0);
            const idx_t pe = tp * C + (ch + 1) * CH;
            const idx_t pb = pe < p1 ? pe : p1;
            int f = 0;
            if (producer) {
                while (ld_acquire(flags + tp * NCH + ch) != epoch) __nanosleep(32);
                f = *(volatile int32_t*)fail;
                if (TMA && !f && pa < pb) {
                    // the chunk's bulk copies go out first, so their L2 round trip
                    // overlaps the denominators' loads below
                    fence_proxy_async_global();  // peer CTA's generic stores -> our TMA reads
                    apply_prologue(pp, cols, a, pa, (int)(pb - pa), m);
                }
            }
            // the flag's acquire and the fail word are read by one thread; the
            // barrier hands both to the CTA (block-uniform exit)
            const bool hop_here = hop_con && prev && ch == NCH - 1;
            (void)hop_here;
            HOP_MARK(hop_here, 3);
            const int broken = __syncthreads_or(f != 0);
            PANEL_LAP(t_wait);
            if (broken) {
                dead = true;
                break;
            }
            if (pa >= pb) continue;
            if (threadIdx.x < pb - pa) {
                const double den = __ldcg(denoms + pa + threadIdx.x);
                pp.sden[pa + threadIdx.x - q0] = den;
                pp.sy[pa + threadIdx.x - q0] = div_recip(den);
            }
            __syncthreads();
            HOP_MARK(hop_here, 4);
            if (!pubw) apply_global<TMA>(tl, pp, cols, a, q0, pa, pb, producer, true);
            HOP_MARK(hop_here, 5);
            PANEL_LAP(t_apply);
        }
    }
    bool stored = false;
    HOP_MARK(hop_con, 6);
    if (!dead && pubw) {
        // the publisher warp: one barrier per mid-triangle publication point
        int* cf = NCH > 1 ? flags + tile * NCH : nullptr;
        const int cnt = (int)((col0 + C < p1 ? col0 + C : p1) - col0);
        constexpr int CHP = C / kPanelChunks > 0 ? C / kPanelChunks : 1;
        for (int cl = 0; cl < C; ++cl) {
            if (cl < cnt && cf && (cl + 1) % CHP == 0 && cl + 1 < C && cl + 1 < cnt) {
                named_bar(2, T + 32);
                if ((threadIdx.x & 31) == 0 && s_pub) {
                    __threadfence();
                    st_relaxed(cf + (cl + 1) / CHP - 1, epoch);
                }
            }
        }
    } else if (!dead) {
        const bool broken = panel_triangle<TMA, S, T, R, C, GEN>(
            tl, pp, a, denoms, m, col0, p1, q0, fail, bc, producer, cols, n,
            NCH > 1 ? flags + tile * NCH : nullptr, epoch, hop_con, PW > 0 ? &s_pub : nullptr);
        HOP_MARK(hop_pub, 0);
        if (!broken) {
            // the earlier chunks went out mid-triangle (a chunk goes out iff it
            // ends before the tile's last pivot): store only the rest
            const int cnt = (int)((col0 + C < p1 ? col0 + C : p1) - col0);
            const int first = NCH > 1 ? (cnt - 1) / CH * CH : 0;
            tl.store(cols, col0, n + 1, first, C);
            stored = true;
        }
#if PDAS_PANEL_TRACE
        if (trace) {
            long long t_tri = 0;
            PANEL_LAP(t_tri);
            g_panel_trace[0] = t_wait;
            g_panel_trace[1] = t_apply;
            g_panel_trace[2] = t_tri;
            g_panel_trace[3] = (long long)(tile - p0 / C) * C;  // apply steps
            g_panel_trace[4] = C;                                 // triangle steps
        }
#endif
    }
    __syncthreads();
    HOP_MARK(hop_pub, 1);
    if (peers.count > 0) {
        // multi-GPU exchange fused into the panel: the tile's final columns go
        // from registers straight into every peer's [Y|x] over NVLink, with
        // their denominators; then one system-scope flag per peer and tile
        if (stored && !pubw) {
            for (int q = 0; q < peers.count; ++q) tl.store(peers.cols[q], col0, n + 1);
            if (threadIdx.x < C && col0 + threadIdx.x < p1) {
                const double den = __ldcg(denoms + col0 + threadIdx.x);
                for (int q = 0; q < peers.count; ++q) peers.denoms[q][col0 + threadIdx.x] = den;
            }
        }
        __threadfence_system();
        __syncthreads();
        if (producer) peer_signal(peers, fail, flags, tile * NCH + NCH - 1, epoch);
    }
    if (producer) {
        // one gpu-scope fence after the CTA barrier covers every thread's stores
        // (cumulative release); the chunk flags then go out as relaxed stores
        __threadfence();
        for (int ch = 0; ch < NCH; ++ch) st_relaxed(flags + tile * NCH + ch, epoch);
    }
    HOP_MARK(hop_pub, 2);
    __syncthreads();  // shared reduction rows and scalars reused by the next tile
    }
}

// ------------------------------------------------------------ warp-per-column panel
// The panel as a latency chain of 8-column tiles (c2, c4, c5: 64 <= H <= 512;
// one pivot block, nothing of the previous block left to apply).  Each of the
// tile's columns lives in ONE warp (Tile<32, H/32, 1>: rows lane + 32 r and
// + H, the same reference tree: in-lane levels, then the 32-lane butterfly),
// so a pivot step needs no CTA barrier: each warp reduces, divides and updates
// its own column as soon as the pivot's [P | A] stage has landed.  A ninth
// warp is the producer: it acquires the earlier tiles' chunk flags, stages
// their denominators and streams [P_l | A_l] (A_l alone for the tile's own
// pivots) through an S-stage bulk-copy ring (full: producer arrive + bytes,
// empty: one arrival per column warp).  Triangle step cl: warp cl writes its
// final column into the stage's P half, reduces its own denominator and
// releases tri[cl]; warps c > cl reduce their columns meanwhile and apply the
// step after tri[cl].  A chunk of columns that ends before the tile's last
// pivot is published by the last of its warps to finish (shared-memory count,
// one gpu-scope fence), the rest at the end.  Breakdown and a failed earlier
// tile keep the stage protocol going
// with the arithmetic skipped, so no warp waits on a stage that never comes.
constexpr int kPwCols = 8;                        // columns per tile (CT)
// + a producer warpgroup (one active warp): 168 registers at launch, column
// warps 200, producer warpgroup 88 (40 spilled its flag/denominator loop)
constexpr int kPwThreads = 32 * kPwCols + 128;
// its final columns go out in kPwChunks chunks of two (flags[tile * kPwChunks +
// ch]): a column warp that has finished its own step has nothing left but stage
// bookkeeping, so finer publication costs the working warps nothing (2 chunks:
// c2 10.5 ms, 4: 9.8, 8: 10.9 -- a flag per pivot is more consumer overhead)
constexpr int kPwChunks = 4;
static_assert(kPwCols % kPwChunks == 0, "chunks");

__host__ __device__ inline size_t panel_w_smem(int S, int m) {
    const size_t mp = (size_t)((m + 1) & ~1);
    return (size_t)S * 2 * mp * 8 + 6 * (size_t)kMaxBlock * 8 + kPwCols * 8 + kPwCols * 4 +
           (2 * (size_t)S + kPwCols) * 8 + 4 * (1 + kPwChunks) + 16;
}

template <int R, int S, bool FULL>
__global__ void __launch_bounds__(kPwThreads, 1)
    k_casc_panel_w(double* __restrict__ cols, const double* __restrict__ a,
                   const double* __restrict__ d, double* __restrict__ denoms, int m, idx_t n,
                   idx_t p0, idx_t p1, int32_t* __restrict__ fail, int* __restrict__ flags,
                   int epoch, const int* __restrict__ uflag, int utag) {
    constexpr int C = kPwCols, NCH = kPwChunks, CH = C / NCH;
    const idx_t tile = p0 / C + blockIdx.x;
    if (__syncthreads_or(threadIdx.x == 0 && *(volatile int32_t*)fail != 0)) {
        if (threadIdx.x == 0)
            for (int ch = 0; ch < NCH; ++ch) st_release(flags + tile * NCH + ch, epoch);
        return;
    }
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int mp = (m + 1) & ~1;
    double* buf = reinterpret_cast<double*>(smem_raw);  // S x [P | A]
    double* sd = buf + (size_t)S * 2 * mp;               // d, window base p0
    double* sden = sd + 2 * kMaxBlock;                   // earlier tiles' denominators
    double* sy = sden + 2 * kMaxBlock;                   // and their div_recip
    double* stden = sy + 2 * kMaxBlock;                  // this tile's denominators
    int* stbrk = reinterpret_cast<int*>(stden + C);      // step cl broke down
    uint64_t* full = reinterpret_cast<uint64_t*>(stbrk + C);
    uint64_t* empty = full + S;
    uint64_t* tri = empty + S;
    int* s_state = reinterpret_cast<int*>(tri + C);      // [0] dead, [1 + ch] chunk counts
    const uint32_t full_a = smem_addr(full), empty_a = smem_addr(empty), tri_a = smem_addr(tri);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, C);
        }
        for (int k = 0; k < C; ++k) mbar_init(tri + k, 1);
        for (int k = 0; k <= NCH; ++k) s_state[k] = 0;
        mbar_fence_init();
    }
    for (idx_t l = p0 + threadIdx.x; l < p1; l += blockDim.x) sd[l - p0] = __ldg(d + l);
    // this tile's last update (the previous block's update kernel, running
    // concurrently) must have landed before the tile is read
    if (uflag && threadIdx.x == 0)
        while (ld_acquire(uflag + tile) != utag) {
            if (*(volatile int32_t*)fail) break;
            __nanosleep(64);
        }
    const bool dead0 =
        __syncthreads_or(uflag != nullptr && threadIdx.x == 0 && *(volatile int32_t*)fail != 0);
    const idx_t col0 = tile * C;
    const int cnt = (int)((col0 + C < p1 ? col0 + C : p1) - col0);
    const idx_t ncols = n + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bytes = (uint32_t)m * 8u;
    const bool hop_pub = gridDim.x == 32 && blockIdx.x == 15 && p0 == 5 * (p1 - p0);
    const bool hop_con = gridDim.x == 32 && blockIdx.x == 16 && p0 == 5 * (p1 - p0);
    (void)hop_pub;
    (void)hop_con;
    if (warp >= C) {
        // ---- producer warpgroup (one lane works)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
        if (warp == C && !dead0) {
            unsigned use = 0;
            bool dead = false;
            auto issue = [&](idx_t l, bool with_p) {  // lane 0
                const uint32_t sl = use % S;
                if (use >= (unsigned)S) mbar_wait_a(empty_a + 8 * sl, ((use / S) - 1u) & 1u);
                const uint32_t fb = full_a + 8 * sl;
                if (dead) {
                    mbar_arrive_a(fb);  // drain: the column warps skip the step
                } else {
                    double* dst = buf + (size_t)sl * 2 * mp;
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                                 "r"(with_p ? 2 * bytes : bytes)
                                 : "memory");
                    if (with_p) tma_load_1d(dst, cols + l * m, bytes, full + sl);
                    tma_load_1d(dst + mp, a + l * m, bytes, full + sl);
                }
                ++use;
            };
            for (idx_t tp = p0 / C; tp < tile; ++tp) {
                // the previous tile chunk by chunk (its triangle may still run);
                // older tiles are complete: one wait on their last chunk
                const bool prev = tp == tile - 1;
                for (int ch = prev ? 0 : NCH - 1; ch < NCH; ++ch) {
                    const idx_t pa = tp * C + (prev ? ch * CH : 0);
                    const idx_t pe = tp * C + (ch + 1) * CH;
                    const idx_t pb = pe < p1 ? pe : p1;
                    if (!dead) {
                        int f = 0;
                        if (lane == 0) {
                            while (ld_acquire(flags + tp * NCH + ch) != epoch) __nanosleep(32);
                            PW_MARK(hop_con && prev && ch == NCH - 1, 2);
                            f = *(volatile int32_t*)fail;
                            if (f) *(volatile int*)s_state = 1;
                            else fence_proxy_async_global();  // their stores -> our bulk reads
                        }
                        dead = __shfl_sync(0xffffffffu, f, 0) != 0;
                        // the chunk's denominators, one lane per pivot (after the
                        // flag: __syncwarp orders lane 0's acquire before the loads)
                        __syncwarp();
                        if (!dead)
                            for (idx_t l = pa + lane; l < pb; l += 32) {
                                const double den = __ldcg(denoms + l);
                                sden[l - p0] = den;
                                sy[l - p0] = div_recip(den);
                            }
                        __syncwarp();
                        PW_MARK(hop_con && prev && ch == NCH - 1 && lane == 0, 3);
                    }
                    if (lane == 0)
                        for (idx_t l = pa; l < pb; ++l)
                            if (sd[l - p0] != 1.0) issue(l, true);  // _kernels.pyx:242-243
                    __syncwarp();
                }
            }
            if (lane == 0)
                for (int cl = 0; cl < cnt; ++cl)
                    if (sd[col0 + cl - p0] != 1.0) issue(col0 + cl, false);
        }
    } else {
        // ---- column warp: column col0 + warp of the tile
        asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
        const idx_t col = col0 + warp;
        const bool have = col < ncols;
        Tile<32, R, 1, false> tl;
        tl.init(lane, m, 0, nullptr, nullptr);
        const int H = tl.H;
        if (have && !dead0) tl.load(cols, col, ncols);
        // inner product of v = A_l (d_l - 1) with this column (reference tree)
        auto dot = [&](const double* ac, double f) {
            const double t = stream_tree<R>([&](int r) {
                const int row = lane + 32 * r;
                const double vl = ac[row] * f;
                const double lo = vl * tl.xl[r][0];
                const double vh = (FULL || tl.vhi(r)) ? ac[row + H] * f : 0.0;
                const double hi = vh * tl.xh[r][0];
                return lo + hi;
            });
            return warp_butterfly32(t);
        };
        auto axpy = [&](double g, const double* pc) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int row = lane + 32 * r;
                const double q0 = g * pc[row];
                tl.xl[r][0] = tl.xl[r][0] - q0;
                if (FULL || tl.vhi(r)) {
                    const double q1 = g * pc[row + H];
                    tl.xh[r][0] = tl.xh[r][0] - q1;
                }
            }
        };
        unsigned use = 0;
        bool dead = dead0, broken = false, stored = false;
#if PDAS_HOP_TRACE
        const bool acc = hop_con && lane == 0 && (warp == 0 || warp == C - 1);
        const int ab = warp == 0 ? 16 : 24;
        long long tw = clock64();
#define PW_ACC(k)                                             \
    do {                                                      \
        if (acc) {                                            \
            const long long tn = clock64();                   \
            g_hop_trace[ab + (k)] += (unsigned long long)(tn - tw); \
            tw = tn;                                          \
        }                                                     \
    } while (0)
#else
#define PW_ACC(k) \
    do {          \
    } while (0)
#endif
        auto wait_stage = [&](uint32_t& sl) {
            sl = use % S;
            PW_ACC(0);  // work since the last mark
            mbar_wait_a(full_a + 8 * sl, (use / S) & 1u);
            PW_ACC(1);  // stage wait
            if (!dead) dead = *(volatile int*)s_state != 0;
        };
        auto release_stage = [&](uint32_t sl) {
            __syncwarp();
            if (lane == 0) mbar_arrive_a(empty_a + 8 * sl);
            ++use;
        };
        if (!dead0) {
            // earlier tiles' pivots, ascending
            for (idx_t l = p0; l < col0; ++l) {
                const double dl = sd[l - p0];
                if (dl == 1.0) continue;
                uint32_t sl;
                wait_stage(sl);
                PW_MARK(hop_con && warp == 0 && lane == 0 && l == col0 - CH, 9);
                if (!dead && have) {
                    const double* pc = buf + (size_t)sl * 2 * mp;
                    const double inner = dot(pc + mp, dl - 1.0);
                    const double g = div_by(inner, sden[l - p0], sy[l - p0]);
                    axpy(g, pc);
                }
                release_stage(sl);
            }
            PW_ACC(0);
#if PDAS_HOP_TRACE
            if (acc) g_hop_trace[ab + 3] += (unsigned long long)(col0 - p0);  // apply steps
#endif
            PW_MARK(hop_con && warp == 0 && lane == 0, 4);
            // the triangle over the tile's own pivots
            const int wch = warp / CH;  // this column's chunk, out before the triangle
            const bool mid = (wch + 1) * CH < cnt;  // ends iff it ends before the last pivot
            for (int cl = 0; cl < cnt; ++cl) {
                const idx_t l = col0 + cl;
                const double dl = sd[l - p0];
                if (dl != 1.0) {  // _kernels.pyx:242-243
                uint32_t sl;
                wait_stage(sl);
                double* pc = buf + (size_t)sl * 2 * mp;
                const bool live = !dead && !broken;
                if (warp == cl) {
                    int brk = broken ? 1 : 0;
                    if (live) {
#pragma unroll
                        for (int r = 0; r < R; ++r) {  // P_l for the later columns
                            pc[lane + 32 * r] = tl.xl[r][0];
                            if (FULL || tl.vhi(r)) pc[lane + 32 * r + H] = tl.xh[r][0];
                        }
                        const double inner = dot(pc + mp, dl - 1.0);
                        const double denom = 1.0 + inner;
                        if (fabs(denom) <= kDenomEpsRel * (1.0 + fabs(inner))) {
                            brk = 1;
                            broken = true;
                            if (lane == 0) *fail = (int32_t)(l + 1);
                        } else if (lane == 0) {
                            denoms[l] = denom;
                            stden[cl] = denom;
                        }
                    }
                    if (lane == 0) stbrk[cl] = brk;
                    __syncwarp();
                    if (lane == 0) mbar_arrive_a(tri_a + 8 * cl);
                    PW_MARK(hop_con && lane == 0 && (cl == 0 || cl == C - 1), cl == 0 ? 5 : 7);
                } else if (warp > cl) {
                    double inner = 0.0;
                    if (live && have) inner = dot(pc + mp, dl - 1.0);
                    PW_ACC(0);
                    mbar_wait_a(tri_a + 8 * cl, 0);
                    PW_ACC(2);  // triangle hand-off wait
                    if (stbrk[cl]) broken = true;
                    if (!dead && !broken && have) axpy(inner / stden[cl], pc);
                }
                release_stage(sl);
                }
                if (cl == warp && mid && !dead && !broken) {
                    // column and denominator final: store the column; the last
                    // of the chunk's warps releases the chunk flag (shared
                    // count, then one cumulative gpu-scope fence)
                    tl.store(cols, col, ncols);
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence_block();
                        if (atomicAdd(s_state + 1 + wch, 1) == CH - 1) {
                            __threadfence();
                            st_relaxed(flags + tile * NCH + wch, epoch);
                            PW_MARK(hop_con && wch == 0, 6);
                        }
                    }
                    stored = true;
                }
            }
            PW_ACC(0);
            if (!stored && !dead && !broken && have) tl.store(cols, col, ncols);
        }
    }
    // the remaining columns are stored: one gpu-scope fence after the CTA
    // barrier covers every warp's stores (cumulative), then the chunk flags
    __syncthreads();
    PW_MARK(threadIdx.x == 0 && (hop_pub || hop_con), hop_pub ? 0 : 8);
    if (threadIdx.x == 0) {
        __threadfence();
        for (int ch = 0; ch < NCH; ++ch) st_relaxed(flags + tile * NCH + ch, epoch);
    }
    PW_MARK(threadIdx.x == 0 && hop_pub, 1);
}

// Non-owner side of the fused exchange: wait until every tile of columns
// [c0, c1) has been signalled by its owner's panel for this epoch.  Bounded:
// a peer that never signals traps after 30 s instead of hanging the device.
__global__ void k_peer_wait(const int* __restrict__ flags, idx_t t0, idx_t t1, int nch, int epoch) {
    for (idx_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        const int* f = flags + t * nch + nch - 1;
        const unsigned long long start = global_ns();
        while (ld_acquire_sys(f) != epoch) {
            __nanosleep(64);
            if (global_ns() - start > 30000000000ull) __trap();
        }
    }
}

// ------------------------------------------------------------ small cascade
// m <= 64 (H <= 32) with [Y | x] and A both resident in one SM's shared
// memory (c1: 80 KB + 80 KB): the whole cascade in ONE CTA, step by step,
// no panels, no flags, no global memory between steps.  A column's tree
// lives in a group of LPC lanes: lane j of the group owns s-indices
// j + LPC r (r < RPL = H / LPC), i.e. rows j + LPC r and j + LPC r + H, so the
// levels h >= LPC are in-lane register adds and the last log2(LPC) are xor
// shuffles inside the group -- a warp reduces 32 / LPC columns with the same
// shuffles.  Step l: warp 0 finds denom_l from the pivot column while every
// group reduces its columns k > l; barrier; each group divides (all of its
// lanes: same bits) and updates its column; barrier (column l+1 is final).
// Computing inner_k then updating column k per column equals the reference's
// phase 1 / phase 2 split (_kernels.pyx:247-266): the pivot column is not
// written in step l.
// 512 threads: 64 column groups, ~1.6 passes per step at c1 (256: 0.37 ms per
// c1 cascade, 512: 0.32, 1024: 0.50 -- 64 registers spill the tile)
constexpr int kSmallThreads = 512;
constexpr int KB = 1;  // columns per group and pass (k_casc_small; 2 and 4 measured slower)

// shared-memory column stride: m rounded up to 8 (mod 16) doubles, so the four
// 8-lane groups of a warp (consecutive columns) fall into two bank halves
__host__ __device__ inline idx_t small_stride(idx_t m) { return (m + 7) / 16 * 16 + 8; }

__host__ __device__ inline size_t small_cascade_smem(idx_t m, idx_t n) {
    const idx_t mp = small_stride(m);
    return (size_t)((n + 1) * mp + n * mp + n + mp) * sizeof(double);  // + x0 scratch
}

// x0 = L^-T L^-1 rhs for column x of [Y | x] in shared memory, by one warp
// (m <= 64: rows lane and lane + 32), with exactly the operations of
// k_fwd_one / k_bwd_one (solve_kernels.cu): forward column sweeps
// x_j /= L_jj, x_i -= L_ij x_j; backward rows s = y_r - L_{r+1,r} x_{r+1}
// - L_{r+2,r} x_{r+2} - ... in ascending order, x_r = s / L_rr.  q: m doubles.
__device__ __forceinline__ void small_x0_warp(const double* __restrict__ L, int m, double* x,
                                              double* q) {
    const int lane = threadIdx.x & 31;
    double xr[2];
    for (int k = 0; k < 2; ++k) xr[k] = lane + 32 * k < m ? x[lane + 32 * k] : 0.0;
    for (int j = 0; j < m; ++j) {
        const int owner = j & 31, slot = j >> 5;
        double l[2];
        for (int k = 0; k < 2; ++k) {
            const int i = lane + 32 * k;
            l[k] = i < m ? __ldg(L + (size_t)j * m + i) : 0.0;
        }
        if (lane == owner) xr[slot] = xr[slot] / l[slot];
        const double xj = __shfl_sync(0xffffffffu, xr[slot], owner);
        for (int k = 0; k < 2; ++k) {
            const int i = lane + 32 * k;
            if (i > j && i < m) {
                const double p = l[k] * xj;
                xr[k] = xr[k] - p;
            }
        }
    }
    for (int k = 0; k < 2; ++k)
        if (lane + 32 * k < m) x[lane + 32 * k] = xr[k];
    __syncwarp();
    for (int r = m - 1; r >= 0; --r) {
        const double* lc = L + (size_t)r * m;  // column r: L_jr at lc[j]
        for (int j = r + 2 + lane; j < m; j += 32) {
            const double p = __ldg(lc + j) * x[j];
            q[j] = p;
        }
        __syncwarp();
        if (lane == 0) {
            double s = x[r];
            if (r + 1 < m) {
                const double p = __ldg(lc + r + 1) * x[r + 1];
                s = s - p;
            }
            for (int j = r + 2; j < m; ++j) s = s - q[j];
            x[r] = s / __ldg(lc + r);
        }
        __syncwarp();
    }
}

template <int LPC, int RPL>
__global__ void __launch_bounds__(kSmallThreads, 1)
    k_casc_small(double* __restrict__ cols, const double* __restrict__ a,
                 const double* __restrict__ d, int m, int n, int32_t* __restrict__ fail,
                 const double* __restrict__ x0_low) {
    extern __shared__ __align__(16) double smx[];
    const int mp = (int)small_stride(m);
    double* sc = smx;                          // [n + 1][mp]
    double* sa = smx + (size_t)(n + 1) * mp;   // [n][mp]
    double* sdv = sa + (size_t)n * mp;         // d
    const int tid = threadIdx.x;
    constexpr int NG = kSmallThreads / LPC;    // column groups per CTA
    const int grp = tid / LPC, j = tid % LPC;
    for (idx_t e = tid; e < (idx_t)(n + 1) * m; e += kSmallThreads)
        sc[(e / m) * mp + e % m] = __ldcg(cols + e);
    for (idx_t e = tid; e < (idx_t)n * m; e += kSmallThreads) sa[(e / m) * mp + e % m] = __ldg(a + e);
    for (int i = tid; i < n; i += kSmallThreads) sdv[i] = __ldg(d + i);
    __syncthreads();
    if (x0_low) {  // the initial x column (init_workspace's x0 solve) first
        if (tid < 32) small_x0_warp(x0_low, m, sc + (size_t)n * mp, sdv + n);
        __syncthreads();
    }
    const bool m1 = m == 1;
    const int H = m > 1 ? (int)(pow2_ceil(m) >> 1) : 0;
    // rows of this lane: lo = j + LPC r, hi = lo + H (absent rows: +0.0 terms)
    bool lo_ok[RPL], hi_ok[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
        const int lo = j + LPC * r;
        lo_ok[r] = m1 ? lo == 0 : lo < H;
        hi_ok[r] = !m1 && lo < H && lo + H < m;
    }
    // tree over a column (its values left in xl/xh for the update): level 0 per
    // s-index (+0.0 pad, _kernels.pyx:46), in-lane levels, then the group's xor
    // butterfly; every lane of the group ends with the result
    auto tree = [&](const double (&vl)[RPL], const double (&vh)[RPL], const double* col,
                    double (&xl)[RPL], double (&xh)[RPL]) {
        double q[RPL];
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            xl[r] = lo_ok[r] ? col[j + LPC * r] : 0.0;
            xh[r] = hi_ok[r] ? col[j + LPC * r + H] : 0.0;
            const double lo = lo_ok[r] ? vl[r] * xl[r] : 0.0;
            const double hi = hi_ok[r] ? vh[r] * xh[r] : 0.0;
            q[r] = m1 ? lo : lo + hi;
        }
        double t = lane_tree<RPL>(q);
#pragma unroll
        for (int sft = LPC / 2; sft >= 1; sft >>= 1) t = t + __shfl_xor_sync(0xffffffffu, t, sft);
        return t;
    };
    int32_t f = 0;
    for (int l = 0; l < n; ++l) {
        const double dl = sdv[l];
        if (dl == 1.0) continue;  // _kernels.pyx:242-243 (uniform)
        const double fl = dl - 1.0;
        const double* al = sa + (size_t)l * mp;
        const double* pl = sc + (size_t)l * mp;
        double vl[RPL], vh[RPL], pv_lo[RPL], pv_hi[RPL];
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int lo = j + LPC * r;
            vl[r] = lo_ok[r] ? al[lo] * fl : 0.0;
            vh[r] = hi_ok[r] ? al[lo + H] * fl : 0.0;
        }
        // every warp finds denom_l itself (same bits everywhere: no barrier)
        const double inner_l = tree(vl, vh, pl, pv_lo, pv_hi);
        const double denom = 1.0 + inner_l;
        if (fabs(denom) <= kDenomEpsRel * (1.0 + fabs(inner_l))) {
            f = l + 1;  // the same test in every thread: uniform exit
            break;
        }
        // this group's columns past l: k0, k0 + NG, ...; shuffles stay
        // warp-uniform (a group past n reduces the pivot column and drops it)
        const int k0 = l + 1 + ((grp - (l + 1)) % NG + NG) % NG;
        // KB columns per pass, their chains (loads, tree, divide, update) overlapped
        for (int kb = k0; __any_sync(0xffffffffu, kb <= n); kb += KB * NG) {
            double xl[KB][RPL], xh[KB][RPL], g[KB];
#pragma unroll
            for (int b = 0; b < KB; ++b) {
                const int k = kb + b * NG;
                const double* ck = sc + (size_t)(k <= n ? k : l) * mp;
                g[b] = tree(vl, vh, ck, xl[b], xh[b]);
            }
#pragma unroll
            for (int b = 0; b < KB; ++b) g[b] = g[b] / denom;
#pragma unroll
            for (int b = 0; b < KB; ++b) {
                const int k = kb + b * NG;
                if (k > n) continue;
                double* ck = sc + (size_t)k * mp;
#pragma unroll
                for (int r = 0; r < RPL; ++r) {
                    const int lo = j + LPC * r;
                    if (lo_ok[r]) {
                        const double q = g[b] * pv_lo[r];
                        ck[lo] = xl[b][r] - q;
                    }
                    if (hi_ok[r]) {
                        const double q = g[b] * pv_hi[r];
                        ck[lo + H] = xh[b][r] - q;
                    }
                }
            }
        }
        __syncthreads();  // column l+1 is final for the next step
    }
    if (f) {
        if (tid == 0) *fail = f;
        return;  // on breakdown only the return code is contractual
    }
    for (idx_t e = tid; e < (idx_t)(n + 1) * m; e += kSmallThreads) cols[e] = sc[(e / m) * mp + e % m];
}

static bool small_cascade_fits(idx_t m, idx_t n) {
    return m >= 1 && m <= 64 && n >= 1 && small_cascade_smem(m, n) <= 200 * 1024;
}

template <int LPC, int RPL>
static int launch_small(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                        int32_t* fail, const double* x0_low, cudaStream_t st) {
    const size_t smem = small_cascade_smem(m, n);
    cudaFuncSetAttribute(k_casc_small<LPC, RPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k_casc_small<LPC, RPL><<<1, kSmallThreads, smem, st>>>(cols, a, d, (int)m, (int)n, fail,
                                                           x0_low);
    return cudaGetLastError() == cudaSuccess ? PDAS_OK : PDAS_ERR_CUDA;
}

// groups of 8 lanes per column (up to 4 s-indices each); fewer for H < 8.
// x0_low: solve the x column in the kernel first (launch_cascade_x0)
static int launch_small_cascade(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                                int32_t* fail, cudaStream_t st, const double* x0_low = nullptr) {
    const idx_t H = m > 1 ? pow2_ceil(m) >> 1 : 0;
    if (H == 32) return launch_small<8, 4>(cols, a, d, m, n, fail, x0_low, st);
    if (H == 16) return launch_small<8, 2>(cols, a, d, m, n, fail, x0_low, st);
    if (H == 8) return launch_small<8, 1>(cols, a, d, m, n, fail, x0_low, st);
    if (H == 4) return launch_small<4, 1>(cols, a, d, m, n, fail, x0_low, st);
    if (H == 2) return launch_small<2, 1>(cols, a, d, m, n, fail, x0_low, st);
    return launch_small<1, 1>(cols, a, d, m, n, fail, x0_low, st);  // m <= 2
}

// ------------------------------------------------------------ host side
struct CascCfg {
    int T, R, Cu, G, CT;
};

static int env_int(const char* name, int dflt) {
    const char* s = getenv(name);
    return s && *s ? atoi(s) : dflt;
}

static CascCfg cascade_cfg(idx_t m) {
    const idx_t H = m > 1 ? pow2_ceil(m) >> 1 : 0;
    if (H <= 32) return {32, 1, 8, 1, 8};
    if (H == 64) return {64, 1, 8, 1, 8};
    if (H == 128) return {128, 1, 8, 1, 8};
    if (H == 256) return {128, 2, 8, 1, 8};   // 2 warp-specialized CTAs per SM
    if (H == 512) return {128, 4, 8, 1, 8};   // 2 warp-specialized CTAs per SM
    if (H == 1024) return {256, 4, 8, 1, 8};  // warp-specialized, 1 CTA per SM
    if (H == 2048) return {256, 8, 4, 1, 4};
    if (H == 4096) return {256, 16, 2, 1, 2};
    if (H == 8192) return {256, 32, 1, 1, 1};
    return {0, 0, 0, 0, 0};
}

idx_t cascade_supported_m() { return 16384; }

bool cascade_one_cta(idx_t m, idx_t n) { return small_cascade_fits(m, n); }

// Side stream (high priority) + events for the panel lookahead, per device.
struct SideStream {
    cudaStream_t ps = nullptr;  // panels (high priority)
    cudaStream_t xs = nullptr;  // x0 solve + the x tile's updates (see CascOp::x0_low)
    cudaEvent_t e0 = nullptr, eP = nullptr, eU = nullptr, eX = nullptr;
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
        cudaStreamCreateWithPriority(&s.xs, cudaStreamNonBlocking, hi);
        cudaEventCreateWithFlags(&s.eX, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&s.e0, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&s.eP, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&s.eU, cudaEventDisableTiming);
    }
    return s;
}

// Diagnostics (env PDAS_CASCADE_PROFILE=1): timing events around every
// update / panel launch of the 1-GPU cascade; the last cascade's rows
// (kind 0 update / 1 panel, block, start ms, end ms) are read back with
// pdas_debug_cascade_profile (tools/cascade_timeline.py).  Off: no events.
struct ProfRow {
    int kind;
    idx_t block;
    cudaEvent_t e[2];
};
static std::vector<double> g_prof_rows;

struct CascProfile {
    bool on;
    cudaEvent_t t0 = nullptr;
    std::vector<ProfRow> rows;
    CascProfile(idx_t nrows, cudaStream_t st) {
        static const bool env = env_int("PDAS_CASCADE_PROFILE", 0) != 0;
        on = env;
        if (!on) return;
        rows.reserve((size_t)nrows);
        cudaEventCreate(&t0);
        cudaEventRecord(t0, st);
    }
    void mark(cudaStream_t s, int kind, idx_t b, int which) {
        if (!on) return;
        if (which == 0) {
            ProfRow r{kind, b, {nullptr, nullptr}};
            cudaEventCreate(&r.e[0]);
            cudaEventCreate(&r.e[1]);
            rows.push_back(r);
            cudaEventRecord(rows.back().e[0], s);
        } else {
            for (size_t i = rows.size(); i-- > 0;)
                if (rows[i].kind == kind && rows[i].block == b) {
                    cudaEventRecord(rows[i].e[1], s);
                    break;
                }
        }
    }
    void finish(cudaStream_t st) {
        if (!on) return;
        cudaStreamSynchronize(st);
        g_prof_rows.clear();
        for (auto& r : rows) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, t0, r.e[0]);
            cudaEventElapsedTime(&b, t0, r.e[1]);
            g_prof_rows.insert(g_prof_rows.end(), {(double)r.kind, (double)r.block, a, b});
            cudaEventDestroy(r.e[0]);
            cudaEventDestroy(r.e[1]);
        }
        cudaEventDestroy(t0);
    }
};

idx_t cascade_profile_rows(double* out, idx_t max_rows) {
    const idx_t nr = (idx_t)(g_prof_rows.size() / 4);
    const idx_t k = nr < max_rows ? nr : max_rows;
    for (idx_t i = 0; i < 4 * k; ++i) out[i] = g_prof_rows[(size_t)i];
    return nr;
}

// What to launch: the full cascade, or one building block of the sharded
// cascade (dist.py): a panel over block [p0,p1) after previous block [q0,p0),
// or an update of a tile list with block [p0,p1).
struct CascOp {
    int kind = 0;  // 0 full, 1 panel, 2 update
    idx_t q0 = 0, p0 = 0, p1 = 0;
    const int64_t* tiles = nullptr;
    idx_t ntiles = 0;
    // kind 0 only: column n holds the right-hand side; x0 = L^-T L^-1 rhs
    // (normal.py:123) is solved here, concurrently with the Y part of the
    // cascade, when column n sits alone in the last tile (n % CT == 0).
    const double* x0_low = nullptr;
    double* x0_work = nullptr;
    PeerSet peers{};  // kind 1 only: fused multi-GPU exchange
    // kinds 1 / 2 of the chained sharded schedule: a panel waits for its tiles'
    // tile_done == utag (kind 1, q0 == p0); an update publishes tile_done = utag
    int* uflag = nullptr;
    int utag = 0;
};

// The panel is a latency chain (one full-tile reduction per pivot step on one
// SM), so its CTA spreads a tile over twice the update's threads (half the
// rows per thread): each step's fp64 work and register tile halve.
template <int T, int R>
struct PanelShape {
    static constexpr int TP = (R >= 2 && 2 * T <= 512) ? 2 * T : T;
    static constexpr int RP = R * T / TP;
};

template <bool TMA, int S, int T, int R, int Cu, int G, int CT>
static int run_cascade_impl(double* cols, const double* a, const double* d, int m, idx_t n,
                            double* denoms, int32_t* fail, int* flags, int epoch, int B,
                            cudaStream_t st, const CascOp& op) {
    constexpr bool GEN = (T == 32);
    static_assert(Cu * G == CT, "tile width");
    const size_t smem_u = casc_smem_bytes<T, Cu, G>(TMA ? S : 0, m);
    constexpr int TP = PanelShape<T, R>::TP, RP = PanelShape<T, R>::RP;
    // The panel's pivot data always comes through the TMA ring when it can
    // (prefetched S stages ahead, also where the update loads straight from
    // L2): a latency chain cannot hide an L2 round trip per step.
    // 4 stages when they fit next to the panel's reduction rows, else 2, else
    // direct loads (m beyond ~6000)
    const bool pok = (TMA || TP >= 128) && !GEN && m % 2 == 0 &&
                     ((uintptr_t)cols | (uintptr_t)a) % 16 == 0;
    constexpr size_t kPanelSmem = 200 * 1024;
    const int sp = pok && casc_smem_bytes<TP, CT, 1>(4, m) <= kPanelSmem   ? 4
                   : pok && casc_smem_bytes<TP, CT, 1>(2, m) <= kPanelSmem ? 2
                                                                           : 0;
    const size_t smem_p = casc_smem_bytes<TP, CT, 1>(sp, m);
    auto ku = k_casc_update<TMA, S, T, R, Cu, G, GEN>;
    // a publisher warp where the registers allow it (TP <= 256: c2, c4, c5;
    // 512 + 32 threads are allocated as 20 warps -> 96 registers, spills)
    constexpr int PW = (TP <= 256 && !GEN) ? 32 : 0;
    constexpr int TPB = TP + PW;  // panel block size
    auto kp = sp == 4   ? k_casc_panel<!GEN, 4, TP, RP, CT, GEN, PW>
              : sp == 2 ? k_casc_panel<!GEN, 2, TP, RP, CT, GEN, PW>
                        : k_casc_panel<false, 1, TP, RP, CT, GEN, PW>;
    cudaFuncSetAttribute(ku, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_u);
    cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
    // warp-specialized update for the 256-thread single-group layouts
    // (R >= 16 spills the compute warpgroups' 232-register budget)
    constexpr bool kWs256 = TMA && T == kWsT && G == 1 && CT % 2 == 0 && S >= 2 && R <= 8;
    constexpr bool kWs128 = T == 128 && G == 1 && CT % 2 == 0 && R >= 2 &&
                            (R <= 4 || (TMA && R <= 8 && S >= 2 && S <= 3));
    constexpr bool kUseWs = kWs256 || kWs128;
    constexpr int CW = kUseWs ? CT : 2;
    constexpr int RW = kUseWs ? R : 1;
    constexpr int TCW = kWs128 ? 128 : kWsT;
    const int ws_threads = TCW + 128;
    auto kws = k_casc_update_ws<S, RW, CW, TCW>;
    const size_t smem_ws = casc_smem_bytes<TCW, CW, 1>(S, m);
    constexpr bool use_ws = kUseWs;
    if (use_ws)
        cudaFuncSetAttribute(kws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_ws);
    // the warp-per-column panel (k_casc_panel_w) for the 1-GPU chain, m <= 1024:
    // every column warp reads each pivot's [P | A] in full, 8x the shared-memory
    // traffic of the CTA-wide panel -- at H = 1024 (c3) that is ~2000 cycles of
    // shared bandwidth per step and the two panels tie (163.7 vs 164.0 ms)
    constexpr int RPW = T * R / 32;  // H / 32
    constexpr bool kPwOk = !GEN && CT == kPwCols && G == 1 && RPW >= 2 && RPW <= 16;
    constexpr int SPW = 8;
    const bool pw = kPwOk && pok && panel_w_smem(SPW, m) <= kPanelSmem;
    const bool pw_full = m == 2 * (T * R);
    auto kpw = pw_full ? k_casc_panel_w<kPwOk ? RPW : 2, SPW, true>
                       : k_casc_panel_w<kPwOk ? RPW : 2, SPW, false>;
    const size_t smem_w = panel_w_smem(SPW, m);
    if (pw) cudaFuncSetAttribute(kpw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_w);
    // panel of block [p0, p1) on stream s_ (nothing of an earlier block pending)
    auto panel = [&](cudaStream_t s_, idx_t p0_, idx_t p1_, const int* uf, int ut) {
        const unsigned nt_ = (unsigned)((p1_ - p0_ + CT - 1) / CT);
        if (pw)
            kpw<<<nt_, kPwThreads, smem_w, s_>>>(cols, a, d, denoms, m, n, p0_, p1_, fail, flags,
                                                 epoch, uf, ut);
        else  // more than 32 tiles (512-pivot blocks): two tiles per CTA
            kp<<<nt_ > 32 ? (nt_ + 1) / 2 : nt_, TPB, smem_p, s_>>>(
                cols, a, d, denoms, m, n, p0_, p0_, p1_, fail, flags, epoch, uf, ut, PeerSet{});
    };
    const idx_t ntiles = (n + 1 + CT - 1) / CT;
    if (op.kind == 1) {
        if (op.p0 % CT || op.p1 <= op.p0 || op.p1 - op.q0 > 2 * kMaxBlock) return PDAS_ERR_ARG;
        // a chained block of the NCCL-exchange schedule: nothing outside this
        // launch reads its chunk flags (the fused exchange's k_peer_wait reads
        // them in the CTA-wide panel's layout, so it keeps that panel)
        if (op.q0 == op.p0 && op.peers.count == 0 && op.uflag != nullptr)
            panel(st, op.p0, op.p1, op.uflag, op.utag);
        else
            kp<<<(unsigned)((op.p1 - op.p0 + CT - 1) / CT), TPB, smem_p, st>>>(
                cols, a, d, denoms, m, n, op.q0, op.p0, op.p1, fail, flags, epoch, op.uflag,
                op.utag, op.peers);
        return cudaGetLastError() == cudaSuccess ? PDAS_OK : PDAS_ERR_CUDA;
    }
    if (op.kind == 2) {
        if (op.p1 - op.p0 > kMaxBlock || op.p1 <= op.p0) return PDAS_ERR_ARG;
        if (op.ntiles > 0) {
            if (use_ws)
                kws<<<(unsigned)op.ntiles, ws_threads, smem_ws, st>>>(
                    cols, a, d, denoms, m, n, op.p0, op.p1, 0, fail, op.tiles, op.uflag, op.utag,
                    0, nullptr, 0);
            else
                ku<<<(unsigned)op.ntiles, T * G, smem_u, st>>>(cols, a, d, denoms, m, n, op.p0,
                                                               op.p1, 0, fail, op.tiles, op.uflag,
                                                               op.utag, 0, nullptr, 0);
        }
        return cudaGetLastError() == cudaSuccess ? PDAS_OK : PDAS_ERR_CUDA;
    }
    // pivot blocks: the first one B (its panel runs alone), the others 2B:
    // half the update CTAs, their start-up and tile reloads (c3 161.5 -> 160.8
    // ms, c4 1929 -> 1915; 2B only over the first half of n: c3 161.0)
    std::vector<idx_t> bst{0};
    {
        const idx_t big = 2 * B <= 2 * kMaxBlock ? 2 * B : B;
        while (bst.back() < n) {
            const idx_t at = bst.back();
            const idx_t len = at > 0 ? big : B;
            bst.push_back(at + len < n ? at + len : n);
        }
    }
    const idx_t nb = (idx_t)bst.size() - 1;
    auto bs = [&](idx_t b) { return bst[(size_t)b]; };
    auto blk_end = [&](idx_t b) { return bst[(size_t)b + 1]; };
    auto tiles_of = [&](idx_t b) { return (blk_end(b) - bs(b) + CT - 1) / CT; };
    SideStream& ss = side_stream();
    {
        // U(b) covers block b+1's tiles too (its lowest CTAs) and flags each
        // tile as it lands; panel(b+1) -- only the block's own chain and
        // triangle -- waits on those flags inside the kernel, so it starts as
        // soon as its 16-odd tiles are done instead of after all of U(b).
        int* uflag = flags + panel_flag_ints(n);
        cudaMemsetAsync(uflag, 0, sizeof(int) * (size_t)panel_flag_ints(n), st);
        CascProfile prof(2 * nb + 1, st);
        // x lane: column n alone in the last tile -> the x0 solve and that
        // tile's updates run on their own stream, off the Y critical path
        const bool xlane = op.x0_low != nullptr && n % CT == 0;
        const idx_t nt_y = xlane ? ntiles - 1 : ntiles;  // tiles U(b) covers
        auto update_x = [&](idx_t b) {  // block b -> the x tile (1 CTA)
            if (use_ws)
                kws<<<1, ws_threads, smem_ws, ss.xs>>>(cols, a, d, denoms, m, n, bs(b), blk_end(b),
                                                       ntiles - 1, fail, nullptr, nullptr, 0, 0,
                                                       nullptr, 0);
            else
                ku<<<1, T * G, smem_u, ss.xs>>>(cols, a, d, denoms, m, n, bs(b), blk_end(b),
                                                ntiles - 1, fail, nullptr, nullptr, 0, 0, nullptr,
                                                0);
        };
        cudaEventRecord(ss.e0, st);
        cudaStreamWaitEvent(ss.ps, ss.e0, 0);
        if (op.x0_low) {
            cudaStreamWaitEvent(ss.xs, ss.e0, 0);
            launch_solve_one(op.x0_low, m, cols + (size_t)n * m, op.x0_work, xlane ? ss.xs : st);
            if (!xlane) {  // sequential fallback: the panels wait for x0 too
                cudaEventRecord(ss.e0, st);
                cudaStreamWaitEvent(ss.ps, ss.e0, 0);
            }
        }
        prof.mark(ss.ps, 1, 0, 0);
        panel(ss.ps, 0, blk_end(0), nullptr, 0);
        prof.mark(ss.ps, 1, 0, 1);
        cudaEventRecord(ss.eP, ss.ps);
        if (xlane) {
            cudaStreamWaitEvent(ss.xs, ss.eP, 0);
            update_x(0);
        }
        // U(b) for b >= 1 is chained to U(b-1) by programmatic dependent
        // launch: its CTAs may start on the SMs U(b-1)'s last (partial) wave
        // leaves idle, as soon as every U(b-1) CTA is resident (they signal at
        // their start).  Ordering then comes from flags, not from the stream:
        // each CTA waits for panel(b)'s last chunk flag and for its tile's
        // U(b-1) (tile_done = uflag[tile] >= b, set by every update CTA).
        const int nch = pw ? kPwChunks : panel_flag_chunks(CT);
        auto upd = [&](cudaStream_t s_, idx_t b, idx_t ta, idx_t tb, int* uf) {
            if (ta >= tb) return;
            const bool chained = b > 0;
            const int* pflag = chained ? flags + (bs(b) / CT + tiles_of(b) - 1) * nch + nch - 1
                                       : nullptr;
            const int need = chained ? (int)b : 0;
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)(tb - ta));
            lc.stream = s_;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = chained ? 1 : 0;
            lc.attrs = at;
            lc.numAttrs = 1;
            const double* dd = d;
            const double* dn = denoms;
            const int64_t* no_tiles = nullptr;
            const int utag = (int)(b + 1);
            if (use_ws) {
                lc.blockDim = dim3(ws_threads);
                lc.dynamicSmemBytes = smem_ws;
                cudaLaunchKernelEx(&lc, kws, cols, a, dd, dn, m, n, bs(b), blk_end(b), ta,
                                   (const int32_t*)fail, no_tiles, uf, utag, need, pflag, epoch);
            } else {
                lc.blockDim = dim3(T * G);
                lc.dynamicSmemBytes = smem_u;
                cudaLaunchKernelEx(&lc, ku, cols, a, dd, dn, m, n, bs(b), blk_end(b), ta,
                                   (const int32_t*)fail, no_tiles, uf, utag, need, pflag, epoch);
            }
        };
        for (idx_t b = 0; b < nb; ++b) {
            // panel(b): block b is final.  U(0) waits for it on the stream; the
            // chained U(b >= 1) wait inside the kernel (pflag), because a stream
            // wait between two kernels defeats the programmatic early launch
            // (tools/micro/pdl_probe2.cu).  No deadlock: panel(b) runs on the
            // high-priority stream and is resident before U(b) can launch.
            if (b == 0) cudaStreamWaitEvent(st, ss.eP, 0);
            // eU: the main stream up to U(b-1); panel(b+1) must not be resident
            // (spinning on its SMs) while U(b-1) still runs
            cudaEventRecord(ss.eU, st);
            const idx_t t0 = b + 1 < nb ? bs(b + 1) / CT : (n + CT - 1) / CT;
            prof.mark(st, 0, b, 0);
            upd(st, b, t0, nt_y, uflag);
            prof.mark(st, 0, b, 1);
            if (b + 1 < nb) {
                const idx_t p0 = bs(b + 1);
                cudaStreamWaitEvent(ss.ps, ss.eU, 0);
                prof.mark(ss.ps, 1, b + 1, 0);
                panel(ss.ps, p0, blk_end(b + 1), uflag, (int)(b + 1));
                prof.mark(ss.ps, 1, b + 1, 1);
                cudaEventRecord(ss.eP, ss.ps);
                if (xlane) {
                    cudaStreamWaitEvent(ss.xs, ss.eP, 0);
                    update_x(b + 1);
                }
            }
        }
        // join: the caller's stream sees every panel and the x lane
        cudaEventRecord(ss.eP, ss.ps);
        cudaStreamWaitEvent(st, ss.eP, 0);
        if (op.x0_low) {
            cudaEventRecord(ss.eX, ss.xs);
            cudaStreamWaitEvent(st, ss.eX, 0);
        }
        prof.finish(st);
        return cudaGetLastError() == cudaSuccess ? PDAS_OK : PDAS_ERR_CUDA;
    }
}

template <int T, int R, int Cu, int G, int CT>
static int run_cascade(double* cols, const double* a, const double* d, int m, idx_t n,
                       double* denoms, int32_t* fail, int* flags, int epoch, int B,
                       cudaStream_t st, const CascOp& op) {
    B = (B + CT - 1) / CT * CT;
    if (B > kMaxBlock) B = kMaxBlock / CT * CT;
    // TMA pivot staging pays off only for the 256-thread tiles (m > 256); for
    // smaller m the per-pivot bulk-copy + mbarrier round trip dominates the
    // step (measured 3-5x slower than direct L2 loads at m = 50 / 64).
    const bool aligned = (T == 256 || (T == 128 && R == 8)) && (m % 2 == 0) &&
                         (((uintptr_t)cols | (uintptr_t)a) % 16 == 0);
    // two warp-specialized CTAs per SM for the 128-thread layouts
    const size_t budget = (T == 128 ? 110 : 210) * 1024;
    if (aligned &&
        casc_smem_bytes<PanelShape<T, R>::TP, CT, 1>(5, m) <= budget &&
        casc_smem_bytes<T, Cu, G>(5, m) <= budget)
        return run_cascade_impl<true, 5, T, R, Cu, G, CT>(cols, a, d, m, n, denoms, fail, flags,
                                                          epoch, B, st, op);
    if (aligned && casc_smem_bytes<PanelShape<T, R>::TP, CT, 1>(4, m) <= budget &&
        casc_smem_bytes<T, Cu, G>(4, m) <= budget)
        return run_cascade_impl<true, 4, T, R, Cu, G, CT>(cols, a, d, m, n, denoms, fail, flags,
                                                          epoch, B, st, op);
    if (T == 128 && aligned && casc_smem_bytes<PanelShape<T, R>::TP, CT, 1>(3, m) <= budget &&
        casc_smem_bytes<T, Cu, G>(3, m) <= budget)
        return run_cascade_impl<true, 3, T, R, Cu, G, CT>(cols, a, d, m, n, denoms, fail, flags,
                                                          epoch, B, st, op);
    if (aligned && casc_smem_bytes<PanelShape<T, R>::TP, CT, 1>(2, m) <= budget &&
        casc_smem_bytes<T, Cu, G>(2, m) <= budget)
        return run_cascade_impl<true, 2, T, R, Cu, G, CT>(cols, a, d, m, n, denoms, fail, flags,
                                                          epoch, B, st, op);
    return run_cascade_impl<false, 1, T, R, Cu, G, CT>(cols, a, d, m, n, denoms, fail, flags,
                                                       epoch, B, st, op);
}

idx_t cascade_flags_count(idx_t m, idx_t n) { return 2 * panel_flag_ints(n); }  // panel + update

#if PDAS_PANEL_TRACE
}  // namespace pdas
extern "C" int pdas_debug_panel_trace(long long* host_out) {
    return cudaMemcpyFromSymbol(host_out, pdas::g_panel_trace, sizeof(pdas::g_panel_trace)) ==
                   cudaSuccess
               ? 0
               : -2;
}
namespace pdas {
#endif
#if PDAS_HOP_TRACE
}  // namespace pdas
extern "C" int pdas_debug_hop_trace(unsigned long long* host_out) {
    return cudaMemcpyFromSymbol(host_out, pdas::g_hop_trace, sizeof(pdas::g_hop_trace)) ==
                   cudaSuccess
               ? 0
               : -2;
}
namespace pdas {
#endif
#if PDAS_WS_TRACE
}  // namespace pdas
extern "C" int pdas_debug_ws_trace(long long* host_out) {
    return cudaMemcpyFromSymbol(host_out, pdas::g_ws_trace, sizeof(pdas::g_ws_trace)) ==
                   cudaSuccess
               ? 0
               : -2;
}
namespace pdas {
#endif

int cascade_tile_width(idx_t m) { return cascade_cfg(m).CT; }

static int dispatch_cascade(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                            double* denoms, int32_t* fail_dev, int* flags, int epoch, int B,
                            cudaStream_t st, const CascOp& op) {
    const CascCfg cfg = cascade_cfg(m);
#define PDAS_CASC(T_, R_, C_, G_, CT_)                                                       \
    if (cfg.T == T_ && cfg.R == R_ && cfg.Cu == C_ && cfg.G == G_)                           \
        return run_cascade<T_, R_, C_, G_, CT_>(cols, a, d, (int)m, n, denoms, fail_dev, flags, \
                                                epoch, B, st, op);
    PDAS_CASC(32, 1, 8, 1, 8)
    PDAS_CASC(64, 1, 8, 1, 8)
    PDAS_CASC(128, 1, 8, 1, 8)
    PDAS_CASC(128, 4, 8, 1, 8)
    PDAS_CASC(128, 2, 8, 1, 8)
    PDAS_CASC(256, 4, 8, 1, 8)
    PDAS_CASC(256, 8, 4, 1, 4)
    PDAS_CASC(256, 16, 2, 1, 2)
    PDAS_CASC(256, 32, 1, 1, 1)
#undef PDAS_CASC
    return PDAS_ERR_UNSUPPORTED;
}

int launch_cascade(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                   double* denoms, int32_t* fail_dev, int* flags, int epoch, int block_pivots,
                   cudaStream_t st) {
    if (m < 1 || n < 0 || m > INT_MAX / 4) return PDAS_ERR_ARG;
    cudaMemsetAsync(fail_dev, 0, sizeof(int32_t), st);
    if (n == 0) return PDAS_OK;
    if (small_cascade_fits(m, n)) return launch_small_cascade(cols, a, d, m, n, fail_dev, st);
    const int B = block_pivots > 0 ? block_pivots : kSolveBlock;
    return dispatch_cascade(cols, a, d, m, n, denoms, fail_dev, flags, epoch, B, st, CascOp{});
}

int launch_cascade_x0(double* cols, const double* a, const double* d, const double* low, idx_t m,
                      idx_t n, double* denoms, int32_t* fail_dev, int* flags, int epoch,
                      double* work, cudaStream_t st) {
    if (m < 1 || n < 0 || m > INT_MAX / 4) return PDAS_ERR_ARG;
    cudaMemsetAsync(fail_dev, 0, sizeof(int32_t), st);
    if (n == 0) return launch_solve_one(low, m, cols, work, st);
    if (small_cascade_fits(m, n))  // x0 solved inside the one-CTA cascade, first
        return launch_small_cascade(cols, a, d, m, n, fail_dev, st, low);
    CascOp op;
    op.x0_low = low;
    op.x0_work = work;
    return dispatch_cascade(cols, a, d, m, n, denoms, fail_dev, flags, epoch, kSolveBlock, st,
                            op);
}

int launch_cascade_panel(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                         idx_t q0, idx_t p0, idx_t p1, double* denoms, int32_t* fail_dev,
                         int* flags, int epoch, cudaStream_t st, const PeerSet* peers,
                         int utag) {
    if (m < 1 || m > INT_MAX / 4 || q0 < 0 || q0 > p0 || p1 > n) return PDAS_ERR_ARG;
    CascOp op;
    op.kind = 1;
    op.q0 = q0;
    op.p0 = p0;
    op.p1 = p1;
    if (utag > 0) {  // chained: wait for this rank's own update of the tiles
        op.uflag = flags + panel_flag_ints(n);
        op.utag = utag;
    }
    if (peers) {
        if (peers->count < 0 || peers->count > kMaxPeers) return PDAS_ERR_ARG;
        op.peers = *peers;
    }
    return dispatch_cascade(cols, a, d, m, n, denoms, fail_dev, flags, epoch, kMaxBlock, st, op);
}

int launch_cascade_panel_peers(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                               idx_t q0, idx_t p0, idx_t p1, double* denoms, int32_t* fail_dev,
                               int* flags, int epoch, int npeers, double* const* peer_cols,
                               double* const* peer_denoms, int32_t* const* peer_fail,
                               int* const* peer_flags, cudaStream_t st) {
    if (npeers < 0 || npeers > kMaxPeers) return PDAS_ERR_ARG;
    PeerSet ps{};
    ps.count = npeers;
    for (int q = 0; q < npeers; ++q) {
        if (!peer_cols[q] || !peer_denoms[q] || !peer_fail[q] || !peer_flags[q]) return PDAS_ERR_ARG;
        ps.cols[q] = peer_cols[q];
        ps.denoms[q] = peer_denoms[q];
        ps.fail[q] = peer_fail[q];
        ps.flags[q] = peer_flags[q];
    }
    return launch_cascade_panel(cols, a, d, m, n, q0, p0, p1, denoms, fail_dev, flags, epoch, st,
                                &ps);
}

int panel_flag_chunks(int ct) {
    const int ch = ct / kPanelChunks > 0 ? ct / kPanelChunks : 1;
    return ct / ch;
}

int launch_peer_wait(const int* flags, idx_t m, idx_t c0, idx_t c1, int epoch, cudaStream_t st) {
    const int ct = cascade_cfg(m).CT;
    if (ct < 1 || c0 < 0 || c1 < c0) return PDAS_ERR_ARG;
    if (c1 == c0) return PDAS_OK;
    const idx_t t0 = c0 / ct, t1 = (c1 + ct - 1) / ct;
    k_peer_wait<<<1, 64, 0, st>>>(flags, t0, t1, panel_flag_chunks(ct), epoch);
    return cudaGetLastError() == cudaSuccess ? PDAS_OK : PDAS_ERR_CUDA;
}

int launch_cascade_update(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                          idx_t p0, idx_t p1, const int64_t* tiles, idx_t ntiles, double* denoms,
                          int32_t* fail_dev, cudaStream_t st, int* flags, int utag) {
    if (m < 1 || m > INT_MAX / 4 || p0 < 0 || p1 > n || ntiles < 0) return PDAS_ERR_ARG;
    CascOp op;
    op.kind = 2;
    op.p0 = p0;
    op.p1 = p1;
    op.tiles = tiles;
    op.ntiles = ntiles;
    if (flags && utag > 0) {  // publish tile_done = utag for every tile updated
        op.uflag = flags + panel_flag_ints(n);
        op.utag = utag;
    }
    return dispatch_cascade(cols, a, d, m, n, denoms, fail_dev, nullptr, 0, kMaxBlock, st, op);
}

}  // namespace pdas

