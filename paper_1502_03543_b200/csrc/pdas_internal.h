// pdas_internal.h -- launcher prototypes and the device-resident iteration
// state shared by the kernels and the C-ABI layer (abi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pdas_b200.h"

namespace pdas {

typedef int64_t idx_t;

constexpr double kCapAlpha = 1e6;  // solver.py:28-29

// k_scaling flag bits (model.py:116-119 with np.min NaN semantics)
enum : unsigned {
    IT_X_NAN = 1u,
    IT_X_LE0 = 2u,
    IT_S_NAN = 4u,
    IT_S_LE0 = 8u,
};

__host__ __device__ inline bool not_interior(unsigned f) {
    return ((f & IT_X_LE0) && !(f & IT_X_NAN)) || ((f & IT_S_LE0) && !(f & IT_S_NAN));
}

typedef PdasIterState IterState;

// vec_kernels.cu
int launch_dot_tree(const double* u, idx_t su, const double* v, idx_t sv, idx_t L, double* out,
                    cudaStream_t st);
int launch_mat_t_vec(const double* a, idx_t m, idx_t n, const double* y, double* out,
                     cudaStream_t st);
idx_t mat_vec_scratch(idx_t m, idx_t n);
int launch_mat_vec(const double* a, idx_t m, idx_t n, const double* x, double* out,
                   double* scratch, cudaStream_t st);
int launch_scaling(const double* x, const double* s, idx_t n, double* d, unsigned* flags,
                   cudaStream_t st);
int launch_directions(const double* a, idx_t m, idx_t n, const double* dy, const double* d,
                      const double* x, const double* s, double* dx, double* ds, void* partials,
                      cudaStream_t st);
idx_t directions_partials_bytes(idx_t n);
idx_t ratio_partials_bytes(idx_t n);
int launch_ratio_test(const double* x, const double* s, const double* dx, const double* ds,
                      idx_t n, double rho, void* partials, IterState* state, cudaStream_t st);
int launch_dir_finish(const void* partials, idx_t n, const double* adx, idx_t m, const double* dy,
                      double rho, IterState* state, cudaStream_t st);
int launch_update(double* x, double* y, double* s, const double* dx, const double* dy,
                  const double* ds, idx_t n, idx_t m, const IterState* state, cudaStream_t st);
int launch_dot3(const double* u0, const double* v0, idx_t l0, double* o0, const double* u1,
                const double* v1, idx_t l1, double* o1, const double* u2, const double* v2,
                idx_t l2, double* o2, cudaStream_t st);

int launch_fp64_probe(double* sink, idx_t iters, idx_t* ops, cudaStream_t st);
int launch_div_selftest(const double* a, const double* b, idx_t n, double* fast, double* ref,
                        cudaStream_t st);

// factor_kernels.cu
int launch_gram(const double* a, idx_t m, idx_t n, const double* d, double* g, cudaStream_t st);
int launch_cholesky(const double* g, idx_t nn, double eps_rel, double* low, int64_t* fail_dev,
                    double* work, cudaStream_t st);
idx_t cholesky_work_doubles(idx_t nn);
int launch_solve_many(const double* low, idx_t m, double* x, idx_t k, double* work,
                      cudaStream_t st);
idx_t solve_many_work_doubles(idx_t m, idx_t k);

// cascade.cu
int launch_build_v(const double* a, idx_t m, idx_t l0, double dl, double* v, cudaStream_t st);
int launch_sweep_phase1(const double* cols, idx_t m, const double* v, double* inner, idx_t k0,
                        idx_t k1, cudaStream_t st);
int launch_sweep_phase2(double* cols, idx_t m, idx_t l0, const double* inner, double denom,
                        idx_t k0, idx_t k1, cudaStream_t st);
int launch_cascade(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                   double* denoms, int32_t* fail_dev, int* flags, int epoch, int block_pivots,
                   cudaStream_t st);
int launch_cascade_x0(double* cols, const double* a, const double* d, const double* low, idx_t m,
                      idx_t n, double* denoms, int32_t* fail_dev, int* flags, int epoch,
                      double* work, cudaStream_t st);
constexpr int kMaxPeers = 7;  // one box: 8 GPUs
struct PeerSet;              // cascade.cu
int launch_cascade_panel(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                         idx_t q0, idx_t p0, idx_t p1, double* denoms, int32_t* fail_dev,
                         int* flags, int epoch, cudaStream_t st, const PeerSet* peers = nullptr,
                         int utag = 0);
int launch_cascade_panel_peers(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                               idx_t q0, idx_t p0, idx_t p1, double* denoms, int32_t* fail_dev,
                               int* flags, int epoch, int npeers, double* const* peer_cols,
                               double* const* peer_denoms, int32_t* const* peer_fail,
                               int* const* peer_flags, cudaStream_t st);
int launch_peer_wait(const int* flags, idx_t m, idx_t c0, idx_t c1, int epoch, cudaStream_t st);
int launch_cascade_update(double* cols, const double* a, const double* d, idx_t m, idx_t n,
                          idx_t p0, idx_t p1, const int64_t* tiles, idx_t ntiles, double* denoms,
                          int32_t* fail_dev, cudaStream_t st, int* flags = nullptr, int utag = 0);
idx_t cascade_supported_m();
bool cascade_one_cta(idx_t m, idx_t n);  // the one-CTA shared-memory cascade runs (m, n)

idx_t cascade_flags_count(idx_t m, idx_t n);
// the workspace's int flags: [0, panel_flag_ints(n)) panel chunk flags (up to
// 8 per 8-column tile), then as many update tile tags (cascade_flags_count = 2x)
inline idx_t panel_flag_ints(idx_t n) { return n + 16; }
int cascade_tile_width(idx_t m);
idx_t cascade_profile_rows(double* out, idx_t max_rows);
// Pivot blocks (B, pivots per panel/update round): the 1-GPU cascade uses
// kSolveBlock (pdas_cascade_solve_block), the sharded building blocks of
// dist.py kShardBlock (pdas_cascade_block_pivots: a shorter panel per
// exchange); kernels size their shared scalar windows for kMaxBlock.
constexpr int kMaxBlock = 256;
constexpr int kSolveBlock = 256;  // c3: 2 % faster than 128 (per-tile reload, launches)
constexpr int kShardBlock = 128;
static_assert(kSolveBlock <= kMaxBlock && 2 * kShardBlock <= 2 * kMaxBlock, "block sizes");
// pivot blocks of the 1-GPU cascade (run_cascade_impl): kSolveBlock, then
// 2 * kSolveBlock each
inline idx_t cascade_solve_blocks(idx_t n) {
    return n <= kSolveBlock ? 1 : 1 + (n - kSolveBlock + 2 * kSolveBlock - 1) / (2 * kSolveBlock);
}

// solve_kernels.cu (single right-hand side, latency-optimised)
int launch_solve_one(const double* low, idx_t m, double* x, double* work, cudaStream_t st);
idx_t solve_one_work_doubles(idx_t m);

}  // namespace pdas
