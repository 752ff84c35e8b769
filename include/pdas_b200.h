/*
 * pdas_b200.h -- C-ABI of the B200-native PDAS / Egidi-Maponi hot path.
 *
 * This is the drop-in boundary for the reference's kernel core: the function
 * table that adascale/_core.py:10-16 exposes as `kernels` (implemented by
 * adascale/_kernels.pyx, the compiled core).  Every entry point below names
 * the reference routine it replaces.  The host side (paper_1502_03543_b200,
 * Python) binds it with ctypes exactly as the reference binds its Cython core.
 *
 * Conventions
 *   - fp64 throughout; every matrix is column-contiguous, element (i,j) at
 *     j*rows + i (reference linalg.py:1-7).
 *   - all array pointers are DEVICE pointers on the current CUDA device;
 *     `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - launches are asynchronous on `stream`; data-dependent results
 *     (Cholesky fail column, cascade breakdown step) are written to a device
 *     word the caller reads after synchronising.
 *   - arithmetic is bitwise-identical to the reference compiled core (fixed
 *     pairwise tree, no fused multiply-add, sequential orders of gram /
 *     Cholesky / triangular solves).
 *   - return value: PDAS_OK or a negative PDAS_ERR_*; pdas_last_error()
 *     gives the message of the last failure on the calling thread.
 */
#ifndef PDAS_B200_H
#define PDAS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDAS_ABI_VERSION 1

#define PDAS_OK 0
#define PDAS_ERR_ARG (-1)         /* bad argument / shape */
#define PDAS_ERR_CUDA (-2)        /* CUDA runtime error (message in pdas_last_error) */
#define PDAS_ERR_UNSUPPORTED (-3) /* size outside the compiled configurations */
#define PDAS_ERR_NOMEM (-4)

/* Device-resident state of one PDAS iteration (solver.py:152-279).  Written
 * by the pdas_iter_* kernels, read back by the host once per iteration. */
typedef struct PdasIterState {
    int64_t chol_fail;       /* -1 ok, else failing column (linalg.py:120-122)   */
    int64_t blocking;        /* ratio-test argmin in [0,2n): j = x_j, n+j = s_j    */
    int32_t cascade_fail;    /* 0 or 1-based breakdown step (normal.py:172-173)  */
    uint32_t interior_flags; /* bit0 x NaN, bit1 x<=0, bit2 s NaN, bit3 s<=0       */
    int32_t nonfinite;       /* 1: dx, dy or ds has a non-finite entry (:229-235)  */
    int32_t stepped;         /* 1: x, y, s were updated this iteration             */
    int32_t fallback;        /* 1: dy came from the direct solve (:161-165)       */
    int32_t reserved;
    double alpha, gap, pobj, dobj, r_primal, r_dual, r_comp, min_ratio;
} PdasIterState;

int pdas_abi_version(void);
const char* pdas_last_error(void);
/* SM count and compute capability of the current device. */
int pdas_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* Largest m the rank-one cascade kernels are compiled for. */
int64_t pdas_cascade_max_m(void);

/* ---- kernel table (adascale/_kernels.pyx) --------------------------------- */

/* dot_tree, _kernels.pyx:55-71.  *out_dev = tree_i u[i*su]*v[i*sv], n >= 1. */
int pdas_dot_tree(const double* u, int64_t su, const double* v, int64_t sv, int64_t n,
                  double* out_dev, void* stream);

/* mat_vec, _kernels.pyx:74-88.  out[i] = tree_k a[i,k]*x[k]; a is m x n. */
int pdas_mat_vec(const double* a, int64_t m, int64_t n, const double* x, double* out,
                 void* stream);

/* mat_t_vec, _kernels.pyx:91-105.  out[j] = tree_i a[i,j]*y[i]. */
int pdas_mat_t_vec(const double* a, int64_t m, int64_t n, const double* y, double* out,
                   void* stream);

/* gram, _kernels.pyx:108-123.  g (m x m) = A A^T, sequential k, mirrored. */
int pdas_gram(const double* a, int64_t m, int64_t n, double* g, void* stream);

/* scaled_gram, _kernels.pyx:126-141.  g = A diag(d) A^T (w = a[j,k]*d[k]). */
int pdas_scaled_gram(const double* a, int64_t m, int64_t n, const double* d, double* g,
                     void* stream);

/* cholesky_factor, _kernels.pyx:144-171.  low (nn x nn) is fully written
 * (zeros above the diagonal and in columns >= the failing one);
 * *fail_dev = -1 on success, else the first failing column. */
int pdas_cholesky_factor(const double* g, int64_t nn, double eps_rel, double* low,
                         int64_t* fail_dev, void* stream);

/* cholesky_solve_many, _kernels.pyx:174-193.  Solves (L L^T) X = B in place
 * on x (m x k). */
int pdas_cholesky_solve_many(const double* low, int64_t m, double* x, int64_t k, void* stream);

/* build_v, _kernels.pyx:196-202.  v[i] = a[i,l0]*(dl - 1). */
int pdas_build_v(const double* a, int64_t m, int64_t l0, double dl, double* v, void* stream);

/* sweep_phase1, _kernels.pyx:205-218.  inner[k] = tree(v, cols[:,k]), k in [k0,k1). */
int pdas_sweep_phase1(const double* cols, int64_t m, const double* v, double* inner, int64_t k0,
                      int64_t k1, void* stream);

/* sweep_phase2, _kernels.pyx:221-231.  cols[:,k] -= (inner[k]/denom)*cols[:,l0]. */
int pdas_sweep_phase2(double* cols, int64_t m, int64_t l0, const double* inner, double denom,
                      int64_t k0, int64_t k1, void* stream);

/* solve_sweeps / _cascade, _kernels.pyx:234-291.  The full Egidi-Maponi
 * cascade in place on cols (m x (n+1)) = [Y | x]; *fail_dev = 0 or the
 * 1-based breakdown step.  `inner` and `v` are accepted for interface parity
 * (scratch, contents unspecified afterwards, as in the reference);
 * `workers` is accepted and ignored (results never depend on it). */
int pdas_solve_sweeps(double* cols, const double* a, const double* d, double* inner, double* v,
                      int64_t m, int64_t n, int workers, int32_t* fail_dev, void* stream);

/* Same cascade with a caller-owned workspace (no per-call allocation): ws
 * holds the step denominators and the inter-CTA panel flags; it must be
 * zeroed once, then reused with epoch = 1, 2, 3, ... (strictly increasing on
 * that ws).  Used by the solver engine once per PDAS iteration. */
int64_t pdas_cascade_ws_bytes(int64_t m, int64_t n);
int pdas_solve_sweeps_ws(double* cols, const double* a, const double* d, int64_t m, int64_t n,
                         void* ws, int32_t epoch, int32_t* fail_dev, void* stream);

/* init_workspace's x0 solve fused with the cascade (normal.py:115-124 then
 * :163-175): on entry column n of cols holds the right-hand side A x; the
 * library solves x0 = L0^-T L0^-1 rhs into it (same rounding sequence as
 * cholesky_solve_many with k = 1) and runs the cascade.  When column n sits
 * alone in the last column tile the x0 solve and that tile's updates run on
 * their own stream, overlapped with the Y part of the cascade. */
int pdas_solve_sweeps_ws_x0(double* cols, const double* a, const double* d, const double* low,
                            int64_t m, int64_t n, void* ws, int32_t epoch, int32_t* fail_dev,
                            void* stream);

/* Building blocks of the cascade for column-sharded (multi-GPU) execution,
 * parallel.py:1-7 / the per-step column independence of _kernels.pyx:260-289.
 * Pivots come in blocks of pdas_cascade_block_pivots(); columns in tiles of
 * pdas_cascade_tile_width(m) (tile t = columns [t*w, t*w+w) of [Y|x]).
 *
 * panel: for block [p0, p1) whose tiles have had every pivot < q0 applied,
 * apply the previous block [q0, p0) (denominators in ws), then run the
 * block's own steps in order: after it, columns [p0, p1) are final, their
 * denominators are in ws and a breakdown sets *fail_dev = l + 1.  The tiles
 * touched are those covering [p0, p1) (including column n when it shares the
 * last tile).  No-op when *fail_dev != 0 on entry.
 *
 * update: apply pivots [p0, p1) (final columns + denominators already in
 * cols/ws) to the listed tiles (device int64 array, any order, each tile past
 * p1).  No-op when *fail_dev != 0.  ws/epoch follow pdas_solve_sweeps_ws. */
int pdas_cascade_tile_width(int64_t m);
int pdas_cascade_block_pivots(void);
/* The chained (early-panel) form of the two blocks, as on one GPU: an update
 * that also publishes tile_done[t] = utag for every tile it updates, and a
 * panel over block [p0, p1) that applies no previous block itself but waits
 * in-kernel until each of its tiles reports tile_done == utag (the rank's own
 * update of the previous block).  utag = b + 1 for block b's update; the
 * tags are zeroed per cascade with pdas_cascade_reset_tags.  dist.py. */
int pdas_cascade_panel_chained(double* cols, const double* a, const double* d, int64_t m,
                               int64_t n, int64_t p0, int64_t p1, void* ws, int32_t epoch,
                               int32_t* fail_dev, int32_t utag, void* stream);
int pdas_cascade_update_tagged(double* cols, const double* a, const double* d, int64_t m,
                               int64_t n, int64_t p0, int64_t p1, const int64_t* tiles_dev,
                               int64_t ntiles, void* ws, int32_t* fail_dev, int32_t utag,
                               void* stream);
int pdas_cascade_reset_tags(void* ws, int64_t n, void* stream);
/* Pivots in the first block of the 1-GPU cascade (pdas_solve_sweeps_ws / _x0);
 * the later blocks have twice as many. */
int pdas_cascade_solve_block(void);
/* Pivot blocks (panel + update launches each) of the 1-GPU cascade of (m, n);
 * 0 for the one-CTA cascade (a single kernel). */
int64_t pdas_cascade_solve_blocks(int64_t m, int64_t n);
/* 1 when pdas_solve_sweeps_ws(_x0) runs (m, n) as the one-CTA shared-memory
 * cascade (m <= 64, [Y|x] + A in 200 KB): no pivot-block flags, so the call
 * is independent of the epoch and can be replayed from a CUDA graph. */
int pdas_cascade_one_cta(int64_t m, int64_t n);
int pdas_cascade_panel(double* cols, const double* a, const double* d, int64_t m, int64_t n,
                       int64_t q0, int64_t p0, int64_t p1, void* ws, int32_t epoch,
                       int32_t* fail_dev, void* stream);
int pdas_cascade_update(double* cols, const double* a, const double* d, int64_t m, int64_t n,
                        int64_t p0, int64_t p1, const int64_t* tiles_dev, int64_t ntiles,
                        void* ws, int32_t* fail_dev, void* stream);

/* The block exchange of the sharded cascade fused into the panel (SURVEY.md
 * §8(e): the pivot owner's finished columns go to every peer by in-kernel
 * NVLink stores instead of an NCCL broadcast per block; replaces the
 * torch.distributed.broadcast calls of dist.run_collective, which stand where
 * the reference's thread pool shares one address space, parallel.py:169-209).
 * panel_peers: pdas_cascade_panel, plus each panel tile stores its final
 * columns from registers into every peer's cols, its denominators into the
 * peer's ws, a breakdown into the peer's fail word, then releases a
 * system-scope flag per tile in the peer's ws.  peer_cols / peer_ws /
 * peer_fail: HOST arrays of npeers (<= 7) device addresses valid in this
 * process (CUDA IPC / symmetric-memory peer mappings).
 * peer_wait: on a non-owner, block the stream until every tile covering
 * columns [c0, c1) has been released for `epoch` (traps after 30 s). */
int pdas_cascade_panel_peers(double* cols, const double* a, const double* d, int64_t m, int64_t n,
                             int64_t q0, int64_t p0, int64_t p1, void* ws, int32_t epoch,
                             int32_t* fail_dev, int32_t npeers, const uint64_t* peer_cols,
                             const uint64_t* peer_ws, const uint64_t* peer_fail, void* stream);
int pdas_cascade_peer_wait(void* ws, int64_t m, int64_t n, int64_t c0, int64_t c1, int32_t epoch,
                           void* stream);

/* cholesky_solve (linalg.py:126-132) for ONE right-hand side, in place on
 * x (m): the per-iteration x0 = L0^-T L0^-1 (A x) of init_workspace
 * (normal.py:123).  Same rounding sequence as cholesky_solve_many with k=1,
 * scheduled for latency (one CTA: right-looking forward sweep, backward
 * chain fed by helper warps). */
int pdas_cholesky_solve_one(const double* low, int64_t m, double* x, void* stream);

/* ---- fused per-iteration path (adascale/solver.py) ------------------------- */

/* Reset *state (all zero, chol_fail = -1). */
int pdas_iter_reset(PdasIterState* state, void* stream);

/* scaling_diag + check_interior, solver.py:142-145 / model.py:116-119:
 * d = x/s, interior flags into state. */
int pdas_iter_scaling(const double* x, const double* s, int64_t n, double* d,
                      PdasIterState* state, void* stream);

/* compute_directions tail + step_length, solver.py:166-189: t = A^T dy,
 * ds = -t, dx = d*t - x, residuals, finiteness, ratio test, alpha and the
 * step decision.  Needs state->cascade_fail / chol_fail already final. */
int pdas_iter_directions(const double* a, int64_t m, int64_t n, const double* dy,
                         const double* d, const double* x, const double* s, double* dx,
                         double* ds, double rho, PdasIterState* state, void* stream);

/* The damped ratio test alone on given directions (the public step_length,
 * solver.py:175-189): state->alpha = rho * min(-x/dx | dx < 0, -s/ds | ds < 0),
 * CAP_ALPHA (1e6) when no component blocks; state->blocking = first argmin over
 * [x ratios | s ratios] (-1 if none).  state is reset by the caller. */
int pdas_ratio_test(const double* x, const double* s, const double* dx, const double* ds,
                    int64_t n, double rho, PdasIterState* state, void* stream);

/* x += alpha*dx, y += alpha*dy, s += alpha*ds when state->stepped (solver.py:257-259). */
int pdas_iter_update(double* x, double* y, double* s, const double* dx, const double* dy,
                     const double* ds, int64_t n, int64_t m, const PdasIterState* state,
                     void* stream);

/* gap = tree(x,s), pobj = tree(c,x), dobj = tree(b,y)  (solver.py:192-194, 246-247). */
int pdas_iter_objectives(const double* x, const double* s, const double* c, const double* b,
                         const double* y, int64_t n, int64_t m, PdasIterState* state,
                         void* stream);

/* ---- diagnostics ----------------------------------------------------------- */

/* Sustained separately-rounded fp64 multiply+add rate probe (the cascade's
 * instruction mix); *ops = number of fp64 operations the launch performs.
 * Time it with events on `stream` to get the roofline denominator. */
int pdas_probe_fp64(double* sink, int64_t iters, int64_t* ops, void* stream);

/* The cascade divides every column's inner product by the step denominator
 * with the reciprocal refinement hoisted per pivot (common.cuh div_by); this
 * writes that result and the plain IEEE a/b side by side for n operand pairs
 * so tests can check they are the same bits. */
int pdas_selftest_div(const double* a, const double* b, int64_t n, double* out_fast,
                      double* out_ref, void* stream);

/* With PDAS_CASCADE_PROFILE=1 in the environment the 1-GPU cascade records
 * CUDA events around each update / panel launch (and synchronises at its
 * end).  Copies the last cascade's rows {kind (0 update, 1 panel), block,
 * start ms, end ms} (host memory, up to max_rows) and returns the row count. */
int64_t pdas_debug_cascade_profile(double* out, int64_t max_rows);

#ifdef __cplusplus
}
#endif

#endif /* PDAS_B200_H */
