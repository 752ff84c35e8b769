// abi.cu -- extern "C" entry points declared in include/pdas_b200.h.
// Thin: validate arguments, allocate stream-ordered scratch, launch, map
// CUDA errors to PDAS_ERR_CUDA with a per-thread message.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include "pdas_internal.h"

namespace {

thread_local char g_err[512] = "";

int set_err(int code, const char* what) {
    snprintf(g_err, sizeof g_err, "%s", what);
    return code;
}

int check_cuda(int rc, const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "%s: %s", where, cudaGetErrorString(e));
        return PDAS_ERR_CUDA;
    }
    if (rc == PDAS_ERR_UNSUPPORTED) return set_err(rc, where);
    if (rc == PDAS_ERR_ARG) return set_err(rc, where);
    if (rc != PDAS_OK) {
        snprintf(g_err, sizeof g_err, "%s: error %d", where, rc);
        return rc;
    }
    return PDAS_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Keep freed stream-ordered scratch in the device pool across synchronisations
// (the default release threshold of 0 hands it back to the driver at every
// sync, turning each per-call scratch allocation into a real allocation).
void retain_pool() {
    static thread_local int done[16] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    if (done[dev & 15]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done[dev & 15] = 1;
}

template <class T>
int scratch(T** p, size_t count, cudaStream_t st) {
    *p = nullptr;
    if (count == 0) return PDAS_OK;
    retain_pool();
    if (cudaMallocAsync((void**)p, count * sizeof(T), st) != cudaSuccess) {
        cudaGetLastError();
        return set_err(PDAS_ERR_NOMEM, "cudaMallocAsync failed");
    }
    return PDAS_OK;
}

}  // namespace

using pdas::idx_t;

extern "C" {

int pdas_abi_version(void) { return PDAS_ABI_VERSION; }

const char* pdas_last_error(void) { return g_err; }

int pdas_device_info(int* sm_count, int* cc_major, int* cc_minor) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return check_cuda(PDAS_OK, "cudaGetDevice");
    if (sm_count) cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    return check_cuda(PDAS_OK, "pdas_device_info");
}

int64_t pdas_cascade_max_m(void) { return pdas::cascade_supported_m(); }

int pdas_dot_tree(const double* u, int64_t su, const double* v, int64_t sv, int64_t n,
                  double* out_dev, void* stream) {
    if (n < 1) return set_err(PDAS_ERR_ARG, "dot_tree requires length >= 1");
    return check_cuda(pdas::launch_dot_tree(u, su, v, sv, n, out_dev, S(stream)), "dot_tree");
}

int pdas_mat_vec(const double* a, int64_t m, int64_t n, const double* x, double* out,
                 void* stream) {
    if (m < 0 || n < 1) return set_err(PDAS_ERR_ARG, "mat_vec: bad shape");
    double* work = nullptr;
    int rc = scratch(&work, (size_t)pdas::mat_vec_scratch(m, n), S(stream));
    if (rc) return rc;
    rc = pdas::launch_mat_vec(a, m, n, x, out, work, S(stream));
    if (work) cudaFreeAsync(work, S(stream));
    return check_cuda(rc, "mat_vec");
}

int pdas_mat_t_vec(const double* a, int64_t m, int64_t n, const double* y, double* out,
                   void* stream) {
    if (m < 1 || n < 0) return set_err(PDAS_ERR_ARG, "mat_t_vec: bad shape");
    return check_cuda(pdas::launch_mat_t_vec(a, m, n, y, out, S(stream)), "mat_t_vec");
}

int pdas_gram(const double* a, int64_t m, int64_t n, double* g, void* stream) {
    if (m < 1 || n < 0) return set_err(PDAS_ERR_ARG, "gram: bad shape");
    return check_cuda(pdas::launch_gram(a, m, n, nullptr, g, S(stream)), "gram");
}

int pdas_scaled_gram(const double* a, int64_t m, int64_t n, const double* d, double* g,
                     void* stream) {
    if (m < 1 || n < 0 || d == nullptr) return set_err(PDAS_ERR_ARG, "scaled_gram: bad args");
    return check_cuda(pdas::launch_gram(a, m, n, d, g, S(stream)), "scaled_gram");
}

int pdas_cholesky_factor(const double* g, int64_t nn, double eps_rel, double* low,
                         int64_t* fail_dev, void* stream) {
    if (nn < 1) return set_err(PDAS_ERR_ARG, "cholesky_factor: bad shape");
    double* work = nullptr;
    int rc = scratch(&work, (size_t)pdas::cholesky_work_doubles(nn), S(stream));
    if (rc) return rc;
    rc = pdas::launch_cholesky(g, nn, eps_rel, low, fail_dev, work, S(stream));
    cudaFreeAsync(work, S(stream));
    return check_cuda(rc, "cholesky_factor");
}

int pdas_cholesky_solve_many(const double* low, int64_t m, double* x, int64_t k, void* stream) {
    if (m < 1 || k < 0) return set_err(PDAS_ERR_ARG, "cholesky_solve_many: bad shape");
    double* work = nullptr;
    int rc = scratch(&work, (size_t)pdas::solve_many_work_doubles(m, k), S(stream));
    if (rc) return rc;
    rc = pdas::launch_solve_many(low, m, x, k, work, S(stream));
    if (work) cudaFreeAsync(work, S(stream));
    return check_cuda(rc, "cholesky_solve_many");
}

int pdas_build_v(const double* a, int64_t m, int64_t l0, double dl, double* v, void* stream) {
    if (m < 1 || l0 < 0) return set_err(PDAS_ERR_ARG, "build_v: bad args");
    return check_cuda(pdas::launch_build_v(a, m, l0, dl, v, S(stream)), "build_v");
}

int pdas_sweep_phase1(const double* cols, int64_t m, const double* v, double* inner, int64_t k0,
                      int64_t k1, void* stream) {
    if (m < 1 || k0 < 0) return set_err(PDAS_ERR_ARG, "sweep_phase1: bad args");
    return check_cuda(pdas::launch_sweep_phase1(cols, m, v, inner, k0, k1, S(stream)),
                      "sweep_phase1");
}

int pdas_sweep_phase2(double* cols, int64_t m, int64_t l0, const double* inner, double denom,
                      int64_t k0, int64_t k1, void* stream) {
    if (m < 1 || k0 <= l0) return set_err(PDAS_ERR_ARG, "sweep_phase2: needs k0 > l0");
    return check_cuda(pdas::launch_sweep_phase2(cols, m, l0, inner, denom, k0, k1, S(stream)),
                      "sweep_phase2");
}

int pdas_solve_sweeps(double* cols, const double* a, const double* d, double* inner, double* v,
                      int64_t m, int64_t n, int workers, int32_t* fail_dev, void* stream) {
    (void)inner;
    (void)v;
    (void)workers;
    if (m < 1 || n < 0 || fail_dev == nullptr) return set_err(PDAS_ERR_ARG, "solve_sweeps: bad args");
    if (m > pdas::cascade_supported_m())
        return set_err(PDAS_ERR_UNSUPPORTED, "solve_sweeps: m above the compiled configurations");
    unsigned char* ws = nullptr;
    const size_t bytes = (size_t)pdas_cascade_ws_bytes(m, n);
    int rc = scratch(&ws, bytes, S(stream));
    if (rc) return rc;
    cudaMemsetAsync(ws, 0, bytes, S(stream));
    rc = pdas_solve_sweeps_ws(cols, a, d, m, n, ws, 1, fail_dev, stream);
    cudaFreeAsync(ws, S(stream));
    return rc;
}

int64_t pdas_cascade_ws_bytes(int64_t m, int64_t n) {
    const int64_t nd = n > 0 ? n : 1;
    return (int64_t)(((nd * 8 + 255) / 256) * 256 + pdas::cascade_flags_count(m, n) * 4);
}

int pdas_solve_sweeps_ws(double* cols, const double* a, const double* d, int64_t m, int64_t n,
                         void* ws, int32_t epoch, int32_t* fail_dev, void* stream) {
    if (m < 1 || n < 0 || fail_dev == nullptr || ws == nullptr || epoch < 1)
        return set_err(PDAS_ERR_ARG, "solve_sweeps_ws: bad args");
    if (m > pdas::cascade_supported_m())
        return set_err(PDAS_ERR_UNSUPPORTED, "solve_sweeps: m above the compiled configurations");
    const int64_t nd = n > 0 ? n : 1;
    double* denoms = static_cast<double*>(ws);
    int* flags = reinterpret_cast<int*>(static_cast<unsigned char*>(ws) + ((nd * 8 + 255) / 256) * 256);
    return check_cuda(
        pdas::launch_cascade(cols, a, d, m, n, denoms, fail_dev, flags, epoch, 0, S(stream)),
        "solve_sweeps");
}

int pdas_solve_sweeps_ws_x0(double* cols, const double* a, const double* d, const double* low,
                            int64_t m, int64_t n, void* ws, int32_t epoch, int32_t* fail_dev,
                            void* stream) {
    if (m < 1 || n < 0 || fail_dev == nullptr || ws == nullptr || epoch < 1 || low == nullptr)
        return set_err(PDAS_ERR_ARG, "solve_sweeps_ws_x0: bad args");
    if (m > pdas::cascade_supported_m())
        return set_err(PDAS_ERR_UNSUPPORTED, "solve_sweeps: m above the compiled configurations");
    const int64_t nd = n > 0 ? n : 1;
    double* denoms = static_cast<double*>(ws);
    int* flags = reinterpret_cast<int*>(static_cast<unsigned char*>(ws) + ((nd * 8 + 255) / 256) * 256);
    double* work = nullptr;
    int rc = scratch(&work, (size_t)pdas::solve_one_work_doubles(m), S(stream));
    if (rc) return rc;
    rc = pdas::launch_cascade_x0(cols, a, d, low, m, n, denoms, fail_dev, flags, epoch, work,
                                 S(stream));
    if (work) cudaFreeAsync(work, S(stream));
    return check_cuda(rc, "solve_sweeps_ws_x0");
}

int pdas_cascade_tile_width(int64_t m) {
    if (m < 1 || m > pdas::cascade_supported_m()) return 0;
    return pdas::cascade_tile_width(m);
}

int pdas_cascade_block_pivots(void) { return pdas::kShardBlock; }
int pdas_cascade_solve_block(void) { return pdas::kSolveBlock; }
int pdas_cascade_one_cta(int64_t m, int64_t n) { return pdas::cascade_one_cta(m, n) ? 1 : 0; }
int64_t pdas_cascade_solve_blocks(int64_t m, int64_t n) {
    if (m < 1 || n < 1 || pdas::cascade_one_cta(m, n)) return 0;
    return pdas::cascade_solve_blocks(n);
}

int64_t pdas_debug_cascade_profile(double* out, int64_t max_rows) {
    if (max_rows < 0 || (max_rows > 0 && out == nullptr)) return -1;
    return pdas::cascade_profile_rows(out, max_rows);
}

static int split_ws(void* ws, int64_t n, double** denoms, int** flags) {
    const int64_t nd = n > 0 ? n : 1;
    *denoms = static_cast<double*>(ws);
    *flags = reinterpret_cast<int*>(static_cast<unsigned char*>(ws) + ((nd * 8 + 255) / 256) * 256);
    return 0;
}

int pdas_cascade_panel(double* cols, const double* a, const double* d, int64_t m, int64_t n,
                       int64_t q0, int64_t p0, int64_t p1, void* ws, int32_t epoch,
                       int32_t* fail_dev, void* stream) {
    if (m < 1 || n < 1 || fail_dev == nullptr || ws == nullptr || epoch < 1)
        return set_err(PDAS_ERR_ARG, "cascade_panel: bad args");
    if (m > pdas::cascade_supported_m())
        return set_err(PDAS_ERR_UNSUPPORTED, "cascade_panel: m above the compiled configurations");
    const int ct = pdas::cascade_tile_width(m);
    if (q0 < 0 || q0 > p0 || p0 >= p1 || p1 > n || p0 % ct != 0 || q0 % ct != 0 ||
        p1 - p0 > pdas::kShardBlock || p0 - q0 > pdas::kShardBlock)
        return set_err(PDAS_ERR_ARG, "cascade_panel: block bounds");
    double* denoms;
    int* flags;
    split_ws(ws, n, &denoms, &flags);
    return check_cuda(pdas::launch_cascade_panel(cols, a, d, m, n, q0, p0, p1, denoms, fail_dev,
                                                 flags, epoch, S(stream)),
                      "cascade_panel");
}

int pdas_cascade_panel_peers(double* cols, const double* a, const double* d, int64_t m, int64_t n,
                             int64_t q0, int64_t p0, int64_t p1, void* ws, int32_t epoch,
                             int32_t* fail_dev, int32_t npeers, const uint64_t* peer_cols,
                             const uint64_t* peer_ws, const uint64_t* peer_fail, void* stream) {
    if (m < 1 || n < 1 || fail_dev == nullptr || ws == nullptr || epoch < 1 || npeers < 0 ||
        npeers > pdas::kMaxPeers ||
        (npeers > 0 && (peer_cols == nullptr || peer_ws == nullptr || peer_fail == nullptr)))
        return set_err(PDAS_ERR_ARG, "cascade_panel_peers: bad args");
    if (m > pdas::cascade_supported_m())
        return set_err(PDAS_ERR_UNSUPPORTED,
                       "cascade_panel_peers: m above the compiled configurations");
    const int ct = pdas::cascade_tile_width(m);
    if (q0 < 0 || q0 > p0 || p0 >= p1 || p1 > n || p0 % ct != 0 || q0 % ct != 0 ||
        p1 - p0 > pdas::kShardBlock || p0 - q0 > pdas::kShardBlock)
        return set_err(PDAS_ERR_ARG, "cascade_panel_peers: block bounds");
    double* denoms;
    int* flags;
    split_ws(ws, n, &denoms, &flags);
    double* pc[pdas::kMaxPeers];
    double* pd[pdas::kMaxPeers];
    int32_t* pf[pdas::kMaxPeers];
    int* pg[pdas::kMaxPeers];
    for (int q = 0; q < npeers; ++q) {
        pc[q] = reinterpret_cast<double*>(peer_cols[q]);
        pf[q] = reinterpret_cast<int32_t*>(peer_fail[q]);
        split_ws(reinterpret_cast<void*>(peer_ws[q]), n, &pd[q], &pg[q]);
    }
    return check_cuda(pdas::launch_cascade_panel_peers(cols, a, d, m, n, q0, p0, p1, denoms,
                                                       fail_dev, flags, epoch, npeers, pc, pd, pf,
                                                       pg, S(stream)),
                      "cascade_panel_peers");
}

int pdas_cascade_peer_wait(void* ws, int64_t m, int64_t n, int64_t c0, int64_t c1, int32_t epoch,
                           void* stream) {
    if (m < 1 || n < 1 || ws == nullptr || epoch < 1 || c0 < 0 || c1 < c0 || c1 > n + 1)
        return set_err(PDAS_ERR_ARG, "cascade_peer_wait: bad args");
    if (m > pdas::cascade_supported_m())
        return set_err(PDAS_ERR_UNSUPPORTED, "cascade_peer_wait: m above the compiled configurations");
    double* denoms;
    int* flags;
    split_ws(ws, n, &denoms, &flags);
    return check_cuda(pdas::launch_peer_wait(flags, m, c0, c1, epoch, S(stream)),
                      "cascade_peer_wait");
}

int pdas_cascade_update(double* cols, const double* a, const double* d, int64_t m, int64_t n,
                        int64_t p0, int64_t p1, const int64_t* tiles_dev, int64_t ntiles,
                        void* ws, int32_t* fail_dev, void* stream) {
    if (m < 1 || n < 1 || fail_dev == nullptr || ws == nullptr || ntiles < 0 ||
        (ntiles > 0 && tiles_dev == nullptr))
        return set_err(PDAS_ERR_ARG, "cascade_update: bad args");
    if (m > pdas::cascade_supported_m())
        return set_err(PDAS_ERR_UNSUPPORTED, "cascade_update: m above the compiled configurations");
    if (p0 < 0 || p0 >= p1 || p1 > n || p1 - p0 > pdas::kShardBlock)
        return set_err(PDAS_ERR_ARG, "cascade_update: block bounds");
    double* denoms;
    int* flags;
    split_ws(ws, n, &denoms, &flags);
    return check_cuda(pdas::launch_cascade_update(cols, a, d, m, n, p0, p1, tiles_dev, ntiles,
                                                  denoms, fail_dev, S(stream)),
                      "cascade_update");
}

int pdas_cascade_panel_chained(double* cols, const double* a, const double* d, int64_t m,
                               int64_t n, int64_t p0, int64_t p1, void* ws, int32_t epoch,
                               int32_t* fail_dev, int32_t utag, void* stream) {
    if (m < 1 || n < 1 || fail_dev == nullptr || ws == nullptr || epoch < 1 || utag < 0)
        return set_err(PDAS_ERR_ARG, "cascade_panel_chained: bad args");
    if (m > pdas::cascade_supported_m())
        return set_err(PDAS_ERR_UNSUPPORTED,
                       "cascade_panel_chained: m above the compiled configurations");
    const int ct = pdas::cascade_tile_width(m);
    if (p0 < 0 || p0 >= p1 || p1 > n || p0 % ct != 0 || p1 - p0 > pdas::kShardBlock)
        return set_err(PDAS_ERR_ARG, "cascade_panel_chained: block bounds");
    double* denoms;
    int* flags;
    split_ws(ws, n, &denoms, &flags);
    return check_cuda(pdas::launch_cascade_panel(cols, a, d, m, n, p0, p0, p1, denoms, fail_dev,
                                                 flags, epoch, S(stream), nullptr, utag),
                      "cascade_panel_chained");
}

int pdas_cascade_update_tagged(double* cols, const double* a, const double* d, int64_t m,
                               int64_t n, int64_t p0, int64_t p1, const int64_t* tiles_dev,
                               int64_t ntiles, void* ws, int32_t* fail_dev, int32_t utag,
                               void* stream) {
    if (m < 1 || n < 1 || fail_dev == nullptr || ws == nullptr || ntiles < 0 || utag < 1 ||
        (ntiles > 0 && tiles_dev == nullptr))
        return set_err(PDAS_ERR_ARG, "cascade_update_tagged: bad args");
    if (m > pdas::cascade_supported_m())
        return set_err(PDAS_ERR_UNSUPPORTED,
                       "cascade_update_tagged: m above the compiled configurations");
    if (p0 < 0 || p0 >= p1 || p1 > n || p1 - p0 > pdas::kShardBlock)
        return set_err(PDAS_ERR_ARG, "cascade_update_tagged: block bounds");
    double* denoms;
    int* flags;
    split_ws(ws, n, &denoms, &flags);
    return check_cuda(pdas::launch_cascade_update(cols, a, d, m, n, p0, p1, tiles_dev, ntiles,
                                                  denoms, fail_dev, S(stream), flags, utag),
                      "cascade_update_tagged");
}

int pdas_cascade_reset_tags(void* ws, int64_t n, void* stream) {
    if (ws == nullptr || n < 1) return set_err(PDAS_ERR_ARG, "cascade_reset_tags: bad args");
    double* denoms;
    int* flags;
    split_ws(ws, n, &denoms, &flags);
    return check_cuda(
        cudaMemsetAsync(flags + pdas::panel_flag_ints(n), 0,
                        sizeof(int) * (size_t)pdas::panel_flag_ints(n), S(stream)) == cudaSuccess
            ? PDAS_OK
            : PDAS_ERR_CUDA,
        "cascade_reset_tags");
}

int pdas_cholesky_solve_one(const double* low, int64_t m, double* x, void* stream) {
    if (m < 1) return set_err(PDAS_ERR_ARG, "cholesky_solve_one: bad shape");
    double* work = nullptr;
    int rc = scratch(&work, (size_t)pdas::solve_one_work_doubles(m), S(stream));
    if (rc) return rc;
    rc = pdas::launch_solve_one(low, m, x, work, S(stream));
    if (work) cudaFreeAsync(work, S(stream));
    return check_cuda(rc, "cholesky_solve_one");
}

// ------------------------------------------------------------------ iteration
__global__ void k_iter_reset(PdasIterState* st) {
    PdasIterState z;
    memset(&z, 0, sizeof z);
    z.chol_fail = -1;
    z.blocking = -1;
    *st = z;
}

int pdas_iter_reset(PdasIterState* state, void* stream) {
    k_iter_reset<<<1, 1, 0, S(stream)>>>(state);
    return check_cuda(PDAS_OK, "iter_reset");
}

int pdas_iter_scaling(const double* x, const double* s, int64_t n, double* d,
                      PdasIterState* state, void* stream) {
    if (n < 1) return set_err(PDAS_ERR_ARG, "iter_scaling: n < 1");
    unsigned* flags = &state->interior_flags;
    return check_cuda(pdas::launch_scaling(x, s, n, d, flags, S(stream)), "iter_scaling");
}

int pdas_iter_directions(const double* a, int64_t m, int64_t n, const double* dy,
                         const double* d, const double* x, const double* s, double* dx,
                         double* ds, double rho, PdasIterState* state, void* stream) {
    if (m < 1 || n < 1) return set_err(PDAS_ERR_ARG, "iter_directions: bad shape");
    cudaStream_t st = S(stream);
    void* parts = nullptr;
    double* adx = nullptr;
    double* mvw = nullptr;
    int rc = scratch((unsigned char**)&parts, (size_t)pdas::directions_partials_bytes(n), st);
    if (!rc) rc = scratch(&adx, (size_t)m, st);
    if (!rc) rc = scratch(&mvw, (size_t)pdas::mat_vec_scratch(m, n), st);
    if (!rc) rc = pdas::launch_directions(a, m, n, dy, d, x, s, dx, ds, parts, st);
    if (!rc) rc = pdas::launch_mat_vec(a, m, n, dx, adx, mvw, st);
    if (!rc) rc = pdas::launch_dir_finish(parts, n, adx, m, dy, rho, state, st);
    if (parts) cudaFreeAsync(parts, st);
    if (adx) cudaFreeAsync(adx, st);
    if (mvw) cudaFreeAsync(mvw, st);
    return check_cuda(rc, "iter_directions");
}

int pdas_ratio_test(const double* x, const double* s, const double* dx, const double* ds,
                    int64_t n, double rho, PdasIterState* state, void* stream) {
    if (n < 1) return set_err(PDAS_ERR_ARG, "ratio_test: bad shape");
    cudaStream_t st = S(stream);
    void* parts = nullptr;
    int rc = scratch((unsigned char**)&parts, (size_t)pdas::ratio_partials_bytes(n), st);
    if (!rc) rc = pdas::launch_ratio_test(x, s, dx, ds, n, rho, parts, state, st);
    if (parts) cudaFreeAsync(parts, st);
    return check_cuda(rc, "ratio_test");
}

int pdas_iter_update(double* x, double* y, double* s, const double* dx, const double* dy,
                     const double* ds, int64_t n, int64_t m, const PdasIterState* state,
                     void* stream) {
    if (n < 1 || m < 1 || m > n) return set_err(PDAS_ERR_ARG, "iter_update: bad shape");
    return check_cuda(pdas::launch_update(x, y, s, dx, dy, ds, n, m, state, S(stream)),
                      "iter_update");
}

int pdas_iter_objectives(const double* x, const double* s, const double* c, const double* b,
                         const double* y, int64_t n, int64_t m, PdasIterState* state,
                         void* stream) {
    if (n < 1 || m < 1) return set_err(PDAS_ERR_ARG, "iter_objectives: bad shape");
    return check_cuda(pdas::launch_dot3(x, s, n, &state->gap, c, x, n, &state->pobj, b, y, m,
                                        &state->dobj, S(stream)),
                      "iter_objectives");
}

int pdas_probe_fp64(double* sink, int64_t iters, int64_t* ops, void* stream) {
    if (iters < 1 || ops == nullptr) return set_err(PDAS_ERR_ARG, "probe_fp64: bad args");
    int64_t o = 0;
    int rc = pdas::launch_fp64_probe(sink, iters, &o, S(stream));
    *ops = o;
    return check_cuda(rc, "probe_fp64");
}

int pdas_selftest_div(const double* a, const double* b, int64_t n, double* out_fast,
                      double* out_ref, void* stream) {
    if (n < 0 || (n > 0 && (!a || !b || !out_fast || !out_ref)))
        return set_err(PDAS_ERR_ARG, "selftest_div: bad args");
    return check_cuda(pdas::launch_div_selftest(a, b, n, out_fast, out_ref, S(stream)),
                      "selftest_div");
}

}  // extern "C"
