// extern "C" entry points: transforms (transform.hpp:54-96) and the ImexOde operators
// (swe.hpp:44-79). All data pointers are device pointers; see include/pswe.h.
#include "pswe_internal.h"

using namespace pswe;

namespace {

void need(const void* p, const char* what) {
    if (!p) throw std::invalid_argument(std::string(what) + " is NULL");
}
// data pointers of a batch of n: an empty batch (n <= 0) is a no-op and may pass NULL
void need(const void* p, const char* what, int n) {
    if (n > 0 && !p) throw std::invalid_argument(std::string(what) + " is NULL");
}

inline const double2* c2(const double* p) { return reinterpret_cast<const double2*>(p); }
inline double2* c2(double* p) { return reinterpret_cast<double2*>(p); }

int batch_groups(int n, int per) { return (n + per - 1) / per; }

}  // namespace

namespace pswe {

// eval_implicit + eval_explicit of n states: the hot path (swe.cpp:9-69).
// 4 launches: inverse Legendre (Phi, zeta, U, V) -> fused FFT/products/FFT -> forward Legendre
// (5 projections) -> tail (tendency assembly + linear operator).
// the evaluation up to the five projections in P.d_proj ([5n][Kx]); the tail (eval_tail, or the
// SDC sweep's fused tail + node update) turns them into F_E / F_I
// xprep: the state's X tiles were written by the preceding kernel (the SDC sweep's node update,
// n = 1, xtiles_by_sweep_ok) - the prep launch is skipped
void eval_imex_proj(pswe_plan& P, const pswe_params& prm, const double2* state, int n, cudaStream_t st, bool xprep) {
    P.reserve(n);
    if (xprep) legendre_inverse_prepared(P, P.d_four_a, st);
    else legendre_inverse(P, INV_EVAL, state, nullptr, n, prm.radius, P.d_four_a, st);
    if (gt_path_ok(P, n)) {  // grid stage writes forward G tiles directly
        fft_eval_products_gt(P, prm, P.d_four_a, n, st);
        legendre_forward_gt(P, n, P.d_proj, st);
    } else {
        fft_eval_products(P, prm, P.d_four_a, P.d_four_b, n, st);
        legendre_forward(P, P.d_four_b, 5, n, P.d_proj, true, st);
    }
}

void eval_imex(pswe_plan& P, const pswe_params& prm, const double2* state, double2* f_imp, double2* f_exp,
               int n, cudaStream_t st) {
    eval_imex_proj(P, prm, state, n, st);
    eval_tail(P, prm, P.d_proj, state, f_imp, f_exp, n, st);
}

}  // namespace pswe

extern "C" {

int pswe_device_alloc(unsigned long long bytes, void** out) {
    return guarded([&] {
        need(out, "out");
        PSWE_CUDA(cudaMalloc(out, bytes));
    });
}
int pswe_device_free(void* ptr) {
    return guarded([&] { PSWE_CUDA(cudaFree(ptr)); });
}
int pswe_memcpy_h2d(void* dst, const void* src, unsigned long long bytes, void* stream) {
    return guarded([&] { PSWE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream))); });
}
int pswe_memcpy_d2h(void* dst, const void* src, unsigned long long bytes, void* stream) {
    return guarded([&] { PSWE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream))); });
}
int pswe_stream_synchronize(void* stream) {
    return guarded([&] { PSWE_CUDA(cudaStreamSynchronize(as_stream(stream))); });
}

int pswe_synthesise(pswe_plan* P, const double* coeffs, double* grid, int n, void* stream) {
    PSWE_NVTX("pswe.synthesise");
    return guarded([&] {
        need(P, "plan");
        need(coeffs, "coeffs", n);
        need(grid, "grid", n);
        if (n <= 0) return;
        P->reserve(batch_groups(n, 5));
        legendre_inverse(*P, INV_PLAIN, c2(coeffs), nullptr, n, 1.0, P->d_four_a, as_stream(stream));
        fft_rows_c2r(*P, P->d_four_a, 1, 0, grid, n, false, as_stream(stream));
    });
}

int pswe_analyse(pswe_plan* P, const double* grid, double* coeffs, int n, void* stream) {
    PSWE_NVTX("pswe.analyse");
    return guarded([&] {
        need(P, "plan");
        need(coeffs, "coeffs", n);
        need(grid, "grid", n);
        if (n <= 0) return;
        P->reserve(batch_groups(n, 5));
        const GtLayout gl = gt_layout_fields(P->R, P->J, n);
        if (analyse_gt_ok(*P, gl) && fft_r2c_gt(*P, grid, gl, n, as_stream(stream))) {
            legendre_forward_fields_gt(*P, gl, n, c2(coeffs), as_stream(stream));
            return;
        }
        fft_rows_r2c(*P, grid, P->d_four_a, 1, 0, n, false, 0, 1.0, as_stream(stream));
        legendre_forward(*P, P->d_four_a, n, 1, c2(coeffs), false, as_stream(stream));
    });
}

int pswe_uv_from_vortdiv(pswe_plan* P, const double* vort, const double* div, double radius, double* u,
                         double* v, int n, void* stream) {
    PSWE_NVTX("pswe.uv_from_vortdiv");
    return guarded([&] {
        need(P, "plan");
        need(vort, "vort", n);
        need(div, "div", n);
        need(u, "u", n);
        need(v, "v", n);
        if (n <= 0) return;
        P->reserve(batch_groups(2 * n, 5));
        const cudaStream_t st = as_stream(stream);
        legendre_inverse(*P, INV_UV, c2(vort), c2(div), n, radius, P->d_four_a, st);
        fft_rows_c2r(*P, P->d_four_a, 2, 0, u, n, true, st);
        fft_rows_c2r(*P, P->d_four_a, 2, 1, v, n, true, st);
    });
}

int pswe_vortdiv_from_uv(pswe_plan* P, const double* u, const double* v, double radius, double* vort,
                         double* div, int n, void* stream) {
    PSWE_NVTX("pswe.vortdiv_from_uv");
    return guarded([&] {
        need(P, "plan");
        need(vort, "vort", n);
        need(div, "div", n);
        need(u, "u", n);
        need(v, "v", n);
        if (n <= 0) return;
        P->reserve(batch_groups(2 * n, 5));
        const cudaStream_t st = as_stream(stream);
        fft_rows_r2c(*P, u, P->d_four_a, 2, 0, n, true, 1, radius, st);
        fft_rows_r2c(*P, v, P->d_four_a, 2, 1, n, true, 1, radius, st);
        legendre_forward(*P, P->d_four_a, 2, n, P->d_proj, true, st);
        vortdiv_tail(*P, P->d_proj, c2(vort), c2(div), n, st);
    });
}

int pswe_laplacian(int R, const double* x, double radius, double* y, int n, int inverse, void* stream) {
    return guarded([&] {
        need(x, "x", n);
        need(y, "y", n);
        if (R < 1) throw std::invalid_argument("laplacian: truncation must be >= 1");
        laplacian(R, c2(x), radius, c2(y), n, inverse != 0, as_stream(stream));
    });
}

int pswe_eval_explicit(pswe_plan* P, const pswe_params* p, const double* state, double* f_exp, int n,
                       void* stream) {
    PSWE_NVTX("pswe.eval_explicit");
    return guarded([&] {
        need(P, "plan");
        need(p, "params");
        need(state, "state", n);
        need(f_exp, "f_exp", n);
        if (n <= 0) return;
        eval_imex(*P, *p, c2(state), nullptr, c2(f_exp), n, as_stream(stream));
    });
}

int pswe_eval_implicit(int R, const pswe_params* p, const double* state, double* f_imp, int n, void* stream) {
    return guarded([&] {
        need(p, "params");
        need(state, "state", n);
        need(f_imp, "f_imp", n);
        if (R < 1) throw std::invalid_argument("eval_implicit: truncation must be >= 1");
        eval_linear(R, *p, c2(state), c2(f_imp), n, as_stream(stream));
    });
}

int pswe_eval_imex(pswe_plan* P, const pswe_params* p, const double* state, double* f_imp, double* f_exp, int n,
                   void* stream) {
    PSWE_NVTX("pswe.eval_imex");
    return guarded([&] {
        need(P, "plan");
        need(p, "params");
        need(state, "state", n);
        need(f_imp, "f_imp", n);
        need(f_exp, "f_exp", n);
        if (n <= 0) return;
        eval_imex(*P, *p, c2(state), c2(f_imp), c2(f_exp), n, as_stream(stream));
    });
}

// eval_imex with CUDA events between its 4 launches on `stream`; synchronises and writes the
// per-stage device times (ms) to ms_out[4]: inverse Legendre, fused FFT/products, forward
// Legendre, tail. Used by bench.py for the per-kernel roofline.
int pswe_eval_imex_timed(pswe_plan* P, const pswe_params* p, const double* state, double* f_imp, double* f_exp,
                         int n, void* stream, float* ms_out) {
    return guarded([&] {
        need(P, "plan");
        need(p, "params");
        need(ms_out, "ms_out");
        const cudaStream_t st = as_stream(stream);
        P->reserve(n);
        cudaEvent_t ev[5];
        for (auto& e : ev) PSWE_CUDA(cudaEventCreate(&e));
        PSWE_CUDA(cudaEventRecord(ev[0], st));
        legendre_inverse(*P, INV_EVAL, c2(state), nullptr, n, p->radius, P->d_four_a, st);
        PSWE_CUDA(cudaEventRecord(ev[1], st));
        const bool gt = gt_path_ok(*P, n);
        if (gt) fft_eval_products_gt(*P, *p, P->d_four_a, n, st);
        else fft_eval_products(*P, *p, P->d_four_a, P->d_four_b, n, st);
        PSWE_CUDA(cudaEventRecord(ev[2], st));
        if (gt) legendre_forward_gt(*P, n, P->d_proj, st);
        else legendre_forward(*P, P->d_four_b, 5, n, P->d_proj, true, st);
        PSWE_CUDA(cudaEventRecord(ev[3], st));
        eval_tail(*P, *p, P->d_proj, c2(state), c2(f_imp), c2(f_exp), n, st);
        PSWE_CUDA(cudaEventRecord(ev[4], st));
        PSWE_CUDA(cudaEventSynchronize(ev[4]));
        for (int i = 0; i < 4; ++i) PSWE_CUDA(cudaEventElapsedTime(&ms_out[i], ev[i], ev[i + 1]));
        for (auto& e : ev) cudaEventDestroy(e);
    });
}

// Per-kernel device times (ms) of one eval_imex: ms_out[5] = prep, inverse contraction, grid stage,
// forward contraction, tail (prep = 0 and the inverse time covers both when the recurrence
// inverse runs: single states on grids above 768 latitudes). CUDA events between the launches on `stream`; synchronises.
int pswe_eval_imex_kernel_times(pswe_plan* P, const pswe_params* p, const double* state, double* f_imp,
                                double* f_exp, int n, void* stream, float* ms_out) {
    return guarded([&] {
        need(P, "plan");
        need(p, "params");
        need(ms_out, "ms_out");
        const cudaStream_t st = as_stream(stream);
        P->reserve(n);
        cudaEvent_t ev[6];
        for (auto& e : ev) PSWE_CUDA(cudaEventCreate(&e));
        PSWE_CUDA(cudaEventRecord(ev[0], st));
        if (!P->simt && use_stream_inverse(*P, 4 * n)) {
            legendre_inverse_stream(*P, INV_EVAL, c2(state), nullptr, 4 * n, p->radius, P->d_four_a, st, ev[1]);
        } else {
            PSWE_CUDA(cudaEventRecord(ev[1], st));
            legendre_inverse(*P, INV_EVAL, c2(state), nullptr, n, p->radius, P->d_four_a, st);
        }
        PSWE_CUDA(cudaEventRecord(ev[2], st));
        const bool gt = gt_path_ok(*P, n);
        if (gt) fft_eval_products_gt(*P, *p, P->d_four_a, n, st);
        else fft_eval_products(*P, *p, P->d_four_a, P->d_four_b, n, st);
        PSWE_CUDA(cudaEventRecord(ev[3], st));
        if (gt) legendre_forward_gt(*P, n, P->d_proj, st);
        else legendre_forward(*P, P->d_four_b, 5, n, P->d_proj, true, st);
        PSWE_CUDA(cudaEventRecord(ev[4], st));
        eval_tail(*P, *p, P->d_proj, c2(state), c2(f_imp), c2(f_exp), n, st);
        PSWE_CUDA(cudaEventRecord(ev[5], st));
        PSWE_CUDA(cudaEventSynchronize(ev[5]));
        for (int i = 0; i < 5; ++i) PSWE_CUDA(cudaEventElapsedTime(&ms_out[i], ev[i], ev[i + 1]));
        for (auto& e : ev) cudaEventDestroy(e);
    });
}

int pswe_solve_implicit(int R, const pswe_params* p, const double* b, double c, double* out, int n, void* stream) {
    return guarded([&] {
        need(p, "params");
        need(b, "b", n);
        need(out, "out", n);
        if (R < 1) throw std::invalid_argument("solve_implicit: truncation must be >= 1");
        solve_implicit(R, *p, c2(b), c, c2(out), n, as_stream(stream));
    });
}

}  // extern "C"
