// GpuImexOde: the reference's plugin interface pintswe::ImexOde (proj/include/pintswe/swe.hpp:47-55)
// implemented over libpswe's C ABI (include/pswe.h) — the binding a maintainer of the reference
// would add to run its UNMODIFIED sdc / multilevel / pfasst code (proj/src/sdc.cpp,
// multilevel.cpp, pfasst.cpp) on the B200 right-hand side. See INTEGRATION.md.
//
// TEST INFRASTRUCTURE ONLY: it is compiled together with the reference sources into
// oracle/_ref/libpintswe_gpu.so (oracle/build_ref.sh) and driven by tests/test_gpu_dropin.py.
// Every call copies the state host->device and the result back (the by-value contract of
// ImexOde); the production path keeps states resident on the device (pswe_level / pswe_pfasst).
// Thread safety: the reference shares one ImexOde between its PFASST worker threads
// (Mode::threaded, pfasst.cpp:219-234, runner.cpp:143-144), while a pswe_plan and the adapter's
// staging buffers are single-stream; every method therefore holds the adapter's mutex across
// upload, evaluation and download (tests/test_gpu_dropin.py runs the threaded mode).
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "pintswe/multilevel.hpp"
#include "pintswe/pfasst.hpp"
#include "pintswe/quadrature.hpp"
#include "pintswe/sdc.hpp"
#include "pintswe/swe.hpp"
#include "pswe.h"

using namespace pintswe;

namespace {

void ck(int rc) {
    if (rc != 0) throw std::runtime_error(std::string("libpswe: ") + pswe_last_error());
}

class GpuImexOde final : public ImexOde {
public:
    GpuImexOde(int R, int nlat, int nlon, const ModelParams& p) : R_(R) {
        prm_ = {p.radius, p.omega, p.gravity, p.phi_bar, p.nu};
        ck(pswe_plan_create(R, nlat, nlon, PSWE_LEGENDRE_RECOMPUTE, &plan_));
        bytes_ = 3 * SpectralField::size(R) * 2 * sizeof(double);
        ck(pswe_device_alloc(bytes_, &d_in_));
        ck(pswe_device_alloc(bytes_, &d_out_));
    }
    ~GpuImexOde() override {
        pswe_device_free(d_in_);
        pswe_device_free(d_out_);
        pswe_plan_destroy(plan_);
    }
    int truncation() const override { return R_; }
    PrognosticState eval_implicit(const PrognosticState& s) const override {
        std::lock_guard<std::mutex> lock(mu_);
        upload(s);
        ck(pswe_eval_implicit(R_, &prm_, (const double*)d_in_, (double*)d_out_, 1, nullptr));
        return download();
    }
    PrognosticState eval_explicit(const PrognosticState& s) const override {
        std::lock_guard<std::mutex> lock(mu_);
        upload(s);
        ck(pswe_eval_explicit(plan_, &prm_, (const double*)d_in_, (double*)d_out_, 1, nullptr));
        return download();
    }
    PrognosticState solve_implicit(const PrognosticState& b, double c) const override {
        std::lock_guard<std::mutex> lock(mu_);
        upload(b);
        ck(pswe_solve_implicit(R_, &prm_, (const double*)d_in_, c, (double*)d_out_, 1, nullptr));
        return download();
    }

private:
    void upload(const PrognosticState& s) const {
        const std::size_t K = SpectralField::size(R_);
        std::vector<double> h(6 * K);
        std::memcpy(h.data(), s.phi.data(), 16 * K);
        std::memcpy(h.data() + 2 * K, s.vort.data(), 16 * K);
        std::memcpy(h.data() + 4 * K, s.div.data(), 16 * K);
        ck(pswe_memcpy_h2d(d_in_, h.data(), bytes_, nullptr));
    }
    PrognosticState download() const {
        const std::size_t K = SpectralField::size(R_);
        std::vector<double> h(6 * K);
        ck(pswe_memcpy_d2h(h.data(), d_out_, bytes_, nullptr));
        ck(pswe_stream_synchronize(nullptr));
        PrognosticState s(R_);
        std::memcpy(s.phi.data(), h.data(), 16 * K);
        std::memcpy(s.vort.data(), h.data() + 2 * K, 16 * K);
        std::memcpy(s.div.data(), h.data() + 4 * K, 16 * K);
        return s;
    }
    mutable std::mutex mu_;
    int R_;
    pswe_params prm_{};
    pswe_plan* plan_ = nullptr;
    void* d_in_ = nullptr;
    void* d_out_ = nullptr;
    std::size_t bytes_ = 0;
};

struct Params {
    double radius, omega, gravity, phi_bar, nu;
};
ModelParams mp(const Params* p) {
    ModelParams m;
    m.radius = p->radius;
    m.omega = p->omega;
    m.gravity = p->gravity;
    m.phi_bar = p->phi_bar;
    m.nu = p->nu;
    return m;
}
PrognosticState state_in(int R, const double* d) {
    const std::size_t K = SpectralField::size(R);
    PrognosticState s(R);
    std::memcpy(s.phi.data(), d, 16 * K);
    std::memcpy(s.vort.data(), d + 2 * K, 16 * K);
    std::memcpy(s.div.data(), d + 4 * K, 16 * K);
    return s;
}
void state_out(const PrognosticState& s, double* d) {
    const std::size_t K = SpectralField::size(s.truncation());
    std::memcpy(d, s.phi.data(), 16 * K);
    std::memcpy(d + 2 * K, s.vort.data(), 16 * K);
    std::memcpy(d + 4 * K, s.div.data(), 16 * K);
}
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // namespace

extern "C" {

const char* gpuref_last_error() { return g_err.c_str(); }

// reference sdc::sdc_step (sdc.cpp:66-72) x n_steps with the B200 right-hand side
int gpuref_sdc_run(int R, int nlat, int nlon, const Params* prm, int nodes, int n_sweeps, double dt, int n_steps,
                   const double* theta0, double* final_state, double* residuals) {
    return guard([&] {
        GpuImexOde ode(R, nlat, nlon, mp(prm));
        const auto tables = build_tables(nodes);
        PrognosticState s = state_in(R, theta0);
        for (int n = 0; n < n_steps; ++n) {
            double res = 0.0;
            s = sdc::sdc_step(s, dt, tables, n_sweeps, ode, &res);
            residuals[n] = res;
        }
        state_out(s, final_state);
    });
}

// reference pf::run_block (pfasst.cpp:194-251) in serial emulation with B200 right-hand sides
int gpuref_pfasst_run_mode(int Rf, int nlat_f, int nlon_f, int Rc, int nlat_c, int nlon_c, const Params* prm,
                           int nodes_f, int nodes_c, int n_ts, double dt, int n_iter, int n_blocks,
                           const double* theta0, double* final_state, double* residuals, int threaded) {
    return guard([&] {
        const ModelParams m = mp(prm);
        auto fo = std::make_shared<GpuImexOde>(Rf, nlat_f, nlon_f, m);
        auto co = std::make_shared<GpuImexOde>(Rc, nlat_c, nlon_c, m);
        ml::LevelSpec fine{Rf, nullptr, build_tables(nodes_f), fo};
        ml::LevelSpec coarse{Rc, nullptr, build_tables(nodes_c), co};
        pf::BlockConfig block;
        block.n_time_steps = n_ts;
        block.dt = dt;
        block.n_iter = n_iter;
        block.levels = ml::make_transfer_pair(std::move(fine), std::move(coarse));
        PrognosticState s = state_in(Rf, theta0);
        std::size_t ri = 0;
        for (int b = 0; b < n_blocks; ++b) {
            pf::BlockResult br =
                pf::run_block(block, s, threaded ? pf::Mode::threaded : pf::Mode::serial_emulation);
            s = br.step_final.back();
            for (const auto& wr : br.residuals)
                for (double r : wr) residuals[ri++] = r;
        }
        state_out(s, final_state);
    });
}

int gpuref_pfasst_run(int Rf, int nlat_f, int nlon_f, int Rc, int nlat_c, int nlon_c, const Params* prm, int nodes_f,
                      int nodes_c, int n_ts, double dt, int n_iter, int n_blocks, const double* theta0,
                      double* final_state, double* residuals) {
    return gpuref_pfasst_run_mode(Rf, nlat_f, nlon_f, Rc, nlat_c, nlon_c, prm, nodes_f, nodes_c, n_ts, dt, n_iter,
                                  n_blocks, theta0, final_state, residuals, 0);
}

}  // extern "C"
