// extern "C" harness over the REFERENCE implementation compiled from /root/reference/proj/src.
//
// TEST INFRASTRUCTURE ONLY (oracle/_ref). Used by tests/ as the parity checker, by
// oracle/make_golden.py to generate tests/golden/*, and by bench.py's reference arm /
// cpu_baseline leg. Never linked into or called by the product path.
//
// Every entry point forwards to the reference's own public API:
//   TransformPlan (proj/include/pintswe/transform.hpp:27-96), reference:: direct sums
//   (proj/src/reference.cpp:28-108), eval_linear/eval_nonlinear/solve_implicit
//   (proj/src/swe.cpp:9-98), build_tables (proj/src/quadrature.cpp:74-106),
//   sdc::sdc_step (proj/src/sdc.cpp:66-72), ml::* (proj/src/multilevel.cpp), pf::run_block
//   (proj/src/pfasst.cpp:194-251).
//
// LABELLED DEVIATION (grid override): the reference derives the grid from R
// (proj/src/transform.cpp:45-48, dealiased_nlon). To evaluate BASELINE.json's linear grids
// (e.g. T255 on 256x512) the harness can rebuild a plan's grid-dependent members for an
// explicit (nlat, nlon), repeating the constructor's own steps (transform.cpp:51-88) through
// the reference's public helpers gauss_latitudes / legendre_column / legendre_eps. Plans made
// with nlat = nlon = 0 are the unmodified reference plans.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <fftw3.h>
#include <omp.h>

#define private public
#include "pintswe/transform.hpp"
#undef private
#include "pintswe/legendre.hpp"
#include "pintswe/multilevel.hpp"
#include "pintswe/pfasst.hpp"
#include "pintswe/quadrature.hpp"
#include "pintswe/reference.hpp"
#include "pintswe/sdc.hpp"
#include "pintswe/swe.hpp"

using namespace pintswe;
using cd = std::complex<double>;

namespace {

thread_local std::string g_err;
double g_last_wall = 0.0;  // wall seconds of the last ref_pfasst_run / ref_sdc_run loop

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

void override_grid(TransformPlan& plan, int R, int nlat, int nlon) {
    plan.truncation_ = R;
    plan.nlat_ = nlat;
    plan.nlon_ = nlon;
    auto lats = std::make_shared<GaussLatitudes>(gauss_latitudes(nlat));
    plan.lats_ = lats;
    plan.cos_phi_.assign(nlat, 0.0);
    for (int i = 0; i < nlat; ++i) plan.cos_phi_[i] = std::sqrt(1.0 - lats->mu[i] * lats->mu[i]);
    plan.p_tab_.assign(R + 1, {});
    plan.h_tab_.assign(R + 1, {});
#pragma omp parallel for schedule(static, 1)
    for (int r = 0; r <= R; ++r) {
        const int np = R + 2 - r, nh = R + 1 - r;
        plan.p_tab_[r].resize(static_cast<std::size_t>(nlat) * np);
        plan.h_tab_[r].resize(static_cast<std::size_t>(nlat) * nh);
        for (int i = 0; i < nlat; ++i) {
            double* p = plan.p_tab_[r].data() + static_cast<std::size_t>(i) * np;
            double* h = plan.h_tab_[r].data() + static_cast<std::size_t>(i) * nh;
            legendre_column(r, R + 1, lats->mu[i], p);
            for (int s = r; s <= R; ++s) {
                const double upper = -s * legendre_eps(r, s + 1) * p[s + 1 - r];
                const double lower = (s > r) ? (s + 1.0) * legendre_eps(r, s) * p[s - 1 - r] : 0.0;
                h[s - r] = upper + lower;
            }
        }
    }
    if (plan.fwd_) fftw_destroy_plan(reinterpret_cast<fftw_plan>(plan.fwd_));
    if (plan.bwd_) fftw_destroy_plan(reinterpret_cast<fftw_plan>(plan.bwd_));
    plan.fwd_ = reinterpret_cast<fftw_plan_s*>(fftw_plan_dft_r2c_1d(nlon, nullptr, nullptr, 0));
    plan.bwd_ = reinterpret_cast<fftw_plan_s*>(fftw_plan_dft_c2r_1d(nlon, nullptr, nullptr, 0));
}

std::shared_ptr<TransformPlan> make_plan(int R, int nlat, int nlon) {
    if (nlat <= 0 || nlon <= 0) return std::make_shared<TransformPlan>(R);
    if (nlat == dealiased_nlon(R) / 2 && nlon == dealiased_nlon(R))
        return std::make_shared<TransformPlan>(R);
    auto plan = std::make_shared<TransformPlan>(1);
    override_grid(*plan, R, nlat, nlon);
    return plan;
}

struct Handle {
    std::shared_ptr<TransformPlan> plan;
};

SpectralField field_in(int R, const double* d) {
    SpectralField x(R);
    std::memcpy(x.data(), d, sizeof(cd) * x.num_coeffs());
    return x;
}
void field_out(const SpectralField& x, double* d) {
    std::memcpy(d, x.data(), sizeof(cd) * x.num_coeffs());
}
PrognosticState state_in(int R, const double* d) {
    const std::size_t K = SpectralField::size(R);
    PrognosticState s(R);
    s.phi = field_in(R, d);
    s.vort = field_in(R, d + 2 * K);
    s.div = field_in(R, d + 4 * K);
    return s;
}
void state_out(const PrognosticState& s, double* d) {
    const std::size_t K = SpectralField::size(s.truncation());
    field_out(s.phi, d);
    field_out(s.vort, d + 2 * K);
    field_out(s.div, d + 4 * K);
}

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

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_max_threads() { return omp_get_max_threads(); }
int ref_dealiased_nlon(int R) { return dealiased_nlon(R); }

int ref_gauss(int n, double* mu, double* w) {
    return guard([&] {
        const auto g = gauss_latitudes(n);
        std::copy(g.mu.begin(), g.mu.end(), mu);
        std::copy(g.weight.begin(), g.weight.end(), w);
    });
}

int ref_legendre_column(int r, int smax, double mu, double* out) {
    return guard([&] { legendre_column(r, smax, mu, out); });
}

void* ref_plan_create(int R, int nlat, int nlon) {
    try {
        auto* h = new Handle;
        h->plan = make_plan(R, nlat, nlon);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_plan_destroy(void* h) { delete static_cast<Handle*>(h); }
int ref_plan_nlat(void* h) { return static_cast<Handle*>(h)->plan->nlat(); }
int ref_plan_nlon(void* h) { return static_cast<Handle*>(h)->plan->nlon(); }
int ref_plan_latitudes(void* h, double* mu, double* w) {
    const auto& l = static_cast<Handle*>(h)->plan->latitudes();
    std::copy(l.mu.begin(), l.mu.end(), mu);
    std::copy(l.weight.begin(), l.weight.end(), w);
    return 0;
}

int ref_synthesise(void* h, const double* coeffs, double* grid) {
    return guard([&] {
        auto& p = *static_cast<Handle*>(h)->plan;
        const GridField g = p.synthesise(field_in(p.truncation(), coeffs));
        std::copy(g.values.begin(), g.values.end(), grid);
    });
}

int ref_analyse(void* h, const double* grid, double* coeffs) {
    return guard([&] {
        auto& p = *static_cast<Handle*>(h)->plan;
        GridField g = p.make_grid();
        std::copy(grid, grid + g.values.size(), g.values.begin());
        field_out(p.analyse(g), coeffs);
    });
}

int ref_uv_from_vortdiv(void* h, const double* vort, const double* div, double radius, double* u,
                        double* v) {
    return guard([&] {
        auto& p = *static_cast<Handle*>(h)->plan;
        GridField gu, gv;
        p.uv_from_vortdiv(field_in(p.truncation(), vort), field_in(p.truncation(), div), radius, gu,
                          gv);
        std::copy(gu.values.begin(), gu.values.end(), u);
        std::copy(gv.values.begin(), gv.values.end(), v);
    });
}

int ref_vortdiv_from_uv(void* h, const double* u, const double* v, double radius, double* vort,
                        double* div) {
    return guard([&] {
        auto& p = *static_cast<Handle*>(h)->plan;
        GridField gu = p.make_grid(), gv = p.make_grid();
        std::copy(u, u + gu.values.size(), gu.values.begin());
        std::copy(v, v + gv.values.size(), gv.values.begin());
        auto [z, d] = p.vortdiv_from_uv(gu, gv, radius);
        field_out(z, vort);
        field_out(d, div);
    });
}

// Direct-sum transforms of proj/src/reference.cpp on an arbitrary latitude set.
int ref_direct_synthesise(int R, const double* mu, int nlat, int nlon, const double* coeffs,
                          double* grid) {
    return guard([&] {
        std::vector<double> m(mu, mu + nlat);
        const auto g = reference::synthesise(field_in(R, coeffs), m, nlon);
        std::copy(g.begin(), g.end(), grid);
    });
}
int ref_direct_analyse(int R, const double* mu, const double* w, int nlat, int nlon,
                       const double* grid, double* coeffs) {
    return guard([&] {
        std::vector<double> m(mu, mu + nlat), ww(w, w + nlat);
        std::vector<double> vals(grid, grid + static_cast<std::size_t>(nlat) * nlon);
        field_out(reference::analyse(vals, m, ww, nlon, R), coeffs);
    });
}
int ref_direct_uv(int R, const double* vort, const double* div, double radius, const double* mu,
                  int nlat, int nlon, double* u, double* v) {
    return guard([&] {
        std::vector<double> m(mu, mu + nlat), uo, vo;
        reference::uv(field_in(R, vort), field_in(R, div), radius, m, nlon, uo, vo);
        std::copy(uo.begin(), uo.end(), u);
        std::copy(vo.begin(), vo.end(), v);
    });
}

int ref_laplacian(int R, const double* x, double radius, double* y) {
    return guard([&] { field_out(laplacian(field_in(R, x), radius), y); });
}
int ref_inv_laplacian(int R, const double* x, double radius, double* y) {
    return guard([&] { field_out(inv_laplacian(field_in(R, x), radius), y); });
}

int ref_eval_linear(int R, const Params* prm, const double* state, double* out) {
    return guard([&] { state_out(eval_linear(state_in(R, state), mp(prm)), out); });
}
int ref_eval_nonlinear(void* h, const Params* prm, const double* state, double* out) {
    return guard([&] {
        auto& p = *static_cast<Handle*>(h)->plan;
        state_out(eval_nonlinear(state_in(p.truncation(), state), mp(prm), p), out);
    });
}
int ref_solve_implicit(int R, const Params* prm, const double* b, double c, double* out) {
    return guard([&] { state_out(solve_implicit(state_in(R, b), c, mp(prm)), out); });
}

// Best-of-reps wall time (s) of eval_nonlinear + eval_linear, the method of
// proj/tools/bench_transform.cpp:32-41.
double ref_time_eval(void* h, const Params* prm, const double* state, int reps) {
    auto& p = *static_cast<Handle*>(h)->plan;
    const PrognosticState s = state_in(p.truncation(), state);
    const ModelParams m = mp(prm);
    double best = 1e300;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        volatile double sink = eval_nonlinear(s, m, p).max_abs() + eval_linear(s, m).max_abs();
        (void)sink;
        const auto t1 = std::chrono::steady_clock::now();
        best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    }
    return best;
}

// Best-of-reps wall time (s) of n_fields x (synthesise + analyse).
double ref_time_roundtrip(void* h, const double* coeffs, int n_fields, int reps) {
    auto& p = *static_cast<Handle*>(h)->plan;
    const std::size_t K = SpectralField::size(p.truncation());
    std::vector<SpectralField> xs;
    for (int f = 0; f < n_fields; ++f) xs.push_back(field_in(p.truncation(), coeffs + 2 * K * f));
    double best = 1e300;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        double acc = 0.0;
        for (int f = 0; f < n_fields; ++f) acc += p.analyse(p.synthesise(xs[f])).max_abs();
        volatile double sink = acc;
        (void)sink;
        const auto t1 = std::chrono::steady_clock::now();
        best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    }
    return best;
}

int ref_build_tables(int n, double* nodes, double* q, double* qe, double* qi) {
    return guard([&] {
        const auto t = build_tables(n);
        std::copy(t.nodes.begin(), t.nodes.end(), nodes);
        std::copy(t.q.a.begin(), t.q.a.end(), q);
        std::copy(t.q_exp.a.begin(), t.q_exp.a.end(), qe);
        std::copy(t.q_imp.a.begin(), t.q_imp.a.end(), qi);
    });
}

int ref_transfer_matrices(int nf, int nc, double* restrict_m, double* interp_m, double* qf_r) {
    return guard([&] {
        ml::LevelSpec f{1, nullptr, build_tables(nf), nullptr};
        ml::LevelSpec c{1, nullptr, build_tables(nc), nullptr};
        auto pair = ml::make_transfer_pair(f, c);
        std::copy(pair.time_restrict.a.begin(), pair.time_restrict.a.end(), restrict_m);
        std::copy(pair.time_interp.a.begin(), pair.time_interp.a.end(), interp_m);
        std::copy(pair.qf_time_restricted.a.begin(), pair.qf_time_restricted.a.end(), qf_r);
    });
}

// Serial SDC: n_steps x sdc::sdc_step. residuals[n_steps] receives each step's final residual.
int ref_sdc_run(void* h, const Params* prm, int nodes, int n_sweeps, double dt, int n_steps,
                const double* theta0, double* final_state, double* residuals) {
    return guard([&] {
        auto plan = static_cast<Handle*>(h)->plan;
        SweOde ode(plan, mp(prm));
        const auto tables = build_tables(nodes);
        PrognosticState s = state_in(plan->truncation(), theta0);
        const auto t0 = std::chrono::steady_clock::now();
        for (int n = 0; n < n_steps; ++n) {
            double res = 0.0;
            s = sdc::sdc_step(s, dt, tables, n_sweeps, ode, &res);
            if (residuals) residuals[n] = res;
        }
        g_last_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        state_out(s, final_state);
    });
}

// One SDC sweep on a full space-time state (for sweep-level parity).
// sts layout: [3][nodes][state] i.e. state nodes, then f_imp nodes, then f_exp nodes.
int ref_sdc_sweep(void* h, const Params* prm, int nodes, double dt, double* sts, const double* tau) {
    return guard([&] {
        auto plan = static_cast<Handle*>(h)->plan;
        const int R = plan->truncation();
        const std::size_t S = 6 * SpectralField::size(R);
        SweOde ode(plan, mp(prm));
        const auto tables = build_tables(nodes);
        sdc::SpaceTimeState st;
        for (int m = 0; m < nodes; ++m) {
            st.state.push_back(state_in(R, sts + S * m));
            st.f_imp.push_back(state_in(R, sts + S * (nodes + m)));
            st.f_exp.push_back(state_in(R, sts + S * (2 * nodes + m)));
        }
        std::vector<PrognosticState> fas;
        if (tau)
            for (int m = 0; m < nodes; ++m) fas.push_back(state_in(R, tau + S * m));
        sdc::sweep(st, dt, tables, ode, tau ? &fas : nullptr);
        for (int m = 0; m < nodes; ++m) {
            state_out(st.state[m], sts + S * m);
            state_out(st.f_imp[m], sts + S * (nodes + m));
            state_out(st.f_exp[m], sts + S * (2 * nodes + m));
        }
    });
}

double ref_collocation_residual(int R, int nodes, double dt, const double* sts) {
    const std::size_t S = 6 * SpectralField::size(R);
    const auto tables = build_tables(nodes);
    sdc::SpaceTimeState st;
    for (int m = 0; m < nodes; ++m) {
        st.state.push_back(state_in(R, sts + S * m));
        st.f_imp.push_back(state_in(R, sts + S * (nodes + m)));
        st.f_exp.push_back(state_in(R, sts + S * (2 * nodes + m)));
    }
    return sdc::collocation_residual(st, dt, tables);
}

// Two-level PFASST over n_blocks blocks of n_ts steps (runner.cpp:145-151 chaining).
// final_state: state after the last block; residuals: [n_blocks][n_ts][n_iter+1];
// messages (optional): [max_msgs][7] ints (phase, iteration, step char, sender, receiver,
// level, node) for the FIRST block; returns the message count through *n_msgs.
int ref_pfasst_run(int Rf, int nlat_f, int nlon_f, int Rc, int nlat_c, int nlon_c,
                   const Params* prm, int nodes_f, int nodes_c, int n_ts, double dt, int n_iter,
                   int n_blocks, int serial_mode, const double* theta0, double* final_state,
                   double* residuals, int* messages, int max_msgs, int* n_msgs) {
    return guard([&] {
        auto pf_plan = make_plan(Rf, nlat_f, nlon_f);
        auto pc_plan = (Rc == Rf && nlat_c == nlat_f && nlon_c == nlon_f) ? pf_plan
                                                                          : make_plan(Rc, nlat_c, nlon_c);
        const ModelParams m = mp(prm);
        ml::LevelSpec fine{Rf, pf_plan, build_tables(nodes_f), std::make_shared<SweOde>(pf_plan, m)};
        ml::LevelSpec coarse{Rc, pc_plan, build_tables(nodes_c), std::make_shared<SweOde>(pc_plan, m)};
        pf::BlockConfig block;
        block.n_time_steps = n_ts;
        block.dt = dt;
        block.n_iter = n_iter;
        block.levels = ml::make_transfer_pair(std::move(fine), std::move(coarse));
        PrognosticState s = state_in(Rf, theta0);
        std::size_t ri = 0;
        const auto t0 = std::chrono::steady_clock::now();
        for (int b = 0; b < n_blocks; ++b) {
            pf::BlockResult br = pf::run_block(
                block, s, serial_mode ? pf::Mode::serial_emulation : pf::Mode::threaded);
            s = br.step_final.back();
            for (const auto& wr : br.residuals)
                for (double r : wr) residuals[ri++] = r;
            if (b == 0 && messages) {
                int k = 0;
                for (const auto& mr : br.messages) {
                    if (k >= max_msgs) break;
                    int* o = messages + 7 * k;
                    o[0] = mr.phase; o[1] = mr.iteration; o[2] = mr.step; o[3] = mr.sender;
                    o[4] = mr.receiver; o[5] = mr.level; o[6] = mr.node;
                    ++k;
                }
                if (n_msgs) *n_msgs = static_cast<int>(br.messages.size());
            }
        }
        g_last_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        state_out(s, final_state);
    });
}

// Serial two-level MLSDC (multilevel.cpp:160-194), n_steps steps.
int ref_mlsdc_run(int Rf, int nlat_f, int nlon_f, int Rc, int nlat_c, int nlon_c,
                  const Params* prm, int nodes_f, int nodes_c, double dt, int n_iter, int n_steps,
                  const double* theta0, double* final_state, double* residuals) {
    return guard([&] {
        auto pf_plan = make_plan(Rf, nlat_f, nlon_f);
        auto pc_plan = make_plan(Rc, nlat_c, nlon_c);
        const ModelParams m = mp(prm);
        ml::LevelSpec fine{Rf, pf_plan, build_tables(nodes_f), std::make_shared<SweOde>(pf_plan, m)};
        ml::LevelSpec coarse{Rc, pc_plan, build_tables(nodes_c), std::make_shared<SweOde>(pc_plan, m)};
        auto pair = ml::make_transfer_pair(std::move(fine), std::move(coarse));
        PrognosticState s = state_in(Rf, theta0);
        for (int n = 0; n < n_steps; ++n) {
            double res = 0.0;
            s = ml::mlsdc_step(s, dt, pair, n_iter, &res);
            if (residuals) residuals[n] = res;
        }
        state_out(s, final_state);
    });
}

// Wall seconds of the timed loop of the last ref_pfasst_run / ref_sdc_run (plan setup excluded).
double ref_last_wall() { return g_last_wall; }

}  // extern "C"

// ---- io.cpp (JSON checkpoints, io.cpp:48-67): compiled only when nlohmann/json is available
#ifdef PSWE_REF_WITH_IO
#include "pintswe/io.hpp"
extern "C" {
int ref_save_checkpoint(const char* path, int R, const double* state, double time) {
    return guard([&] { io::save_checkpoint(path, state_in(R, state), time); });
}
int ref_load_checkpoint(const char* path, int R, double* state, double* time) {
    return guard([&] {
        const PrognosticState s = io::load_checkpoint(path, time);
        if (s.truncation() != R) throw std::invalid_argument("checkpoint truncation mismatch");
        state_out(s, state);
    });
}
}
#endif
