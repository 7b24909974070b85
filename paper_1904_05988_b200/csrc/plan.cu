// Plan construction: the host-side numerical setup of TransformPlan (transform.cpp:45-89) and
// the device constant tables it feeds the kernels.
//
// Host setup restates the reference's algorithms:
//   gauss_latitudes  gauss.cpp:11-50 (Newton on P_n, |dx| < 1e-15, w = 2/((1-x^2)P_n'^2))
//   legendre_eps     legendre.cpp:7-11
//   sectoral seed    legendre.cpp:16-29 (log-space P^m_m, underflows to 0 near the poles)
//   dealiased_nlon   transform.cpp:38-43
// Device tables are laid out for the kernels.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <complex>
#include <cstring>
#include <mutex>

#include "pswe_internal.h"

namespace pswe {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }
const char* last_error() { return g_error.c_str(); }

// ---- host numerical setup -----------------------------------------------------------------

static void legendre_pn(int n, double x, double& p, double& dp) {
    double p0 = 1.0, p1 = x;
    for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
    }
    p = p1;
    dp = n * (x * p1 - p0) / (x * x - 1.0);
}

void gauss_latitudes(int n, double* mu, double* wt) {
    if (n < 1) throw std::invalid_argument("gauss_latitudes: need n >= 1");
    const int half = (n + 1) / 2;
    for (int i = 0; i < half; ++i) {
        double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        double p = 0.0, dp = 1.0;
        for (int it = 0; it < 100; ++it) {
            legendre_pn(n, x, p, dp);
            const double dx = p / dp;
            x -= dx;
            if (std::abs(dx) < 1e-15) break;
        }
        legendre_pn(n, x, p, dp);
        const double w = 2.0 / ((1.0 - x * x) * dp * dp);
        mu[n - 1 - i] = x;
        mu[i] = -x;
        wt[n - 1 - i] = w;
        wt[i] = w;
    }
    if (n % 2 == 1) mu[n / 2] = 0.0;
}

double legendre_eps(int r, int s) {
    if (s <= r) return 0.0;
    const double sd = s, rd = r;
    return std::sqrt((sd * sd - rd * rd) / (4.0 * sd * sd - 1.0));
}

static double sectoral_log_amplitude(int r) {
    double acc = 0.5 * std::log(0.5);
    for (int k = 1; k <= r; ++k) acc += 0.5 * std::log((2.0 * k + 1.0) / (2.0 * k));
    return acc;
}

static bool five_smooth(int n) {
    for (int p : {2, 3, 5})
        while (n % p == 0) n /= p;
    return n == 1;
}

int dealiased_nlon(int R) {
    int n = 3 * R + 1;
    if (n % 2) ++n;
    while (!five_smooth(n)) n += 2;
    return n;
}

// ---- device table builders ------------------------------------------------------------------

// P^m_s(mu_j) for s = m..R+1 by the normalised 3-term recurrence (legendre.cpp:30-37), one
// thread per (m, j); table block m is [j][s] (s contiguous) for the coalesced forward contraction.
__global__ void build_ptab_kernel(int R, int J, const double* __restrict__ mu_n,
                                  const double* __restrict__ seed, const double2* __restrict__ rec,
                                  double* __restrict__ ptab) {
    const int m = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= J) return;
    const double mu = mu_n[j];
    const long base = off_ext(R, m);
    const int len = R + 2 - m;
    double* out = ptab + base * J + (long)j * len;
    double p = seed[(long)m * J + j], pm1 = 0.0;
    for (int t = 0; t < len; ++t) {
        out[t] = p;
        if (t + 1 < len) {
            const double2 ab = rec[base + t];
            const double pn = ab.x * (mu * p) - ab.y * pm1;
            pm1 = p;
            p = pn;
        }
    }
}

static std::complex<double> expi_neg(long num, long den) {
    long r = num % den;
    if (r < 0) r += den;
    const long double a = -2.0L * 3.141592653589793238462643383279502884L * r / den;
    return {static_cast<double>(std::cos(a)), static_cast<double>(std::sin(a))};
}

}  // namespace pswe

using namespace pswe;

void pswe_plan::reserve(int batch) {
    if (batch <= cap_batch) return;
    PSWE_CUDA(cudaSetDevice(device));
    // grow-only; callers must not resize during graph capture (pswe_plan_reserve first)
    ++generation;
    if (d_four_a) cudaFree(d_four_a);
    if (d_four_b) cudaFree(d_four_b);
    if (d_proj) cudaFree(d_proj);
    if (d_xcoef) cudaFree(d_xcoef);
    d_four_a = d_four_b = d_proj = d_xcoef = nullptr;
    const size_t four = (size_t)batch * 5 * (R + 1) * nlat;
    PSWE_CUDA(cudaMalloc(&d_four_a, four * sizeof(double2)));
    PSWE_CUDA(cudaMalloc(&d_four_b, four * sizeof(double2)));
    PSWE_CUDA(cudaMalloc(&d_proj, (size_t)batch * 5 * Kx * sizeof(double2)));
    PSWE_CUDA(cudaMalloc(&d_xcoef, (size_t)batch * 5 * Kx * sizeof(double2)));
    if (n_chunks > 0) {  // STREAM inverse X tiles for up to 5 batch columns, any column tiling
        const int nq = 5 * batch;
        size_t need = 0;
        for (int nt = 1; nt <= 5; ++nt) {
            const size_t d = (size_t)((nq + 4 * nt - 1) / (4 * nt)) * (8 * nt + 2) * n_chunks * 16;
            need = d > need ? d : need;
        }
        if (need > xtile_cap) {
            if (d_xtile) cudaFree(d_xtile);
            d_xtile = nullptr;
            PSWE_CUDA(cudaMalloc(&d_xtile, need * sizeof(double)));
            xtile_cap = need;
        }
    }
    if (n_chunks > 0) {  // G tiles of the eval grid stage (batch states) or of analyse (5 batch
                         // fields); zeroed once: never-written slots stay finite
        const size_t need = std::max(pswe::gt_layout(R, J, batch).doubles,
                                     pswe::gt_layout_fields(R, J, 5 * batch).doubles);
        if (need > gtile_cap) {
            if (d_gtile) cudaFree(d_gtile);
            d_gtile = nullptr;
            PSWE_CUDA(cudaMalloc(&d_gtile, need * sizeof(double)));
            PSWE_CUDA(cudaMemset(d_gtile, 0, need * sizeof(double)));
            gtile_cap = need;
        }
    }
    cap_batch = batch;
}

static void plan_free(pswe_plan* p) {
    void* ptrs[] = {p->d_mu_n, p->d_seed, p->d_rec, p->d_eps, p->d_rlap, p->d_ptab, p->d_rowc, p->d_roww,
                    p->d_rowmu, p->d_fft_tw, p->d_fft_post, p->d_four_a, p->d_four_b, p->d_proj,
                    p->d_xcoef, p->d_chk, p->d_chk_off, p->d_fft_roots, p->d_fft_iptw, p->d_fft_iptw1, p->d_ptab2, p->d_cstart, p->d_chunk_m, p->d_xtile, p->d_fwd_ta, p->d_fwd_tb, p->d_gtile};
    for (void* q : ptrs)
        if (q) cudaFree(q);
}

namespace pswe {
bool pdl_enabled() {
    static const bool on = [] { const char* e = std::getenv("PSWE_NO_PDL"); return !(e && std::atoi(e) != 0); }();
    return on;
}
}  // namespace pswe

template <class T>
static T* upload(const std::vector<T>& v) {
    T* d = nullptr;
    PSWE_CUDA(cudaMalloc(&d, v.size() * sizeof(T)));
    PSWE_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

static void plan_build(pswe_plan* p, int R, int nlat, int nlon, int mode) {
    if (R < 1) throw std::invalid_argument("TransformPlan: truncation must be >= 1");
    if (nlat <= 0 || nlon <= 0) {
        nlon = dealiased_nlon(R);
        nlat = nlon / 2;
    }
    if (nlon % 2 || !five_smooth(nlon / 2))
        throw std::invalid_argument("pswe_plan_create: nlon must be even with nlon/2 5-smooth");
    if (nlon <= 2 * R) throw std::invalid_argument("pswe_plan_create: nlon must exceed 2R");
    if (nlat <= R) throw std::invalid_argument("pswe_plan_create: nlat must exceed R");
    if (mode != PSWE_LEGENDRE_RECOMPUTE && mode != PSWE_LEGENDRE_STREAM)
        throw std::invalid_argument("pswe_plan_create: unknown legendre_mode");
    PSWE_CUDA(cudaGetDevice(&p->device));
    p->R = R;
    p->nlat = nlat;
    p->nlon = nlon;
    p->J = (nlat + 1) / 2;  // latitude pairs (+ the equator row when nlat is odd)
    p->N = nlon / 2;
    p->legendre_mode = mode;
    if (const char* e = std::getenv("PSWE_LEGENDRE_SIMT")) p->simt = std::atoi(e) != 0;
    p->K = num_coeffs(R);
    p->Kx = num_ext(R);
    const int J = p->J;

    p->mu.resize(nlat);
    p->w.resize(nlat);
    p->cosphi.resize(nlat);
    gauss_latitudes(nlat, p->mu.data(), p->w.data());
    for (int i = 0; i < nlat; ++i) p->cosphi[i] = std::sqrt(1.0 - p->mu[i] * p->mu[i]);

    // north-half latitudes, seeds (legendre.cpp:26-29)
    std::vector<double> mu_n(J), seed((size_t)(R + 1) * J);
    for (int j = 0; j < J; ++j) mu_n[j] = p->mu[nlat - J + j];
    for (int m = 0; m <= R; ++m) {
        const double la = sectoral_log_amplitude(m);
        for (int j = 0; j < J; ++j) {
            const double cos2 = 1.0 - mu_n[j] * mu_n[j];
            seed[(size_t)m * J + j] = std::exp(la + 0.5 * m * std::log(cos2));
        }
    }
    // recurrence coefficients and eps, extended layout s = m..R+1
    std::vector<double2> rec(p->Kx);
    std::vector<double> eps(p->Kx);
    for (int m = 0; m <= R; ++m) {
        const long b = off_ext(R, m);
        for (int s = m; s <= R + 1; ++s) {
            eps[b + s - m] = legendre_eps(m, s);
            if (s <= R) {
                const double e1 = legendre_eps(m, s + 1);
                rec[b + s - m] = make_double2(1.0 / e1, legendre_eps(m, s) / e1);
            } else {
                rec[b + s - m] = make_double2(0.0, 0.0);
            }
        }
    }
    p->d_mu_n = upload(mu_n);
    p->d_seed = upload(seed);
    p->d_rec = upload(rec);
    p->d_eps = upload(eps);
    {
        std::vector<double> rl(p->R + 2, 0.0);
        for (int s = 1; s <= p->R + 1; ++s) rl[s] = 1.0 / ((double)s * (s + 1.0));
        p->d_rlap = upload(rl);
    }
    p->d_rowc = upload(p->cosphi);
    p->d_roww = upload(p->w);
    p->d_rowmu = upload(p->mu);

    // FFT plan: N = nlon/2, radices 4, 2, 3, 5 (Stockham DIF, see fft.cu)
    FftDesc fd{};
    fd.N = p->N;
    std::vector<double2> tw;
    {
        int n = p->N, s = 1;
        while (n > 1) {
            int r = (n % 4 == 0) ? 4 : (n % 2 == 0) ? 2 : (n % 3 == 0) ? 3 : 5;
            if (fd.nst >= kMaxFftStages) throw std::runtime_error("fft: too many stages");
            const int m = n / r;
            FftStage st{r, m, s, (int)tw.size()};
            for (int j = 0; j < m; ++j)
                for (int t = 0; t < r; ++t) {
                    const auto c = expi_neg((long)j * t, n);
                    tw.push_back(make_double2(c.real(), c.imag()));
                }
            fd.st[fd.nst++] = st;
            n = m;
            s *= r;
        }
    }
    if (tw.empty()) tw.push_back(make_double2(1.0, 0.0));
    std::vector<double2> post(p->N + 1);
    for (int k = 0; k <= p->N; ++k) {
        const auto c = expi_neg(k, nlon);
        post[k] = make_double2(c.real(), c.imag());
    }
    std::vector<double2> roots(p->N);
    for (int k = 0; k < p->N; ++k) {
        const auto c = expi_neg(k, p->N);
        roots[k] = make_double2(c.real(), c.imag());
    }
    p->fft = fd;
    p->d_fft_tw = upload(tw);
    p->d_fft_post = upload(post);
    p->d_fft_roots = upload(roots);
    p->d_fft_iptw = upload(fft_ip_twiddles(p->N));
    p->d_fft_iptw1 = upload(fft_ip_twiddles(p->N, 1));

    if (mode == PSWE_LEGENDRE_STREAM && p->simt) {  // table of the DFMA (SIMT) stream kernel
        PSWE_CUDA(cudaMalloc(&p->d_ptab, (size_t)p->Kx * J * sizeof(double)));
        dim3 grid((J + 127) / 128, R + 1);
        build_ptab_kernel<<<grid, 128>>>(R, J, p->d_mu_n, p->d_seed, p->d_rec, p->d_ptab);
        PSWE_LAUNCH_CHECK();
    }
    build_legendre_checkpoints(*p);
    if (mode == PSWE_LEGENDRE_STREAM) build_legendre_table2(*p);
    p->reserve(1);
    PSWE_CUDA(cudaDeviceSynchronize());
}

extern "C" {

const char* pswe_last_error(void) { return pswe::last_error(); }
int pswe_abi_version(void) { return PSWE_ABI_VERSION; }
int pswe_dealiased_nlon(int truncation) { return pswe::dealiased_nlon(truncation); }

int pswe_gauss_latitudes(int n, double* mu, double* weight) {
    return guarded([&] { pswe::gauss_latitudes(n, mu, weight); });
}

int pswe_plan_create(int truncation, int nlat, int nlon, int legendre_mode, pswe_plan** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("pswe_plan_create: out is NULL");
        auto* p = new pswe_plan;
        try {
            plan_build(p, truncation, nlat, nlon, legendre_mode);
        } catch (...) {
            plan_free(p);
            delete p;
            throw;
        }
        *out = p;
    });
}

int pswe_plan_destroy(pswe_plan* plan) {
    return guarded([&] {
        if (!plan) return;
        plan_free(plan);
        delete plan;
    });
}

int pswe_plan_info(const pswe_plan* p, int* R, int* nlat, int* nlon, int* mode) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("pswe_plan_info: NULL plan");
        if (R) *R = p->R;
        if (nlat) *nlat = p->nlat;
        if (nlon) *nlon = p->nlon;
        if (mode) *mode = p->legendre_mode;
    });
}

int pswe_plan_latitudes(const pswe_plan* p, double* mu, double* weight) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("pswe_plan_latitudes: NULL plan");
        std::memcpy(mu, p->mu.data(), sizeof(double) * p->nlat);
        std::memcpy(weight, p->w.data(), sizeof(double) * p->nlat);
    });
}

int pswe_plan_reserve(pswe_plan* p, int max_batch) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("pswe_plan_reserve: NULL plan");
        p->reserve(max_batch);
    });
}

}  // extern "C"
