// FFTW3-API shim for building the reference CPU path (oracle/_ref) in this image.
//
// TEST INFRASTRUCTURE ONLY. FFTW3 (no pinned version; `proj/CMakeLists.txt:15-16`) is not
// installed here, so this header implements exactly the subset the reference calls
// (`proj/src/transform.cpp:82-87,93-94,108-109,129-130`):
//   fftw_plan_dft_r2c_1d / fftw_plan_dft_c2r_1d / fftw_execute_dft_r2c / fftw_execute_dft_c2r /
//   fftw_destroy_plan, FFTW_ESTIMATE, FFTW_UNALIGNED.
// Semantics follow FFTW's published definition: unnormalised transforms;
// r2c: X[k] = sum_j x[j] exp(-2 pi i jk/n), k = 0..n/2;
// c2r: y[j] = sum_{k=0}^{n-1} X[k] exp(+2 pi i jk/n) with Hermitian extension, the imaginary
// parts of X[0] and X[n/2] ignored. Parity of this shim is pinned by the reference's own
// "production vs direct-sum" test (`proj/tests/test_transform.cpp:219-245`), re-run in
// tests/test_oracle_ref.py.
//
// Algorithm: the real transform of even length n is computed through one complex FFT of
// length n/2 (even/odd packing) and a post/pre-processing twiddle pass; the complex FFT is a
// self-sorting Stockham DIF with radices 4, 2, 3, 5 and precomputed twiddles.
#pragma once

#include <cmath>
#include <complex>
#include <cstddef>
#include <vector>

typedef double fftw_complex[2];

#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

struct fftw_plan_s {
    int n = 0;       // real length
    int nh = 0;      // complex length n/2
    bool r2c = true;
    std::vector<int> radix;                          // factorisation of nh
    std::vector<std::vector<std::complex<double>>> tw;  // per stage: w^(j t), j<m, t<p
    std::vector<std::complex<double>> post;          // exp(-2 pi i k / n), k = 0..nh
};
typedef fftw_plan_s* fftw_plan;

namespace pswe_fftw_shim {

using cd = std::complex<double>;

inline cd expi(long num, long den) {
    // exp(-2 pi i num/den) with reduced argument for accuracy
    long r = num % den;
    if (r < 0) r += den;
    const long double a = -2.0L * 3.141592653589793238462643383279502884L * r / den;
    return cd(static_cast<double>(std::cos(a)), static_cast<double>(std::sin(a)));
}

inline void build(fftw_plan p) {
    int m = p->nh;
    while (m > 1) {
        int r = 0;
        if (m % 4 == 0) r = 4;
        else if (m % 2 == 0) r = 2;
        else if (m % 3 == 0) r = 3;
        else if (m % 5 == 0) r = 5;
        else r = m;  // generic odd prime factor
        p->radix.push_back(r);
        m /= r;
    }
    int n = p->nh;
    for (int r : p->radix) {
        const int mm = n / r;
        std::vector<cd> t(static_cast<std::size_t>(mm) * r);
        for (int j = 0; j < mm; ++j)
            for (int q = 0; q < r; ++q) t[static_cast<std::size_t>(j) * r + q] = expi(static_cast<long>(j) * q, n);
        p->tw.push_back(std::move(t));
        n = mm;
    }
    p->post.resize(p->nh + 1);
    for (int k = 0; k <= p->nh; ++k) p->post[k] = expi(k, p->n);
}

// Forward complex DFT (sign -1) of length nh, x -> out, using scratch y.
inline void cfft(const fftw_plan p, cd* x, cd* y, bool inverse) {
    int n = p->nh;
    int s = 1;
    cd* src = x;
    cd* dst = y;
    const double sg = inverse ? -1.0 : 1.0;
    for (std::size_t st = 0; st < p->radix.size(); ++st) {
        const int r = p->radix[st];
        const int m = n / r;
        const cd* tw = p->tw[st].data();
        if (r == 4) {
            for (int j = 0; j < m; ++j) {
                cd w1 = tw[j * 4 + 1], w2 = tw[j * 4 + 2], w3 = tw[j * 4 + 3];
                if (inverse) { w1 = std::conj(w1); w2 = std::conj(w2); w3 = std::conj(w3); }
                for (int q = 0; q < s; ++q) {
                    const cd a0 = src[q + s * (j + 0 * m)];
                    const cd a1 = src[q + s * (j + 1 * m)];
                    const cd a2 = src[q + s * (j + 2 * m)];
                    const cd a3 = src[q + s * (j + 3 * m)];
                    const cd b0 = a0 + a2, b1 = a0 - a2, b2 = a1 + a3;
                    const cd d = a1 - a3;
                    const cd b3(sg * d.imag(), -sg * d.real());  // -i*d (fwd) / +i*d (inv)
                    dst[q + s * (4 * j + 0)] = b0 + b2;
                    dst[q + s * (4 * j + 1)] = (b1 + b3) * w1;
                    dst[q + s * (4 * j + 2)] = (b0 - b2) * w2;
                    dst[q + s * (4 * j + 3)] = (b1 - b3) * w3;
                }
            }
        } else if (r == 2) {
            for (int j = 0; j < m; ++j) {
                cd w1 = tw[j * 2 + 1];
                if (inverse) w1 = std::conj(w1);
                for (int q = 0; q < s; ++q) {
                    const cd a0 = src[q + s * j];
                    const cd a1 = src[q + s * (j + m)];
                    dst[q + s * (2 * j + 0)] = a0 + a1;
                    dst[q + s * (2 * j + 1)] = (a0 - a1) * w1;
                }
            }
        } else {
            // generic radix r (3, 5, other odd primes): direct r-point DFT
            std::vector<cd> root(r);
            for (int t = 0; t < r; ++t) root[t] = inverse ? std::conj(expi(t, r)) : expi(t, r);
            std::vector<cd> a(r);
            for (int j = 0; j < m; ++j) {
                for (int q = 0; q < s; ++q) {
                    for (int k = 0; k < r; ++k) a[k] = src[q + s * (j + k * m)];
                    for (int t = 0; t < r; ++t) {
                        cd acc = a[0];
                        for (int k = 1; k < r; ++k) acc += a[k] * root[(k * t) % r];
                        cd w = tw[j * r + t];
                        if (inverse) w = std::conj(w);
                        dst[q + s * (r * j + t)] = acc * w;
                    }
                }
            }
        }
        std::swap(src, dst);
        s *= r;
        n = m;
    }
    if (src != x)
        for (int i = 0; i < p->nh; ++i) x[i] = src[i];
}

inline std::vector<cd>& scratch(std::size_t n, int which) {
    thread_local std::vector<cd> buf[2];
    if (buf[which].size() < n) buf[which].resize(n);
    return buf[which];
}

}  // namespace pswe_fftw_shim

inline fftw_plan fftw_plan_dft_r2c_1d(int n, double*, fftw_complex*, unsigned) {
    if (n < 2 || n % 2) return nullptr;
    auto* p = new fftw_plan_s;
    p->n = n;
    p->nh = n / 2;
    p->r2c = true;
    pswe_fftw_shim::build(p);
    return p;
}

inline fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex*, double*, unsigned) {
    fftw_plan p = fftw_plan_dft_r2c_1d(n, nullptr, nullptr, 0);
    if (p) p->r2c = false;
    return p;
}

inline void fftw_destroy_plan(fftw_plan p) { delete p; }

inline void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
    using namespace pswe_fftw_shim;
    const int N = p->nh;
    auto& z = scratch(N, 0);
    auto& y = scratch(N, 1);
    for (int k = 0; k < N; ++k) z[k] = cd(in[2 * k], in[2 * k + 1]);
    cfft(p, z.data(), y.data(), false);
    cd* X = reinterpret_cast<cd*>(out);
    for (int k = 0; k <= N; ++k) {
        const cd zk = z[k % N];
        const cd zc = std::conj(z[(N - k) % N]);
        const cd e = 0.5 * (zk + zc);
        const cd o = cd(0.0, -0.5) * (zk - zc);
        X[k] = e + p->post[k] * o;
    }
}

inline void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
    using namespace pswe_fftw_shim;
    const int N = p->nh;
    const cd* X = reinterpret_cast<const cd*>(in);
    auto& z = scratch(N, 0);
    auto& y = scratch(N, 1);
    const cd x0(X[0].real(), 0.0), xn(X[N].real(), 0.0);
    for (int k = 0; k < N; ++k) {
        const cd a = (k == 0) ? x0 : X[k];
        const cd b = std::conj((k == 0) ? xn : X[N - k]);
        const cd e = a + b;
        const cd o = (a - b) * std::conj(p->post[k]);  // divide by W^k
        z[k] = e + cd(0.0, 1.0) * o;
    }
    cfft(p, z.data(), y.data(), true);
    for (int k = 0; k < N; ++k) {
        out[2 * k] = z[k].real();
        out[2 * k + 1] = z[k].imag();
    }
}
