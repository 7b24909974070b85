// Compile-time-sized shared-memory FFT (sm_100a, fp64): self-sorting Stockham DIF over G
// sequences of length NT. Each pass is one radix-P butterfly per thread computed entirely in
// registers (P in {16, 8, 4, 2, 3, 5}; largest first, so e.g. N = 384 = 16*8*3 takes 3 passes and
// N = 256 = 16*16 takes 2), followed by the inter-pass twiddles w_n^(j t) from a per-pass table
// in global memory ([t][j] layout, L1-resident). Shared buffers use padded indexing (pidx).
// Every index is compile-time; one __syncthreads per pass.
#pragma once

#include "pswe_internal.h"

namespace pswe {
namespace fftt {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
template <bool INV>
__device__ __forceinline__ double2 rot(double2 a) {  // -i a (forward), +i a (inverse)
    return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
template <bool INV>
__device__ __forceinline__ double2 root(const double2* W, int k) {
    const double2 w = W[k];
    return INV ? cconj(w) : w;
}

// cos / sin (2 pi k / 16), k = 0..15
__device__ constexpr double kC16[16] = {1.0,
                                        0.92387953251128675613,
                                        0.70710678118654752440,
                                        0.38268343236508977173,
                                        0.0,
                                        -0.38268343236508977173,
                                        -0.70710678118654752440,
                                        -0.92387953251128675613,
                                        -1.0,
                                        -0.92387953251128675613,
                                        -0.70710678118654752440,
                                        -0.38268343236508977173,
                                        0.0,
                                        0.38268343236508977173,
                                        0.70710678118654752440,
                                        0.92387953251128675613};

// multiply by w_16^k = exp(-+2 pi i k / 16) (compile-time k)
template <int K, bool INV>
__device__ __forceinline__ double2 w16(double2 a) {
    constexpr int k = K % 16;
    if constexpr (k == 0) return a;
    if constexpr (k == 4) return rot<INV>(a);
    if constexpr (k == 8) return make_double2(-a.x, -a.y);
    if constexpr (k == 12) return rot<!INV>(a);
    const double c = kC16[k], s = INV ? kC16[(k + 12) % 16] : -kC16[(k + 12) % 16];  // sin = cos(k - 4)
    return make_double2(a.x * c - a.y * s, a.x * s + a.y * c);
}

// multiply by w_12^k = exp(-+2 pi i k / 12) (compile-time k)
__device__ constexpr double kC12[12] = {1.0,
                                        0.86602540378443864676,
                                        0.5,
                                        0.0,
                                        -0.5,
                                        -0.86602540378443864676,
                                        -1.0,
                                        -0.86602540378443864676,
                                        -0.5,
                                        0.0,
                                        0.5,
                                        0.86602540378443864676};
template <int K, bool INV>
__device__ __forceinline__ double2 w12(double2 a) {
    constexpr int k = K % 12;
    if constexpr (k == 0) return a;
    if constexpr (k == 3) return rot<INV>(a);
    if constexpr (k == 6) return make_double2(-a.x, -a.y);
    if constexpr (k == 9) return rot<!INV>(a);
    const double c = kC12[k], s = INV ? kC12[(k + 9) % 12] : -kC12[(k + 9) % 12];  // sin = cos(k - 3)
    return make_double2(a.x * c - a.y * s, a.x * s + a.y * c);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
    const double2 b0 = cadd(x0, x2), b1 = csub(x0, x2), b2 = cadd(x1, x3);
    const double2 b3 = rot<INV>(csub(x1, x3));
    x0 = cadd(b0, b2);
    x1 = cadd(b1, b3);
    x2 = csub(b0, b2);
    x3 = csub(b1, b3);
}

// natural-order in-register DFTs: x[k] <- sum_n x[n] w_P^(n k)
template <int P, bool INV>
__device__ __forceinline__ void dft(double2 (&x)[P]) {
    if constexpr (P == 2) {
        const double2 a = x[0], b = x[1];
        x[0] = cadd(a, b);
        x[1] = csub(a, b);
    } else if constexpr (P == 3) {
        const double c1 = -0.5, s1 = 0.86602540378443864676372317075294;
        const double2 t1 = cadd(x[1], x[2]);
        const double2 t2 = make_double2(x[0].x + c1 * t1.x, x[0].y + c1 * t1.y);
        const double2 d = csub(x[1], x[2]);
        const double2 t3 = rot<INV>(make_double2(s1 * d.x, s1 * d.y));
        x[0] = cadd(x[0], t1);
        x[1] = cadd(t2, t3);
        x[2] = csub(t2, t3);
    } else if constexpr (P == 4) {
        dft4<INV>(x[0], x[1], x[2], x[3]);
    } else if constexpr (P == 5) {
        const double c1 = 0.30901699437494742410229341718282, c2 = -0.80901699437494742410229341718282;
        const double s1 = 0.95105651629515357211643933337938, s2 = 0.58778525229247312916870595463907;
        const double2 a0 = x[0];
        const double2 b1 = cadd(x[1], x[4]), b2 = cadd(x[2], x[3]), d1 = csub(x[1], x[4]), d2 = csub(x[2], x[3]);
        const double2 e1 = make_double2(a0.x + c1 * b1.x + c2 * b2.x, a0.y + c1 * b1.y + c2 * b2.y);
        const double2 e2 = make_double2(a0.x + c2 * b1.x + c1 * b2.x, a0.y + c2 * b1.y + c1 * b2.y);
        const double2 f1 = rot<INV>(make_double2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y));
        const double2 f2 = rot<INV>(make_double2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y));
        x[0] = cadd(a0, cadd(b1, b2));
        x[1] = cadd(e1, f1);
        x[4] = csub(e1, f1);
        x[2] = cadd(e2, f2);
        x[3] = csub(e2, f2);
    } else if constexpr (P == 6) {
        // 3 x 2: a = DFT3(x0, x2, x4), b = DFT3(x1, x3, x5) w6^k; y_k = a_k + b_k, y_{k+3} = a_k - b_k
        double2 a[3] = {x[0], x[2], x[4]}, b[3] = {x[1], x[3], x[5]};
        dft<3, INV>(a);
        dft<3, INV>(b);
        b[1] = w12<2, INV>(b[1]);
        b[2] = w12<4, INV>(b[2]);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            x[k] = cadd(a[k], b[k]);
            x[k + 3] = csub(a[k], b[k]);
        }
    } else if constexpr (P == 12) {
        // 3 x 4: n = n2 + 4 n1; A[n2] = DFT3 over n1, twiddle w12^(n2 k1), DFT4 over n2 -> k1 + 3 k2
        double2 f[4][3];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            f[r][0] = x[r];
            f[r][1] = x[r + 4];
            f[r][2] = x[r + 8];
            dft<3, INV>(f[r]);
        }
        f[1][1] = w12<1, INV>(f[1][1]);
        f[1][2] = w12<2, INV>(f[1][2]);
        f[2][1] = w12<2, INV>(f[2][1]);
        f[2][2] = w12<4, INV>(f[2][2]);
        f[3][1] = w12<3, INV>(f[3][1]);
        f[3][2] = w12<6, INV>(f[3][2]);
#pragma unroll
        for (int k1 = 0; k1 < 3; ++k1) {
            double2 a = f[0][k1], b = f[1][k1], c = f[2][k1], d = f[3][k1];
            dft4<INV>(a, b, c, d);
            x[k1] = a;
            x[k1 + 3] = b;
            x[k1 + 6] = c;
            x[k1 + 9] = d;
        }
    } else if constexpr (P == 8) {
        // DIT 2 x 4: E = DFT4(even), O = DFT4(odd); y_k = E_k + w8^k O_k, y_{k+4} = E_k - w8^k O_k
        double2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
        double2 o0 = x[1], o1 = x[3], o2 = x[5], o3 = x[7];
        dft4<INV>(e0, e1, e2, e3);
        dft4<INV>(o0, o1, o2, o3);
        o1 = w16<2, INV>(o1);
        o2 = w16<4, INV>(o2);
        o3 = w16<6, INV>(o3);
        x[0] = cadd(e0, o0);
        x[4] = csub(e0, o0);
        x[1] = cadd(e1, o1);
        x[5] = csub(e1, o1);
        x[2] = cadd(e2, o2);
        x[6] = csub(e2, o2);
        x[3] = cadd(e3, o3);
        x[7] = csub(e3, o3);
    } else if constexpr (P == 16) {
        // 4 x 4: n = r + 4 n2, k = k1 + 4 k2; F_r = DFT4 over n2, twiddle w16^(r k1), DFT4 over r
        double2 f[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            f[r][0] = x[r];
            f[r][1] = x[r + 4];
            f[r][2] = x[r + 8];
            f[r][3] = x[r + 12];
            dft4<INV>(f[r][0], f[r][1], f[r][2], f[r][3]);
        }
        f[1][1] = w16<1, INV>(f[1][1]);
        f[1][2] = w16<2, INV>(f[1][2]);
        f[1][3] = w16<3, INV>(f[1][3]);
        f[2][1] = w16<2, INV>(f[2][1]);
        f[2][2] = w16<4, INV>(f[2][2]);
        f[2][3] = w16<6, INV>(f[2][3]);
        f[3][1] = w16<3, INV>(f[3][1]);
        f[3][2] = w16<6, INV>(f[3][2]);
        f[3][3] = w16<9, INV>(f[3][3]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            double2 a = f[0][k1], b = f[1][k1], c = f[2][k1], d = f[3][k1];
            dft4<INV>(a, b, c, d);
            x[k1] = a;
            x[k1 + 4] = b;
            x[k1 + 8] = c;
            x[k1 + 12] = d;
        }
    }
}

__host__ __device__ constexpr int radix_of(int n) {
    return (n % 16 == 0) ? 16 : (n % 8 == 0) ? 8 : (n % 4 == 0) ? 4 : (n % 2 == 0) ? 2 : (n % 3 == 0) ? 3 : 5;
}

// padded shared-memory index: one element of padding every 16 makes the strided accesses of the
// first Stockham pass (stride P elements) conflict-free (4 wavefronts for 32 x 16-byte accesses)
__host__ __device__ constexpr int pidx(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded(int n) { return n + (n >> 4) + 1; }

// one radix-P pass: current length n = P*M, stride S; twiddles w_n^(j t) from the per-pass table
// TW[OFF + (t-1) M + j] (layout [t][j]: consecutive threads read consecutive entries)
template <int NT, int P, int M, int S, int G, int OFF, bool INV>
__device__ __forceinline__ void stage(const double2* __restrict__ src, double2* __restrict__ dst,
                                      const double2* __restrict__ TW) {
    constexpr int PER = NT / P;  // butterflies per sequence
    for (int it = threadIdx.x; it < G * PER; it += blockDim.x) {
        const int g = it / PER;
        const int r = it - g * PER;
        const int j = r / S;
        const int q = r - j * S;
        const int xb = g * NT + q + S * j;
        const int yb = g * NT + q + S * P * j;
        double2 v[P];
#pragma unroll
        for (int k = 0; k < P; ++k) v[k] = src[pidx(xb + k * S * M)];
        dft<P, INV>(v);
        dst[pidx(yb)] = v[0];
#pragma unroll
        for (int t = 1; t < P; ++t) {
            double2 o = v[t];
            if constexpr (M > 1) {
                const double2 w = __ldg(TW + OFF + (t - 1) * M + j);
                o = cmul(o, INV ? cconj(w) : w);
            }
            dst[pidx(yb + t * S)] = o;
        }
    }
}

template <int NT, int N, int S, int G, int OFF, bool INV>
struct Stages {
    static constexpr int P = radix_of(N);
    static constexpr int M = N / P;
    static constexpr int count = 1 + Stages<NT, M, S * P, G, OFF + (P - 1) * M, INV>::count;
    __device__ static void run(double2* a, double2* b, const double2* TW) {
        stage<NT, P, M, S, G, OFF, INV>(a, b, TW);
        __syncthreads();
        Stages<NT, M, S * P, G, OFF + (P - 1) * M, INV>::run(b, a, TW);
    }
};
template <int NT, int S, int G, int OFF, bool INV>
struct Stages<NT, 1, S, G, OFF, INV> {
    static constexpr int count = 0;
    __device__ static void run(double2*, double2*, const double2*) {}
};

// Complex FFT of G sequences in buf (padded indexing; scratch tmp); returns the buffer holding
// the result. Caller synchronises before (inputs ready); returns after a barrier.
template <int NT, int G, bool INV>
__device__ __forceinline__ double2* fft(double2* buf, double2* tmp, const double2* TW) {
    Stages<NT, NT, 1, G, 0, INV>::run(buf, tmp, TW);
    return (Stages<NT, NT, 1, G, 0, INV>::count & 1) ? tmp : buf;
}

}  // namespace fftt
}  // namespace pswe
