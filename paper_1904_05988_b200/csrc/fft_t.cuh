// Compile-time-sized shared-memory FFT (sm_100a, fp64): self-sorting Stockham DIF over G
// sequences of length NT, radices 4/2/3/5 chosen at compile time, twiddles from one table of
// the NT roots exp(-2 pi i k/NT) held in shared memory. Every index is a compile-time
// shift/multiply; one __syncthreads per stage.
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

constexpr int radix_of(int n) { return (n % 4 == 0) ? 4 : (n % 2 == 0) ? 2 : (n % 3 == 0) ? 3 : 5; }

// one radix-P stage: current length n = P*M, stride S; twiddle w_n^(j t) = W[j t (NT/n)]
template <int NT, int P, int M, int S, int G, bool INV>
__device__ __forceinline__ void stage(const double2* __restrict__ src, double2* __restrict__ dst,
                                      const double2* __restrict__ W) {
    constexpr int PER = NT / P;       // butterflies per sequence
    constexpr int TWS = NT / (P * M); // root-table stride of this stage
    for (int it = threadIdx.x; it < G * PER; it += blockDim.x) {
        const int g = it / PER;
        const int r = it - g * PER;
        const int j = r / S;
        const int q = r - j * S;
        const double2* x = src + g * NT + q + S * j;
        double2* y = dst + g * NT + q + S * P * j;
        if (P == 4) {
            const double2 a0 = x[0], a1 = x[S * M], a2 = x[2 * S * M], a3 = x[3 * S * M];
            const double2 b0 = cadd(a0, a2), b1 = csub(a0, a2), b2 = cadd(a1, a3);
            const double2 b3 = rot<INV>(csub(a1, a3));
            y[0] = cadd(b0, b2);
            y[S] = cmul(cadd(b1, b3), root<INV>(W, j * TWS));
            y[2 * S] = cmul(csub(b0, b2), root<INV>(W, 2 * j * TWS));
            y[3 * S] = cmul(csub(b1, b3), root<INV>(W, 3 * j * TWS));
        } else if (P == 2) {
            const double2 a0 = x[0], a1 = x[S * M];
            y[0] = cadd(a0, a1);
            y[S] = cmul(csub(a0, a1), root<INV>(W, j * TWS));
        } else if (P == 3) {
            const double c1 = -0.5, s1 = 0.86602540378443864676372317075294;
            const double2 a0 = x[0], a1 = x[S * M], a2 = x[2 * S * M];
            const double2 t1 = cadd(a1, a2);
            const double2 t2 = make_double2(a0.x + c1 * t1.x, a0.y + c1 * t1.y);
            const double2 d = csub(a1, a2);
            const double2 t3 = rot<INV>(make_double2(s1 * d.x, s1 * d.y));
            y[0] = cadd(a0, t1);
            y[S] = cmul(cadd(t2, t3), root<INV>(W, j * TWS));
            y[2 * S] = cmul(csub(t2, t3), root<INV>(W, 2 * j * TWS));
        } else {
            const double c1 = 0.30901699437494742410229341718282, c2 = -0.80901699437494742410229341718282;
            const double s1 = 0.95105651629515357211643933337938, s2 = 0.58778525229247312916870595463907;
            const double2 a0 = x[0], a1 = x[S * M], a2 = x[2 * S * M], a3 = x[3 * S * M], a4 = x[4 * S * M];
            const double2 b1 = cadd(a1, a4), b2 = cadd(a2, a3), d1 = csub(a1, a4), d2 = csub(a2, a3);
            const double2 e1 = make_double2(a0.x + c1 * b1.x + c2 * b2.x, a0.y + c1 * b1.y + c2 * b2.y);
            const double2 e2 = make_double2(a0.x + c2 * b1.x + c1 * b2.x, a0.y + c2 * b1.y + c1 * b2.y);
            const double2 f1 = rot<INV>(make_double2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y));
            const double2 f2 = rot<INV>(make_double2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y));
            y[0] = cadd(a0, cadd(b1, b2));
            y[S] = cmul(cadd(e1, f1), root<INV>(W, j * TWS));
            y[4 * S] = cmul(csub(e1, f1), root<INV>(W, 4 * j * TWS));
            y[2 * S] = cmul(cadd(e2, f2), root<INV>(W, 2 * j * TWS));
            y[3 * S] = cmul(csub(e2, f2), root<INV>(W, 3 * j * TWS));
        }
    }
}

template <int NT, int N, int S, int G, bool INV>
struct Stages {
    static constexpr int P = radix_of(N);
    static constexpr int M = N / P;
    static constexpr int count = 1 + Stages<NT, M, S * P, G, INV>::count;
    __device__ static void run(double2* a, double2* b, const double2* W) {
        stage<NT, P, M, S, G, INV>(a, b, W);
        __syncthreads();
        Stages<NT, M, S * P, G, INV>::run(b, a, W);
    }
};
template <int NT, int S, int G, bool INV>
struct Stages<NT, 1, S, G, INV> {
    static constexpr int count = 0;
    __device__ static void run(double2*, double2*, const double2*) {}
};

// Complex FFT of G sequences in buf (scratch tmp); returns the buffer holding the result.
// Caller synchronises before (inputs ready); returns after a barrier.
template <int NT, int G, bool INV>
__device__ __forceinline__ double2* fft(double2* buf, double2* tmp, const double2* W) {
    Stages<NT, NT, 1, G, INV>::run(buf, tmp, W);
    return (Stages<NT, NT, 1, G, INV>::count & 1) ? tmp : buf;
}

}  // namespace fftt
}  // namespace pswe
