// SDC sweeper and two-level transfers on device-resident space-time states.
//
// Reference: sdc.cpp:7-72 (spread, refresh_node, sweep, collocation_residual, sdc_step),
// quadrature.cpp:57-106 (tables), multilevel.cpp:9-158 (transfer matrices, restrict_states,
// fas_correction, interpolate_increment, interpolate_states).
//
// Kernels:
//   sweep_node_kernel   one SDC node update (sdc.cpp:31-46) fused with solve_implicit
//                       (swe.cpp:77-98): reads up to 4(M+1)+2 node arrays, writes state[m+1].
//   residual_kernel     collocation residual over all nodes, block max + atomicMax on the bit
//                       pattern of a non-negative double (order-independent => deterministic).
//   restrict/fas/interp coefficient gather kernels between the r-major triangles of Rf and Rc.
// The node refresh is one batched eval_imex call (4 launches) for any number of nodes.
#include <cmath>
#include <cstring>

#include "pswe_internal.h"
#include "tail.cuh"
#include "xrow.cuh"

#ifndef PSWE_SWEEP_PREP
#define PSWE_SWEEP_PREP 1
#endif

namespace pswe {
void eval_imex(pswe_plan& P, const pswe_params& prm, const double2* state, double2* f_imp, double2* f_exp, int n,
               cudaStream_t st);

// ---- quadrature tables (quadrature.cpp:19-106) ---------------------------------------------

static std::vector<double> lobatto_nodes(int n) {
    switch (n) {
        case 2: return {0.0, 1.0};
        case 3: return {0.0, 0.5, 1.0};
        case 5: {
            const double c = std::sqrt(3.0 / 7.0);
            return {0.0, 0.5 * (1.0 - c), 0.5, 0.5 * (1.0 + c), 1.0};
        }
        default: throw std::invalid_argument("build_tables: supported node counts are 2, 3, 5");
    }
}

double lagrange_basis(const std::vector<double>& nodes, int j, double x) {
    double acc = 1.0;
    for (int i = 0; i < (int)nodes.size(); ++i) {
        if (i == j) continue;
        acc *= (x - nodes[i]) / (nodes[j] - nodes[i]);
    }
    return acc;
}

static std::vector<double> lagrange_monomial(const std::vector<double>& nodes, int j) {
    std::vector<double> c{1.0};
    double denom = 1.0;
    for (int i = 0; i < (int)nodes.size(); ++i) {
        if (i == j) continue;
        denom *= nodes[j] - nodes[i];
        std::vector<double> next(c.size() + 1, 0.0);
        for (size_t k = 0; k < c.size(); ++k) {
            next[k] -= nodes[i] * c[k];
            next[k + 1] += c[k];
        }
        c = std::move(next);
    }
    for (double& v : c) v /= denom;
    return c;
}

static double integrate_monomial(const std::vector<double>& c, double upper) {
    double acc = 0.0, xp = upper;
    for (size_t k = 0; k < c.size(); ++k) {
        acc += c[k] * xp / static_cast<double>(k + 1);
        xp *= upper;
    }
    return acc;
}

Tables build_tables(int n) {
    Tables t;
    t.n = n;
    t.nodes = lobatto_nodes(n);
    t.q.assign((size_t)n * n, 0.0);
    t.qe.assign((size_t)n * n, 0.0);
    t.qi.assign((size_t)n * n, 0.0);
    for (int j = 0; j < n; ++j) {
        const auto c = lagrange_monomial(t.nodes, j);
        for (int m = 0; m < n; ++m) t.q[(size_t)m * n + j] = integrate_monomial(c, t.nodes[m]);
    }
    for (int m = 1; m < n; ++m)
        for (int j = 0; j < m; ++j) t.qe[(size_t)m * n + j] = t.nodes[j + 1] - t.nodes[j];
    const int mm = n - 1;
    std::vector<double> qt((size_t)mm * mm);
    for (int i = 0; i < mm; ++i)
        for (int j = 0; j < mm; ++j) qt[(size_t)i * mm + j] = t.q[(size_t)(1 + j) * n + 1 + i];
    for (int k = 0; k < mm; ++k)
        for (int i = k + 1; i < mm; ++i) {
            const double l = qt[(size_t)i * mm + k] / qt[(size_t)k * mm + k];
            for (int j = k; j < mm; ++j) qt[(size_t)i * mm + j] -= l * qt[(size_t)k * mm + j];
        }
    for (int i = 0; i < mm; ++i)
        for (int j = 0; j <= i; ++j) t.qi[(size_t)(1 + i) * n + 1 + j] = qt[(size_t)j * mm + i];
    return t;
}

// ---- kernels -------------------------------------------------------------------------------

constexpr int kMaxNodes = 5;

struct SweepNodeArgs {
    const double2* theta0;
    const double2* tau;  // tau[m+1] or nullptr
    double2* out;
    double2* fe_new[kMaxNodes];  // written at node m by the fused tail
    const double2* fe_old[kMaxNodes];
    double2* fi_new[kMaxNodes];
    const double2* fi_old[kMaxNodes];
    double ae[kMaxNodes], ai[kMaxNodes];  // dt*qE(m+1,j), dt*qI(m+1,j), j = 1..m
    double aq[kMaxNodes];                 // dt*q(m+1,j), j = 0..M
    double aii;                           // dt*qI(m+1,m+1)
    // quadrature of the OLD right-hand sides, S_m = sum_j dt q(m+1,j) (F_I^old_j + F_E^old_j): the same
    // ten arrays for every node of the sweep, so the first node's kernel (which reads them anyway)
    // forms S_1 .. S_{M-1} for the later nodes, which read one array instead of ten
    double aq_all[kMaxNodes][kMaxNodes];  // first node: dt*q(m'+1, j) for m' = 1..M-1
    double2* qsum_out;                    // first node: S_1 .. S_{M-1}, [M-1][3K]
    const double2* qsum_in;               // later nodes: S_m (or nullptr: the ten-array sum)
    double2* fi0_dst;                     // node 0's F_I, F_E copied old -> new buffer (first node only)
    double2* fe0_dst;
    const double2* proj;                  // fused tail: projections of state m ([5][Kx]), the state,
    const double2* st_m;                  // and the degree recurrence eps
    const double* eps;
    int m, M, R;
    double inv_a2, phi_bar, nu;
    double* xt;           // XP: the new state's X tiles (one column tile, [16][10] per chunk)
    const int* cbase;     //     chunk base per order m
    const double* rtab;   //     1/(s(s+1))
    double radius;
};

namespace {

__device__ __forceinline__ void axpy(double2& acc, double a, double2 x) {
    acc.x += a * x.x;
    acc.y += a * x.y;
}

// (r, s) of r-major index k (field.hpp:29-32)
using tailc::decode_rs;
__device__ __forceinline__ int degree_of(int R, long k) {
    int m, s;
    decode_rs(R, k, m, s);
    return s;
}

// rhs (sdc.cpp:31-44, same axpy order) then solve_implicit (swe.cpp:77-98). Block (128, 3): thread
// (x, f) accumulates field f of coefficient k (node loops unrolled over NN nodes, loads predicated on
// j <= m so they all issue together); field 0's thread then solves the coupled (Phi, delta) system.
// TAIL: the same kernel first finishes node m's evaluation (tail.cuh, the five projections of
// state m in proj) and writes F_new[m], which the node-m+1 update then takes from registers -
// one launch fewer per node, the same expressions as eval_tail + sweep_node (tail.cuh).
// XP: the block also writes the new state's inverse-Legendre X tiles (the next evaluation's
// prep, xrow.cuh) - block (130, 3) with one halo coefficient on either side, so the degree
// neighbours s-1, s+1 of every owned coefficient are in shared memory; the evaluation then skips
// its prep launch (PSWE_SWEEP_PREP).
template <int NN, bool TAIL, bool XP>
__global__ void __launch_bounds__(XP ? 390 : 384) sweep_node_kernel(SweepNodeArgs A) {
    constexpr int BX = XP ? 130 : 128;
    __shared__ double2 rs[3][BX];
    __shared__ double2 snew[XP ? 3 : 1][XP ? BX : 1];
    const long K = (long)(A.R + 1) * (A.R + 2) / 2;
    const long k = (long)blockIdx.x * 128 + threadIdx.x - (XP ? 1 : 0);
    const bool owned = !XP || (threadIdx.x >= 1 && threadIdx.x <= 128);
    const bool valid = k >= 0 && k < K;
    const int f = threadIdx.y;
    pdl_trigger();
    // XP: the plan constants of this coefficient's X-tile row(s) load before the wait
    int xm = 0, xs = 0, xcb = 0;
    xrow::Fac xF{}, xF1{};
    // TAIL: node m's (order, degree) and its eps pair are plan constants too
    int tm = 0, ts = 0;
    double teu = 0.0, tel = 0.0;
    if constexpr (TAIL) {
        if (valid) {
            tailc::decode_rs(A.R, k, tm, ts);
            teu = A.eps[off_ext(A.R, tm) + ts - tm + 1];
            tel = A.eps[off_ext(A.R, tm) + ts - tm];
        }
    }
    if constexpr (XP) {
        if (f == 0 && valid && owned) {
            tailc::decode_rs(A.R, k, xm, xs);
            const long bx = off_ext(A.R, xm);
            xcb = A.cbase[xm];
            xF = xrow::factors(A.R, xm, xs, bx, A.eps, A.rtab, A.radius);
            if (xs == A.R) xF1 = xrow::factors(A.R, xm, A.R + 1, bx, A.eps, A.rtab, A.radius);
        }
    }
    pdl_wait();  // F and states (TAIL: the projections) come from the preceding kernel
    if (valid) {
        const long i = f * K + k;
        double2 fe_m = make_double2(0.0, 0.0), fi_m = make_double2(0.0, 0.0);
        if constexpr (TAIL) {
            const long Kx = (long)(A.R + 1) * (A.R + 4) / 2;
            tailc::tail_field(f, teu, tel, A.proj, Kx, off_ext(A.R, tm), tm, ts, -ts * (ts + 1.0) * A.inv_a2,
                              A.st_m, K, k, A.phi_bar, A.nu, true, fe_m, fi_m);
            if (owned) {
                A.fe_new[A.m][i] = fe_m;
                A.fi_new[A.m][i] = fi_m;
            }
        }
        double2 acc = A.theta0[i];
#pragma unroll
        for (int j = 1; j < NN; ++j) {
            if (j <= A.m) {
                const bool reg = TAIL && j == A.m;
                axpy(acc, A.ae[j], reg ? fe_m : A.fe_new[j][i]);
                axpy(acc, -A.ae[j], A.fe_old[j][i]);
                axpy(acc, A.ai[j], reg ? fi_m : A.fi_new[j][i]);
                axpy(acc, -A.ai[j], A.fi_old[j][i]);
            }
        }
        axpy(acc, -A.aii, A.fi_old[A.m + 1][i]);
        if (A.qsum_in) {
            const double2 q = A.qsum_in[i];
            acc.x += q.x;
            acc.y += q.y;
        } else {
            double2 qs[NN];  // S_{m'} of the later nodes (first node only)
#pragma unroll
            for (int mm = 0; mm < NN; ++mm) qs[mm] = make_double2(0.0, 0.0);
            double2 qm = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < NN; ++j) {
                const double2 fij = A.fi_old[j][i], fej = A.fe_old[j][i];
                axpy(qm, A.aq[j], fij);
                axpy(qm, A.aq[j], fej);
                if (A.qsum_out) {
#pragma unroll
                    for (int mm = 1; mm < NN - 1; ++mm) {
                        axpy(qs[mm], A.aq_all[mm][j], fij);
                        axpy(qs[mm], A.aq_all[mm][j], fej);
                    }
                }
                if (j == 0 && A.fi0_dst && owned) {  // node 0 keeps its right-hand sides (sdc.cpp:22-29)
                    A.fi0_dst[i] = fij;
                    A.fe0_dst[i] = fej;
                }
            }
            acc.x += qm.x;
            acc.y += qm.y;
            if (A.qsum_out && owned) {
#pragma unroll
                for (int mm = 1; mm < NN - 1; ++mm)
                    if (mm < A.M) A.qsum_out[(size_t)(mm - 1) * 3 * K + i] = qs[mm];
            }
        }
        if (A.tau) {
            const double2 t = A.tau[i];
            acc.x += t.x;
            acc.y += t.y;
        }
        rs[f][threadIdx.x] = acc;
    }
    __syncthreads();
    int s = 0;
    if (f == 0 && valid) {
        const double2 r0 = rs[0][threadIdx.x], r1 = rs[1][threadIdx.x], r2 = rs[2][threadIdx.x];
        s = degree_of(A.R, k);
        const double c = A.aii;
        const double lam = -s * (s + 1.0) * A.inv_a2;
        const double diff = 1.0 - c * A.nu * lam;
        const double2 bp = make_double2(r0.x / diff, r0.y / diff);
        const double2 bz = make_double2(r1.x / diff, r1.y / diff);
        const double2 bd = make_double2(r2.x / diff, r2.y / diff);
        const double ce = c / diff;
        const double det = 1.0 - ce * ce * A.phi_bar * lam;
        const double2 nph = make_double2((bp.x - ce * A.phi_bar * bd.x) / det, (bp.y - ce * A.phi_bar * bd.y) / det);
        const double2 ndv = make_double2((bd.x - ce * lam * bp.x) / det, (bd.y - ce * lam * bp.y) / det);
        if (owned) {
            A.out[k] = nph;
            A.out[2 * K + k] = ndv;
            A.out[K + k] = bz;
        }
        if constexpr (XP) {
            snew[0][threadIdx.x] = nph;
            snew[1][threadIdx.x] = bz;
            snew[2][threadIdx.x] = ndv;
        }
    }
    if constexpr (XP) {
        __syncthreads();
        if (f != 0 || !valid || !owned) return;
        const int m = xm, R = A.R, x = threadIdx.x, cb = xcb;
        s = xs;
        // degree s' of this order: shared-memory slot of the clamped neighbour (the halo holds the
        // coefficients k0 - 1 and k0 + 128; clamped positions are never used by xrow::columns)
        auto at = [&](int fld, int sp) { return snew[fld][x + (min(max(sp, m), R) - s)]; };
        auto emit = [&](int sd, const xrow::Fac& F) {  // X-tile row of degree sd (s or R+1)
            const int t = sd - m;
            double2 v[4];
            xrow::columns(F, R, m, sd, A.radius, at(0, sd), at(1, sd - 1), at(1, sd), at(1, sd + 1), at(2, sd - 1),
                          at(2, sd), at(2, sd + 1), v);
            double2* row = reinterpret_cast<double2*>(A.xt + ((long)(cb + t / 16) * 16 + (t & 15)) * 10);
            row[0] = v[0];
            row[1] = v[1];
            row[2] = v[2];
            row[3] = v[3];
            row[4] = make_double2(0.0, 0.0);
        };
        emit(s, xF);
        if (s == R) {  // the extra degree R+1 (H-sum terms), then zero rows to the end of the chunk
            emit(R + 1, xF1);
            const int nrow = (R + 2 - m + 15) / 16 * 16;
            for (int t = R + 2 - m; t < nrow; ++t) {
                double2* row = reinterpret_cast<double2*>(A.xt + ((long)(cb + t / 16) * 16 + (t & 15)) * 10);
#pragma unroll
                for (int c = 0; c < 5; ++c) row[c] = make_double2(0.0, 0.0);
            }
        }
    }
}

struct ResidualArgs {
    const double2* state[kMaxNodes];
    const double2* fi[kMaxNodes];
    const double2* fe[kMaxNodes];
    double w[kMaxNodes][kMaxNodes];  // -dt*q(m,j)
    int nn;
    long n3;  // 3K
    unsigned long long* bmax;  // per-block maxima (bit patterns of non-negative doubles)
    unsigned int* count;       // blocks done; the last block reduces and resets it to 0
};

// collocation residual of flat index i (sdc.cpp:46-62): F_I, F_E of every node loaded once and
// reused for all NN rows (same axpy order). LAST: node NN-1's right-hand sides come from registers.
template <int NN, bool LAST>
__device__ __forceinline__ double residual_at(const ResidualArgs& A, long i, double2 fi_last, double2 fe_last) {
    double2 fi[NN], fe[NN], st[NN];
#pragma unroll
    for (int j = 0; j < NN; ++j) {
        if (LAST && j == NN - 1) {
            fi[j] = fi_last;
            fe[j] = fe_last;
        } else {
            fi[j] = A.fi[j][i];
            fe[j] = A.fe[j][i];
        }
        st[j] = A.state[j][i];
    }
    const double2 s0 = st[0];
    double mx = 0.0;
#pragma unroll
    for (int m = 0; m < NN; ++m) {
        double2 acc = make_double2(st[m].x - s0.x, st[m].y - s0.y);
#pragma unroll
        for (int j = 0; j < NN; ++j) {
            axpy(acc, A.w[m][j], fi[j]);
            axpy(acc, A.w[m][j], fe[j]);
        }
        mx = fmax(mx, hypot(acc.x, acc.y));
    }
    return mx;
}

// block max, then the last block to finish reduces the block maxima (max is order-independent, so
// the result is deterministic whatever the block shape) - no zeroing of *out beforehand
__device__ __forceinline__ void residual_finish(double mx, const ResidualArgs& A, unsigned long long* out) {
    const unsigned tid = threadIdx.x + threadIdx.y * blockDim.x;
    const unsigned nthr = blockDim.x * blockDim.y;
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ double wm[32];
    if ((tid & 31) == 0) wm[tid >> 5] = mx;
    __syncthreads();
    if (tid < 32) {
        mx = tid < (nthr >> 5) ? wm[tid] : 0.0;
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (tid == 0) {
            A.bmax[blockIdx.x] = (unsigned long long)__double_as_longlong(mx);
            __threadfence();
            wm[0] = atomicAdd(A.count, 1u) == gridDim.x - 1 ? 1.0 : 0.0;
        }
    }
    __syncthreads();
    if (wm[0] == 0.0) return;
    __threadfence();
    unsigned long long b = 0ull;
    for (unsigned j = tid; j < gridDim.x; j += nthr) b = max(b, __ldcg(A.bmax + j));
    for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    __shared__ unsigned long long wb[32];
    if ((tid & 31) == 0) wb[tid >> 5] = b;
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < (int)(nthr >> 5); ++w) b = max(b, wb[w]);
        *out = b;
        *A.count = 0u;
    }
}

template <int NN>
__global__ void residual_kernel(ResidualArgs A, unsigned long long* out) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    pdl_trigger();
    pdl_wait();
    const double2 z = make_double2(0.0, 0.0);
    const double mx = i < A.n3 ? residual_at<NN, false>(A, i, z, z) : 0.0;
    residual_finish(mx, A, out);
}

// the sweep's last evaluation tail (eval_tail_kernel's expressions, tail.cuh) fused with the
// collocation residual that follows it in the PFASST schedule (pfasst.cpp OP_SWEEP_FINE +
// OP_RESIDUAL): block (128, 3), thread (x, f) finishes field f of coefficient k of the last node,
// stores it and takes it from registers into that index's residual rows - one launch and one
// round trip of F[M] fewer; every value is the one the two separate kernels produce
template <int NN>
__global__ void __launch_bounds__(384) tail_residual_kernel(ResidualArgs A, const double* __restrict__ eps,
                                                            const double2* __restrict__ proj,
                                                            double2* __restrict__ fi_last,
                                                            double2* __restrict__ fe_last, int R, double inv_a2,
                                                            double phi_bar, double nu, unsigned long long* out) {
    const long K = (long)(R + 1) * (R + 2) / 2;
    const long Kx = (long)(R + 1) * (R + 4) / 2;
    const long k = (long)blockIdx.x * 128 + threadIdx.x;
    const int f = threadIdx.y;
    pdl_trigger();
    int m = 0, s = 0;
    double eu = 0.0, el = 0.0;
    if (k < K) {
        decode_rs(R, k, m, s);
        eu = eps[off_ext(R, m) + s - m + 1];
        el = eps[off_ext(R, m) + s - m];
    }
    pdl_wait();  // the projections come from the forward Legendre kernel
    double mx = 0.0;
    if (k < K) {
        double2 e, i;
        tailc::tail_field(f, eu, el, proj, Kx, off_ext(R, m), m, s, -s * (s + 1.0) * inv_a2, A.state[NN - 1], K, k,
                          phi_bar, nu, true, e, i);
        const long ix = f * K + k;
        fe_last[ix] = e;
        fi_last[ix] = i;
        mx = residual_at<NN, true>(A, ix, i, e);
    }
    residual_finish(mx, A, out);
}

struct CopyArgs {
    double2* dst[8];
    const double2* src[8];
    long len;  // double2 per pair
};
// n device-to-device copies in one launch (blockIdx.y = pair): a kernel rather than memcpy nodes,
// so the stream / graph chain keeps its programmatic-launch overlap
__global__ void copy_kernel(CopyArgs A) {
    pdl_trigger();
    pdl_wait();
    const int p = blockIdx.y;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < A.len; i += (long)gridDim.x * blockDim.x)
        A.dst[p][i] = A.src[p][i];
}

// coarse coefficient kc of a state (3 fields) -> fine coefficient index
__device__ __forceinline__ long fine_index(int Rf, int Rc, long kc3, long Kc, long Kf) {
    const int f = (int)(kc3 / Kc);
    const long kc = kc3 - f * Kc;
    int m, s;
    decode_rs(Rc, kc, m, s);
    return f * Kf + off_std(Rf, m) + (s - m);
}

struct TimeMatArgs {
    const double2* src[kMaxNodes];
    const double2* src2[kMaxNodes];  // optional second operand (added / subtracted)
    double w[kMaxNodes][kMaxNodes];
    int rows, cols;
};

// y[i] = restrict( sum_j w(i,j) x[j] ) for every coarse node i (multilevel.cpp:100-107); row i = blockIdx.y
__global__ void restrict_states_kernel(TimeMatArgs A, double2* out0, long stride_out, int Rf, int Rc) {
    const long Kc = (long)(Rc + 1) * (Rc + 2) / 2, Kf = (long)(Rf + 1) * (Rf + 2) / 2;
    const long kc3 = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    pdl_trigger();
    pdl_wait();
    if (kc3 >= 3 * Kc) return;
    const long kf3 = fine_index(Rf, Rc, kc3, Kc, Kf);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < kMaxNodes; ++j)
        if (j < A.cols && A.w[i][j] != 0.0) axpy(acc, A.w[i][j], A.src[j][kf3]);
    out0[i * stride_out + kc3] = acc;
}

// tau_i = dt * [ restrict(sum_j qfr(i,j)(FI_f[j] + FE_f[j])) - sum_j qc(i,j)(FI_c[j] + FE_c[j]) ]
// (multilevel.cpp:109-137, same operation order)
// Multi-level (Eq. 19): tau_c += R tau_f for a fine level that itself carries a
// FAS term (three-level PFASST): the cumulative-form tau_f is restricted like a state (time matrix
// tr at the coarse nodes, then spectral truncation).
struct FasArgs {
    const double2* fi_f[kMaxNodes];
    const double2* fe_f[kMaxNodes];
    const double2* fi_c[kMaxNodes];
    const double2* fe_c[kMaxNodes];
    double qfr[kMaxNodes][kMaxNodes];
    double qc[kMaxNodes][kMaxNodes];
    const double2* tau_f;  // nullable: [mf][3 Kf]
    double tr[kMaxNodes][kMaxNodes];
    int mc, mf, Rf, Rc;
    double dt;
};
// row i = blockIdx.y; node loops unrolled over kMaxNodes with predicated loads (same order as before)
__global__ void fas_kernel(FasArgs A, double2* tau) {
    const long Kc = (long)(A.Rc + 1) * (A.Rc + 2) / 2, Kf = (long)(A.Rf + 1) * (A.Rf + 2) / 2;
    const long kc3 = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    pdl_trigger();
    pdl_wait();
    if (kc3 >= 3 * Kc) return;
    const long kf3 = fine_index(A.Rf, A.Rc, kc3, Kc, Kf);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < kMaxNodes; ++j) {
        const double w = A.qfr[i][j];
        if (j < A.mf && w != 0.0) {
            axpy(acc, w, A.fi_f[j][kf3]);
            axpy(acc, w, A.fe_f[j][kf3]);
        }
    }
#pragma unroll
    for (int j = 0; j < kMaxNodes; ++j) {
        const double w = A.qc[i][j];
        if (j < A.mc && w != 0.0) {
            axpy(acc, -w, A.fi_c[j][kc3]);
            axpy(acc, -w, A.fe_c[j][kc3]);
        }
    }
    double2 t = make_double2(acc.x * A.dt, acc.y * A.dt);
    if (A.tau_f) {
#pragma unroll
        for (int j = 0; j < kMaxNodes; ++j) {
            const double w = A.tr[i][j];
            if (j < A.mf && w != 0.0) axpy(t, w, A.tau_f[j * 3 * Kf + kf3]);
        }
    }
    tau[i * 3 * Kc + kc3] = t;
}

// fine[i] (+)= sum_j ti(i,j) pad(a[j] - b[j])  (interpolate_increment / interpolate_states,
// multilevel.cpp:139-158). mode 0: add increments to 3 families (state, F_I, F_E);
// mode 1: assign interpolated states.
struct InterpArgs {
    const double2* a[3][kMaxNodes];
    const double2* b[3][kMaxNodes];  // saved (mode 0)
    double2* dst[3][kMaxNodes];
    double w[kMaxNodes][kMaxNodes];  // ti: (mf x mc)
    int mf, mc, Rf, Rc, nfam;
    double2* dstate0;  // optional: node-0 state increment (fine layout)
};
// one (family, fine node) pair per blockIdx.y: blockIdx.y = fam * mf + i
__global__ void interp_kernel(InterpArgs A, int mode) {
    const long Kc = (long)(A.Rc + 1) * (A.Rc + 2) / 2, Kf = (long)(A.Rf + 1) * (A.Rf + 2) / 2;
    const long kf3 = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int fam = blockIdx.y / A.mf, i = blockIdx.y - fam * A.mf;
    pdl_trigger();
    pdl_wait();
    if (kf3 >= 3 * Kf) return;
    const int f = (int)(kf3 / Kf);
    const long kf = kf3 - f * Kf;
    int m, s;
    decode_rs(A.Rf, kf, m, s);
    const bool inside = (m <= A.Rc && s <= A.Rc);
    double2 acc = make_double2(0.0, 0.0);
    if (inside) {
        const long kc3 = f * Kc + off_std(A.Rc, m) + (s - m);
#pragma unroll
        for (int j = 0; j < kMaxNodes; ++j) {
            const double w = A.w[i][j];
            if (j < A.mc && w != 0.0) {
                double2 d = A.a[fam][j][kc3];
                if (mode == 0) {
                    const double2 sv = A.b[fam][j][kc3];
                    d = make_double2(d.x - sv.x, d.y - sv.y);
                }
                axpy(acc, w, d);
            }
        }
    }
    double2* o = A.dst[fam][i] + kf3;
    if (mode == 0) {
        const double2 cur = *o;
        *o = make_double2(cur.x + acc.x, cur.y + acc.y);
        if (fam == 0 && i == 0 && A.dstate0) A.dstate0[kf3] = acc;
    } else {
        *o = acc;
    }
}

// interpolate_increment_add restricted to the coefficients that can change: the increment is the
// zero-padded coarse difference, so fine coefficients outside the coarse triangle (3/4 of them for
// T255 -> T127) receive exactly zero - the full-range kernel above read and rewrote them anyway.
// One thread per (coarse coefficient, field); blockIdx.y = fam * mf + i. dstate0 (optional) gets
// the node-0 state increment inside the triangle; zero_out_kernel writes its zeros outside.
__global__ void interp_inc_kernel(InterpArgs A) {
    const long Kc = (long)(A.Rc + 1) * (A.Rc + 2) / 2, Kf = (long)(A.Rf + 1) * (A.Rf + 2) / 2;
    const long kc3 = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int fam = blockIdx.y / A.mf, i = blockIdx.y - fam * A.mf;
    pdl_trigger();
    pdl_wait();
    if (kc3 >= 3 * Kc) return;
    const int f = (int)(kc3 / Kc);
    const long kc = kc3 - f * Kc;
    int m, s;
    decode_rs(A.Rc, kc, m, s);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < kMaxNodes; ++j) {
        const double w = A.w[i][j];
        if (j < A.mc && w != 0.0) {
            const double2 a = A.a[fam][j][kc3], b = A.b[fam][j][kc3];
            axpy(acc, w, make_double2(a.x - b.x, a.y - b.y));
        }
    }
    const long kf3 = f * Kf + off_std(A.Rf, m) + (s - m);
    double2* o = A.dst[fam][i] + kf3;
    const double2 cur = *o;
    *o = make_double2(cur.x + acc.x, cur.y + acc.y);
    if (fam == 0 && i == 0 && A.dstate0) A.dstate0[kf3] = acc;
}

__global__ void zero_out_kernel(int Rf, int Rc, double2* __restrict__ y) {
    const long Kf = (long)(Rf + 1) * (Rf + 2) / 2;
    const long kf3 = (long)blockIdx.x * blockDim.x + threadIdx.x;
    pdl_trigger();
    pdl_wait();
    if (kf3 >= 3 * Kf) return;
    int m, s;
    decode_rs(Rf, kf3 % Kf, m, s);
    if (m > Rc || s > Rc) y[kf3] = make_double2(0.0, 0.0);
}

}  // namespace
}  // namespace pswe

using namespace pswe;

namespace pswe {

static void copies(const std::vector<std::pair<double2*, const double2*>>& cp, long len, cudaStream_t st) {
    for (size_t b = 0; b < cp.size(); b += 8) {
        CopyArgs A{};
        const int n = (int)std::min<size_t>(8, cp.size() - b);
        for (int i = 0; i < n; ++i) {
            A.dst[i] = cp[b + i].first;
            A.src[i] = cp[b + i].second;
        }
        A.len = len;
        const unsigned gx = (unsigned)std::min<long>((len + 255) / 256, 296);
        launch_pdl(copy_kernel, dim3(gx, n), dim3(256), 0, st, A);
        PSWE_LAUNCH_CHECK();
    }
}

static void refresh(pswe_level* L, int first, int count, cudaStream_t st) {
    if (count <= 0) return;
    eval_imex(*L->plan, L->prm, L->st(first), L->fi(first), L->fe(first), count, st);
}

void level_spread(pswe_level* L, const double2* theta0, cudaStream_t st) {
    std::vector<std::pair<double2*, const double2*>> cp;
    for (int m = 0; m < L->nn; ++m)
        if (L->st(m) != theta0) cp.push_back({L->st(m), theta0});
    copies(cp, 3 * L->K, st);
    refresh(L, 0, 1, st);
    cp.clear();
    for (int m = 1; m < L->nn; ++m) {
        cp.push_back({L->fi(m), L->fi(0)});
        cp.push_back({L->fe(m), L->fe(0)});
    }
    copies(cp, 3 * L->K, st);
}

void level_refresh(pswe_level* L, int first, int count, cudaStream_t st) { refresh(L, first, count, st); }

static ResidualArgs residual_args(pswe_level* L, double dt, int set) {
    ResidualArgs A{};
    A.nn = L->nn;
    A.n3 = 3 * L->K;
    for (int m = 0; m < L->nn; ++m) {
        A.state[m] = L->st(m);
        A.fi[m] = L->fi(m, set);
        A.fe[m] = L->fe(m, set);
        for (int j = 0; j < L->nn; ++j) A.w[m][j] = -dt * L->tab.Q(m, j);
    }
    A.bmax = L->d_bmax;
    A.count = L->d_count;
    return A;
}

void level_sweep(pswe_level* L, double dt, const double2* tau, cudaStream_t st, double* res_out) {
    const int M = L->nn - 1;
    const int old = L->cur, nw = 1 - L->cur;
    const size_t bytes = 3 * L->K * sizeof(double2);
    // node 0 keeps its right-hand sides (sdc.cpp:22-29: F_old is a copy; node 0 is not refreshed):
    // the first node's update kernel copies them into the new buffer
    (void)bytes;
    const Tables& t = L->tab;
    // the node update also writes the next evaluation's X tiles (its prep launch is skipped)
    static const bool xp_env = [] { const char* e = getenv("PSWE_NO_SWEEP_PREP"); return !(e && atoi(e) != 0); }();
    // (measured per level size: T255 5-node sweep -5.6%, T255 3-node -5%, T127 even, T511 +4.8% - the
    // larger update kernel then costs more than the prep launch it saves)
    const bool xp = PSWE_SWEEP_PREP && xp_env && L->K <= 65536 && xtiles_by_sweep_ok(*L->plan);
    if (xp) xtile_reserve(*L->plan, 4, INV_EVAL);
    for (int m = 0; m < M; ++m) {
        SweepNodeArgs A{};
        A.theta0 = L->st(0);
        A.tau = tau ? tau + (size_t)(m + 1) * 3 * L->K : nullptr;
        A.out = L->st(m + 1);
        for (int j = 0; j <= M; ++j) {
            A.fe_new[j] = L->fe(j, nw);
            A.fi_new[j] = L->fi(j, nw);
            A.fe_old[j] = L->fe(j, old);
            A.fi_old[j] = L->fi(j, old);
            A.aq[j] = dt * t.Q(m + 1, j);
            if (j >= 1 && j <= m) {
                A.ae[j] = dt * t.QE(m + 1, j);
                A.ai[j] = dt * t.QI(m + 1, j);
            }
        }
        A.aii = dt * t.QI(m + 1, m + 1);
        if (L->d_qsum && M >= 2) {
            if (m == 0) {
                A.qsum_out = L->d_qsum;
                for (int mm = 1; mm < M; ++mm)
                    for (int j = 0; j <= M; ++j) A.aq_all[mm][j] = dt * t.Q(mm + 1, j);
            } else {
                A.qsum_in = L->d_qsum + (size_t)(m - 1) * 3 * L->K;
            }
        }
        A.fi0_dst = m == 0 ? L->fi(0, nw) : nullptr;
        A.fe0_dst = m == 0 ? L->fe(0, nw) : nullptr;
        A.m = m;
        A.M = M;
        A.R = L->R;
        A.inv_a2 = 1.0 / (L->prm.radius * L->prm.radius);
        A.phi_bar = L->prm.phi_bar;
        A.nu = L->prm.nu;
        const dim3 grid((unsigned)((L->K + 127) / 128)), block(xp ? 130 : 128, 3);
        A.eps = L->plan->d_eps;
        if (xp) {
            A.xt = L->plan->d_xtile;
            A.cbase = L->plan->d_chk_off;
            A.rtab = L->plan->d_rlap;
            A.radius = L->prm.radius;
        }
        if (m > 0) {  // finish node m's evaluation in the same kernel
            A.proj = L->plan->d_proj;
            A.st_m = L->st(m);
        }
#define PSWE_SWEEP_LAUNCH(NN)                                                                   \
    if (m > 0 && xp) launch_pdl(sweep_node_kernel<NN, true, true>, grid, block, 0, st, A);      \
    else if (m > 0) launch_pdl(sweep_node_kernel<NN, true, false>, grid, block, 0, st, A);      \
    else if (xp) launch_pdl(sweep_node_kernel<NN, false, true>, grid, block, 0, st, A);         \
    else launch_pdl(sweep_node_kernel<NN, false, false>, grid, block, 0, st, A);
        switch (L->nn) {
            case 2: PSWE_SWEEP_LAUNCH(2) break;
            case 3: PSWE_SWEEP_LAUNCH(3) break;
            default: PSWE_SWEEP_LAUNCH(5) break;
        }
#undef PSWE_SWEEP_LAUNCH
        PSWE_LAUNCH_CHECK();
        eval_imex_proj(*L->plan, L->prm, L->st(m + 1), 1, st, xp);
    }
    if (res_out) {  // the last node's tail and the residual after the sweep in one launch
        const ResidualArgs A = residual_args(L, dt, nw);
        const dim3 grid((unsigned)((L->K + 127) / 128)), block(128, 3);
        auto* o = reinterpret_cast<unsigned long long*>(res_out);
        const pswe_plan& P = *L->plan;
        const double ia2 = 1.0 / (L->prm.radius * L->prm.radius);
#define PSWE_TR_LAUNCH(NN)                                                                                  \
    launch_pdl(tail_residual_kernel<NN>, grid, block, 0, st, A, P.d_eps, P.d_proj, L->fi(M, nw), L->fe(M, nw), \
               L->R, ia2, L->prm.phi_bar, L->prm.nu, o);
        switch (L->nn) {
            case 2: PSWE_TR_LAUNCH(2) break;
            case 3: PSWE_TR_LAUNCH(3) break;
            default: PSWE_TR_LAUNCH(5) break;
        }
#undef PSWE_TR_LAUNCH
        PSWE_LAUNCH_CHECK();
    } else {
        eval_tail(*L->plan, L->prm, L->plan->d_proj, L->st(M), L->fi(M, nw), L->fe(M, nw), 1, st);
    }
    L->cur = nw;
}

void level_residual(pswe_level* L, double dt, double* out, cudaStream_t st) {
    const ResidualArgs A = residual_args(L, dt, L->cur);
    const int bs = 256;
    const unsigned g = (unsigned)((A.n3 + bs - 1) / bs);
    auto* o = reinterpret_cast<unsigned long long*>(out);
    switch (L->nn) {
        case 2: launch_pdl(residual_kernel<2>, dim3(g), dim3(bs), 0, st, A, o); break;
        case 3: launch_pdl(residual_kernel<3>, dim3(g), dim3(bs), 0, st, A, o); break;
        default: launch_pdl(residual_kernel<5>, dim3(g), dim3(bs), 0, st, A, o); break;
    }
    PSWE_LAUNCH_CHECK();
}

void pair_restrict_states(pswe_pair* P, cudaStream_t st) {
    pswe_level *F = P->fine, *C = P->coarse;
    TimeMatArgs A{};
    A.rows = C->nn;
    A.cols = F->nn;
    for (int j = 0; j < F->nn; ++j) A.src[j] = F->st(j);
    for (int i = 0; i < C->nn; ++i)
        for (int j = 0; j < F->nn; ++j) A.w[i][j] = P->tr[(size_t)i * F->nn + j];
    const long n = 3 * C->K;
    launch_pdl(restrict_states_kernel, dim3((unsigned)((n + 127) / 128), C->nn), dim3(128), 0, st, A, C->st(0),
               3 * C->K, F->R, C->R);
    PSWE_LAUNCH_CHECK();
}

void pair_fas(pswe_pair* P, double dt, double2* tau, cudaStream_t st, const double2* tau_f) {
    pswe_level *F = P->fine, *C = P->coarse;
    FasArgs A{};
    A.tau_f = tau_f;
    A.mc = C->nn;
    A.mf = F->nn;
    A.Rf = F->R;
    A.Rc = C->R;
    A.dt = dt;
    for (int j = 0; j < F->nn; ++j) {
        A.fi_f[j] = F->fi(j);
        A.fe_f[j] = F->fe(j);
    }
    for (int j = 0; j < C->nn; ++j) {
        A.fi_c[j] = C->fi(j);
        A.fe_c[j] = C->fe(j);
    }
    for (int i = 0; i < C->nn; ++i) {
        for (int j = 0; j < F->nn; ++j) A.qfr[i][j] = P->qfr[(size_t)i * F->nn + j];
        for (int j = 0; j < F->nn; ++j) A.tr[i][j] = P->tr[(size_t)i * F->nn + j];
        for (int j = 0; j < C->nn; ++j) A.qc[i][j] = C->tab.Q(i, j);
    }
    const long n = 3 * C->K;
    launch_pdl(fas_kernel, dim3((unsigned)((n + 127) / 128), C->nn), dim3(128), 0, st, A, tau);
    PSWE_LAUNCH_CHECK();
}

void pair_save(pswe_pair* P, cudaStream_t st) {
    pswe_level* C = P->coarse;
    copies({{P->saved(0, 0), C->st(0)}, {P->saved(1, 0), C->fi(0)}, {P->saved(2, 0), C->fe(0)}},
           (long)C->nn * 3 * C->K, st);
}

void pair_interp_increment_add(pswe_pair* P, double2* dstate0, cudaStream_t st, bool dstate0_outside_zero) {
    pswe_level *F = P->fine, *C = P->coarse;
    InterpArgs A{};
    A.mf = F->nn;
    A.mc = C->nn;
    A.Rf = F->R;
    A.Rc = C->R;
    A.nfam = 3;
    A.dstate0 = dstate0;
    for (int j = 0; j < C->nn; ++j) {
        A.a[0][j] = C->st(j);
        A.a[1][j] = C->fi(j);
        A.a[2][j] = C->fe(j);
        for (int fam = 0; fam < 3; ++fam) A.b[fam][j] = P->saved(fam, j);
    }
    for (int i = 0; i < F->nn; ++i) {
        A.dst[0][i] = F->st(i);
        A.dst[1][i] = F->fi(i);
        A.dst[2][i] = F->fe(i);
        for (int j = 0; j < C->nn; ++j) A.w[i][j] = P->ti[(size_t)i * C->nn + j];
    }
    static const bool full = [] { const char* e = getenv("PSWE_INTERP_FULL"); return e && atoi(e) != 0; }();
    if (full) {  // A/B: the full-range kernel
        const long n = 3 * F->K;
        launch_pdl(interp_kernel, dim3((unsigned)((n + 127) / 128), 3 * F->nn), dim3(128), 0, st, A, 0);
        PSWE_LAUNCH_CHECK();
        return;
    }
    const long nc = 3 * C->K;
    launch_pdl(interp_inc_kernel, dim3((unsigned)((nc + 127) / 128), 3 * F->nn), dim3(128), 0, st, A);
    PSWE_LAUNCH_CHECK();
    if (dstate0 && !dstate0_outside_zero && F->R > C->R) {
        const long n = 3 * F->K;
        launch_pdl(zero_out_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, F->R, C->R, dstate0);
        PSWE_LAUNCH_CHECK();
    }
}

void pair_interp_states(pswe_pair* P, cudaStream_t st) {
    pswe_level *F = P->fine, *C = P->coarse;
    InterpArgs A{};
    A.mf = F->nn;
    A.mc = C->nn;
    A.Rf = F->R;
    A.Rc = C->R;
    A.nfam = 1;
    for (int j = 0; j < C->nn; ++j) A.a[0][j] = C->st(j);
    for (int i = 0; i < F->nn; ++i) {
        A.dst[0][i] = F->st(i);
        for (int j = 0; j < C->nn; ++j) A.w[i][j] = P->ti[(size_t)i * C->nn + j];
    }
    const long n = 3 * F->K;
    launch_pdl(interp_kernel, dim3((unsigned)((n + 127) / 128), F->nn), dim3(128), 0, st, A, 1);
    PSWE_LAUNCH_CHECK();
}

// restrict_space / interpolate_space of n states
__global__ void space_copy_kernel(int Rf, int Rc, const double2* __restrict__ x, double2* __restrict__ y, int down) {
    const long Kc = (long)(Rc + 1) * (Rc + 2) / 2, Kf = (long)(Rf + 1) * (Rf + 2) / 2;
    const int b = blockIdx.y;
    if (down) {
        const long kc3 = (long)blockIdx.x * blockDim.x + threadIdx.x;
        if (kc3 >= 3 * Kc) return;
        y[b * 3 * Kc + kc3] = x[b * 3 * Kf + fine_index(Rf, Rc, kc3, Kc, Kf)];
    } else {
        const long kf3 = (long)blockIdx.x * blockDim.x + threadIdx.x;
        if (kf3 >= 3 * Kf) return;
        const int f = (int)(kf3 / Kf);
        int m, s;
        tailc::decode_rs(Rf, kf3 - f * Kf, m, s);
        y[b * 3 * Kf + kf3] = (m <= Rc && s <= Rc) ? x[b * 3 * Kc + f * Kc + off_std(Rc, m) + (s - m)]
                                                   : make_double2(0.0, 0.0);
    }
}

}  // namespace pswe

namespace {
std::vector<double> lagrange_matrix(const std::vector<double>& from, const std::vector<double>& to) {
    std::vector<double> pi(to.size() * from.size());
    for (size_t i = 0; i < to.size(); ++i)
        for (size_t j = 0; j < from.size(); ++j) pi[i * from.size() + j] = lagrange_basis(from, (int)j, to[i]);
    return pi;
}
}  // namespace

extern "C" {

int pswe_quadrature_tables(int n, double* nodes, double* q, double* qe, double* qi) {
    return guarded([&] {
        const Tables t = build_tables(n);
        std::memcpy(nodes, t.nodes.data(), sizeof(double) * n);
        std::memcpy(q, t.q.data(), sizeof(double) * n * n);
        std::memcpy(qe, t.qe.data(), sizeof(double) * n * n);
        std::memcpy(qi, t.qi.data(), sizeof(double) * n * n);
    });
}

int pswe_level_create(pswe_plan* plan, const pswe_params* p, int num_nodes, pswe_level** out) {
    return guarded([&] {
        if (!plan || !p || !out) throw std::invalid_argument("pswe_level_create: NULL argument");
        if (num_nodes != 2 && num_nodes != 3 && num_nodes != 5)  // the kernels' node arrays hold kMaxNodes
            throw std::invalid_argument("pswe_level_create: supported node counts are 2, 3, 5");
        auto* L = new pswe_level;
        try {
            L->plan = plan;
            L->prm = *p;
            L->R = plan->R;
            L->K = plan->K;
            L->nn = num_nodes;
            L->tab = build_tables(num_nodes);
            const size_t bytes = (size_t)num_nodes * 3 * L->K * sizeof(double2);
            PSWE_CUDA(cudaMalloc(&L->d_state, bytes));
            for (int b = 0; b < 2; ++b)
                for (int k = 0; k < 2; ++k) PSWE_CUDA(cudaMalloc(&L->d_f[b][k], bytes));
            PSWE_CUDA(cudaMemset(L->d_state, 0, bytes));
            const size_t nblk = (size_t)(3 * L->K + 255) / 256;  // residual_kernel's grid
            PSWE_CUDA(cudaMalloc(&L->d_bmax, nblk * sizeof(unsigned long long)));
            PSWE_CUDA(cudaMalloc(&L->d_count, sizeof(unsigned int)));
            PSWE_CUDA(cudaMemset(L->d_count, 0, sizeof(unsigned int)));
            static const bool qsum_off = [] { const char* e = getenv("PSWE_NO_QSUM"); return e && atoi(e) != 0; }();
            if (num_nodes >= 4 && !qsum_off)
                PSWE_CUDA(cudaMalloc(&L->d_qsum, (size_t)(num_nodes - 2) * 3 * L->K * sizeof(double2)));
            plan->reserve(num_nodes);
        } catch (...) {
            if (L->d_state) cudaFree(L->d_state);
            if (L->d_qsum) cudaFree(L->d_qsum);
            if (L->d_bmax) cudaFree(L->d_bmax);
            if (L->d_count) cudaFree(L->d_count);
            for (auto& b : L->d_f)
                for (auto* q : b)
                    if (q) cudaFree(q);
            delete L;
            throw;
        }
        *out = L;
    });
}

int pswe_level_destroy(pswe_level* L) {
    return guarded([&] {
        if (!L) return;
        cudaFree(L->d_state);
        if (L->d_bmax) cudaFree(L->d_bmax);
        if (L->d_count) cudaFree(L->d_count);
        if (L->d_qsum) cudaFree(L->d_qsum);
        for (auto& b : L->d_f)
            for (auto* q : b) cudaFree(q);
        delete L;
    });
}

double* pswe_level_ptr(pswe_level* L, int which, int node) {
    if (!L || node < 0 || node >= L->nn) return nullptr;
    switch (which) {
        case 0: return reinterpret_cast<double*>(L->st(node));
        case 1: return reinterpret_cast<double*>(L->fi(node));
        case 2: return reinterpret_cast<double*>(L->fe(node));
        default: return nullptr;
    }
}

int pswe_level_info(const pswe_level* L, int* R, int* nn) {
    return guarded([&] {
        if (!L) throw std::invalid_argument("NULL level");
        if (R) *R = L->R;
        if (nn) *nn = L->nn;
    });
}

int pswe_spread(pswe_level* L, const double* theta0, void* stream) {
    PSWE_NVTX("pswe.spread");
    return guarded([&] {
        if (!L || !theta0) throw std::invalid_argument("pswe_spread: NULL argument");
        level_spread(L, reinterpret_cast<const double2*>(theta0), as_stream(stream));
    });
}

int pswe_refresh_nodes(pswe_level* L, int first, int count, void* stream) {
    PSWE_NVTX("pswe.refresh_nodes");
    return guarded([&] {
        if (!L) throw std::invalid_argument("NULL level");
        if (first < 0 || count < 0 || first + count > L->nn) throw std::invalid_argument("refresh: node range");
        level_refresh(L, first, count, as_stream(stream));
    });
}

int pswe_sweep(pswe_level* L, double dt, const double* tau, void* stream) {
    PSWE_NVTX("pswe.sweep");
    return guarded([&] {
        if (!L) throw std::invalid_argument("NULL level");
        level_sweep(L, dt, reinterpret_cast<const double2*>(tau), as_stream(stream), nullptr);
    });
}

int pswe_collocation_residual(pswe_level* L, double dt, double* out, void* stream) {
    PSWE_NVTX("pswe.collocation_residual");
    return guarded([&] {
        if (!L || !out) throw std::invalid_argument("NULL argument");
        level_residual(L, dt, out, as_stream(stream));
    });
}

int pswe_sdc_step(pswe_level* L, const double* theta0, double dt, int n_sweeps, double* out_res, void* stream) {
    PSWE_NVTX("pswe.sdc_step");
    return guarded([&] {
        if (!L || !theta0) throw std::invalid_argument("NULL argument");
        const cudaStream_t st = as_stream(stream);
        level_spread(L, reinterpret_cast<const double2*>(theta0), st);
        for (int k = 0; k < n_sweeps; ++k) level_sweep(L, dt, nullptr, st, k == n_sweeps - 1 ? out_res : nullptr);
        if (out_res && n_sweeps == 0) level_residual(L, dt, out_res, st);
    });
}

int pswe_pair_create(pswe_level* fine, pswe_level* coarse, pswe_pair** out) {
    return guarded([&] {
        if (!fine || !coarse || !out) throw std::invalid_argument("pswe_pair_create: NULL argument");
        if (coarse->R > fine->R) throw std::invalid_argument("make_transfer_pair: coarse truncation exceeds fine");
        if (coarse->R < 1) throw std::invalid_argument("make_transfer_pair: coarse truncation must be >= 1");
        const int nf = fine->nn, nc = coarse->nn;
        if (!(nf == nc || (nf == 3 && nc == 2) || (nf == 5 && nc == 3)))
            throw std::invalid_argument("make_transfer_pair: unsupported node pair");
        auto* P = new pswe_pair;
        P->fine = fine;
        P->coarse = coarse;
        P->tr = lagrange_matrix(fine->tab.nodes, coarse->tab.nodes);
        P->ti = lagrange_matrix(coarse->tab.nodes, fine->tab.nodes);
        // matmul (quadrature.cpp:8-17), i-k-j order
        P->qfr.assign((size_t)nc * nf, 0.0);
        for (int i = 0; i < nc; ++i)
            for (int k = 0; k < nf; ++k) {
                const double xv = P->tr[(size_t)i * nf + k];
                for (int j = 0; j < nf; ++j) P->qfr[(size_t)i * nf + j] += xv * fine->tab.Q(k, j);
            }
        const size_t bytes = (size_t)3 * nc * 3 * coarse->K * sizeof(double2);
        try {
            PSWE_CUDA(cudaMalloc(&P->d_saved, bytes));
        } catch (...) {
            delete P;
            throw;
        }
        *out = P;
    });
}

int pswe_pair_destroy(pswe_pair* P) {
    return guarded([&] {
        if (!P) return;
        cudaFree(P->d_saved);
        delete P;
    });
}

int pswe_restrict_space(int rf, int rc, const double* x, double* y, int n, void* stream) {
    return guarded([&] {
        if (rc > rf || rc < 1) throw std::invalid_argument("restrict_space: bad truncations");
        if (n <= 0) return;
        const long Kc = num_coeffs(rc);
        space_copy_kernel<<<dim3((unsigned)((3 * Kc + 127) / 128), n), 128, 0, as_stream(stream)>>>(
            rf, rc, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), 1);
        PSWE_LAUNCH_CHECK();
    });
}

int pswe_interpolate_space(int rc, int rf, const double* x, double* y, int n, void* stream) {
    return guarded([&] {
        if (rc > rf || rc < 1) throw std::invalid_argument("interpolate_space: bad truncations");
        if (n <= 0) return;
        const long Kf = num_coeffs(rf);
        space_copy_kernel<<<dim3((unsigned)((3 * Kf + 127) / 128), n), 128, 0, as_stream(stream)>>>(
            rf, rc, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), 0);
        PSWE_LAUNCH_CHECK();
    });
}

int pswe_restrict_states(pswe_pair* P, void* stream) {
    return guarded([&] {
        if (!P) throw std::invalid_argument("NULL pair");
        pair_restrict_states(P, as_stream(stream));
    });
}

int pswe_fas_correction(pswe_pair* P, double dt, double* tau, void* stream) {
    return guarded([&] {
        if (!P || !tau) throw std::invalid_argument("NULL argument");
        pair_fas(P, dt, reinterpret_cast<double2*>(tau), as_stream(stream), nullptr);
    });
}

int pswe_fas_correction_ml(pswe_pair* P, double dt, const double* tau_fine, double* tau, void* stream) {
    return guarded([&] {
        if (!P || !tau) throw std::invalid_argument("NULL argument");
        pair_fas(P, dt, reinterpret_cast<double2*>(tau), as_stream(stream),
                 reinterpret_cast<const double2*>(tau_fine));
    });
}

int pswe_save_coarse(pswe_pair* P, void* stream) {
    return guarded([&] {
        if (!P) throw std::invalid_argument("NULL pair");
        pair_save(P, as_stream(stream));
    });
}

int pswe_interpolate_increment_add(pswe_pair* P, double* dstate0, void* stream) {
    return guarded([&] {
        if (!P) throw std::invalid_argument("NULL pair");
        pair_interp_increment_add(P, reinterpret_cast<double2*>(dstate0), as_stream(stream), false);
    });
}

int pswe_interpolate_states(pswe_pair* P, void* stream) {
    return guarded([&] {
        if (!P) throw std::invalid_argument("NULL pair");
        pair_interp_states(P, as_stream(stream));
    });
}

}  // extern "C"
