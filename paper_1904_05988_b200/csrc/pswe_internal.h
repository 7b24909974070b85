// Internal declarations of libpswe (B200 / sm_100a, fp64). See include/pswe.h for the ABI and
// DESIGN.md for the data layout and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pswe.h"

namespace pswe {

// ------------------------------------------------------------------------------------------
// errors

void set_error(const std::string& msg);

#define PSWE_CUDA(x)                                                                          \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess)                                                                \
            throw std::runtime_error(std::string(#x) + " failed: " + cudaGetErrorString(e_)); \
    } while (0)

#define PSWE_LAUNCH_CHECK() PSWE_CUDA(cudaGetLastError())

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        set_error(e.what());
        return 1;
    }
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// NVTX ranges on the host API (nsys / ncu --nvtx timelines: per ABI call, per PFASST op, per message);
// header-only NVTX v3, a no-op without an attached tool
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define PSWE_NVTX_CAT2(a, b) a##b
#define PSWE_NVTX_CAT(a, b) PSWE_NVTX_CAT2(a, b)
#define PSWE_NVTX(name) ::pswe::NvtxRange PSWE_NVTX_CAT(pswe_nvtx_, __LINE__)(name)

// Programmatic dependent launch (PDL) of the eval chain prep -> inverse -> grid stage -> forward
// -> tail: each kernel is launched with programmatic stream serialisation, runs its independent
// prologue (mbarrier init, plan tables, twiddles), calls pdl_wait() before touching its
// predecessor's output (every thread of every kernel waits, so completion stays transitive) and
// pdl_trigger() early, so the next kernel's blocks become resident during this kernel's tail.
// Without the launch attribute both instructions are no-ops. PSWE_NO_PDL=1 disables it.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::); }
#endif
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    PSWE_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// ------------------------------------------------------------------------------------------
// spectral indexing (field.hpp:29-32) and the "extended" triangle s = m..R+1 used internally

__host__ __device__ inline long off_std(int R, int m) { return (long)m * (2 * R + 3 - m) / 2; }
__host__ __device__ inline long off_ext(int R, int m) { return (long)m * (2 * R + 5 - m) / 2; }
inline long num_coeffs(int R) { return (long)(R + 1) * (R + 2) / 2; }
inline long num_ext(int R) { return (long)(R + 1) * (R + 4) / 2; }

// ------------------------------------------------------------------------------------------
// FFT descriptor: complex Stockham DIF of length N = nlon/2, radices 4/2/3/5

struct FftStage {
    int p;       // radix
    int m;       // sub-length after this stage (n/p)
    int s;       // stride
    int tw_off;  // offset of this stage's twiddles tw[j*p + t] in Plan::d_fft_tw
};
constexpr int kMaxFftStages = 16;
struct FftDesc {
    int N;
    int nst;
    FftStage st[kMaxFftStages];
};

// ------------------------------------------------------------------------------------------
// kernel launchers (defined in legendre.cu / fft.cu / ops.cu)

struct DevPlan;  // POD view of the plan passed to kernels

}  // namespace pswe

// The plan: TransformPlan (transform.hpp:27-96) on one device. Immutable after creation except
// for the grow-only scratch, which makes it single-stream (one host thread) like the ABI says.
struct pswe_plan {
    int R = 0, nlat = 0, nlon = 0, J = 0, N = 0;
    int legendre_mode = PSWE_LEGENDRE_RECOMPUTE;
    int simt = 0;  // PSWE_LEGENDRE_SIMT=1 at plan creation: DFMA (CUDA-core) Legendre kernels
    int device = 0;
    long K = 0, Kx = 0;
    // host copies
    std::vector<double> mu, w, cosphi;
    // device constants
    double* d_mu_n = nullptr;    // [J] mu at north-half latitude j (row nlat/2 + j)
    double* d_seed = nullptr;    // [(R+1) * J] P^m_m(mu_j) (legendre.cpp:26-29)
    double2* d_rec = nullptr;    // [Kx] (1/eps(m,s+1), eps(m,s)/eps(m,s+1)) at off_ext(m)+s-m
    double* d_eps = nullptr;     // [Kx] eps(m, s) at off_ext(m)+s-m, s = m..R+1
    double* d_rlap = nullptr;    // [R+2] 1/(s(s+1)), s >= 1 (inverse Laplacian factor)
    double* d_ptab = nullptr;    // STREAM mode: [Kx * J] P^m_s(mu_j), block m: [j][s]
    double2* d_chk = nullptr;    // [sum_m ceil((R+2-m)/16)][J] (P_t, P_{t-1}) at t = 16c (forward DMMA)
    int* d_chk_off = nullptr;    // [R+2] chunk offsets per m into d_chk
    double* d_ptab2 = nullptr;   // STREAM mode: P tiles [m][chunk][Jp][16] swizzled (legendre_stream.cu)
    int* d_cstart = nullptr;     // STREAM mode: [m][slice] first chunk with |P| >= 1e-20 (polar skip)
    int n_chunks = 0;            // STREAM mode: 16-degree chunks over all m (= d_chk_off[R+1])
    int* d_chunk_m = nullptr;    // STREAM mode: [n_chunks] int2 (order m, chunk within m)
    mutable double* d_xtile = nullptr;  // STREAM mode: inverse X tiles (grow-only scratch)
    mutable size_t xtile_cap = 0;       // doubles
    int4* d_fwd_ta = nullptr;     // STREAM mode: forward tasks (m_a, first chunk, chunks of m_a, m_b)
    int2* d_fwd_tb = nullptr;     //   (first chunk of m_b, chunks of m_b)
    int n_fwd_tasks = 0;
    int fwd_cfg = 0;              // index into kFwdCfg the task table was cut for
    double* d_gtile = nullptr;    // STREAM mode: grid-stage products as forward G tiles (GtLayout)
    size_t gtile_cap = 0;         // doubles
    double* d_rowc = nullptr;    // [nlat] cos(phi_i)
    double* d_roww = nullptr;    // [nlat] Gauss weight w_i
    double* d_rowmu = nullptr;   // [nlat] mu_i
    double2* d_fft_tw = nullptr; // stage twiddles
    double2* d_fft_post = nullptr;  // [N+1] exp(-2 pi i k / nlon)
    double2* d_fft_roots = nullptr; // [N] exp(-2 pi i k / N)
    double2* d_fft_iptw = nullptr;  // per-pass twiddles of the in-place DIF/DIT plan (fft_ip.cu)
    double2* d_fft_iptw1 = nullptr; // the same for plan 1 (narrow evaluations, plain row transforms)
    pswe::FftDesc fft{};
    // scratch (grow-only)
    int cap_batch = 0;
    double2* d_four_a = nullptr;  // [cap * 5 * (R+1) * nlat] Fourier rows, [b][f][m][i]
    double2* d_four_b = nullptr;  // [cap * 5 * (R+1) * nlat]
    double2* d_proj = nullptr;    // [cap * 5 * Kx] Legendre projections, extended layout
    double2* d_xcoef = nullptr;   // [cap * 5 * Kx] inverse-Legendre coefficients (U/V derived), ext layout
    // bumped on every scratch reallocation: a CUDA graph captured over this plan's scratch
    // (pswe_pfasst's serial-emulation block) is stale once it changes
    mutable unsigned long long generation = 0;
    void reserve(int batch);
};

namespace pswe {

// Forward-Legendre G tiles written by the fused grid stage (fft_ip.cu) and read by bulk copies in
// legendre_stream.cu: per column group z (spg states = 10 spg real columns), order m, 8-latitude
// slice s, hemisphere h (0 = north row nlat-J+j, 1 = south row J-1-j), latitude row r:
//   gt[((((z (R+1) + m) ns8 + s) 2 + h) 8 + r) sgc + 10 b' + 2 f + {re, im}]
// for state b = spg z + b', field f of (Phi'U, Phi'V, qU, qV, ke), the column XOR-swizzled per
// row by gt_swz (sgc = 8 ntc doubles, no padding; the forward's fragment reads are then
// conflict-free).
// Plain analyse (gt_layout_fields): the same tiles with apg single FIELDS per column group (2
// real columns each, column 2 f' + {re, im} for field f = apg z + f'), and the forward writes
// the standard coefficient layout out[f K + off_std(m) + s - m] (plain = 1) instead of the
// extended projections out[q Kx + off_ext(m) + s - m].
struct GtLayout {
    int spg = 0, groups = 0, ntc = 0, sgc = 0, ns8 = 0;
    int apg = 0;    // complex arrays (projections / fields) per column group
    int plain = 0;  // 1: fields in the standard layout (analyse)
    size_t doubles = 0;
};
// forward tasks: runs of <= warps x cpw chunks of <= 2 orders m, ~per_sm runs per SM. Two
// configurations (measured, tools/stage_times.py): one chunk per warp, 8 warps, 2 blocks/SM,
// 4 stages when every chunk fits one wave (T255 and below); two chunks per warp (fragment reuse),
// 4 warps, 3 blocks/SM, 3 stages otherwise.
struct FwdCfg {
    int warps, cpw, per_sm, stages;
};
constexpr FwdCfg kFwdCfg[2] = {{8, 1, 2, 4}, {4, 2, 3, 3}};
// column swizzle of latitude row r (0..7) of a G tile with ntc 8-column tiles
__host__ __device__ inline int gt_swz(int ntc, int r) { return (ntc & 1) ? 4 * ((r >> 1) & 1) : 4 * (r & 3); }
inline GtLayout gt_layout(int R, int J, int n) {
    GtLayout g;
    g.spg = n < 5 ? n : 5;
    g.groups = (n + g.spg - 1) / g.spg;
    g.apg = 5 * g.spg;
    g.ntc = (10 * g.spg + 7) / 8;
    g.sgc = 8 * g.ntc;
    g.ns8 = ((J + 31) / 32) * 4;
    g.doubles = (size_t)g.groups * (R + 1) * g.ns8 * 2 * 8 * g.sgc;
    return g;
}
// nf plain fields: groups of at most 16 fields (4 column tiles), at least 2 column tiles
inline GtLayout gt_layout_fields(int R, int J, int nf) {
    GtLayout g;
    g.groups = (nf + 15) / 16;
    g.apg = (nf + g.groups - 1) / g.groups;
    g.ntc = (2 * g.apg + 7) / 8 < 2 ? 2 : (2 * g.apg + 7) / 8;
    g.plain = 1;
    g.sgc = 8 * g.ntc;
    g.ns8 = ((J + 31) / 32) * 4;
    g.doubles = (size_t)g.groups * (R + 1) * g.ns8 * 2 * 8 * g.sgc;
    return g;
}

// legendre.cu
enum InvKind { INV_PLAIN = 0, INV_UV = 1, INV_EVAL = 2 };
// Inverse Legendre (synthesis) into Fourier rows out[b][f][m][i].
// PLAIN: in = n fields [K] (in2 unused); UV: in = n vort fields, in2 = n div fields;
// EVAL: in = n states [3][K]. out rows: PLAIN [f][m][i], UV [b][2][m][i], EVAL [b][4][m][i].
void legendre_inverse(const pswe_plan& P, int kind, const double2* in, const double2* in2, int n,
                      double radius, double2* out, cudaStream_t st);
// Forward Legendre (analysis) from Fourier rows four[b][f][m][i] (nf fields per batch item) into
// projections; out_ext: extended layout [b][f][Kx] (s = m..R+1); else standard [b][f][K].
void legendre_forward(const pswe_plan& P, const double2* four, int nf, int n_batch, double2* out,
                      bool out_ext, cudaStream_t st);
// DMMA (FP64 tensor core) variants over nq complex columns (legendre_mma.cu)
void legendre_inverse_mma(const pswe_plan& P, int kind, const double2* in, const double2* in2, int nq,
                          double radius, double2* out, cudaStream_t st);
void legendre_forward_mma(const pswe_plan& P, const double2* four, int nq, double2* out, bool ext,
                          cudaStream_t st);
void build_legendre_checkpoints(pswe_plan& P);
// STREAM mode (legendre_stream.cu): DMMA contractions on a streamed P table
void build_legendre_table2(pswe_plan& P);
void legendre_forward_stream(const pswe_plan& P, const double2* four, int nq, double2* out, bool ext,
                             cudaStream_t st);
// streamed (TMA) inverse chosen over the recurrence inverse for nq columns (legendre_mma.cu)
bool use_stream_inverse(const pswe_plan& P, int nq);
void xtile_reserve(const pswe_plan& P, int nq, int kind);
bool xtiles_by_sweep_ok(const pswe_plan& P);
void legendre_inverse_prepared(const pswe_plan& P, double2* out, cudaStream_t st);
// legendre_rec.cu: single-state inverse on large grids on the CUDA cores, P recomputed in registers
bool inv_rec_big(const pswe_plan& P, int nq);
void inv_rec_launch(const pswe_plan& P, const double* Xt, int nq, int NT, double2* out, cudaStream_t st);
// capi.cu: an evaluation up to the five projections in P.d_proj
void eval_imex_proj(pswe_plan& P, const pswe_params& prm, const double2* state, int n, cudaStream_t st,
                    bool xprep = false);
// after_prep (optional): recorded between the prep and the contraction kernel (timing)
void legendre_inverse_stream(const pswe_plan& P, int kind, const double2* in, const double2* in2, int nq,
                             double radius, double2* out, cudaStream_t st, cudaEvent_t after_prep = nullptr);

// fft.cu
// Fourier rows [b][m][i] -> grid [b][i][j] (c2r, Im G_0 := 0), optional per-row 1/cos(phi).
// Row b of the batch reads Fourier rows four[(b*in_stride + in_off)][m][i].
void fft_rows_c2r(const pswe_plan& P, const double2* four, int in_stride, int in_off, double* grid, int n,
                  bool div_cos, cudaStream_t st);
// grid [b][i][j] -> Fourier rows [b][m][i], x pre (cos(phi) if pre_cos) then x post-scale:
// mode 0: w_i/nlon (analyse), mode 1: w_i/(a cos^2 phi_i nlon) (vortdiv_from_uv).
void fft_rows_r2c(const pswe_plan& P, const double* grid, double2* four, int out_stride, int out_off, int n,
                  bool pre_cos, int scale_mode, double radius, cudaStream_t st);
// Fused grid stage of eval_nonlinear (swe.cpp:41-54 + the FFT halves of uv_from_vortdiv /
// synthesise / vortdiv_from_uv / analyse): four_in [b][4][m][i] (Phi, zeta, U, V) ->
// four_out [b][5][m][i] (Phi'U, Phi'V, qU, qV, ke), weights folded in.
void fft_eval_products(const pswe_plan& P, const pswe_params& prm, const double2* four_in,
                       double2* four_out, int n_batch, cudaStream_t st);

// G-tile path of the eval grid stage (STREAM mode): fft_ip.cu writes P.d_gtile, the forward
// reads it (legendre_stream.cu). gt_path_ok: every precondition of the pair holds for n states.
bool gt_path_ok(const pswe_plan& P, int n);
void fft_eval_products_gt(const pswe_plan& P, const pswe_params& prm, const double2* fin, int n, cudaStream_t st);
void legendre_forward_gt(const pswe_plan& P, int n, double2* out, cudaStream_t st);
// analyse on G tiles: fft_r2c_gt writes the nf fields' tiles (gt_layout_fields), the column-warp
// forward writes the coefficients (standard layout); analyse_gt_ok: the pair applies
bool analyse_gt_ok(const pswe_plan& P, const GtLayout& gl);
bool fft_r2c_gt(const pswe_plan& P, const double* grid, const GtLayout& gl, int nf, cudaStream_t st);
void legendre_forward_fields_gt(const pswe_plan& P, const GtLayout& gl, int nf, double2* out, cudaStream_t st);
// fft_ip.cu: in-place fused grid stage; false if nlon/2 has no in-place plan
std::vector<double2> fft_ip_twiddles(int N, int pl = 0);
bool fft_eval_products_ip(const pswe_plan& P, const pswe_params& prm, const double2* fin, double2* fout, int n,
                          cudaStream_t st);
// in-place plain row transforms (fft_ip.cu); false when nlon/2 has no in-place plan
bool fft_rows_ip(const pswe_plan& P, bool c2r, const double2* four_in, const double* grid_in, double2* four_out,
                 double* grid_out, int stride, int off, int n, bool cos_flag, int scale_mode, double radius,
                 cudaStream_t st);

// ops.cu
void eval_tail(const pswe_plan& P, const pswe_params& prm, const double2* proj, const double2* state,
               double2* f_imp, double2* f_exp, int n_batch, cudaStream_t st);
void vortdiv_tail(const pswe_plan& P, const double2* proj, double2* vort, double2* div, int n_pairs,
                  cudaStream_t st);
void eval_linear(int R, const pswe_params& prm, const double2* state, double2* out, int n_states,
                 cudaStream_t st);
void solve_implicit(int R, const pswe_params& prm, const double2* b, double c, double2* out,
                    int n_states, cudaStream_t st);
void laplacian(int R, const double2* x, double radius, double2* y, int n_fields, bool inverse,
               cudaStream_t st);

}  // namespace pswe

namespace pswe {
// SDC collocation tables (QuadratureTables, quadrature.hpp:16-22), row-major n x n.
struct Tables {
    int n = 0;
    std::vector<double> nodes, q, qe, qi;  // row-major n x n
    double Q(int i, int j) const { return q[(size_t)i * n + j]; }
    double QE(int i, int j) const { return qe[(size_t)i * n + j]; }
    double QI(int i, int j) const { return qi[(size_t)i * n + j]; }
};

Tables build_tables(int n);
}  // namespace pswe

// LevelSpec + SpaceTimeState (multilevel.hpp:16-23, sdc.hpp:14-20) on the device.
struct pswe_level {
    pswe_plan* plan = nullptr;
    pswe_params prm{};
    int R = 0, nn = 0;
    long K = 0;
    pswe::Tables tab;
    double2* d_state = nullptr;  // [nn][3K]
    double2* d_f[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [buffer][0=imp,1=exp] -> [nn][3K]
    int cur = 0;
    unsigned long long* d_res = nullptr;
    unsigned long long* d_bmax = nullptr;  // residual: per-block maxima
    unsigned int* d_count = nullptr;       // residual: blocks done (0 between launches)
    double2* d_qsum = nullptr;             // sweep: quadrature of the old right-hand sides, [nn-2][3K]
    double2* st(int node) const { return d_state + (size_t)node * 3 * K; }
    double2* fi(int node, int buf = -1) const { return d_f[buf < 0 ? cur : buf][0] + (size_t)node * 3 * K; }
    double2* fe(int node, int buf = -1) const { return d_f[buf < 0 ? cur : buf][1] + (size_t)node * 3 * K; }
};

struct pswe_pair {
    pswe_level* fine = nullptr;
    pswe_level* coarse = nullptr;
    std::vector<double> tr, ti, qfr;  // (mc x mf), (mf x mc), (mc x mf)
    double2* d_saved = nullptr;       // [3 families][mc][3Kc]
    double2* saved(int fam, int node) const {
        return d_saved + ((size_t)fam * coarse->nn + node) * 3 * coarse->K;
    }
};

