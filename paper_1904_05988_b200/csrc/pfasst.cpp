// PFASST block controller (host C++), the B200 replacement of pf::run_block
// (proj/src/pfasst.cpp:78-251, Algorithm 1 of PAPER.md:709-766).
//
// The per-worker control flow is generated once as data (build_schedule, mirroring
// worker_predict :78-120 and worker_iterate :122-176 op for op) and executed by
//   * SerialExec  — all workers on this GPU in worker order with in-process message queues
//                   (the reference's Mode::serial_emulation, :212-216);
//   * NcclExec    — one process per GPU, worker w = rank, messages carried by NCCL send/recv
//                   over NVLink. The reference's two forward-only channels (fine_ch/coarse_ch,
//                   :65-66) become two NCCL communicators per direction parity: rank w sends on
//                   comm[level][w%2] from a dedicated send stream (the reference's send never
//                   blocks, :31-37) and receives on comm[level][(w+1)%2] on the compute stream,
//                   so no communicator is ever used from two streams and sends can never block
//                   the compute pipeline (which would deadlock Step C against Step A).
// The same schedule is exported through pswe_pfasst_schedule() so the multi-rank host logic is
// tested on CPU with gloo (tests/test_pfasst_schedule.py).
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <tuple>

#include "pswe_internal.h"

namespace pswe {
void level_spread(pswe_level* L, const double2* theta0, cudaStream_t st);
void level_refresh(pswe_level* L, int first, int count, cudaStream_t st);
void level_sweep(pswe_level* L, double dt, const double2* tau, cudaStream_t st);
void level_residual(pswe_level* L, double dt, double* out, cudaStream_t st);
void pair_restrict_states(pswe_pair* P, cudaStream_t st);
void pair_fas(pswe_pair* P, double dt, double2* tau, cudaStream_t st, const double2* tau_f = nullptr);
void pair_save(pswe_pair* P, cudaStream_t st);
void pair_interp_increment_add(pswe_pair* P, double2* dstate0, cudaStream_t st);
void pair_interp_states(pswe_pair* P, cudaStream_t st);
}  // namespace pswe

extern "C" {
double* pswe_level_ptr(pswe_level* L, int which, int node);
int pswe_level_info(const pswe_level* L, int* R, int* nn);
int pswe_restrict_space(int rf, int rc, const double* x, double* y, int n, void* stream);
}

namespace pswe {

// ---- schedule -------------------------------------------------------------------------------

enum OpCode : int {
    OP_PREDICT_INIT = 1,       // coarse = spread(restrict_space(theta0))          pfasst.cpp:91-92
    OP_RECV_COARSE_IC = 2,     // coarse.state[0] = recv(coarse_ch)                :98-99, :149-150
    OP_REFRESH_COARSE0 = 3,    // refresh_node(coarse, 0)                           :100, :152
    OP_SWEEP_COARSE = 4,       // sweep(coarse[, tau])                              :102, :153
    OP_SEND_COARSE = 5,        // send(coarse.state[mc-1]) -> w+1                   :104-106, :155-156
    OP_INTERP_STATES = 6,      // fine.state = interpolate_states(coarse.state)     :112
    OP_REFRESH_FINE_ALL = 7,   // refresh all fine nodes                            :116
    OP_RESIDUAL = 8,           // residuals[k] = collocation_residual(fine)         :118, :132
    OP_SWEEP_FINE = 9,         // sweep(fine)                                       :131
    OP_SEND_FINE = 10,         // send(fine.state[mf-1]) -> w+1                     :134-137
    OP_RESTRICT = 11,          // coarse.state = restrict_states(fine.state)        :141
    OP_REFRESH_COARSE_ALL = 12,// refresh all coarse nodes                          :142
    OP_SAVE = 13,              // saved = coarse                                    :143
    OP_FAS = 14,               // tau = fas_correction(fine, coarse)                :144
    OP_INTERP_INC = 15,        // fine.{state,F} += interpolate_increment(...)      :162-170
    OP_RECV_FINE_IC = 16,      // fine.state[0] = recv(fine_ch) + dstate[0]         :171-174
    OP_REFRESH_FINE0 = 17,     // refresh_node(fine, 0)                             :175
    // three-level chain (config 4; the reference is two-level only, multilevel.hpp:29-35): a
    // V-cycle per iteration, fine -> mid -> coarse -> mid -> fine, with the FAS of Eq. 19
    // (tau_f != 0 on the mid level). Ops on the (fine, mid) pair reuse the
    // two-level codes (RESTRICT, SAVE, INTERP_INC, INTERP_STATES); the coarse ops act on the
    // coarsest level.
    OP_INTERP_STATES_MC = 18,  // mid.state = interpolate_states(coarse.state)
    OP_REFRESH_MID_ALL = 19,   // refresh all mid nodes
    OP_RESTRICT_MC = 20,       // coarse.state = restrict_states(mid.state)
    OP_SAVE_MC = 21,           // saved_mc = coarse
    OP_FAS_MC = 22,            // tau_c = fas_correction(mid, coarse) + R tau_mid
    OP_SWEEP_MID = 23,         // sweep(mid, tau_mid)
    OP_SEND_MID = 24,          // send(mid.state[mm-1]) -> w+1
    OP_INTERP_INC_MC = 25,     // mid.{state,F} += interpolate_increment(coarse - saved_mc)
    OP_RECV_MID_IC = 26,       // mid.state[0] = recv(mid_ch), modes <= R_c from coarse.state[0]
    OP_REFRESH_MID0 = 27,      // refresh_node(mid, 0)
    OP_FAS_FM = 28,            // tau_mid = fas_correction(fine, mid)
};

struct Op {
    int code, phase, iter, arg;  // arg: use_tau for sweeps, residual index, message step char
};

std::vector<Op> build_schedule3(int w, int n, int n_iter);

std::vector<Op> build_schedule(int w, int n, int n_iter, int nlev = 2) {
    if (nlev == 3) return build_schedule3(w, n, n_iter);
    std::vector<Op> ops;
    ops.push_back({OP_PREDICT_INIT, 0, 0, 0});
    for (int q = 0; q <= w; ++q) {
        if (q >= 1) {
            ops.push_back({OP_RECV_COARSE_IC, 0, q - 1, 0});
            ops.push_back({OP_REFRESH_COARSE0, 0, q, 0});
        }
        ops.push_back({OP_SWEEP_COARSE, 0, q, 0});
        if (w < n - 1) ops.push_back({OP_SEND_COARSE, 0, q, 'P'});
    }
    ops.push_back({OP_INTERP_STATES, 0, 0, 0});
    ops.push_back({OP_REFRESH_FINE_ALL, 0, 0, 0});
    ops.push_back({OP_RESIDUAL, 0, 0, 0});
    for (int k = 1; k <= n_iter; ++k) {
        ops.push_back({OP_SWEEP_FINE, 1, k, 0});
        ops.push_back({OP_RESIDUAL, 1, k, k});
        if (k == n_iter) break;
        if (w < n - 1) ops.push_back({OP_SEND_FINE, 1, k, 'A'});
        ops.push_back({OP_RESTRICT, 1, k, 0});
        ops.push_back({OP_REFRESH_COARSE_ALL, 1, k, 0});
        ops.push_back({OP_SAVE, 1, k, 0});
        ops.push_back({OP_FAS, 1, k, 0});
        if (w > 0) ops.push_back({OP_RECV_COARSE_IC, 1, k, 0});
        ops.push_back({OP_REFRESH_COARSE0, 1, k, 0});
        ops.push_back({OP_SWEEP_COARSE, 1, k, 1});
        if (w < n - 1) ops.push_back({OP_SEND_COARSE, 1, k, 'C'});
        ops.push_back({OP_INTERP_INC, 1, k, 0});
        if (w > 0) ops.push_back({OP_RECV_FINE_IC, 1, k, 0});
        ops.push_back({OP_REFRESH_FINE0, 1, k, 0});
    }
    return ops;
}

// Three levels: predictor on the coarsest level (pipelined as in the two-level case), states
// interpolated up level by level; each iteration sweeps the fine level, restricts to the mid
// level (FAS), sweeps it (down) and sends its end state, restricts to the coarse level (FAS with
// R tau_mid), runs the pipelined coarse sweep, then goes back up: coarse increment -> mid, mid IC
// from w-1 (low modes from the coarse node 0), mid sweep (up), mid increment -> fine, fine IC from
// w-1 (low modes from the mid node 0).
std::vector<Op> build_schedule3(int w, int n, int n_iter) {
    std::vector<Op> ops;
    ops.push_back({OP_PREDICT_INIT, 0, 0, 0});
    for (int q = 0; q <= w; ++q) {
        if (q >= 1) {
            ops.push_back({OP_RECV_COARSE_IC, 0, q - 1, 0});
            ops.push_back({OP_REFRESH_COARSE0, 0, q, 0});
        }
        ops.push_back({OP_SWEEP_COARSE, 0, q, 0});
        if (w < n - 1) ops.push_back({OP_SEND_COARSE, 0, q, 'P'});
    }
    ops.push_back({OP_INTERP_STATES_MC, 0, 0, 0});
    ops.push_back({OP_REFRESH_MID_ALL, 0, 0, 0});
    ops.push_back({OP_INTERP_STATES, 0, 0, 0});
    ops.push_back({OP_REFRESH_FINE_ALL, 0, 0, 0});
    ops.push_back({OP_RESIDUAL, 0, 0, 0});
    for (int k = 1; k <= n_iter; ++k) {
        ops.push_back({OP_SWEEP_FINE, 1, k, 0});
        ops.push_back({OP_RESIDUAL, 1, k, k});
        if (k == n_iter) break;
        if (w < n - 1) ops.push_back({OP_SEND_FINE, 1, k, 'A'});
        ops.push_back({OP_RESTRICT, 1, k, 0});
        ops.push_back({OP_REFRESH_MID_ALL, 1, k, 0});
        ops.push_back({OP_SAVE, 1, k, 0});
        ops.push_back({OP_FAS_FM, 1, k, 0});
        ops.push_back({OP_SWEEP_MID, 1, k, 0});
        if (w < n - 1) ops.push_back({OP_SEND_MID, 1, k, 'M'});
        ops.push_back({OP_RESTRICT_MC, 1, k, 0});
        ops.push_back({OP_REFRESH_COARSE_ALL, 1, k, 0});
        ops.push_back({OP_SAVE_MC, 1, k, 0});
        ops.push_back({OP_FAS_MC, 1, k, 0});
        if (w > 0) ops.push_back({OP_RECV_COARSE_IC, 1, k, 0});
        ops.push_back({OP_REFRESH_COARSE0, 1, k, 0});
        ops.push_back({OP_SWEEP_COARSE, 1, k, 1});
        if (w < n - 1) ops.push_back({OP_SEND_COARSE, 1, k, 'C'});
        ops.push_back({OP_INTERP_INC_MC, 1, k, 0});
        if (w > 0) ops.push_back({OP_RECV_MID_IC, 1, k, 0});
        ops.push_back({OP_REFRESH_MID0, 1, k, 0});
        ops.push_back({OP_SWEEP_MID, 1, k, 0});
        ops.push_back({OP_INTERP_INC, 1, k, 0});
        if (w > 0) ops.push_back({OP_RECV_FINE_IC, 1, k, 0});
        ops.push_back({OP_REFRESH_FINE0, 1, k, 0});
    }
    return ops;
}

struct MsgRec {
    int phase, iteration, step, sender, receiver, level, node;
};

// Message log of a block (MessageRecord, pfasst.hpp:22-31), merged in the reference's order.
// Three levels: level 0 fine, 1 mid, 2 coarse; step 'M' for the mid down-sweep message.
std::vector<MsgRec> message_log(int n, int n_iter, int mf, int mc, int nlev = 2, int mm = 0) {
    std::vector<MsgRec> log;
    for (int r = 1; r < n; ++r) log.push_back({0, 0, 'B', 0, r, 0, 0});
    for (int w = 0; w < n; ++w)
        for (const Op& o : build_schedule(w, n, n_iter, nlev)) {
            if (o.code == OP_SEND_COARSE) log.push_back({o.phase, o.iter, o.arg, w, w + 1, nlev - 1, mc - 1});
            if (o.code == OP_SEND_FINE) log.push_back({o.phase, o.iter, o.arg, w, w + 1, 0, mf - 1});
            if (o.code == OP_SEND_MID) log.push_back({o.phase, o.iter, o.arg, w, w + 1, 1, mm - 1});
        }
    auto rank = [](int s) { return s == 'B' ? 0 : s == 'P' ? 1 : s == 'A' ? 2 : s == 'M' ? 3 : 4; };
    std::stable_sort(log.begin(), log.end(), [&](const MsgRec& a, const MsgRec& b) {
        return std::make_tuple(a.phase, a.iteration, a.sender, rank(a.step)) <
               std::make_tuple(b.phase, b.iteration, b.sender, rank(b.step));
    });
    return log;
}

// ---- NCCL (resolved at run time so libpswe.so loads on machines without NCCL) --------------

typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
enum { ncclFloat64 = 8, ncclUint8 = 1 };
typedef int ncclResult_t;

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    void load() {
        if (h) return;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) throw std::runtime_error("NCCL not available (dlopen libnccl.so.2 failed)");
        auto sym = [&](const char* s) {
            void* p = dlsym(h, s);
            if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + s);
            return p;
        };
        GetUniqueId = (decltype(GetUniqueId))sym("ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))sym("ncclCommInitRank");
        CommDestroy = (decltype(CommDestroy))sym("ncclCommDestroy");
        Send = (decltype(Send))sym("ncclSend");
        Recv = (decltype(Recv))sym("ncclRecv");
        Broadcast = (decltype(Broadcast))sym("ncclBroadcast");
        AllGather = (decltype(AllGather))sym("ncclAllGather");
        GetErrorString = (decltype(GetErrorString))sym("ncclGetErrorString");
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != 0) throw std::runtime_error(std::string(what) + ": " + GetErrorString(r));
    }
};
static NcclApi& nccl() {
    static NcclApi api;
    api.load();
    return api;
}

}  // namespace pswe

using namespace pswe;

// One block controller. Owns the comm objects and per-block device buffers; the levels and the
// pair belong to the caller.
struct pswe_pfasst {
    pswe_pair* pair = nullptr;   // (fine, next level)
    pswe_pair* pair2 = nullptr;  // three levels: (mid, coarse)
    int nlev = 2;
    pswe_level *fine = nullptr, *coarse = nullptr, *mid = nullptr;
    int Rf = 0, Rc = 0, mf = 0, mc = 0, Rm = 0, mm = 0;
    long Kf = 0, Kc = 0, Km = 0;
    double2* d_tau_mid = nullptr;      // [mm][3Km]
    double2* d_dstate0_mid = nullptr;  // [3Km]
    pswe_block_config cfg{};
    bool distributed = false;
    int rank = 0, world = 1;
    double2* d_tau = nullptr;      // [mc][3Kc]
    double2* d_dstate0 = nullptr;  // [3Kf]
    double* d_res = nullptr;       // [n_ts][n_iter+1]
    // serial emulation: queues of device buffers per (receiver, level)
    struct Msg {
        double2* buf;
        int phase, iter, level;
    };
    std::map<std::pair<int, int>, std::deque<Msg>> queues;
    std::vector<double2*> pool[3];  // free message buffers per level
    // NCCL
    ncclComm_t comm[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};  // [level][parity]
    ncclComm_t world_comm = nullptr;
    cudaStream_t send_stream[3] = {nullptr, nullptr, nullptr};
    std::vector<double2*> send_bufs[3];
    std::vector<cudaEvent_t> send_done[3];
    size_t send_next[3] = {0, 0, 0};
    long K_of(int level) const { return level == 0 ? Kf : (level == nlev - 1 ? Kc : Km); }
    double* d_res_all = nullptr;
    // serial emulation replays the whole block as one CUDA graph (captured on the 2nd call,
    // after an eager call has sized every pool); theta0 is copied into d_theta first
    bool use_graph = true;
    int eager_runs = 0;
    double2* d_theta = nullptr;
    cudaGraphExec_t graph = nullptr;
    unsigned long long graph_gen = 0;  // plan scratch generations the graph was captured over
    cudaStream_t gstream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
};

namespace {

size_t state_bytes(long K) { return (size_t)3 * K * sizeof(double2); }

// sum of the scratch generations of every level's plan (each only grows)
unsigned long long plans_generation(const pswe_pfasst* pf) {
    unsigned long long g = pf->fine->plan->generation + 3 * pf->coarse->plan->generation;
    if (pf->mid) g += 9 * pf->mid->plan->generation;
    return g;
}

void init_common(pswe_pfasst* pf, pswe_pair* pair, const pswe_block_config* cfg, pswe_pair* pair2 = nullptr) {
    if (!pair || !cfg) throw std::invalid_argument("pswe_pfasst: NULL argument");
    if (cfg->n_time_steps < 1) throw std::invalid_argument("run_block: need n_time_steps >= 1");
    if (cfg->n_iter < 1) throw std::invalid_argument("run_block: need n_iter >= 1");
    if (pair2 && pair2->fine != pair->coarse)
        throw std::invalid_argument("pswe_pfasst3: the second pair must start at the first pair's coarse level");
    pf->pair = pair;
    pf->pair2 = pair2;
    pf->nlev = pair2 ? 3 : 2;
    pf->cfg = *cfg;
    pf->fine = pair->fine;
    pf->coarse = pair2 ? pair2->coarse : pair->coarse;
    if (pair2) {
        pf->mid = pair->coarse;
        pf->Rm = pf->mid->R;
        pf->mm = pf->mid->nn;
        pf->Km = num_coeffs(pf->Rm);
        PSWE_CUDA(cudaMalloc(&pf->d_tau_mid, pf->mm * state_bytes(pf->Km)));
        PSWE_CUDA(cudaMalloc(&pf->d_dstate0_mid, state_bytes(pf->Km)));
    }
    pf->Rf = pf->fine->R;
    pf->mf = pf->fine->nn;
    pf->Rc = pf->coarse->R;
    pf->mc = pf->coarse->nn;
    pf->Kf = num_coeffs(pf->Rf);
    pf->Kc = num_coeffs(pf->Rc);
    PSWE_CUDA(cudaMalloc(&pf->d_tau, pf->mc * state_bytes(pf->Kc)));
    PSWE_CUDA(cudaMalloc(&pf->d_dstate0, state_bytes(pf->Kf)));
    PSWE_CUDA(cudaMalloc(&pf->d_res, sizeof(double) * cfg->n_time_steps * (cfg->n_iter + 1)));
}

double2* st_ptr(pswe_level* L, int node) { return reinterpret_cast<double2*>(pswe_level_ptr(L, 0, node)); }

// execute the schedule of worker w; send/recv through the callbacks
template <class SendF, class RecvF>
void run_worker(pswe_pfasst* pf, int w, const double2* theta0, cudaStream_t st, SendF&& send, RecvF&& recv) {
    const int n = pf->cfg.n_time_steps, N = pf->cfg.n_iter;
    const double dt = pf->cfg.dt;
    pswe_level *F = pf->fine, *C = pf->coarse, *M = pf->mid;
    const int lc = pf->nlev - 1;  // message level of the coarsest level
    for (const Op& o : build_schedule(w, n, N, pf->nlev)) {
        switch (o.code) {
            case OP_PREDICT_INIT:
                pswe_restrict_space(pf->Rf, pf->Rc, reinterpret_cast<const double*>(theta0),
                                    reinterpret_cast<double*>(st_ptr(C, 0)), 1, st);
                level_spread(C, st_ptr(C, 0), st);
                break;
            case OP_RECV_COARSE_IC: recv(w, lc, o.phase, o.iter, st_ptr(C, 0), pf->Kc); break;
            case OP_REFRESH_COARSE0: level_refresh(C, 0, 1, st); break;
            case OP_SWEEP_COARSE: level_sweep(C, dt, o.arg ? pf->d_tau : nullptr, st); break;
            case OP_SEND_COARSE: send(w, lc, o.phase, o.iter, st_ptr(C, pf->mc - 1), pf->Kc); break;
            case OP_INTERP_STATES: pair_interp_states(pf->pair, st); break;
            case OP_REFRESH_FINE_ALL: level_refresh(F, 0, pf->mf, st); break;
            case OP_RESIDUAL: level_residual(F, dt, pf->d_res + (size_t)w * (N + 1) + o.arg, st); break;
            case OP_SWEEP_FINE: level_sweep(F, dt, nullptr, st); break;
            case OP_SEND_FINE: send(w, 0, o.phase, o.iter, st_ptr(F, pf->mf - 1), pf->Kf); break;
            case OP_RESTRICT: pair_restrict_states(pf->pair, st); break;
            case OP_REFRESH_COARSE_ALL: level_refresh(C, 0, pf->mc, st); break;
            case OP_SAVE: pair_save(pf->pair, st); break;
            case OP_FAS: pair_fas(pf->pair, dt, pf->d_tau, st); break;
            case OP_INTERP_INC: pair_interp_increment_add(pf->pair, pf->d_dstate0, st); break;
            case OP_RECV_FINE_IC: recv(w, 0, o.phase, o.iter, st_ptr(F, 0), pf->Kf); break;
            case OP_REFRESH_FINE0: level_refresh(F, 0, 1, st); break;
            case OP_INTERP_STATES_MC: pair_interp_states(pf->pair2, st); break;
            case OP_REFRESH_MID_ALL: level_refresh(M, 0, pf->mm, st); break;
            case OP_RESTRICT_MC: pair_restrict_states(pf->pair2, st); break;
            case OP_SAVE_MC: pair_save(pf->pair2, st); break;
            case OP_FAS_MC: pair_fas(pf->pair2, dt, pf->d_tau, st, pf->d_tau_mid); break;
            case OP_SWEEP_MID: level_sweep(M, dt, pf->d_tau_mid, st); break;
            case OP_SEND_MID: send(w, 1, o.phase, o.iter, st_ptr(M, pf->mm - 1), pf->Km); break;
            case OP_INTERP_INC_MC: pair_interp_increment_add(pf->pair2, pf->d_dstate0_mid, st); break;
            case OP_RECV_MID_IC: recv(w, 1, o.phase, o.iter, st_ptr(M, 0), pf->Km); break;
            case OP_REFRESH_MID0: level_refresh(M, 0, 1, st); break;
            case OP_FAS_FM: pair_fas(pf->pair, dt, pf->d_tau_mid, st); break;
            default: throw std::logic_error("pfasst: unknown op");
        }
    }
}

__global__ void add_state_kernel(double2* dst, const double2* a, const double2* b, long n) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = make_double2(a[i].x + b[i].x, a[i].y + b[i].y);
}

// received IC + the receiver's own interpolated node-0 increment (pfasst.cpp:171-174): the
// reference's two-level form (fine level only). Three-level chains use low-mode replacement
// instead (replace_low_modes below).
bool has_dstate(const pswe_pfasst* pf, int level) { return level == 0 && pf->nlev == 2; }

// Three-level IC update: node 0 of level l := received state with its coefficients (m, s) <= R_{l+1}
// replaced by node 0 of level l+1, i.e. recv + pad(c0 - trunc(recv)). The two-level form above
// measures the coarse increment against the OLD restricted node 0 while the received state is
// already new, so the low-mode part of the IC change is counted twice; nested over two levels that
// diverged (tests/test_gpu_pfasst3.py), while this form has the same fixed point without it.
__global__ void replace_low_kernel(int Rf, int Rc, double2* __restrict__ dst, const double2* __restrict__ src) {
    const int m = blockIdx.y, f = blockIdx.z;
    const int s = m + blockIdx.x * blockDim.x + threadIdx.x;
    if (s > Rc) return;
    const long Kf = (long)(Rf + 1) * (Rf + 2) / 2, Kc = (long)(Rc + 1) * (Rc + 2) / 2;
    dst[f * Kf + off_std(Rf, m) + (s - m)] = src[f * Kc + off_std(Rc, m) + (s - m)];
}
void replace_low_modes(pswe_pfasst* pf, int level, double2* dst, cudaStream_t st) {
    pswe_level* lower = level == 0 ? pf->mid : pf->coarse;
    const int Rf = level == 0 ? pf->Rf : pf->Rm;
    const int Rc = lower->R;
    dim3 grid((Rc + 1 + 127) / 128, Rc + 1, 3);
    replace_low_kernel<<<grid, 128, 0, st>>>(Rf, Rc, dst, st_ptr(lower, 0));
    PSWE_LAUNCH_CHECK();
}
bool has_low_replace(const pswe_pfasst* pf, int level) { return pf->nlev == 3 && level <= 1; }
void add_dstate0(pswe_pfasst* pf, double2* dst, const double2* msg, cudaStream_t st, int level = 0) {
    const long n = 3 * pf->K_of(level);
    add_state_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dst, msg, level ? pf->d_dstate0_mid : pf->d_dstate0,
                                                                  n);
    PSWE_LAUNCH_CHECK();
}

void run_serial(pswe_pfasst* pf, const double2* theta0, cudaStream_t st) {
    pf->queues.clear();
    std::vector<std::pair<int, double2*>> in_use;
    auto get_buf = [&](int level) {
        auto& pool = pf->pool[level];
        double2* b;
        if (!pool.empty()) {
            b = pool.back();
            pool.pop_back();
        } else {
            PSWE_CUDA(cudaMalloc(&b, state_bytes(pf->K_of(level))));
        }
        return b;
    };
    auto send = [&](int w, int level, int phase, int iter, const double2* src, long K) {
        double2* b = get_buf(level);
        PSWE_CUDA(cudaMemcpyAsync(b, src, state_bytes(K), cudaMemcpyDeviceToDevice, st));
        pf->queues[{w + 1, level}].push_back({b, phase, iter, level});
    };
    auto recv = [&](int w, int level, int phase, int iter, double2* dst, long K) {
        auto& q = pf->queues[{w, level}];
        if (q.empty()) throw std::runtime_error("pfasst: receive on an empty channel (schedule bug)");
        const auto m = q.front();
        q.pop_front();
        if (m.phase != phase || m.iter != iter || m.level != level)
            throw std::logic_error("pfasst: message tag mismatch");
        if (has_dstate(pf, level)) add_dstate0(pf, dst, m.buf, st, level);
        else PSWE_CUDA(cudaMemcpyAsync(dst, m.buf, state_bytes(K), cudaMemcpyDeviceToDevice, st));
        if (has_low_replace(pf, level)) replace_low_modes(pf, level, dst, st);
        pf->pool[level].push_back(m.buf);  // stream-ordered reuse
    };
    for (int w = 0; w < pf->cfg.n_time_steps; ++w) run_worker(pf, w, theta0, st, send, recv);
}

void run_nccl(pswe_pfasst* pf, const double2* theta0, cudaStream_t st) {
    auto& api = nccl();
    const int w = pf->rank, n = pf->world;
    auto send = [&](int, int level, int, int, const double2* src, long K) {
        // stage into a ring buffer (the reference's message holds a copy), then send from the
        // level's send stream so the compute stream never waits for the receiver
        const size_t slot = pf->send_next[level]++ % pf->send_bufs[level].size();
        double2* b = pf->send_bufs[level][slot];
        cudaEvent_t ev = pf->send_done[level][slot];
        PSWE_CUDA(cudaStreamWaitEvent(st, ev, 0));  // previous send from this slot finished
        PSWE_CUDA(cudaMemcpyAsync(b, src, state_bytes(K), cudaMemcpyDeviceToDevice, st));
        cudaEvent_t ready;
        PSWE_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        PSWE_CUDA(cudaEventRecord(ready, st));
        PSWE_CUDA(cudaStreamWaitEvent(pf->send_stream[level], ready, 0));
        PSWE_CUDA(cudaEventDestroy(ready));
        api.check(api.Send(b, state_bytes(K) / sizeof(double), ncclFloat64, w + 1, pf->comm[level][w % 2],
                           pf->send_stream[level]),
                  "ncclSend");
        PSWE_CUDA(cudaEventRecord(ev, pf->send_stream[level]));
    };
    auto recv = [&](int, int level, int, int, double2* dst, long K) {
        // fine IC: receive into dst, then add the node-0 increment in place (pfasst.cpp:171-174)
        api.check(api.Recv(dst, state_bytes(K) / sizeof(double), ncclFloat64, w - 1, pf->comm[level][(w + 1) % 2], st),
                  "ncclRecv");
        if (has_dstate(pf, level)) add_dstate0(pf, dst, dst, st, level);
        if (has_low_replace(pf, level)) replace_low_modes(pf, level, dst, st);
    };
    run_worker(pf, w, theta0, st, send, recv);
    // make sure all sends are posted before the block ends
    for (int l = 0; l < pf->nlev; ++l) {
        cudaEvent_t e;
        PSWE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        PSWE_CUDA(cudaEventRecord(e, pf->send_stream[l]));
        PSWE_CUDA(cudaStreamWaitEvent(st, e, 0));
        PSWE_CUDA(cudaEventDestroy(e));
    }
}

}  // namespace

extern "C" {

static void create_serial(pswe_pair* pair, pswe_pair* pair2, const pswe_block_config* cfg, pswe_pfasst** out) {
    if (!out) throw std::invalid_argument("out is NULL");
    auto* pf = new pswe_pfasst;
    if (const char* e = std::getenv("PSWE_NO_GRAPH")) pf->use_graph = std::atoi(e) == 0;
    try {
        init_common(pf, pair, cfg, pair2);
    } catch (...) {
        delete pf;
        throw;
    }
    *out = pf;
}

int pswe_pfasst_create_serial(pswe_pair* pair, const pswe_block_config* cfg, pswe_pfasst** out) {
    return guarded([&] { create_serial(pair, nullptr, cfg, out); });
}

int pswe_pfasst3_create_serial(pswe_pair* fine_mid, pswe_pair* mid_coarse, const pswe_block_config* cfg,
                               pswe_pfasst** out) {
    return guarded([&] {
        if (!mid_coarse) throw std::invalid_argument("pswe_pfasst3: NULL mid-coarse pair");
        create_serial(fine_mid, mid_coarse, cfg, out);
    });
}

int pswe_nccl_unique_id(void* out128) {
    return guarded([&] {
        ncclUniqueId id;
        nccl().check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof(id));
    });
}

static void create_nccl(pswe_pair* pair, pswe_pair* pair2, const pswe_block_config* cfg, int rank, int world,
                        const void* uid, pswe_pfasst** out) {
    {
        if (!out || !uid) throw std::invalid_argument("NULL argument");
        if (cfg && cfg->n_time_steps != world)
            throw std::invalid_argument("pswe_pfasst_create_nccl: n_time_steps must equal world size");
        auto& api = nccl();
        auto* pf = new pswe_pfasst;
        init_common(pf, pair, cfg, pair2);
        pf->distributed = true;
        pf->rank = rank;
        pf->world = world;
        // 5 communicators from one unique id: derive distinct ids by perturbing a byte the
        // bootstrap does not use for addressing is not portable, so every comm is initialised
        // from the same id sequentially (NCCL allows re-using an id once per init round).
        ncclUniqueId base;
        std::memcpy(&base, uid, sizeof(base));
        api.check(api.CommInitRank(&pf->world_comm, world, base, rank), "ncclCommInitRank(world)");
        for (int l = 0; l < pf->nlev; ++l)
            for (int p = 0; p < 2; ++p) {
                // per-comm ids are broadcast through the world communicator
                ncclUniqueId id;
                if (rank == 0) api.check(api.GetUniqueId(&id), "ncclGetUniqueId");
                char* d_id;
                PSWE_CUDA(cudaMalloc(&d_id, sizeof(id)));
                PSWE_CUDA(cudaMemcpy(d_id, &id, sizeof(id), cudaMemcpyHostToDevice));
                api.check(api.Broadcast(d_id, d_id, sizeof(id), ncclUint8, 0, pf->world_comm, 0), "ncclBroadcast(id)");
                PSWE_CUDA(cudaMemcpy(&id, d_id, sizeof(id), cudaMemcpyDeviceToHost));
                cudaFree(d_id);
                api.check(api.CommInitRank(&pf->comm[l][p], world, id, rank), "ncclCommInitRank(p2p)");
            }
        for (int l = 0; l < pf->nlev; ++l) {
            PSWE_CUDA(cudaStreamCreateWithFlags(&pf->send_stream[l], cudaStreamNonBlocking));
            const long K = pf->K_of(l);
            const int nslots = l == pf->nlev - 1 ? world + cfg->n_iter + 2 : cfg->n_iter + 2;
            for (int s = 0; s < nslots; ++s) {
                double2* b;
                PSWE_CUDA(cudaMalloc(&b, state_bytes(K)));
                pf->send_bufs[l].push_back(b);
                cudaEvent_t e;
                PSWE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                PSWE_CUDA(cudaEventRecord(e, pf->send_stream[l]));
                pf->send_done[l].push_back(e);
            }
        }
        PSWE_CUDA(cudaMalloc(&pf->d_res_all, sizeof(double) * world * (cfg->n_iter + 1)));
        *out = pf;
    }
}

int pswe_pfasst_create_nccl(pswe_pair* pair, const pswe_block_config* cfg, int rank, int world,
                            const void* uid, pswe_pfasst** out) {
    return guarded([&] { create_nccl(pair, nullptr, cfg, rank, world, uid, out); });
}

int pswe_pfasst3_create_nccl(pswe_pair* fine_mid, pswe_pair* mid_coarse, const pswe_block_config* cfg, int rank,
                             int world, const void* uid, pswe_pfasst** out) {
    return guarded([&] {
        if (!mid_coarse) throw std::invalid_argument("pswe_pfasst3: NULL mid-coarse pair");
        create_nccl(fine_mid, mid_coarse, cfg, rank, world, uid, out);
    });
}

int pswe_pfasst_destroy(pswe_pfasst* pf) {
    return guarded([&] {
        if (!pf) return;
        cudaDeviceSynchronize();
        if (pf->graph) cudaGraphExecDestroy(pf->graph);
        if (pf->d_theta) cudaFree(pf->d_theta);
        if (pf->gstream) cudaStreamDestroy(pf->gstream);
        if (pf->ev_in) cudaEventDestroy(pf->ev_in);
        if (pf->ev_out) cudaEventDestroy(pf->ev_out);
        cudaFree(pf->d_tau);
        cudaFree(pf->d_dstate0);
        if (pf->d_tau_mid) cudaFree(pf->d_tau_mid);
        if (pf->d_dstate0_mid) cudaFree(pf->d_dstate0_mid);
        cudaFree(pf->d_res);
        if (pf->d_res_all) cudaFree(pf->d_res_all);
        for (int l = 0; l < 3; ++l) {
            for (auto* b : pf->pool[l]) cudaFree(b);
            for (auto* b : pf->send_bufs[l]) cudaFree(b);
            for (auto e : pf->send_done[l]) cudaEventDestroy(e);
            if (pf->send_stream[l]) cudaStreamDestroy(pf->send_stream[l]);
        }
        for (auto& q : pf->queues)
            for (auto& m : q.second) cudaFree(m.buf);
        if (pf->distributed) {
            auto& api = nccl();
            for (auto& l : pf->comm)
                for (auto c : l)
                    if (c) api.CommDestroy(c);
            if (pf->world_comm) api.CommDestroy(pf->world_comm);
        }
        delete pf;
    });
}

int pswe_pfasst_run_block(pswe_pfasst* pf, const double* theta0, double* final_state, double* residuals,
                          void* stream) {
    return guarded([&] {
        if (!pf || !theta0) throw std::invalid_argument("NULL argument");
        const cudaStream_t st = as_stream(stream);
        const double2* th = reinterpret_cast<const double2*>(theta0);
        const int n = pf->cfg.n_time_steps, N = pf->cfg.n_iter;
        PSWE_CUDA(cudaMemsetAsync(pf->d_res, 0, sizeof(double) * n * (N + 1), st));
        if (!pf->distributed) {
            if (!pf->use_graph) {
                run_serial(pf, th, st);
            } else {
                // the block is a fixed sequence of ~10^2-10^3 small launches: capture it once and
                // replay it (no host launch overhead, no host logic per kernel)
                // capture/launch on an internal stream (the caller's may be the legacy default
                // stream, which cannot be captured), ordered after / before the caller's stream
                if (!pf->d_theta) {
                    PSWE_CUDA(cudaMalloc(&pf->d_theta, state_bytes(pf->Kf)));
                    PSWE_CUDA(cudaStreamCreateWithFlags(&pf->gstream, cudaStreamNonBlocking));
                    PSWE_CUDA(cudaEventCreateWithFlags(&pf->ev_in, cudaEventDisableTiming));
                    PSWE_CUDA(cudaEventCreateWithFlags(&pf->ev_out, cudaEventDisableTiming));
                }
                const cudaStream_t gs = pf->gstream;
                // the graph holds raw pointers into the levels' plan scratch, which is grow-only
                // and reallocated by a larger eval/transform batch, pswe_plan_reserve or a level
                // with more nodes: any change since the capture makes it stale -> run eagerly once
                // (re-sizing every pool), then capture again
                const unsigned long long gen = plans_generation(pf);
                if (pf->graph && gen != pf->graph_gen) {
                    PSWE_CUDA(cudaGraphExecDestroy(pf->graph));
                    pf->graph = nullptr;
                    pf->eager_runs = 0;
                }
                PSWE_CUDA(cudaMemcpyAsync(pf->d_theta, th, state_bytes(pf->Kf), cudaMemcpyDeviceToDevice, st));
                PSWE_CUDA(cudaEventRecord(pf->ev_in, st));
                PSWE_CUDA(cudaStreamWaitEvent(gs, pf->ev_in, 0));
                if (!pf->graph && pf->eager_runs >= 1) {
                    cudaGraph_t g = nullptr;
                    PSWE_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
                    try {
                        run_serial(pf, pf->d_theta, gs);
                    } catch (...) {
                        cudaStreamEndCapture(gs, &g);
                        if (g) cudaGraphDestroy(g);
                        throw;
                    }
                    PSWE_CUDA(cudaStreamEndCapture(gs, &g));
                    PSWE_CUDA(cudaGraphInstantiate(&pf->graph, g, 0));
                    cudaGraphDestroy(g);
                    pf->graph_gen = plans_generation(pf);
                }
                if (pf->graph) {
                    PSWE_CUDA(cudaGraphLaunch(pf->graph, gs));
                } else {
                    run_serial(pf, pf->d_theta, gs);
                    ++pf->eager_runs;
                }
                PSWE_CUDA(cudaEventRecord(pf->ev_out, gs));
                PSWE_CUDA(cudaStreamWaitEvent(st, pf->ev_out, 0));
            }
            if (final_state)
                PSWE_CUDA(cudaMemcpyAsync(final_state, st_ptr(pf->fine, pf->mf - 1), state_bytes(pf->Kf),
                                          cudaMemcpyDeviceToDevice, st));
            if (residuals) {
                PSWE_CUDA(cudaMemcpyAsync(residuals, pf->d_res, sizeof(double) * n * (N + 1), cudaMemcpyDeviceToHost, st));
                PSWE_CUDA(cudaStreamSynchronize(st));
            }
        } else {
            auto& api = nccl();
            run_nccl(pf, th, st);
            // BlockResult: the last step's final state goes to every rank (next block's theta0,
            // runner.cpp:145-147); residual rows are gathered everywhere.
            if (final_state) {
                if (pf->rank == pf->world - 1)
                    PSWE_CUDA(cudaMemcpyAsync(final_state, st_ptr(pf->fine, pf->mf - 1), state_bytes(pf->Kf),
                                              cudaMemcpyDeviceToDevice, st));
                api.check(api.Broadcast(final_state, final_state, state_bytes(pf->Kf) / sizeof(double), ncclFloat64,
                                        pf->world - 1, pf->world_comm, st),
                          "ncclBroadcast(final)");
            }
            api.check(api.AllGather(pf->d_res + (size_t)pf->rank * (N + 1), pf->d_res_all, N + 1, ncclFloat64,
                                    pf->world_comm, st),
                      "ncclAllGather(residuals)");
            if (residuals) {
                PSWE_CUDA(cudaMemcpyAsync(residuals, pf->d_res_all, sizeof(double) * n * (N + 1), cudaMemcpyDeviceToHost, st));
                PSWE_CUDA(cudaStreamSynchronize(st));
            }
        }
    });
}

int pswe_pfasst_messages(const pswe_pfasst* pf, int* out, int max_records) {
    if (!pf) return 0;
    const auto log = message_log(pf->cfg.n_time_steps, pf->cfg.n_iter, pf->mf, pf->mc, pf->nlev, pf->mm);
    const int n = (int)log.size();
    if (out)
        for (int i = 0; i < n && i < max_records; ++i) {
            const auto& m = log[i];
            int* o = out + 7 * i;
            o[0] = m.phase; o[1] = m.iteration; o[2] = m.step; o[3] = m.sender;
            o[4] = m.receiver; o[5] = m.level; o[6] = m.node;
        }
    return n;
}

// Schedule of worker w as 4 ints per op (code, phase, iter, arg); returns the op count.
int pswe_pfasst_schedule(int w, int n_time_steps, int n_iter, int* out, int max_ops) {
    return pswe_pfasst_schedule_ml(2, w, n_time_steps, n_iter, out, max_ops);
}

int pswe_pfasst_schedule_ml(int n_levels, int w, int n_time_steps, int n_iter, int* out, int max_ops) {
    if (n_levels != 2 && n_levels != 3) return -1;
    const auto ops = build_schedule(w, n_time_steps, n_iter, n_levels);
    if (out)
        for (int i = 0; i < (int)ops.size() && i < max_ops; ++i) {
            out[4 * i] = ops[i].code;
            out[4 * i + 1] = ops[i].phase;
            out[4 * i + 2] = ops[i].iter;
            out[4 * i + 3] = ops[i].arg;
        }
    return (int)ops.size();
}

}  // extern "C"
