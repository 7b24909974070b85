// PFASST block controller (host C++), the B200 replacement of pf::run_block
// (proj/src/pfasst.cpp:78-251, Algorithm 1 of PAPER.md:709-766).
//
// The per-worker control flow is generated once as data (build_schedule, mirroring
// worker_predict :78-120 and worker_iterate :122-176 op for op) and executed by
//   * SerialExec  — all workers on this GPU in worker order with in-process message queues
//                   (the reference's Mode::serial_emulation, :212-216);
//   * run_dist    — one process per GPU, worker w = rank, messages through a Transport
//                   (transport.h): CUDA IPC over peer memory (NVLink/NVSwitch; also several
//                   processes on one GPU) or NCCL send/recv. Every message carries a
//                   (phase, iteration, level, sender, sequence) trailer checked on receipt
//                   (the reference's expect(), :71-76), receives are bounded by
//                   recv_timeout_seconds (pfasst.hpp:19, :39-47) and a failing rank aborts
//                   the block for its peers (the reference rethrows worker exceptions,
//                   :219-234).
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
#include "transport.h"

namespace pswe {
void level_spread(pswe_level* L, const double2* theta0, cudaStream_t st);
void level_refresh(pswe_level* L, int first, int count, cudaStream_t st);
void level_sweep(pswe_level* L, double dt, const double2* tau, cudaStream_t st, double* res_out = nullptr);
void level_residual(pswe_level* L, double dt, double* out, cudaStream_t st);
void pair_restrict_states(pswe_pair* P, cudaStream_t st);
void pair_fas(pswe_pair* P, double dt, double2* tau, cudaStream_t st, const double2* tau_f = nullptr);
void pair_save(pswe_pair* P, cudaStream_t st);
void pair_interp_increment_add(pswe_pair* P, double2* dstate0, cudaStream_t st, bool dstate0_outside_zero);
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

std::vector<Op> build_schedule3(int w, int n, int n_iter, int mid_sweeps);

std::vector<Op> build_schedule(int w, int n, int n_iter, int nlev = 2, int mid_sweeps = 1) {
    if (nlev == 3) return build_schedule3(w, n, n_iter, mid_sweeps);
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
// mid_sweeps: mid-level sweeps on each leg of the V-cycle (1; 0 only for the degenerate-chain
// check of tests/test_gpu_pfasst3.py, where the mid level equals the fine one)
std::vector<Op> build_schedule3(int w, int n, int n_iter, int mid_sweeps) {
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
        for (int i = 0; i < mid_sweeps; ++i) ops.push_back({OP_SWEEP_MID, 1, k, 0});
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
        for (int i = 0; i < mid_sweeps; ++i) ops.push_back({OP_SWEEP_MID, 1, k, 0});
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
    // distributed: this rank's worker, messages through the transport
    std::unique_ptr<Transport> tr;
    unsigned long long sseq[3] = {0, 0, 0}, rseq[3] = {0, 0, 0};  // messages sent / received per level
    TagError* h_err = nullptr;  // host-mapped: raised by consume kernels on a tag mismatch
    TagError* d_err = nullptr;
    double recv_timeout = 300.0;  // BlockConfig::recv_timeout_seconds (pfasst.hpp:19)
    int fault = 0;                // fault injection for tests (PSWE_PFASST_FAULT): 1 = skew tags
    bool broken = false;          // a block failed: the transport state is undefined
    // distributed: segment graphs (captured on the second block, replayed after; invalidated like
    // the serial graph when a plan's scratch is reallocated)
    std::vector<cudaGraphExec_t> seg_graphs;
    int dist_runs = 0;
    unsigned long long seg_gen = 0;
    // BlockResult.step_final (pfasst.hpp:34-36): serial: every worker's last fine node [n][3Kf]
    double2* d_step_final = nullptr;
    long K_of(int level) const { return level == 0 ? Kf : (level == nlev - 1 ? Kc : Km); }
    // serial emulation replays the whole block as one CUDA graph (captured on the 2nd call,
    // after an eager call has sized every pool); theta0 is copied into d_theta first
    bool use_graph = true;
    // three levels: node-0 update form (PSWE_NODE0_LOWMODE default / PSWE_NODE0_REFERENCE) and
    // mid-level sweeps per V-cycle leg (pswe_pfasst3_configure)
    int node0 = PSWE_NODE0_LOWMODE;
    int mid_sweeps = 1;
    // Worker 0 receives nothing, so in every iteration its node-0 states stay exactly what they
    // were (the interpolated coarse increment at node 0 is exactly zero: coarse node 0 is never
    // changed by a sweep or a receive); the reference still re-evaluates F there after Step C/D
    // (refresh_node(coarse, 0), pfasst.cpp:152; refresh_node(fine, 0), :175) and gets the same
    // bits. The executor skips those evaluations for worker 0 (the schedule and the message log
    // are unchanged); tests/test_gpu_sdc_pfasst.py checks bit-identity with PSWE_PFASST_NO_ELIDE=1.
    bool elide_w0 = true;
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
        // increments are written only inside the coarser triangle: the rest stays zero
        PSWE_CUDA(cudaMemset(pf->d_dstate0_mid, 0, state_bytes(pf->Km)));
    }
    pf->Rf = pf->fine->R;
    pf->mf = pf->fine->nn;
    pf->Rc = pf->coarse->R;
    pf->mc = pf->coarse->nn;
    pf->Kf = num_coeffs(pf->Rf);
    pf->Kc = num_coeffs(pf->Rc);
    PSWE_CUDA(cudaMalloc(&pf->d_tau, pf->mc * state_bytes(pf->Kc)));
    PSWE_CUDA(cudaMalloc(&pf->d_dstate0, state_bytes(pf->Kf)));
    PSWE_CUDA(cudaMemset(pf->d_dstate0, 0, state_bytes(pf->Kf)));
    PSWE_CUDA(cudaMalloc(&pf->d_res, sizeof(double) * cfg->n_time_steps * (cfg->n_iter + 1)));
}

double2* st_ptr(pswe_level* L, int node) { return reinterpret_cast<double2*>(pswe_level_ptr(L, 0, node)); }

// execute the schedule of worker w; send/recv through the callbacks
bool is_comm(int code) {
    return code == OP_SEND_COARSE || code == OP_SEND_FINE || code == OP_SEND_MID || code == OP_RECV_COARSE_IC ||
           code == OP_RECV_FINE_IC || code == OP_RECV_MID_IC;
}

// Segment graphs of the distributed executor: the ops between two messages (sends and receives
// stay eager - they touch host-side counters, events and the transport's rings) are captured once
// per run of compute ops and replayed as one graph launch each.
struct SegCtl {
    enum Mode { EAGER, CAPTURE, REPLAY } mode = EAGER;
    std::vector<cudaGraphExec_t>* graphs = nullptr;
    size_t next = 0;
    bool capturing = false;
    cudaStream_t st = nullptr;
    void close() {  // end the open capture, instantiate, launch
        if (!capturing) return;
        cudaGraph_t g = nullptr;
        PSWE_CUDA(cudaStreamEndCapture(st, &g));
        cudaGraphExec_t e = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&e, g, 0);
        cudaGraphDestroy(g);
        PSWE_CUDA(ie);
        graphs->push_back(e);
        capturing = false;
        PSWE_CUDA(cudaGraphLaunch(e, st));
    }
    // returns true if the compute op must be issued now (eager or being captured)
    bool compute(bool first_of_run) {
        if (mode == EAGER) return true;
        if (mode == CAPTURE) {
            if (!capturing) {
                PSWE_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                capturing = true;
            }
            return true;
        }
        if (first_of_run) {
            if (next >= graphs->size()) throw std::logic_error("pfasst: segment graph missing");
            PSWE_CUDA(cudaGraphLaunch((*graphs)[next++], st));
        }
        return false;
    }
    void comm() {
        if (mode == CAPTURE) close();
    }
    void abort_capture() {
        if (!capturing) return;
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        capturing = false;
    }
};

template <class SendF, class RecvF>
void run_worker(pswe_pfasst* pf, int w, const double2* theta0, cudaStream_t st, SendF&& send, RecvF&& recv,
                SegCtl* seg = nullptr) {
    const int n = pf->cfg.n_time_steps, N = pf->cfg.n_iter;
    const double dt = pf->cfg.dt;
    pswe_level *F = pf->fine, *C = pf->coarse, *M = pf->mid;
    const int lc = pf->nlev - 1;  // message level of the coarsest level
    static const char* const op_name[] = {
        "", "PREDICT_INIT", "RECV_COARSE_IC", "REFRESH_COARSE0", "SWEEP_COARSE", "SEND_COARSE", "INTERP_STATES",
        "REFRESH_FINE_ALL", "RESIDUAL", "SWEEP_FINE", "SEND_FINE", "RESTRICT", "REFRESH_COARSE_ALL", "SAVE", "FAS",
        "INTERP_INC", "RECV_FINE_IC", "REFRESH_FINE0", "INTERP_STATES_MC", "REFRESH_MID_ALL", "RESTRICT_MC",
        "SAVE_MC", "FAS_MC", "SWEEP_MID", "SEND_MID", "INTERP_INC_MC", "RECV_MID_IC", "REFRESH_MID0", "FAS_FM"};
    const std::vector<Op> ops = build_schedule(w, n, N, pf->nlev, pf->mid_sweeps);
    // a fine sweep followed by the residual: its last tail kernel computes the residual too
    static const bool fuse_res = [] { const char* e = getenv("PSWE_NO_TAIL_RES"); return !(e && atoi(e) != 0); }();
    bool res_fused = false;
    for (size_t i = 0; i < ops.size(); ++i) {
        const Op& o = ops[i];
        PSWE_NVTX(op_name[o.code]);
        if (seg) {
            if (is_comm(o.code)) {
                seg->comm();
            } else if (!seg->compute(i == 0 || is_comm(ops[i - 1].code))) {
                continue;  // replayed inside this run's segment graph
            }
        }
        switch (o.code) {
            case OP_PREDICT_INIT:
                pswe_restrict_space(pf->Rf, pf->Rc, reinterpret_cast<const double*>(theta0),
                                    reinterpret_cast<double*>(st_ptr(C, 0)), 1, st);
                level_spread(C, st_ptr(C, 0), st);
                break;
            case OP_RECV_COARSE_IC: recv(w, lc, o.phase, o.iter, st_ptr(C, 0), pf->Kc); break;
            case OP_REFRESH_COARSE0:
                if (!(pf->elide_w0 && w == 0 && o.phase == 1)) level_refresh(C, 0, 1, st);
                break;
            case OP_SWEEP_COARSE: level_sweep(C, dt, o.arg ? pf->d_tau : nullptr, st); break;
            case OP_SEND_COARSE: send(w, lc, o.phase, o.iter, st_ptr(C, pf->mc - 1), pf->Kc); break;
            case OP_INTERP_STATES: pair_interp_states(pf->pair, st); break;
            case OP_REFRESH_FINE_ALL: level_refresh(F, 0, pf->mf, st); break;
            case OP_RESIDUAL:
                if (res_fused) {  // computed by the preceding sweep's last kernel
                    res_fused = false;
                    break;
                }
                level_residual(F, dt, pf->d_res + (size_t)w * (N + 1) + o.arg, st);
                break;
            case OP_SWEEP_FINE: {
                double* r = nullptr;
                if (fuse_res && i + 1 < ops.size() && ops[i + 1].code == OP_RESIDUAL)
                    r = pf->d_res + (size_t)w * (N + 1) + ops[i + 1].arg;
                level_sweep(F, dt, nullptr, st, r);
                res_fused = r != nullptr;
                break;
            }
            case OP_SEND_FINE: send(w, 0, o.phase, o.iter, st_ptr(F, pf->mf - 1), pf->Kf); break;
            case OP_RESTRICT: pair_restrict_states(pf->pair, st); break;
            case OP_REFRESH_COARSE_ALL: level_refresh(C, 0, pf->mc, st); break;
            case OP_SAVE: pair_save(pf->pair, st); break;
            case OP_FAS: pair_fas(pf->pair, dt, pf->d_tau, st); break;
            case OP_INTERP_INC: pair_interp_increment_add(pf->pair, pf->d_dstate0, st, true); break;
            case OP_RECV_FINE_IC: recv(w, 0, o.phase, o.iter, st_ptr(F, 0), pf->Kf); break;
            case OP_REFRESH_FINE0:
                if (!(pf->elide_w0 && w == 0)) level_refresh(F, 0, 1, st);
                break;
            case OP_INTERP_STATES_MC: pair_interp_states(pf->pair2, st); break;
            case OP_REFRESH_MID_ALL: level_refresh(M, 0, pf->mm, st); break;
            case OP_RESTRICT_MC: pair_restrict_states(pf->pair2, st); break;
            case OP_SAVE_MC: pair_save(pf->pair2, st); break;
            case OP_FAS_MC: pair_fas(pf->pair2, dt, pf->d_tau, st, pf->d_tau_mid); break;
            case OP_SWEEP_MID: level_sweep(M, dt, pf->d_tau_mid, st); break;
            case OP_SEND_MID: send(w, 1, o.phase, o.iter, st_ptr(M, pf->mm - 1), pf->Km); break;
            case OP_INTERP_INC_MC: pair_interp_increment_add(pf->pair2, pf->d_dstate0_mid, st, true); break;
            case OP_RECV_MID_IC: recv(w, 1, o.phase, o.iter, st_ptr(M, 0), pf->Km); break;
            case OP_REFRESH_MID0:
                if (!(pf->elide_w0 && w == 0)) level_refresh(M, 0, 1, st);
                break;
            case OP_FAS_FM: pair_fas(pf->pair, dt, pf->d_tau_mid, st); break;
            default: throw std::logic_error("pfasst: unknown op");
        }
    }
    if (seg) seg->close();
}

__global__ void add_state_kernel(double2* dst, const double2* a, const double2* b, long n) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = make_double2(a[i].x + b[i].x, a[i].y + b[i].y);
}

// Node-0 update after the IC receive (pfasst.cpp:171-174). Two levels: the received state + the
// receiver's own interpolated node-0 increment (the reference's form). Three levels:
//   * PSWE_NODE0_REFERENCE — the same additive form on every level, generalised so that a level
//     adds only the correction that came from the COARSEST level: mid node 0 := recv + dstate0_mid
//     (the node-0 part of the coarse increment interpolated into the mid level), fine node 0 :=
//     recv + interpolate_space(dstate0_mid). With a degenerate chain (mid level = fine level, no
//     mid sweeps) this is exactly the two-level reference (tests/test_gpu_pfasst3.py);
//   * PSWE_NODE0_LOWMODE (default) — low-mode replacement, below.
bool node0_additive(const pswe_pfasst* pf) { return pf->nlev == 2 || pf->node0 == PSWE_NODE0_REFERENCE; }
bool has_dstate(const pswe_pfasst* pf, int level) { return node0_additive(pf) && level <= pf->nlev - 2; }
// three-level reference form: the fine IC's increment is the coarse correction's node-0 part,
// carried up from the mid level
void prepare_dstate(pswe_pfasst* pf, int level, cudaStream_t st) {
    if (pf->nlev == 3 && level == 0 && node0_additive(pf))
        if (pswe_interpolate_space(pf->Rm, pf->Rf, reinterpret_cast<const double*>(pf->d_dstate0_mid),
                                   reinterpret_cast<double*>(pf->d_dstate0), 1, st) != 0)
            throw std::runtime_error(pswe_last_error());
}

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
bool has_low_replace(const pswe_pfasst* pf, int level) { return !node0_additive(pf) && level <= 1; }
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
        prepare_dstate(pf, level, st);
        if (has_dstate(pf, level)) add_dstate0(pf, dst, m.buf, st, level);
        else PSWE_CUDA(cudaMemcpyAsync(dst, m.buf, state_bytes(K), cudaMemcpyDeviceToDevice, st));
        if (has_low_replace(pf, level)) replace_low_modes(pf, level, dst, st);
        pf->pool[level].push_back(m.buf);  // stream-ordered reuse
    };
    for (int w = 0; w < pf->cfg.n_time_steps; ++w) {
        run_worker(pf, w, theta0, st, send, recv);
        // BlockResult.step_final[w] (pfasst.cpp:238-241): the workers share the levels in turn
        PSWE_CUDA(cudaMemcpyAsync(pf->d_step_final + (size_t)w * 3 * pf->Kf, st_ptr(pf->fine, pf->mf - 1),
                                  state_bytes(pf->Kf), cudaMemcpyDeviceToDevice, st));
    }
}

void run_dist(pswe_pfasst* pf, const double2* theta0, cudaStream_t st, SegCtl* seg = nullptr) {
    Transport& T = *pf->tr;
    const int w = pf->rank;
    auto tag_of = [&](int level, int phase, int iter, int sender, unsigned long long seq) {
        MsgTag t{};
        t.magic = kMsgMagic;
        t.phase = phase;
        t.iter = iter;
        t.level = level;
        t.sender = sender;
        t.seq_lo = (int)(seq & 0xffffffffu);
        t.seq_hi = (int)(seq >> 32);
        return t;
    };
    auto send = [&](int, int level, int phase, int iter, const double2* src, long) {
        const unsigned long long k = pf->sseq[level]++;
        // fault injection (tests): the first iteration message carries the wrong iteration
        const int skew = (pf->fault == 1 && phase == 1 && iter == 1) ? 1 : 0;
        T.send(level, k, src, tag_of(level, phase, iter + skew, w, k), st);
    };
    auto recv = [&](int, int level, int phase, int iter, double2* dst, long K) {
        const unsigned long long k = pf->rseq[level]++;
        const double2* slot = T.recv(level, k, st);
        prepare_dstate(pf, level, st);
        // copy into place (+ the receiver's node-0 increment for the two-level fine IC,
        // pfasst.cpp:171-174) and check the trailer (pfasst.cpp:71-76) in one kernel
        consume_message(dst, slot, has_dstate(pf, level) ? (level ? pf->d_dstate0_mid : pf->d_dstate0) : nullptr,
                        3 * K, tag_of(level, phase, iter, w - 1, k), pf->d_err, st);
        if (has_low_replace(pf, level)) replace_low_modes(pf, level, dst, st);
    };
    try {
        run_worker(pf, w, theta0, st, send, recv, seg);
    } catch (...) {
        if (seg) seg->abort_capture();
        throw;
    }
}

void check_tags(pswe_pfasst* pf) {
    if (!pf->h_err || !pf->h_err->flag) return;
    const TagError e = *pf->h_err;
    std::memset(pf->h_err, 0, sizeof(TagError));
    throw std::logic_error("pfasst: message tag mismatch (received phase " + std::to_string(e.phase) + " iteration " +
                           std::to_string(e.iter) + " level " + std::to_string(e.level) + " from worker " +
                           std::to_string(e.sender) + ", expected phase " + std::to_string(e.want_phase) +
                           " iteration " + std::to_string(e.want_iter) + " level " + std::to_string(e.want_level) + ")");
}

}  // namespace

extern "C" {

static void create_serial(pswe_pair* pair, pswe_pair* pair2, const pswe_block_config* cfg, pswe_pfasst** out) {
    if (!out) throw std::invalid_argument("out is NULL");
    auto* pf = new pswe_pfasst;
    if (const char* e = std::getenv("PSWE_NO_GRAPH")) pf->use_graph = std::atoi(e) == 0;
    if (const char* e = std::getenv("PSWE_PFASST_NO_ELIDE")) pf->elide_w0 = std::atoi(e) == 0;
    try {
        init_common(pf, pair, cfg, pair2);
        PSWE_CUDA(cudaMalloc(&pf->d_step_final, pf->cfg.n_time_steps * state_bytes(pf->Kf)));
    } catch (...) {
        pswe_pfasst_destroy(pf);
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

int pswe_transport_unique_id(int transport, void* out128) {
    return guarded([&] {
        if (!out128) throw std::invalid_argument("NULL argument");
        if (transport == PSWE_TRANSPORT_IPC) ipc_unique_id(out128);
        else if (transport == PSWE_TRANSPORT_NCCL) nccl_unique_id(out128);
        else throw std::invalid_argument("pswe_transport_unique_id: unknown transport");
    });
}

int pswe_nccl_unique_id(void* out128) { return pswe_transport_unique_id(PSWE_TRANSPORT_NCCL, out128); }

static void create_dist(pswe_pair* pair, pswe_pair* pair2, const pswe_block_config* cfg, int rank, int world,
                        int transport, const void* uid, pswe_pfasst** out) {
    if (!out || !uid) throw std::invalid_argument("NULL argument");
    if (!cfg) throw std::invalid_argument("pswe_pfasst: NULL argument");
    if (cfg->n_time_steps != world)
        throw std::invalid_argument("pswe_pfasst_create_dist: n_time_steps must equal world size");
    if (rank < 0 || rank >= world) throw std::invalid_argument("pswe_pfasst_create_dist: rank out of range");
    std::unique_ptr<pswe_pfasst> pf(new pswe_pfasst);
    try {
        init_common(pf.get(), pair, cfg, pair2);
        pf->distributed = true;
        pf->rank = rank;
        pf->world = world;
        if (const char* e = std::getenv("PSWE_RECV_TIMEOUT")) pf->recv_timeout = std::atof(e);
        if (const char* e = std::getenv("PSWE_PFASST_NO_ELIDE")) pf->elide_w0 = std::atoi(e) == 0;
        if (const char* e = std::getenv("PSWE_PFASST_FAULT")) pf->fault = std::atoi(e);
        PSWE_CUDA(cudaHostAlloc(&pf->h_err, sizeof(TagError), cudaHostAllocMapped));
        std::memset(pf->h_err, 0, sizeof(TagError));
        PSWE_CUDA(cudaHostGetDevicePointer(&pf->d_err, pf->h_err, 0));
        TransportConfig tc;
        tc.rank = rank;
        tc.world = world;
        tc.nlev = pf->nlev;
        for (int l = 0; l < pf->nlev; ++l) tc.K[l] = pf->K_of(l);
        // messages per level and receiver within one block: fine / mid <= n_iter - 1, coarse
        // <= world + n_iter - 1 (prediction rounds + Step C); slots are reused only in the next
        // block, after the block-end synchronisation
        tc.slots = world + cfg->n_iter + 1;
        tc.Kfinal = pf->Kf;
        tc.n_res = cfg->n_iter + 1;
        tc.timeout_s = pf->recv_timeout;
        pf->tr = transport == PSWE_TRANSPORT_IPC ? make_ipc_transport(tc, uid) : make_nccl_transport(tc, uid);
    } catch (...) {
        pswe_pfasst_destroy(pf.release());
        throw;
    }
    *out = pf.release();
}

int pswe_pfasst_create_dist(pswe_pair* pair, pswe_pair* mid_coarse, const pswe_block_config* cfg, int rank,
                            int world, int transport, const void* unique_id, pswe_pfasst** out) {
    return guarded([&] {
        if (transport != PSWE_TRANSPORT_IPC && transport != PSWE_TRANSPORT_NCCL)
            throw std::invalid_argument("pswe_pfasst_create_dist: unknown transport");
        create_dist(pair, mid_coarse, cfg, rank, world, transport, unique_id, out);
    });
}

int pswe_pfasst_create_nccl(pswe_pair* pair, const pswe_block_config* cfg, int rank, int world,
                            const void* uid, pswe_pfasst** out) {
    return guarded([&] { create_dist(pair, nullptr, cfg, rank, world, PSWE_TRANSPORT_NCCL, uid, out); });
}

int pswe_pfasst3_create_nccl(pswe_pair* fine_mid, pswe_pair* mid_coarse, const pswe_block_config* cfg, int rank,
                             int world, const void* uid, pswe_pfasst** out) {
    return guarded([&] {
        if (!mid_coarse) throw std::invalid_argument("pswe_pfasst3: NULL mid-coarse pair");
        create_dist(fine_mid, mid_coarse, cfg, rank, world, PSWE_TRANSPORT_NCCL, uid, out);
    });
}

int pswe_pfasst3_configure(pswe_pfasst* pf, int node0_form, int mid_sweeps) {
    return guarded([&] {
        if (!pf) throw std::invalid_argument("NULL argument");
        if (pf->nlev != 3) throw std::invalid_argument("pswe_pfasst3_configure: not a three-level controller");
        if (node0_form != PSWE_NODE0_LOWMODE && node0_form != PSWE_NODE0_REFERENCE)
            throw std::invalid_argument("pswe_pfasst3_configure: unknown node-0 form");
        if (mid_sweeps < 0 || mid_sweeps > 4) throw std::invalid_argument("pswe_pfasst3_configure: mid_sweeps in 0..4");
        pf->node0 = node0_form;
        pf->mid_sweeps = mid_sweeps;
        if (pf->graph) {  // the captured block follows the old schedule
            PSWE_CUDA(cudaGraphExecDestroy(pf->graph));
            pf->graph = nullptr;
            pf->eager_runs = 0;
        }
    });
}

int pswe_pfasst_set_recv_timeout(pswe_pfasst* pf, double seconds) {
    return guarded([&] {
        if (!pf) throw std::invalid_argument("NULL argument");
        if (!(seconds > 0)) throw std::invalid_argument("pswe_pfasst_set_recv_timeout: need seconds > 0");
        pf->recv_timeout = seconds;
        if (pf->tr) pf->tr->timeout_s = seconds;
    });
}

int pswe_pfasst_destroy(pswe_pfasst* pf) {
    return guarded([&] {
        if (!pf) return;
        cudaDeviceSynchronize();
        if (pf->graph) cudaGraphExecDestroy(pf->graph);
        for (auto e : pf->seg_graphs) cudaGraphExecDestroy(e);
        if (pf->d_theta) cudaFree(pf->d_theta);
        if (pf->gstream) cudaStreamDestroy(pf->gstream);
        if (pf->ev_in) cudaEventDestroy(pf->ev_in);
        if (pf->ev_out) cudaEventDestroy(pf->ev_out);
        if (pf->d_tau) cudaFree(pf->d_tau);
        if (pf->d_dstate0) cudaFree(pf->d_dstate0);
        if (pf->d_tau_mid) cudaFree(pf->d_tau_mid);
        if (pf->d_dstate0_mid) cudaFree(pf->d_dstate0_mid);
        cudaFree(pf->d_res);
        if (pf->d_step_final) cudaFree(pf->d_step_final);
        for (int l = 0; l < 3; ++l)
            for (auto* b : pf->pool[l]) cudaFree(b);
        for (auto& q : pf->queues)
            for (auto& m : q.second) cudaFree(m.buf);
        pf->tr.reset();
        if (pf->h_err) cudaFreeHost(pf->h_err);
        delete pf;
    });
}

// One serial-emulation block on stream st: theta0 -> pf->d_res (residuals, device), final_state /
// step_final (device, optional). No host synchronisation. final_state may alias theta0 (theta0 is
// consumed before final_state is written: graph path copies it first, eager path reads it during
// the block and final_state is written last).
static void serial_block(pswe_pfasst* pf, const double2* th, double* step_final, double* final_state,
                         cudaStream_t st) {
    const int n = pf->cfg.n_time_steps, N = pf->cfg.n_iter;
    PSWE_CUDA(cudaMemsetAsync(pf->d_res, 0, sizeof(double) * n * (N + 1), st));
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
    if (step_final)
        PSWE_CUDA(cudaMemcpyAsync(step_final, pf->d_step_final, n * state_bytes(pf->Kf),
                                  cudaMemcpyDeviceToDevice, st));
}

int pswe_pfasst_run_block_steps(pswe_pfasst* pf, const double* theta0, double* step_final, double* final_state,
                                double* residuals, void* stream) {
    return guarded([&] {
        PSWE_NVTX("pswe.pfasst.run_block");
        if (!pf || !theta0) throw std::invalid_argument("NULL argument");
        if (pf->broken) throw std::runtime_error("pfasst: a previous block failed; destroy and recreate the controller");
        const cudaStream_t st = as_stream(stream);
        const double2* th = reinterpret_cast<const double2*>(theta0);
        const int n = pf->cfg.n_time_steps, N = pf->cfg.n_iter;
        if (!pf->distributed) {
            serial_block(pf, th, step_final, final_state, st);
            if (residuals) {
                PSWE_CUDA(cudaMemcpyAsync(residuals, pf->d_res, sizeof(double) * n * (N + 1), cudaMemcpyDeviceToHost, st));
                PSWE_CUDA(cudaStreamSynchronize(st));
            }
        } else {
            PSWE_CUDA(cudaMemsetAsync(pf->d_res, 0, sizeof(double) * n * (N + 1), st));
            // BlockResult: the last step's final state goes to every rank (next block's theta0,
            // runner.cpp:145-147), step_final (optional) gathers every rank's, residual rows are
            // gathered everywhere; end_block bounds every wait by the receive timeout
            std::vector<double> all((size_t)n * (N + 1));
            try {
                if (pf->use_graph) {
                    // segment graphs on an internal stream (the caller's may be the legacy stream),
                    // ordered after / before the caller's stream; theta0 copied to a fixed buffer
                    if (!pf->d_theta) {
                        PSWE_CUDA(cudaMalloc(&pf->d_theta, state_bytes(pf->Kf)));
                        PSWE_CUDA(cudaStreamCreateWithFlags(&pf->gstream, cudaStreamNonBlocking));
                        PSWE_CUDA(cudaEventCreateWithFlags(&pf->ev_in, cudaEventDisableTiming));
                        PSWE_CUDA(cudaEventCreateWithFlags(&pf->ev_out, cudaEventDisableTiming));
                    }
                    const unsigned long long gen = plans_generation(pf);
                    if (!pf->seg_graphs.empty() && gen != pf->seg_gen) {
                        for (auto e : pf->seg_graphs) cudaGraphExecDestroy(e);
                        pf->seg_graphs.clear();
                        pf->dist_runs = 0;
                    }
                    PSWE_CUDA(cudaMemcpyAsync(pf->d_theta, th, state_bytes(pf->Kf), cudaMemcpyDeviceToDevice, st));
                    PSWE_CUDA(cudaEventRecord(pf->ev_in, st));
                    PSWE_CUDA(cudaStreamWaitEvent(pf->gstream, pf->ev_in, 0));
                    SegCtl seg;
                    seg.graphs = &pf->seg_graphs;
                    seg.st = pf->gstream;
                    seg.mode = !pf->seg_graphs.empty() ? SegCtl::REPLAY
                                                       : (pf->dist_runs >= 1 ? SegCtl::CAPTURE : SegCtl::EAGER);
                    run_dist(pf, pf->d_theta, pf->gstream, &seg);
                    if (seg.mode == SegCtl::CAPTURE) pf->seg_gen = plans_generation(pf);
                    ++pf->dist_runs;
                    PSWE_CUDA(cudaEventRecord(pf->ev_out, pf->gstream));
                    PSWE_CUDA(cudaStreamWaitEvent(st, pf->ev_out, 0));
                } else {
                    run_dist(pf, th, st);
                }
                // tags first: a mismatch must abort the block before the block-end barrier, so
                // the peers stop (and stop touching this rank's buffers) instead of going on
                pf->tr->drain(st);
                check_tags(pf);
                pf->tr->end_block(st_ptr(pf->fine, pf->mf - 1), reinterpret_cast<double2*>(final_state),
                                  reinterpret_cast<double2*>(step_final), pf->d_res + (size_t)pf->rank * (N + 1),
                                  all.data(), st);
            } catch (const std::exception& e) {
                pf->broken = true;
                pf->tr->abort(e.what(), pf->use_graph && pf->gstream ? pf->gstream : st);
                throw;
            }
            if (residuals) std::memcpy(residuals, all.data(), sizeof(double) * all.size());
        }
    });
}

// runner.cpp:145-151: n_blocks blocks chained (block b's theta0 = block b-1's final state). Serial
// emulation: everything is enqueued on the stream without a host synchronisation; residuals
// (device, n_blocks * n_time_steps * (n_iter+1)) are valid once the stream has been synchronised.
// Distributed: one host-synchronising block at a time (the block end gathers over the ranks).
int pswe_pfasst_run_blocks(pswe_pfasst* pf, const double* theta0, int n_blocks, double* final_state,
                           double* residuals_dev, void* stream) {
    return guarded([&] {
        PSWE_NVTX("pswe.pfasst.run_blocks");
        if (!pf || !theta0 || !final_state || n_blocks < 0) throw std::invalid_argument("NULL argument");
        if (pf->broken) throw std::runtime_error("pfasst: a previous block failed; destroy and recreate the controller");
        const cudaStream_t st = as_stream(stream);
        const int n = pf->cfg.n_time_steps, N = pf->cfg.n_iter;
        const size_t rb = sizeof(double) * n * (N + 1);
        const double* th = theta0;
        std::vector<double> host(pf->distributed ? (size_t)n * (N + 1) : 0);
        for (int b = 0; b < n_blocks; ++b) {
            if (!pf->distributed) {
                serial_block(pf, reinterpret_cast<const double2*>(th), nullptr, final_state, st);
                if (residuals_dev)
                    PSWE_CUDA(cudaMemcpyAsync(residuals_dev + (size_t)b * n * (N + 1), pf->d_res, rb,
                                              cudaMemcpyDeviceToDevice, st));
            } else {
                if (pswe_pfasst_run_block_steps(pf, th, nullptr, final_state, host.data(), stream))
                    throw std::runtime_error(pswe_last_error());
                if (residuals_dev)
                    PSWE_CUDA(cudaMemcpy(residuals_dev + (size_t)b * n * (N + 1), host.data(), rb,
                                         cudaMemcpyHostToDevice));
            }
            th = final_state;
        }
    });
}

int pswe_pfasst_run_block(pswe_pfasst* pf, const double* theta0, double* final_state, double* residuals,
                          void* stream) {
    return pswe_pfasst_run_block_steps(pf, theta0, nullptr, final_state, residuals, stream);
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
    const auto ops = build_schedule(w, n_time_steps, n_iter, n_levels, 1);
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
