/*
 * pswe.h — C ABI of the B200-native PFASST-SH hot path (libpswe.so, sm_100a, fp64).
 *
 * Drop-in boundary for the reference's plugin/operator interface (reference paths relative to
 * /root/reference/proj):
 *   TransformPlan                include/pintswe/transform.hpp:27-96   -> pswe_plan_* / pswe_synthesise ...
 *   ImexOde / SweOde             include/pintswe/swe.hpp:44-79         -> pswe_eval_* / pswe_solve_implicit
 *   sdc::SpaceTimeState + sweep  include/pintswe/sdc.hpp:14-45         -> pswe_level_* / pswe_sweep ...
 *   ml::TransferPair + transfers include/pintswe/multilevel.hpp:29-80  -> pswe_pair_* / pswe_restrict_states ...
 *   pf::run_block                include/pintswe/pfasst.hpp:51-56      -> pswe_pfasst_* (host C++ controller)
 * The reference passes host std::vector<complex<double>> by value; this ABI keeps states resident
 * on the device (plain device pointers, explicit cudaStream_t passed as void*), which is why the
 * boundary sits at the sweeper level rather than at ImexOde.
 *
 * Layouts (identical to the reference's, field.hpp:14-111 and grid.hpp:14-37):
 *   spectral field : K = (R+1)(R+2)/2 complex fp64, interleaved (re, im), r-major:
 *                    index(r, s) = r(2R+3-r)/2 + (s-r), 0 <= r <= s <= R.
 *   state          : 3 consecutive fields (Phi, zeta, delta) = 3K complex.
 *   grid field     : nlat x nlon fp64, row-major, rows south -> north at the Gauss latitudes,
 *                    lambda_j = 2 pi j / nlon.
 * Batches are consecutive (n fields / n states / n grids back to back).
 *
 * Errors: every int-returning entry point returns 0 on success, nonzero on failure, and
 * pswe_last_error() (thread-local) describes it — the C translation of the reference's
 * std::invalid_argument / std::runtime_error / std::logic_error (transform.cpp:49,137,156,178,228;
 * multilevel.cpp:38-43; pfasst.cpp:43,74). Handles are not thread-safe; use one host thread per
 * handle (one per GPU rank).
 */
#ifndef PSWE_H
#define PSWE_H

#ifdef __cplusplus
extern "C" {
#endif

#define PSWE_ABI_VERSION 1

/* Associated-Legendre strategy ("streamed from HBM or recomputed on the fly"). */
#define PSWE_LEGENDRE_RECOMPUTE 0 /* recurrence in registers/shared memory; no table */
#define PSWE_LEGENDRE_STREAM 1    /* both contractions stream a P table kept in HBM (bulk-copied tiles) */

typedef struct pswe_plan pswe_plan;     /* TransformPlan (transform.hpp:27) on one GPU */
typedef struct pswe_level pswe_level;   /* LevelSpec + SpaceTimeState (multilevel.hpp:16, sdc.hpp:14) */
typedef struct pswe_pair pswe_pair;     /* TransferPair (multilevel.hpp:29) */

/* ModelParams (swe.hpp:13-19). */
typedef struct pswe_params {
    double radius;  /* a, m */
    double omega;   /* rotation rate, 1/s */
    double gravity; /* g, m/s^2 */
    double phi_bar; /* mean geopotential g*hbar, m^2/s^2 */
    double nu;      /* diffusion, m^2/s */
} pswe_params;

const char* pswe_last_error(void);
int pswe_abi_version(void);

/* ---- device memory / stream helpers for hosts without CUDA bindings (cgo, JNI, ctypes) */
int pswe_device_alloc(unsigned long long bytes, void** out);
int pswe_device_free(void* ptr);
int pswe_memcpy_h2d(void* dst, const void* src, unsigned long long bytes, void* stream); /* async */
int pswe_memcpy_d2h(void* dst, const void* src, unsigned long long bytes, void* stream); /* async */
int pswe_stream_synchronize(void* stream);

/* ---- host-side numerical setup (gauss.cpp:24-50, transform.cpp:38-43, quadrature.cpp:74-106) */
int pswe_dealiased_nlon(int truncation);
int pswe_gauss_latitudes(int n, double* mu, double* weight);
/* nodes[n], q/q_exp/q_imp [n*n] row-major; n in {2, 3, 5} */
int pswe_quadrature_tables(int num_nodes, double* nodes, double* q, double* q_exp, double* q_imp);

/* ---- TransformPlan: TransformPlan(int) ctor (transform.cpp:45-89). nlat = nlon = 0 selects the
 * reference's dealiased grid; otherwise an explicit Gaussian grid (nlat even, nlon even,
 * nlon/2 5-smooth, nlon > 2R). */
int pswe_plan_create(int truncation, int nlat, int nlon, int legendre_mode, pswe_plan** out);
int pswe_plan_destroy(pswe_plan* plan);
int pswe_plan_info(const pswe_plan* plan, int* truncation, int* nlat, int* nlon, int* legendre_mode);
int pswe_plan_latitudes(const pswe_plan* plan, double* mu, double* weight);
/* Pre-size the device scratch for batches of up to n states / n fields (avoids cudaMalloc in
 * the first call and inside CUDA-graph capture). */
int pswe_plan_reserve(pswe_plan* plan, int max_batch);

/* ---- transforms (transform.hpp:54-72); all pointers are device pointers */
int pswe_synthesise(pswe_plan* plan, const double* coeffs, double* grid, int n_fields, void* stream);
int pswe_analyse(pswe_plan* plan, const double* grid, double* coeffs, int n_fields, void* stream);
int pswe_uv_from_vortdiv(pswe_plan* plan, const double* vort, const double* div, double radius,
                         double* u, double* v, int n_pairs, void* stream);
int pswe_vortdiv_from_uv(pswe_plan* plan, const double* u, const double* v, double radius,
                         double* vort, double* div, int n_pairs, void* stream);
/* laplacian / inv_laplacian (transform.cpp:272-290) on n fields */
int pswe_laplacian(int truncation, const double* x, double radius, double* y, int n_fields, int inverse,
                   void* stream);

/* ---- ImexOde / SweOde (swe.hpp:44-79, swe.cpp:9-98); n_states states back to back */
int pswe_eval_explicit(pswe_plan* plan, const pswe_params* p, const double* state, double* f_exp,
                       int n_states, void* stream);
int pswe_eval_implicit(int truncation, const pswe_params* p, const double* state, double* f_imp,
                       int n_states, void* stream);
/* eval_implicit + eval_explicit of the same states in one pass (refresh_node, sdc.cpp:15-18) */
int pswe_eval_imex(pswe_plan* plan, const pswe_params* p, const double* state, double* f_imp,
                   double* f_exp, int n_states, void* stream);
int pswe_solve_implicit(int truncation, const pswe_params* p, const double* b, double c, double* out,
                        int n_states, void* stream);
/* pswe_eval_imex with CUDA events between its four kernels; synchronises `stream` and writes the
 * per-kernel device times in ms to ms_out[4] (inverse Legendre, FFT+products, forward Legendre,
 * tail). Measurement aid for the roofline. */
int pswe_eval_imex_timed(pswe_plan* plan, const pswe_params* p, const double* state, double* f_imp,
                         double* f_exp, int n_states, void* stream, float* ms_out);
/* the same with the inverse stage split into its two kernels: ms_out[5] = coefficient prep,
 * inverse Legendre contraction, FFT+products, forward Legendre, tail (prep = 0 when the
 * recurrence inverse runs: single states on grids above 768 latitudes) */
int pswe_eval_imex_kernel_times(pswe_plan* plan, const pswe_params* p, const double* state, double* f_imp,
                                double* f_exp, int n_states, void* stream, float* ms_out);

/* ---- SDC level: LevelSpec + SpaceTimeState on the device (sdc.hpp:14-45) */
/* num_nodes: 2, 3 or 5 Gauss-Lobatto nodes (quadrature.cpp); any other count is an error */
int pswe_level_create(pswe_plan* plan, const pswe_params* p, int num_nodes, pswe_level** out);
int pswe_level_destroy(pswe_level* lvl);
/* which: 0 = state, 1 = f_imp, 2 = f_exp; returns the device pointer of that node's 3K complex */
double* pswe_level_ptr(pswe_level* lvl, int which, int node);
int pswe_level_info(const pswe_level* lvl, int* truncation, int* num_nodes);
int pswe_spread(pswe_level* lvl, const double* theta0, void* stream);                /* sdc.cpp:7-13 */
int pswe_refresh_nodes(pswe_level* lvl, int first, int count, void* stream);         /* sdc.cpp:15-18 */
/* sdc.cpp:20-49; tau = NULL or num_nodes consecutive coarse states (FAS, added at node m+1) */
int pswe_sweep(pswe_level* lvl, double dt, const double* tau, void* stream);
/* sdc.cpp:51-64: writes the residual (one double) to the DEVICE pointer out */
int pswe_collocation_residual(pswe_level* lvl, double dt, double* out, void* stream);
/* sdc.cpp:66-72: spread + n_sweeps sweeps (+ residual if out_residual != NULL, device pointer);
 * the last-node state stays in the level (pswe_level_ptr(lvl, 0, num_nodes-1)). */
int pswe_sdc_step(pswe_level* lvl, const double* theta0, double dt, int n_sweeps, double* out_residual,
                  void* stream);

/* ---- two-level transfers (multilevel.cpp:37-158) */
int pswe_pair_create(pswe_level* fine, pswe_level* coarse, pswe_pair** out);
int pswe_pair_destroy(pswe_pair* pair);
/* restrict_space / interpolate_space of n states between truncations (multilevel.cpp:53-82) */
int pswe_restrict_space(int rf, int rc, const double* x, double* y, int n_states, void* stream);
int pswe_interpolate_space(int rc, int rf, const double* x, double* y, int n_states, void* stream);
/* coarse.state := restrict_states(fine.state) (multilevel.cpp:100-107) */
int pswe_restrict_states(pswe_pair* pair, void* stream);
/* tau (device, coarse num_nodes states) := fas_correction(fine, coarse) (multilevel.cpp:109-137) */
int pswe_fas_correction(pswe_pair* pair, double dt, double* tau, void* stream);
/* multi-level FAS (Eq. 19): tau := fas_correction(fine, coarse) + R tau_fine,
 * where tau_fine (device, fine num_nodes states, may be NULL) is the fine level's own FAS term
 * (three-level chains; the reference itself is two-level, tau_fine = 0) */
int pswe_fas_correction_ml(pswe_pair* pair, double dt, const double* tau_fine, double* tau, void* stream);
/* save a copy of the coarse space-time state (pfasst.cpp:158) */
int pswe_save_coarse(pswe_pair* pair, void* stream);
/* fine.{state,f_imp,f_exp} += interpolate_increment(coarse - saved) (multilevel.cpp:139-150,
 * pfasst.cpp:177-185); also writes the node-0 state increment to dstate0 (device, may be NULL) */
int pswe_interpolate_increment_add(pswe_pair* pair, double* dstate0, void* stream);
/* fine.state := interpolate_states(coarse.state) (multilevel.cpp:152-158) */
int pswe_interpolate_states(pswe_pair* pair, void* stream);

/* ---- PFASST block controller (pfasst.cpp:78-251), host C++ ---------------------------------
 * A pswe_pfasst runs the worker(s) of one block. Communication between time ranks is
 * pluggable: either in-process (serial emulation of all n_ts workers on this GPU, the
 * reference's Mode::serial_emulation) or through NCCL send/recv between one process per GPU
 * (rank w runs worker w). */
typedef struct pswe_pfasst pswe_pfasst;

typedef struct pswe_block_config {
    int n_time_steps; /* workers per block (BlockConfig, pfasst.hpp:14-20) */
    double dt;
    int n_iter;       /* fixed iteration count N_PF */
} pswe_block_config;

/* Serial emulation: all n_time_steps workers on this device, in worker order. */
int pswe_pfasst_create_serial(pswe_pair* pair, const pswe_block_config* cfg, pswe_pfasst** out);
/* Distributed: this process is worker `rank` of `world`; nccl_unique_id is the 128-byte
 * ncclUniqueId created by rank 0 and shared by the caller (e.g. over torch.distributed). */
int pswe_pfasst_create_nccl(pswe_pair* pair, const pswe_block_config* cfg, int rank, int world,
                            const void* nccl_unique_id, pswe_pfasst** out);
int pswe_nccl_unique_id(void* out128);
/* Distributed controller over a chosen message transport (one process per GPU, rank = worker):
 *   PSWE_TRANSPORT_IPC  — CUDA IPC over peer memory (NVLink/NVSwitch within one node; several
 *                         processes may share one GPU): the sender's kernel writes each message
 *                         into the receiver's ring slot, a POSIX shared-memory segment named by the
 *                         unique id carries counters, handles, a barrier and the abort flag;
 *   PSWE_TRANSPORT_NCCL — ncclSend/ncclRecv (two communicators per level by sender parity).
 * mid_coarse = NULL for two levels. unique_id: 128 bytes from pswe_transport_unique_id on rank 0,
 * shared by the caller. Every message carries a (phase, iteration, level, sender, sequence) tag
 * checked on receipt ("pfasst: message tag mismatch", pfasst.cpp:71-76); every wait is bounded by
 * the receive timeout (BlockConfig::recv_timeout_seconds, pfasst.hpp:19; default 300 s, env
 * PSWE_RECV_TIMEOUT) and fails with "pfasst: receive timed out, pipeline deadlock suspected"
 * (pfasst.cpp:39-47); a rank whose block fails aborts the block for its peers. */
#define PSWE_TRANSPORT_NCCL 0
#define PSWE_TRANSPORT_IPC 1
int pswe_transport_unique_id(int transport, void* out128);
int pswe_pfasst_create_dist(pswe_pair* pair, pswe_pair* mid_coarse, const pswe_block_config* cfg, int rank,
                            int world, int transport, const void* unique_id, pswe_pfasst** out);
int pswe_pfasst_set_recv_timeout(pswe_pfasst* pf, double seconds);
/* Three-level PFASST (BASELINE config 4; the reference implements two levels only,
 * multilevel.hpp:29-35): fine_mid = (fine, mid), mid_coarse = (mid, coarse) with
 * mid_coarse->fine == fine_mid->coarse. Each iteration is a V-cycle fine -> mid -> coarse -> mid
 * -> fine with the FAS of Eq. 19 on the mid and coarse levels; messages on three levels
 * (0 fine, 1 mid, 2 coarse; step 'M' for the mid down-sweep). */
int pswe_pfasst3_create_serial(pswe_pair* fine_mid, pswe_pair* mid_coarse, const pswe_block_config* cfg,
                               pswe_pfasst** out);
int pswe_pfasst3_create_nccl(pswe_pair* fine_mid, pswe_pair* mid_coarse, const pswe_block_config* cfg, int rank,
                             int world, const void* nccl_unique_id, pswe_pfasst** out);
/* Three-level options. node0_form: how a level's node 0 is updated after its IC receive
 * (pfasst.cpp:171-174 is the two-level rule):
 *   PSWE_NODE0_LOWMODE   (default) received state with its modes <= R of the next coarser level
 *                        replaced by that level's node 0;
 *   PSWE_NODE0_REFERENCE the reference's additive form on every level: received state + the
 *                        node-0 increment of the coarsest correction (interpolated up).
 * mid_sweeps: mid-level sweeps per V-cycle leg (default 1; 0..4). */
#define PSWE_NODE0_LOWMODE 0
#define PSWE_NODE0_REFERENCE 1
int pswe_pfasst3_configure(pswe_pfasst* pf, int node0_form, int mid_sweeps);
int pswe_pfasst_destroy(pswe_pfasst* pf);
/* Runs one block from theta0 (device, fine state). On return:
 *   final_state (device): fine last-node state of the LAST time step of the block (the
 *                         next block's theta0, runner.cpp:145-147) — on every rank;
 *   residuals (host, n_time_steps*(n_iter+1)): BlockResult.residuals (pfasst.hpp:36-40),
 *                         gathered to every rank. */
int pswe_pfasst_run_block(pswe_pfasst* pf, const double* theta0, double* final_state, double* residuals,
                          void* stream);
/* The same with BlockResult.step_final (pfasst.hpp:34-36): step_final (device, n_time_steps
 * states, may be NULL) receives the fine last-node state of every time step of the block. */
int pswe_pfasst_run_block_steps(pswe_pfasst* pf, const double* theta0, double* step_final, double* final_state,
                                double* residuals, void* stream);
/* n_blocks blocks chained as the reference's runner does (runner.cpp:145-151): block b starts from
 * block b-1's final state. final_state (device) receives the last block's; residuals_dev (device,
 * may be NULL) n_blocks * n_time_steps * (n_iter+1) doubles, block-major. Serial emulation runs
 * without any host synchronisation (read the results after synchronising the stream). */
int pswe_pfasst_run_blocks(pswe_pfasst* pf, const double* theta0, int n_blocks, double* final_state,
                           double* residuals_dev, void* stream);
/* Message log of the last block (pfasst.hpp:22-31), 7 ints per record:
 * phase, iteration, step ('B','P','A','C'), sender, receiver, level, node. Returns the count. */
int pswe_pfasst_messages(const pswe_pfasst* pf, int* out, int max_records);
/* The control flow of worker w as data: 4 ints per op (code, phase, iteration, arg), codes as in
 * csrc/pfasst.cpp OpCode (worker_predict / worker_iterate, pfasst.cpp:78-176). Returns the op
 * count; writes at most max_ops ops. Host-only (no device work). */
int pswe_pfasst_schedule(int w, int n_time_steps, int n_iter, int* out, int max_ops);
/* the same for a chain of n_levels = 2 or 3 levels (returns -1 otherwise) */
int pswe_pfasst_schedule_ml(int n_levels, int w, int n_time_steps, int n_iter, int* out, int max_ops);

/* FP64 throughput microbenchmark on the current device (roofline denominator; MEASURED_PEAKS.json
 * has no FP64 figure): use_dmma = 0 -> DFMA, 1 -> DMMA m8n8k4. Returns TFLOP/s (< 0 on error). */
double pswe_fp64_peak(int use_dmma, int iters);

#ifdef __cplusplus
}
#endif

#endif /* PSWE_H */
