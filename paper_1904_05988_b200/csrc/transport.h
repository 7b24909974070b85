// Message transports of the distributed PFASST executor (csrc/pfasst.cpp), one process per GPU.
//
// The reference moves PrognosticState values between worker threads through forward-only
// channels (Channel, proj/src/pfasst.cpp:25-48): sends never block, receives block up to
// BlockConfig::recv_timeout_seconds (pfasst.hpp:19) and throw "pipeline deadlock suspected", and
// every message carries (phase, iteration, level) checked by expect() (pfasst.cpp:71-76).
// Here a message is a device state followed by a 64-byte tag trailer (MsgTag): the sender's
// put/stage kernel writes both, the receiver's consume kernel checks the trailer while it copies
// the state into place and raises a flag the host turns into the reference's logic_error.
//
// Two transports behind one interface:
//   * IpcTransport  — CUDA IPC over peer memory (NVLink / NVSwitch, or the same device): the
//                     sender's put kernel stores the message straight into the receiver's ring
//                     slot and records an interprocess event; a shared-memory segment carries the
//                     posted counters, the exported handles, a barrier and an abort flag. Works
//                     for several processes on ONE GPU too (the world = 2 test): then the receiver
//                     waits on the host (event polling) so no GPU work ever waits on another
//                     process; across GPUs the wait is a stream wait on the event.
//   * NcclTransport — ncclSend / ncclRecv on two communicators per level chosen by sender
//                     parity (send stream / compute stream), warm-up connection at creation,
//                     async-error polling, ncclCommAbort on timeout.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>

namespace pswe {

struct MsgTag {
    int magic, phase, iter, level, sender, seq_lo, seq_hi, step;
    int pad[8];
};
static_assert(sizeof(MsgTag) == 64, "tag trailer is 64 bytes");
constexpr int kMsgMagic = 0x50535745;  // "PSWE"
constexpr size_t kTagBytes = sizeof(MsgTag);

// error word raised by consume kernels (host-mapped pinned memory)
struct TagError {
    int flag;  // 0 = none
    int phase, iter, level, sender;
    int want_phase, want_iter, want_level;
};

// dst[0..n) = slot[0..n) (+ add[0..n) if add), check the trailer after slot[n) against `want`
void consume_message(double2* dst, const double2* slot, const double2* add, long n, const MsgTag& want,
                     TagError* err_dev, cudaStream_t st);
// dst[0..n) = src[0..n), trailer := tag (dst may be peer memory)
void put_message(double2* dst, const double2* src, long n, const MsgTag& tag, cudaStream_t st);

struct TransportConfig {
    int rank = 0, world = 1, nlev = 2;
    long K[3] = {0, 0, 0};  // coefficients per field of each message level
    int slots = 0;          // ring slots per level (>= messages per level per block)
    long Kfinal = 0;        // coefficients per field of the block's final (fine) state
    int n_res = 0;          // residual entries per worker
    double timeout_s = 300.0;
};

class Transport {
public:
    virtual ~Transport() = default;
    virtual const char* name() const = 0;
    // message k (0-based, per level, counted over the transport's lifetime) of `level` to rank+1:
    // copy 3K complex from src and the tag (enqueued on st; never waits for the receiver)
    virtual void send(int level, unsigned long long k, const double2* src, const MsgTag& tag, cudaStream_t st) = 0;
    // message k of `level` from rank-1: returns the device slot (3K complex + trailer) that is
    // valid in stream order on st until the next block
    virtual const double2* recv(int level, unsigned long long k, cudaStream_t st) = 0;
    // end of a block: waits (bounded by the timeout) for st to drain, then
    //   final_state (device, may be NULL) := the last rank's `my_final`,
    //   step_finals (device, may be NULL) := every rank's `my_final` in rank order,
    //   res_all (host, world * n_res) := every rank's d_res_mine (device, n_res)
    virtual void end_block(const double2* my_final, double2* final_state, double2* step_finals,
                           const double* d_res_mine, double* res_all, cudaStream_t st) = 0;
    // wait for st with the deadlock guard (throws "pipeline deadlock suspected" after the timeout)
    virtual void drain(cudaStream_t st) = 0;
    // this rank's block failed: tell the peers (they stop waiting for it), and make sure no GPU
    // work of any rank still targets another rank's buffers before the processes go away
    // (st: the stream this rank's block work was issued on; waits are bounded by the timeout)
    virtual void abort(const std::string& why, cudaStream_t st) = 0;
    double timeout_s = 300.0;
};

std::unique_ptr<Transport> make_ipc_transport(const TransportConfig& c, const void* uid128);
std::unique_ptr<Transport> make_nccl_transport(const TransportConfig& c, const void* uid128);
void ipc_unique_id(void* out128);
void nccl_unique_id(void* out128);

}  // namespace pswe
