// Message transports of the distributed PFASST executor — see transport.h.
//
// Reference behaviour mirrored here (paths relative to /root/reference/proj):
//   * sends never block the sender (Channel::send, src/pfasst.cpp:29-35);
//   * a receive waits at most BlockConfig::recv_timeout_seconds (include/pintswe/pfasst.hpp:19)
//     and then throws "pfasst: receive timed out, pipeline deadlock suspected" (pfasst.cpp:39-47);
//   * every message's (phase, iteration, level) is checked on receipt and a mismatch throws
//     "pfasst: message tag mismatch" (pfasst.cpp:71-76);
//   * a failing worker's exception ends the block for everyone (pfasst.cpp:219-234): here the
//     failing rank raises the shared abort flag (IPC) or aborts its communicators (NCCL) so the
//     peers fail fast instead of waiting for the timeout.
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pswe_internal.h"
#include "transport.h"

namespace pswe {

// ---- message kernels ------------------------------------------------------------------------

__global__ void put_message_kernel(double2* __restrict__ dst, const double2* __restrict__ src, long n, MsgTag tag) {
    const long stride = (long)gridDim.x * blockDim.x;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x < kTagBytes / sizeof(int))
        reinterpret_cast<int*>(dst + n)[threadIdx.x] = reinterpret_cast<const int*>(&tag)[threadIdx.x];
}

__global__ void consume_message_kernel(double2* __restrict__ dst, const double2* __restrict__ slot,
                                       const double2* __restrict__ add, long n, MsgTag want, TagError* err) {
    const long stride = (long)gridDim.x * blockDim.x;
    if (add) {
        for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
            const double2 a = slot[i], b = add[i];
            dst[i] = make_double2(a.x + b.x, a.y + b.y);
        }
    } else {
        for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = slot[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const MsgTag got = *reinterpret_cast<const MsgTag*>(slot + n);
        const bool ok = got.magic == want.magic && got.phase == want.phase && got.iter == want.iter &&
                        got.level == want.level && got.sender == want.sender && got.seq_lo == want.seq_lo &&
                        got.seq_hi == want.seq_hi;
        if (!ok && atomicCAS(&err->flag, 0, 1) == 0) {
            err->phase = got.phase;
            err->iter = got.iter;
            err->level = got.level;
            err->sender = got.magic == want.magic ? got.sender : -1;
            err->want_phase = want.phase;
            err->want_iter = want.iter;
            err->want_level = want.level;
            __threadfence_system();
        }
    }
}

static unsigned copy_blocks(long n) {
    const long b = (n + 255) / 256;
    return (unsigned)(b < 592 ? (b < 1 ? 1 : b) : 592);  // 4 x 148 SMs, grid-stride beyond
}

void put_message(double2* dst, const double2* src, long n, const MsgTag& tag, cudaStream_t st) {
    put_message_kernel<<<copy_blocks(n), 256, 0, st>>>(dst, src, n, tag);
    PSWE_LAUNCH_CHECK();
}

void consume_message(double2* dst, const double2* slot, const double2* add, long n, const MsgTag& want,
                     TagError* err_dev, cudaStream_t st) {
    consume_message_kernel<<<copy_blocks(n), 256, 0, st>>>(dst, slot, add, n, want, err_dev);
    PSWE_LAUNCH_CHECK();
}

namespace {

using Clock = std::chrono::steady_clock;

size_t msg_bytes(long K) { return (size_t)3 * K * sizeof(double2) + kTagBytes; }

[[noreturn]] void throw_timeout() {
    throw std::runtime_error("pfasst: receive timed out, pipeline deadlock suspected");
}

void backoff(int& spins) {
    if (++spins < 2000) return;
    struct timespec ts = {0, spins < 20000 ? 2000 : 50000};
    nanosleep(&ts, nullptr);
}

// waits for stream st with a deadline; `poll` is called between queries (may throw)
template <class Poll>
void drain_stream(cudaStream_t st, double timeout_s, Poll&& poll) {
    const auto deadline = Clock::now() + std::chrono::duration<double>(timeout_s);
    int spins = 0;
    for (;;) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e == cudaSuccess) return;
        if (e != cudaErrorNotReady) PSWE_CUDA(e);
        poll();
        if (Clock::now() > deadline) throw_timeout();
        backoff(spins);
    }
}

}  // namespace

// =============================================================================================
// IPC transport
// =============================================================================================

namespace {

constexpr int kMaxRanks = 64;
constexpr int kMaxSlots = 64;
constexpr int kMaxRes = 64;

struct alignas(64) ShmRank {
    std::atomic<int> ready;
    int device_ordinal;
    char bus_id[32];
    cudaIpcMemHandle_t arena;      // receive rings of this rank, all levels
    cudaIpcMemHandle_t final_buf;  // this rank's step-final state
    cudaIpcEventHandle_t ev_send[3][kMaxSlots];  // recorded by this rank after writing rank+1's slot
    cudaIpcEventHandle_t ev_final;
    alignas(64) std::atomic<unsigned long long> posted[3];  // messages written INTO this rank's rings
    alignas(64) std::atomic<unsigned long long> final_seq;  // blocks whose final this rank published
    std::atomic<int> abort_ack;  // this rank saw the abort and its stream is drained
    double res[kMaxRes];
};

struct ShmSeg {
    std::atomic<int> attached;
    std::atomic<int> abort_rank;  // 1 + rank of the first failing rank, 0 = none
    alignas(64) std::atomic<unsigned long long> barrier;
    int world;
    char why[256];
    ShmRank rank[kMaxRanks];
};

class IpcTransport final : public Transport {
public:
    IpcTransport(const TransportConfig& c, const void* uid) : c_(c) {
        timeout_s = c.timeout_s;
        if (c.world > kMaxRanks) throw std::invalid_argument("pfasst ipc: at most 64 ranks");
        if (c.slots > kMaxSlots) throw std::invalid_argument("pfasst ipc: too many ring slots");
        if (c.n_res > kMaxRes) throw std::invalid_argument("pfasst ipc: too many residual entries");
        char name[129];
        std::memcpy(name, uid, 128);
        name[128] = 0;
        if (name[0] != '/') throw std::invalid_argument("pfasst ipc: bad unique id (use pswe_ipc_unique_id)");
        name_ = name;
        attach();
        PSWE_CUDA(cudaGetDevice(&dev_));
        try {
            setup();
        } catch (...) {
            release();
            throw;
        }
    }
    ~IpcTransport() override { release(); }
    const char* name() const override { return "ipc"; }

    void send(int level, unsigned long long k, const double2* src, const MsgTag& tag, cudaStream_t st) override {
        check_abort();
        const int slot = (int)(k % c_.slots);
        put_message(reinterpret_cast<double2*>(peer_arena_ + off_[level] + slot * mb_[level]), src, 3 * c_.K[level], tag,
                    st);
        PSWE_CUDA(cudaEventRecord(ev_send_[level][slot], st));
        seg_->rank[c_.rank + 1].posted[level].store(k + 1, std::memory_order_release);
    }

    const double2* recv(int level, unsigned long long k, cudaStream_t st) override {
        const int slot = (int)(k % c_.slots);
        auto& posted = seg_->rank[c_.rank].posted[level];
        wait_host([&] { return posted.load(std::memory_order_acquire) >= k + 1; });
        wait_event(ev_recv_[level][slot], st, peer_same_dev_prev_);
        return reinterpret_cast<const double2*>(arena_ + off_[level] + slot * mb_[level]);
    }

    void end_block(const double2* my_final, double2* final_state, double2* step_finals, const double* d_res_mine,
                   double* res_all, cudaStream_t st) override {
        ++block_;
        const size_t fb = (size_t)3 * c_.Kfinal * sizeof(double2);
        PSWE_CUDA(cudaMemcpyAsync(final_, my_final, fb, cudaMemcpyDeviceToDevice, st));
        PSWE_CUDA(cudaEventRecord(ev_final_, st));
        seg_->rank[c_.rank].final_seq.store(block_, std::memory_order_release);
        const int last = c_.world - 1;
        if (final_state) copy_final_from(last, final_state, st);
        if (step_finals)
            for (int r = 0; r < c_.world; ++r) copy_final_from(r, step_finals + (size_t)r * 3 * c_.Kfinal, st);
        drain(st);  // bounded wait; the residual copy below then finds the stream idle
        if (d_res_mine)
            PSWE_CUDA(cudaMemcpyAsync(seg_->rank[c_.rank].res, d_res_mine, sizeof(double) * c_.n_res,
                                      cudaMemcpyDeviceToHost, st));
        PSWE_CUDA(cudaStreamSynchronize(st));
        barrier();  // everyone has read every final and published its residuals
        if (res_all)
            for (int r = 0; r < c_.world; ++r) std::memcpy(res_all + (size_t)r * c_.n_res, seg_->rank[r].res,
                                                            sizeof(double) * c_.n_res);
        barrier();  // residual rows read before anyone publishes the next block's
    }

    void drain(cudaStream_t st) override {
        drain_stream(st, timeout_s, [&] { check_abort(); });
    }

    // Abort handshake: the first failing rank raises the abort word; every rank that sees it
    // (including the initiator) drains its own stream - so none of its put kernels or peer copies
    // is still in flight - and acknowledges; the initiator then waits (bounded) for the acks of
    // its peers before its buffers can go away with the process. A peer that never answers (hung)
    // only delays the initiator by min(timeout, 10 s).
    void abort(const std::string& why, cudaStream_t st) override {
        if (!seg_) return;
        int expected = 0;
        const bool initiator = seg_->abort_rank.compare_exchange_strong(expected, c_.rank + 1);
        if (initiator) std::snprintf(seg_->why, sizeof(seg_->why), "%s", why.c_str());
        const double wait_s = std::min(timeout_s, 10.0);
        try {
            drain_stream(st, wait_s, [] {});
        } catch (...) {  // a stream stuck for the whole bound: acknowledge anyway
        }
        seg_->rank[c_.rank].abort_ack.store(1, std::memory_order_release);
        if (!initiator) return;
        const auto deadline = Clock::now() + std::chrono::duration<double>(wait_s);
        int spins = 0;
        for (;;) {
            bool all = true;
            for (int r = 0; r < c_.world; ++r)
                if (!seg_->rank[r].abort_ack.load(std::memory_order_acquire)) all = false;
            if (all || Clock::now() > deadline) break;
            backoff(spins);
        }
    }

private:
    void attach() {
        const size_t bytes = sizeof(ShmSeg);
        int fd = -1;
        if (c_.rank == 0) {
            fd = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
            if (fd < 0) throw std::runtime_error("pfasst ipc: shm_open(create) failed for " + name_);
            if (ftruncate(fd, (off_t)bytes) != 0) {
                close(fd);
                shm_unlink(name_.c_str());
                throw std::runtime_error("pfasst ipc: ftruncate failed");
            }
            owner_ = true;
        } else {
            const auto deadline = Clock::now() + std::chrono::duration<double>(timeout_s);
            int spins = 0;
            for (;;) {
                fd = shm_open(name_.c_str(), O_RDWR, 0600);
                if (fd >= 0) {
                    struct stat sb;
                    if (fstat(fd, &sb) == 0 && (size_t)sb.st_size >= bytes) break;
                    close(fd);
                    fd = -1;
                }
                if (Clock::now() > deadline) throw std::runtime_error("pfasst ipc: rank 0 never created " + name_);
                backoff(spins);
            }
        }
        void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (p == MAP_FAILED) throw std::runtime_error("pfasst ipc: mmap failed");
        seg_ = static_cast<ShmSeg*>(p);
        if (c_.rank == 0) seg_->world = c_.world;  // fresh segment: zero-filled by ftruncate
    }

    void setup() {
        // receive arena: [level][slot] messages of 3K complex + tag trailer
        size_t total = 0;
        for (int l = 0; l < c_.nlev; ++l) {
            mb_[l] = (msg_bytes(c_.K[l]) + 255) / 256 * 256;
            off_[l] = total;
            total += mb_[l] * c_.slots;
        }
        PSWE_CUDA(cudaMalloc(&arena_, total));
        PSWE_CUDA(cudaMemset(arena_, 0, total));
        PSWE_CUDA(cudaMalloc(&final_, (size_t)3 * c_.Kfinal * sizeof(double2)));
        ShmRank& me = seg_->rank[c_.rank];
        PSWE_CUDA(cudaIpcGetMemHandle(&me.arena, arena_));
        PSWE_CUDA(cudaIpcGetMemHandle(&me.final_buf, final_));
        const unsigned evf = cudaEventInterprocess | cudaEventDisableTiming;
        for (int l = 0; l < c_.nlev; ++l)
            for (int s = 0; s < c_.slots; ++s) {
                PSWE_CUDA(cudaEventCreateWithFlags(&ev_send_[l][s], evf));
                PSWE_CUDA(cudaIpcGetEventHandle(&me.ev_send[l][s], ev_send_[l][s]));
            }
        PSWE_CUDA(cudaEventCreateWithFlags(&ev_final_, evf));
        PSWE_CUDA(cudaIpcGetEventHandle(&me.ev_final, ev_final_));
        me.device_ordinal = dev_;
        PSWE_CUDA(cudaDeviceGetPCIBusId(me.bus_id, sizeof(me.bus_id), dev_));
        PSWE_CUDA(cudaDeviceSynchronize());
        me.ready.store(1, std::memory_order_release);
        seg_->attached.fetch_add(1);
        // wait for every rank's exports
        wait_host([&] {
            for (int r = 0; r < c_.world; ++r)
                if (!seg_->rank[r].ready.load(std::memory_order_acquire)) return false;
            return true;
        });
        if (owner_) shm_unlink(name_.c_str());  // every rank has it mapped
        unlinked_ = true;
        peer_same_.assign(c_.world, false);
        for (int r = 0; r < c_.world; ++r) peer_same_[r] = std::strcmp(seg_->rank[r].bus_id, me.bus_id) == 0;
        // the next rank's receive rings (we write them), the previous rank's send events (we
        // wait on them), every rank's final buffer and event
        if (c_.rank + 1 < c_.world) {
            void* p = nullptr;
            PSWE_CUDA(cudaIpcOpenMemHandle(&p, seg_->rank[c_.rank + 1].arena, cudaIpcMemLazyEnablePeerAccess));
            peer_arena_ = static_cast<char*>(p);
        }
        if (c_.rank > 0) {
            peer_same_dev_prev_ = peer_same_[c_.rank - 1];
            for (int l = 0; l < c_.nlev; ++l)
                for (int s = 0; s < c_.slots; ++s)
                    PSWE_CUDA(cudaIpcOpenEventHandle(&ev_recv_[l][s], seg_->rank[c_.rank - 1].ev_send[l][s]));
        }
        peer_final_.assign(c_.world, nullptr);
        peer_ev_final_.assign(c_.world, nullptr);
        for (int r = 0; r < c_.world; ++r) {
            if (r == c_.rank) {
                peer_final_[r] = final_;
                peer_ev_final_[r] = ev_final_;
                continue;
            }
            void* p = nullptr;
            PSWE_CUDA(cudaIpcOpenMemHandle(&p, seg_->rank[r].final_buf, cudaIpcMemLazyEnablePeerAccess));
            peer_final_[r] = static_cast<double2*>(p);
            PSWE_CUDA(cudaIpcOpenEventHandle(&peer_ev_final_[r], seg_->rank[r].ev_final));
        }
        barrier();  // nobody starts sending before every peer has opened its handles
    }

    void release() {
        for (int r = 0; r < (int)peer_final_.size(); ++r)
            if (r != c_.rank && peer_final_[r]) cudaIpcCloseMemHandle(peer_final_[r]);
        for (int r = 0; r < (int)peer_ev_final_.size(); ++r)
            if (r != c_.rank && peer_ev_final_[r]) cudaEventDestroy(peer_ev_final_[r]);
        if (peer_arena_) cudaIpcCloseMemHandle(peer_arena_);
        for (int l = 0; l < 3; ++l)
            for (int s = 0; s < kMaxSlots; ++s) {
                if (ev_send_[l][s]) cudaEventDestroy(ev_send_[l][s]);
                if (ev_recv_[l][s]) cudaEventDestroy(ev_recv_[l][s]);
            }
        if (ev_final_) cudaEventDestroy(ev_final_);
        if (arena_) cudaFree(arena_);
        if (final_) cudaFree(final_);
        if (owner_ && !unlinked_) shm_unlink(name_.c_str());
        if (seg_) munmap(seg_, sizeof(ShmSeg));
        seg_ = nullptr;
    }

    void check_abort() {
        const int a = seg_->abort_rank.load(std::memory_order_acquire);
        if (a != 0 && a != c_.rank + 1)
            throw std::runtime_error("pfasst: worker " + std::to_string(a - 1) + " failed (" + seg_->why +
                                     "); block aborted");
    }

    template <class Pred>
    void wait_host(Pred&& ready) {
        const auto deadline = Clock::now() + std::chrono::duration<double>(timeout_s);
        int spins = 0;
        while (!ready()) {
            check_abort();
            if (Clock::now() > deadline) throw_timeout();
            backoff(spins);
        }
    }

    // make st wait for ev: a GPU-side stream wait across devices; on the same device the host
    // polls the event first (no GPU work of this process ever waits on another process's work)
    void wait_event(cudaEvent_t ev, cudaStream_t st, bool same_device) {
        if (same_device) {
            wait_host([&] {
                const cudaError_t e = cudaEventQuery(ev);
                if (e == cudaSuccess) return true;
                if (e != cudaErrorNotReady) PSWE_CUDA(e);
                return false;
            });
        } else {
            PSWE_CUDA(cudaStreamWaitEvent(st, ev, 0));
        }
    }

    void copy_final_from(int r, double2* dst, cudaStream_t st) {
        const size_t fb = (size_t)3 * c_.Kfinal * sizeof(double2);
        if (r != c_.rank) {
            auto& seq = seg_->rank[r].final_seq;
            wait_host([&] { return seq.load(std::memory_order_acquire) >= block_; });
            wait_event(peer_ev_final_[r], st, peer_same_[r]);
        }
        PSWE_CUDA(cudaMemcpyAsync(dst, peer_final_[r], fb, cudaMemcpyDefault, st));
    }

    void barrier() {
        const unsigned long long arrived = seg_->barrier.fetch_add(1) + 1;
        const unsigned long long target = ((arrived - 1) / c_.world + 1) * c_.world;
        wait_host([&] { return seg_->barrier.load(std::memory_order_acquire) >= target; });
    }

    TransportConfig c_;
    std::string name_;
    ShmSeg* seg_ = nullptr;
    bool owner_ = false, unlinked_ = false;
    int dev_ = 0;
    char* arena_ = nullptr;
    char* peer_arena_ = nullptr;
    double2* final_ = nullptr;
    size_t mb_[3] = {0, 0, 0}, off_[3] = {0, 0, 0};
    cudaEvent_t ev_send_[3][kMaxSlots] = {};
    cudaEvent_t ev_recv_[3][kMaxSlots] = {};
    cudaEvent_t ev_final_ = nullptr;
    std::vector<double2*> peer_final_;
    std::vector<cudaEvent_t> peer_ev_final_;
    std::vector<bool> peer_same_;
    bool peer_same_dev_prev_ = false;
    unsigned long long block_ = 0;
};

}  // namespace

void ipc_unique_id(void* out128) {
    std::random_device rd;
    char buf[128] = {0};
    std::snprintf(buf, sizeof(buf), "/pswe_ipc_%d_%08x%08x", (int)getpid(), rd(), rd());
    std::memcpy(out128, buf, 128);
}

std::unique_ptr<Transport> make_ipc_transport(const TransportConfig& c, const void* uid128) {
    return std::unique_ptr<Transport>(new IpcTransport(c, uid128));
}

// =============================================================================================
// NCCL transport (resolved with dlopen so libpswe.so loads on machines without NCCL)
// =============================================================================================

namespace {

typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
enum { ncclUint8 = 1, ncclFloat64 = 8 };
typedef int ncclResult_t;
constexpr ncclResult_t ncclInProgress = 7;

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
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
        CommAbort = (decltype(CommAbort))sym("ncclCommAbort");
        CommGetAsyncError = (decltype(CommGetAsyncError))sym("ncclCommGetAsyncError");
        Send = (decltype(Send))sym("ncclSend");
        Recv = (decltype(Recv))sym("ncclRecv");
        Broadcast = (decltype(Broadcast))sym("ncclBroadcast");
        AllGather = (decltype(AllGather))sym("ncclAllGather");
        GetErrorString = (decltype(GetErrorString))sym("ncclGetErrorString");
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != 0 && r != ncclInProgress) throw std::runtime_error(std::string(what) + ": " + GetErrorString(r));
    }
};
NcclApi& nccl() {
    static NcclApi api;
    api.load();
    return api;
}

// Two communicators per message level chosen by sender parity: rank w sends on comm[l][w % 2]
// from its send stream and receives on comm[l][(w + 1) % 2] on the compute stream, so each
// communicator is driven by one stream per rank and a send never blocks the compute pipeline
// (with one blocking channel worker w would wait in Step A's fine send while w+1 waits for Step
// C's coarse message; tests/test_pfasst_schedule.py reproduces that deadlock with gloo).
class NcclTransport final : public Transport {
public:
    NcclTransport(const TransportConfig& c, const void* uid) : c_(c) {
        timeout_s = c.timeout_s;
        auto& api = nccl();
        try {
            ncclUniqueId base;
            std::memcpy(&base, uid, sizeof(base));
            api.check(api.CommInitRank(&world_comm_, c.world, base, c.rank), "ncclCommInitRank(world)");
            PSWE_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
            char* d_id = nullptr;
            PSWE_CUDA(cudaMalloc(&d_id, sizeof(ncclUniqueId)));
            for (int l = 0; l < c.nlev; ++l)
                for (int p = 0; p < 2; ++p) {
                    ncclUniqueId id{};
                    if (c.rank == 0) api.check(api.GetUniqueId(&id), "ncclGetUniqueId");
                    PSWE_CUDA(cudaMemcpyAsync(d_id, &id, sizeof(id), cudaMemcpyHostToDevice, aux_));
                    api.check(api.Broadcast(d_id, d_id, sizeof(id), ncclUint8, 0, world_comm_, aux_), "ncclBroadcast(id)");
                    PSWE_CUDA(cudaMemcpyAsync(&id, d_id, sizeof(id), cudaMemcpyDeviceToHost, aux_));
                    drain(aux_);
                    api.check(api.CommInitRank(&comm_[l][p], c.world, id, c.rank), "ncclCommInitRank(p2p)");
                }
            cudaFree(d_id);
            for (int l = 0; l < c.nlev; ++l) {
                PSWE_CUDA(cudaStreamCreateWithFlags(&send_stream_[l], cudaStreamNonBlocking));
                const size_t mb = msg_bytes(c.K[l]);
                for (int s = 0; s < c.slots; ++s) {
                    char* b = nullptr;
                    PSWE_CUDA(cudaMalloc(&b, mb));
                    send_buf_[l].push_back(b);
                    PSWE_CUDA(cudaMalloc(&b, mb));
                    recv_buf_[l].push_back(b);
                    cudaEvent_t e;
                    PSWE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    send_done_[l].push_back(e);
                    PSWE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    staged_[l].push_back(e);
                    PSWE_CUDA(cudaEventRecord(send_done_[l].back(), send_stream_[l]));
                }
            }
            PSWE_CUDA(cudaMalloc(&d_res_all_, sizeof(double) * c.n_res * c.world));
            PSWE_CUDA(cudaMallocHost(&h_res_all_, sizeof(double) * c.n_res * c.world));
            warm_up();
        } catch (...) {
            abort("initialisation failed", nullptr);
            release();
            throw;
        }
    }
    ~NcclTransport() override { release(); }
    const char* name() const override { return "nccl"; }

    void send(int level, unsigned long long k, const double2* src, const MsgTag& tag, cudaStream_t st) override {
        auto& api = nccl();
        const int slot = (int)(k % c_.slots);
        char* b = send_buf_[level][slot];
        PSWE_CUDA(cudaStreamWaitEvent(st, send_done_[level][slot], 0));  // previous send from this slot done
        put_message(reinterpret_cast<double2*>(b), src, 3 * c_.K[level], tag, st);
        PSWE_CUDA(cudaEventRecord(staged_[level][slot], st));
        PSWE_CUDA(cudaStreamWaitEvent(send_stream_[level], staged_[level][slot], 0));
        api.check(api.Send(b, msg_bytes(c_.K[level]), ncclUint8, c_.rank + 1, comm_[level][c_.rank % 2],
                           send_stream_[level]),
                  "ncclSend");
        PSWE_CUDA(cudaEventRecord(send_done_[level][slot], send_stream_[level]));
    }

    const double2* recv(int level, unsigned long long k, cudaStream_t st) override {
        auto& api = nccl();
        const int slot = (int)(k % c_.slots);
        char* b = recv_buf_[level][slot];
        api.check(api.Recv(b, msg_bytes(c_.K[level]), ncclUint8, c_.rank - 1, comm_[level][(c_.rank + 1) % 2], st),
                  "ncclRecv");
        return reinterpret_cast<const double2*>(b);
    }

    void end_block(const double2* my_final, double2* final_state, double2* step_finals, const double* d_res_mine,
                   double* res_all, cudaStream_t st) override {
        auto& api = nccl();
        const size_t fdb = (size_t)3 * c_.Kfinal * 2;  // doubles
        // every send posted before the block's collectives
        for (int l = 0; l < c_.nlev; ++l) {
            PSWE_CUDA(cudaEventRecord(staged_[l][0], send_stream_[l]));  // reuse: nothing waits on it now
            PSWE_CUDA(cudaStreamWaitEvent(st, staged_[l][0], 0));
        }
        if (final_state) {
            if (c_.rank == c_.world - 1)
                PSWE_CUDA(cudaMemcpyAsync(final_state, my_final, fdb * sizeof(double), cudaMemcpyDeviceToDevice, st));
            api.check(api.Broadcast(final_state, final_state, fdb, ncclFloat64, c_.world - 1, world_comm_, st),
                      "ncclBroadcast(final)");
        }
        if (step_finals)
            api.check(api.AllGather(my_final, step_finals, fdb, ncclFloat64, world_comm_, st), "ncclAllGather(finals)");
        if (res_all) {
            api.check(api.AllGather(d_res_mine, d_res_all_, c_.n_res, ncclFloat64, world_comm_, st),
                      "ncclAllGather(residuals)");
            PSWE_CUDA(cudaMemcpyAsync(h_res_all_, d_res_all_, sizeof(double) * c_.n_res * c_.world,
                                      cudaMemcpyDeviceToHost, st));  // pinned: stays asynchronous
        }
        drain(st);
        if (res_all) std::memcpy(res_all, h_res_all_, sizeof(double) * c_.n_res * c_.world);
    }

    void drain(cudaStream_t st) override {
        try {
            drain_stream(st, timeout_s, [&] { poll_async(); });
        } catch (...) {
            abort("timeout or communicator error", st);
            throw;
        }
    }

    // ncclCommAbort ends every outstanding NCCL operation of this rank; peers' blocked operations
    // on these communicators then fail and their own drains report it
    void abort(const std::string&, cudaStream_t) override {
        if (aborted_) return;
        aborted_ = true;
        auto& api = nccl();
        for (auto& l : comm_)
            for (auto& cm : l)
                if (cm) {
                    api.CommAbort(cm);
                    cm = nullptr;
                }
        if (world_comm_) {
            api.CommAbort(world_comm_);
            world_comm_ = nullptr;
        }
    }

private:
    void poll_async() {
        auto& api = nccl();
        auto one = [&](ncclComm_t cm) {
            if (!cm) return;
            ncclResult_t e = 0;
            api.CommGetAsyncError(cm, &e);
            if (e != 0 && e != ncclInProgress)
                throw std::runtime_error(std::string("pfasst: NCCL asynchronous error: ") + api.GetErrorString(e));
        };
        one(world_comm_);
        for (auto& l : comm_)
            for (auto cm : l) one(cm);
    }

    // connect every P2P pair that the schedule uses now, so no send or receive inside a block
    // blocks the host on a lazy connection
    void warm_up() {
        auto& api = nccl();
        char* b = recv_buf_[0][0];
        for (int l = 0; l < c_.nlev; ++l)
            for (int p = 0; p < 2; ++p) {
                if (c_.rank % 2 == p && c_.rank + 1 < c_.world)
                    api.check(api.Send(send_buf_[0][0], 64, ncclUint8, c_.rank + 1, comm_[l][p], aux_), "ncclSend(warm-up)");
                if (c_.rank % 2 != p && c_.rank > 0)
                    api.check(api.Recv(b, 64, ncclUint8, c_.rank - 1, comm_[l][p], aux_), "ncclRecv(warm-up)");
            }
        drain(aux_);
    }

    void release() {
        cudaDeviceSynchronize();
        auto& api = nccl();
        for (auto& l : comm_)
            for (auto& cm : l)
                if (cm) {
                    api.CommDestroy(cm);
                    cm = nullptr;
                }
        if (world_comm_) api.CommDestroy(world_comm_);
        world_comm_ = nullptr;
        for (int l = 0; l < 3; ++l) {
            for (auto b : send_buf_[l]) cudaFree(b);
            for (auto b : recv_buf_[l]) cudaFree(b);
            for (auto e : send_done_[l]) cudaEventDestroy(e);
            for (auto e : staged_[l]) cudaEventDestroy(e);
            send_buf_[l].clear();
            recv_buf_[l].clear();
            send_done_[l].clear();
            staged_[l].clear();
            if (send_stream_[l]) cudaStreamDestroy(send_stream_[l]);
            send_stream_[l] = nullptr;
        }
        if (aux_) cudaStreamDestroy(aux_);
        aux_ = nullptr;
        if (d_res_all_) cudaFree(d_res_all_);
        if (h_res_all_) cudaFreeHost(h_res_all_);
        h_res_all_ = nullptr;
        d_res_all_ = nullptr;
    }

    TransportConfig c_;
    ncclComm_t world_comm_ = nullptr;
    ncclComm_t comm_[3][2] = {};
    cudaStream_t send_stream_[3] = {nullptr, nullptr, nullptr};
    cudaStream_t aux_ = nullptr;
    std::vector<char*> send_buf_[3], recv_buf_[3];
    std::vector<cudaEvent_t> send_done_[3], staged_[3];
    double* d_res_all_ = nullptr;
    double* h_res_all_ = nullptr;
    bool aborted_ = false;
};

}  // namespace

void nccl_unique_id(void* out128) {
    ncclUniqueId id;
    nccl().check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

std::unique_ptr<Transport> make_nccl_transport(const TransportConfig& c, const void* uid128) {
    return std::unique_ptr<Transport>(new NcclTransport(c, uid128));
}

}  // namespace pswe
