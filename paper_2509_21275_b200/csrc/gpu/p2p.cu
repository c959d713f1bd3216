// epp-b200: stage-to-stage P2P channels over peer memory (NVLink on the
// 8 x B200 box) behind include/epp_gpu.h (epp_p2p_*).
//
// The reference models the stage hand-off as a zero-latency event
// (proj/src/pipeline.cpp:168-193); the paper sends activations / gradients
// between adjacent pipeline stages with NCCL.  Here one
// directed channel carries one stream of messages (forward activations
// p -> p+1, or backward gradients p+1 -> p) without NCCL and without host
// synchronisation:
//
//   * the RECEIVER owns a mailbox arena and a `ready` flag; the SENDER owns a
//     `consumed` flag.  Each side exports its allocations as CUDA IPC handles
//     (or raw pointers inside one process); the other side maps them, so the
//     sender can store into the mailbox directly (the producing kernel's
//     epilogue writes over NVLink: no send buffer, no copy) and each side can
//     store into the other's flag;
//   * message k occupies [off_k, off_k + size_k) of the arena, placed by a
//     ring allocator that both sides run on the same size sequence (sizes
//     come from the plan, so both sides know them; no handshake);
//   * send_reserve(k): the sender's stream waits (cuStreamWaitValue32 on its
//     LOCAL consumed flag) until every older message overlapping the region
//     has been released, then returns the peer address;
//     send_commit(k): a one-thread kernel stores k into the receiver's ready
//     flag with release semantics at system scope, after the data writes in
//     stream order;
//   * recv_wait(k): the receiver's stream waits until its LOCAL ready flag
//     >= k (flushing remote writes), then returns the local address;
//     recv_release(k): stores k into the sender's consumed flag.
// Messages are consumed in order on each channel (stage op lists,
// schedule.stage_ops), so the flags are monotonic counters.  A receiver
// releases a message right after the stage call that reads it (the stage
// copies an activation into its own x_in; a gradient is read in place by the
// last layer's backward), so a sender never waits on anything but the
// receiver's progress on that same message: no deadlock for any arena that
// holds the largest message.
#include <cuda.h>
#include <unistd.h>

#include <cstring>
#include <deque>
#include <string>

#include "common.cuh"
#include "epp_gpu.h"

namespace eppk {
std::string& gpu_error_slot();

namespace {

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

// CU_STREAM_WAIT_VALUE_FLUSH where the device supports it: remote (peer)
// writes that reached the device before the flag are visible downstream.
unsigned int wait_flags() {
    static unsigned int f = [] {
        int dev = 0, ok = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&ok, cudaDevAttrCanFlushRemoteWrites, dev) == cudaSuccess && ok)
            return static_cast<unsigned int>(CU_STREAM_WAIT_VALUE_GEQ | CU_STREAM_WAIT_VALUE_FLUSH);
        return static_cast<unsigned int>(CU_STREAM_WAIT_VALUE_GEQ);
    }();
    return f;
}

WaitFn wait_value32() {
    static WaitFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        EPP_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw CudaError("cuStreamWaitValue32 unavailable");
        return reinterpret_cast<WaitFn>(p);
    }();
    return fn;
}

__global__ void p2p_flag_store(unsigned int* flag, unsigned int value) {
    pdl_wait();   // the producing kernel (data writes) has completed
    pdl_trigger();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

constexpr size_t kAlign = 256;

struct HandleBlob {          // EPP_P2P_HANDLE_BYTES, exchanged by the caller
    uint32_t magic;
    int32_t pid;
    int32_t device;
    int32_t role;            // 0 sender, 1 receiver
    uint64_t arena_bytes;
    void* arena_ptr;         // in-process peers map raw pointers
    void* flag_ptr;
    cudaIpcMemHandle_t arena;
    cudaIpcMemHandle_t flag;
};
static_assert(sizeof(HandleBlob) <= EPP_P2P_HANDLE_BYTES, "handle blob too large");
constexpr uint32_t kMagic = 0x45505032u;   // "EPP2"

}  // namespace

struct P2PChannel {
    int role = 0;                 // 0 sender, 1 receiver
    int device = 0;
    uint64_t arena_bytes = 0;
    // own allocations
    void* arena = nullptr;        // receiver: the mailbox
    unsigned int* flag = nullptr; // receiver: ready; sender: consumed
    // peer mappings
    void* peer_arena = nullptr;        // sender: the receiver's mailbox
    unsigned int* peer_flag = nullptr; // sender: receiver's ready; receiver: sender's consumed
    bool peer_ipc = false;
    bool opened = false;
    // ring state (identical on both sides)
    uint64_t next_off = 0;
    unsigned int seq = 0;            // messages placed so far
    unsigned int committed = 0;      // sender: last committed; receiver: last released
    struct Slot { unsigned int seq; uint64_t off, size; };
    std::deque<Slot> live;           // sender: messages not yet known to be released
    int64_t messages = 0, bytes = 0;

    uint64_t place(uint64_t size) {
        const uint64_t b = (size + kAlign - 1) / kAlign * kAlign;
        EPP_REQUIRE(b <= arena_bytes, "p2p: message larger than the channel's arena");
        uint64_t off = next_off;
        if (off + b > arena_bytes) off = 0;
        next_off = off + b;
        return off;
    }
};

}  // namespace eppk

using eppk::P2PChannel;

namespace {
template <typename F>
int pguard(F&& f) {
    eppk::gpu_error_slot().clear();
    try {
        f();
        return EPP_GPU_OK;
    } catch (const eppk::CudaError& e) {
        eppk::gpu_error_slot() = e.what();
        return EPP_GPU_ECUDA;
    } catch (const std::invalid_argument& e) {
        eppk::gpu_error_slot() = e.what();
        return EPP_GPU_EARG;
    } catch (const std::exception& e) {
        eppk::gpu_error_slot() = e.what();
        return EPP_GPU_EOTHER;
    }
}
cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }
}  // namespace

extern "C" {

int epp_p2p_init(int ndev, const int* devs) {
    return pguard([&] {
        EPP_REQUIRE(ndev >= 0 && (ndev == 0 || devs), "p2p_init: bad device list");
        int cur = 0;
        EPP_CUDA(cudaGetDevice(&cur));
        for (int i = 0; i < ndev; ++i)
            for (int j = 0; j < ndev; ++j) {
                if (i == j || devs[i] == devs[j]) continue;
                int ok = 0;
                EPP_CUDA(cudaDeviceCanAccessPeer(&ok, devs[i], devs[j]));
                EPP_REQUIRE(ok, "p2p_init: devices cannot access each other's memory");
                EPP_CUDA(cudaSetDevice(devs[i]));
                const cudaError_t e = cudaDeviceEnablePeerAccess(devs[j], 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
                else EPP_CUDA(e);
            }
        EPP_CUDA(cudaSetDevice(cur));
    });
}

int epp_p2p_create(int role, uint64_t arena_bytes, epp_p2p** out, void* handle_out) {
    return pguard([&] {
        EPP_REQUIRE(out && handle_out, "p2p_create: null argument");
        EPP_REQUIRE(role == EPP_P2P_SENDER || role == EPP_P2P_RECEIVER, "p2p_create: bad role");
        EPP_REQUIRE(role == EPP_P2P_SENDER || arena_bytes >= eppk::kAlign, "p2p_create: arena too small");
        auto* ch = new P2PChannel;
        try {
            ch->role = role;
            ch->arena_bytes = arena_bytes / eppk::kAlign * eppk::kAlign;
            EPP_CUDA(cudaGetDevice(&ch->device));
            EPP_CUDA(cudaMalloc(&ch->flag, 256));
            EPP_CUDA(cudaMemset(ch->flag, 0, 256));
            if (role == EPP_P2P_RECEIVER) EPP_CUDA(cudaMalloc(&ch->arena, ch->arena_bytes));
            eppk::HandleBlob hb{};
            hb.magic = eppk::kMagic;
            hb.pid = static_cast<int32_t>(getpid());
            hb.device = ch->device;
            hb.role = role;
            hb.arena_bytes = ch->arena_bytes;
            hb.arena_ptr = ch->arena;
            hb.flag_ptr = ch->flag;
            EPP_CUDA(cudaIpcGetMemHandle(&hb.flag, ch->flag));
            if (ch->arena) EPP_CUDA(cudaIpcGetMemHandle(&hb.arena, ch->arena));
            std::memset(handle_out, 0, EPP_P2P_HANDLE_BYTES);
            std::memcpy(handle_out, &hb, sizeof(hb));
            EPP_CUDA(cudaDeviceSynchronize());
        } catch (...) {
            if (ch->flag) cudaFree(ch->flag);
            if (ch->arena) cudaFree(ch->arena);
            delete ch;
            throw;
        }
        *out = reinterpret_cast<epp_p2p*>(ch);
    });
}

int epp_p2p_open(epp_p2p* h, const void* peer_handle) {
    return pguard([&] {
        auto* ch = reinterpret_cast<P2PChannel*>(h);
        EPP_REQUIRE(ch && peer_handle, "p2p_open: null argument");
        EPP_REQUIRE(!ch->opened, "p2p_open: channel already open");
        eppk::HandleBlob hb;
        std::memcpy(&hb, peer_handle, sizeof(hb));
        EPP_REQUIRE(hb.magic == eppk::kMagic, "p2p_open: not a channel handle");
        EPP_REQUIRE(hb.role != ch->role, "p2p_open: both ends have the same role");
        // the receiver owns the arena; the sender adopts its size
        if (ch->role == EPP_P2P_SENDER) {
            EPP_REQUIRE(hb.arena_bytes >= eppk::kAlign, "p2p_open: receiver handle without an arena");
            ch->arena_bytes = hb.arena_bytes;
        }
        if (hb.pid == static_cast<int32_t>(getpid())) {
            // same process (one host thread driving several GPUs): raw pointers
            // (epp_p2p_init enabled peer access between the devices)
            ch->peer_flag = static_cast<unsigned int*>(hb.flag_ptr);
            ch->peer_arena = hb.arena_ptr;
        } else {
            void* p = nullptr;
            EPP_CUDA(cudaIpcOpenMemHandle(&p, hb.flag, cudaIpcMemLazyEnablePeerAccess));
            ch->peer_flag = static_cast<unsigned int*>(p);
            if (ch->role == EPP_P2P_SENDER) {
                EPP_CUDA(cudaIpcOpenMemHandle(&p, hb.arena, cudaIpcMemLazyEnablePeerAccess));
                ch->peer_arena = p;
            }
            ch->peer_ipc = true;
        }
        ch->opened = true;
    });
}

int epp_p2p_send_reserve(epp_p2p* h, uint64_t bytes, void* stream, void** dst) {
    return pguard([&] {
        auto* ch = reinterpret_cast<P2PChannel*>(h);
        EPP_REQUIRE(ch && dst && ch->opened && ch->role == EPP_P2P_SENDER, "p2p_send_reserve: not an open sender");
        EPP_REQUIRE(ch->committed == ch->seq, "p2p_send_reserve: previous message not committed");
        const uint64_t off = ch->place(bytes);
        const uint64_t end = off + (bytes + eppk::kAlign - 1) / eppk::kAlign * eppk::kAlign;
        // wait for the newest older message whose bytes overlap [off, end)
        unsigned int need = 0;
        for (const auto& sl : ch->live)
            if (sl.off < end && off < sl.off + sl.size) need = sl.seq;
        if (need) {
            const CUresult r = eppk::wait_value32()(reinterpret_cast<CUstream>(S(stream)),
                                                     reinterpret_cast<CUdeviceptr>(ch->flag), need,
                                                     CU_STREAM_WAIT_VALUE_GEQ);
            if (r != CUDA_SUCCESS) throw eppk::CudaError("cuStreamWaitValue32 failed (" + std::to_string(r) + ")");
            while (!ch->live.empty() && ch->live.front().seq <= need) ch->live.pop_front();
        }
        ch->seq += 1;
        ch->live.push_back({ch->seq, off, end - off});
        ch->messages += 1;
        ch->bytes += static_cast<int64_t>(bytes);
        *dst = static_cast<uint8_t*>(ch->peer_arena) + off;
    });
}

int epp_p2p_send_commit(epp_p2p* h, void* stream) {
    return pguard([&] {
        auto* ch = reinterpret_cast<P2PChannel*>(h);
        EPP_REQUIRE(ch && ch->opened && ch->role == EPP_P2P_SENDER, "p2p_send_commit: not an open sender");
        EPP_REQUIRE(ch->committed + 1 == ch->seq, "p2p_send_commit: no reserved message");
        eppk::launch_k(eppk::p2p_flag_store, 1, 1, 0, S(stream), ch->peer_flag, ch->seq);
        EPP_CHECK_LAUNCH();
        ch->committed = ch->seq;
    });
}

int epp_p2p_recv_wait(epp_p2p* h, uint64_t bytes, void* stream, const void** src) {
    return pguard([&] {
        auto* ch = reinterpret_cast<P2PChannel*>(h);
        EPP_REQUIRE(ch && src && ch->opened && ch->role == EPP_P2P_RECEIVER, "p2p_recv_wait: not an open receiver");
        EPP_REQUIRE(ch->committed == ch->seq, "p2p_recv_wait: previous message not released");
        const uint64_t off = ch->place(bytes);
        ch->seq += 1;
        const CUresult r = eppk::wait_value32()(reinterpret_cast<CUstream>(S(stream)),
                                                 reinterpret_cast<CUdeviceptr>(ch->flag), ch->seq,
                                                 eppk::wait_flags());
        if (r != CUDA_SUCCESS) throw eppk::CudaError("cuStreamWaitValue32 failed (" + std::to_string(r) + ")");
        ch->messages += 1;
        ch->bytes += static_cast<int64_t>(bytes);
        *src = static_cast<const uint8_t*>(ch->arena) + off;
    });
}

int epp_p2p_recv_release(epp_p2p* h, void* stream) {
    return pguard([&] {
        auto* ch = reinterpret_cast<P2PChannel*>(h);
        EPP_REQUIRE(ch && ch->opened && ch->role == EPP_P2P_RECEIVER, "p2p_recv_release: not an open receiver");
        EPP_REQUIRE(ch->committed + 1 == ch->seq, "p2p_recv_release: no message being received");
        eppk::launch_k(eppk::p2p_flag_store, 1, 1, 0, S(stream), ch->peer_flag, ch->seq);
        EPP_CHECK_LAUNCH();
        ch->committed = ch->seq;
    });
}

int epp_p2p_send(epp_p2p* h, const void* src, uint64_t bytes, void* stream) {
    void* dst = nullptr;
    int rc = epp_p2p_send_reserve(h, bytes, stream, &dst);
    if (rc) return rc;
    rc = pguard([&] {
        EPP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, S(stream)));
    });
    if (rc) return rc;
    return epp_p2p_send_commit(h, stream);
}

int epp_p2p_recv(epp_p2p* h, void* dst, uint64_t bytes, void* stream) {
    const void* src = nullptr;
    int rc = epp_p2p_recv_wait(h, bytes, stream, &src);
    if (rc) return rc;
    rc = pguard([&] {
        EPP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, S(stream)));
    });
    if (rc) return rc;
    return epp_p2p_recv_release(h, stream);
}

int epp_p2p_stats(epp_p2p* h, int64_t* messages, int64_t* bytes) {
    return pguard([&] {
        auto* ch = reinterpret_cast<P2PChannel*>(h);
        EPP_REQUIRE(ch != nullptr, "p2p_stats: null channel");
        if (messages) *messages = ch->messages;
        if (bytes) *bytes = ch->bytes;
    });
}

int epp_p2p_destroy(epp_p2p* h) {
    return pguard([&] {
        auto* ch = reinterpret_cast<P2PChannel*>(h);
        if (!ch) return;
        cudaDeviceSynchronize();
        if (ch->peer_ipc) {
            if (ch->peer_flag) cudaIpcCloseMemHandle(ch->peer_flag);
            if (ch->peer_arena) cudaIpcCloseMemHandle(ch->peer_arena);
        }
        if (ch->flag) cudaFree(ch->flag);
        if (ch->arena) cudaFree(ch->arena);
        delete ch;
    });
}

}  // extern "C"
