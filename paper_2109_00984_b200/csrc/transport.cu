// transport.cu — the in-process reveal transport (LocalGroup) and the local
// XOR of an all-gathered binary reveal.  See transport.h.
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "transport.h"

namespace mpc {

namespace {
constexpr int kGroupMax = 16;

struct PartyPtrs {
    const void* send[kGroupMax];
    void* recv[kGroupMax];
};

// Thread = one element for every party: all P inputs are read before any
// output is written, so in-place reveals (send == recv) are safe.
template <RedOp OP>
__global__ void __launch_bounds__(256) local_allreduce_kernel(PartyPtrs ptr, int P, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        if constexpr (OP == RedOp::SumI8) {
            int8_t s = 0;
            for (int q = 0; q < P; ++q) s = (int8_t)(s + static_cast<const int8_t*>(ptr.send[q])[i]);
            for (int q = 0; q < P; ++q) static_cast<int8_t*>(ptr.recv[q])[i] = s;
        } else {
            uint64_t s = 0;
            for (int q = 0; q < P; ++q) {
                const uint64_t v = static_cast<const uint64_t*>(ptr.send[q])[i];
                s = OP == RedOp::XorU64 ? (s ^ v) : (s + v);
            }
            for (int q = 0; q < P; ++q) static_cast<uint64_t*>(ptr.recv[q])[i] = s;
        }
    }
}

__global__ void __launch_bounds__(256) xor_gathered_kernel(const uint64_t* __restrict__ g, int P, int64_t n,
                                                           uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t s = 0;
        for (int q = 0; q < P; ++q) s ^= g[(int64_t)q * n + i];
        out[i] = s;
    }
}

unsigned grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (unsigned)g;
}
}  // namespace

struct LocalGroup {
    struct Slot {
        const void* send = nullptr;
        void* recv = nullptr;
        size_t count = 0;
        RedOp op = RedOp::SumU64;
        cudaEvent_t ready = nullptr;
        cudaStream_t stream = nullptr;
    };
    int P = 0;
    std::mutex m;
    std::condition_variable cv;
    uint64_t gen = 0;
    int arrived = 0;
    int status = 0;                 // result of the last completed collective
    bool broken = false;
    std::vector<Slot> slots;
    std::vector<bool> attached;
    cudaEvent_t done[2] = {nullptr, nullptr};   // per generation parity
};

LocalGroup* local_group_create(int P) {
    if (P < 1 || P > kGroupMax) return nullptr;
    auto* g = new LocalGroup();
    g->P = P;
    g->slots.resize(P);
    g->attached.assign(P, false);
    for (int q = 0; q < P; ++q) {
        if (cudaEventCreateWithFlags(&g->slots[q].ready, cudaEventDisableTiming) != cudaSuccess) {
            local_group_destroy(g);
            return nullptr;
        }
    }
    for (auto& e : g->done)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            local_group_destroy(g);
            return nullptr;
        }
    return g;
}

void local_group_destroy(LocalGroup* g) {
    if (!g) return;
    for (auto& s : g->slots)
        if (s.ready) cudaEventDestroy(s.ready);
    for (auto e : g->done)
        if (e) cudaEventDestroy(e);
    delete g;
}

int local_group_size(const LocalGroup* g) { return g ? g->P : 0; }

bool local_group_attach(LocalGroup* g, int rank) {
    std::lock_guard<std::mutex> lk(g->m);
    if (rank < 0 || rank >= g->P || g->attached[rank]) return false;
    g->attached[rank] = true;
    return true;
}

void local_group_detach(LocalGroup* g, int rank) {
    std::lock_guard<std::mutex> lk(g->m);
    if (rank >= 0 && rank < g->P) g->attached[rank] = false;
}

int local_group_allreduce(LocalGroup* g, int rank, const void* send, void* recv, size_t count, RedOp op,
                          cudaStream_t st) {
    std::unique_lock<std::mutex> lk(g->m);
    if (g->broken) return 4;
    LocalGroup::Slot& me = g->slots[rank];
    if (cudaEventRecord(me.ready, st) != cudaSuccess) { g->broken = true; g->cv.notify_all(); return 3; }
    me.send = send; me.recv = recv; me.count = count; me.op = op; me.stream = st;
    const uint64_t my_gen = g->gen;
    cudaEvent_t done = g->done[my_gen & 1];
    if (++g->arrived == g->P) {
        // last to arrive: check the collective contract, then launch for everyone
        int status = 0;
        for (int q = 0; q < g->P; ++q)
            if (g->slots[q].count != count || g->slots[q].op != op) status = 1;
        if (status == 0 && count > 0) {
            for (int q = 0; q < g->P; ++q)
                if (q != rank && cudaStreamWaitEvent(st, g->slots[q].ready, 0) != cudaSuccess) status = 3;
            PartyPtrs ptr{};
            for (int q = 0; q < g->P; ++q) { ptr.send[q] = g->slots[q].send; ptr.recv[q] = g->slots[q].recv; }
            if (status == 0) {
                const unsigned grid = grid_for((int64_t)count);
                if (op == RedOp::SumI8) local_allreduce_kernel<RedOp::SumI8><<<grid, 256, 0, st>>>(ptr, g->P, (int64_t)count);
                else if (op == RedOp::XorU64) local_allreduce_kernel<RedOp::XorU64><<<grid, 256, 0, st>>>(ptr, g->P, (int64_t)count);
                else local_allreduce_kernel<RedOp::SumU64><<<grid, 256, 0, st>>>(ptr, g->P, (int64_t)count);
                if (cudaGetLastError() != cudaSuccess) status = 3;
            }
        }
        if (status == 0 && cudaEventRecord(done, st) != cudaSuccess) status = 3;
        if (status != 0) g->broken = true;
        g->status = status;
        g->arrived = 0;
        g->gen++;
        g->cv.notify_all();
    } else {
        static const long timeout_s = getenv("MPC_GROUP_TIMEOUT_S") ? atol(getenv("MPC_GROUP_TIMEOUT_S")) : 300;
        const bool ok = g->cv.wait_for(lk, std::chrono::seconds(timeout_s),
                                       [&] { return g->gen != my_gen || g->broken; });
        if (!ok) { g->broken = true; g->cv.notify_all(); return 2; }
        if (g->gen == my_gen) return 4;          // broken while waiting
    }
    if (g->status != 0) return g->status;
    lk.unlock();
    // every party's later work on `st` is ordered after the collective kernel
    return cudaStreamWaitEvent(st, done, 0) == cudaSuccess ? 0 : 3;
}

cudaError_t launch_xor_gathered(const uint64_t* gathered, int P, int64_t n, uint64_t* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    xor_gathered_kernel<<<grid_for(n), 256, 0, st>>>(gathered, P, n, out);
    return cudaGetLastError();
}

}  // namespace mpc
