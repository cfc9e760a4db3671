// transport.h — the reveal transports of one-party contexts.
//
// A reveal is an allreduce over the P parties (§4.1): a mod-2^64 sum
// of arithmetic shares, an int8 sum (Alg. 1's top-nibble reveal, R12)
// or an XOR of binary shares (App. A.1.2, the ReLU path).  Two transports:
//   * NCCL (one process and one GPU per party — the deployment): sums are
//     ncclAllReduce; XOR is an ncclAllGather of the P shares plus a local XOR
//     (NCCL has no XOR reduction);
//   * an in-process group (`LocalGroup`): P one-party contexts of one process,
//     each driven by its own host thread, on one device.  The collective is a
//     host rendezvous: the last party to arrive makes its stream wait on every
//     party's "ready" event, launches one kernel that reduces all P send buffers
//     into all P receive buffers, and publishes a "done" event every party's
//     stream waits on.  It runs the one-party schedule — the same kernels, the
//     same stream and event structure as with NCCL — on a single GPU, which is
//     how the tests exercise P > 1 one-party contexts (one GPU per test box).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace mpc {

enum class RedOp : int { SumU64 = 0, SumI8 = 1, XorU64 = 2 };

struct LocalGroup;

LocalGroup* local_group_create(int P);
void local_group_destroy(LocalGroup* g);
int local_group_size(const LocalGroup* g);
// Attach party `rank` (once per party).  Returns false if the rank is taken or out of range.
bool local_group_attach(LocalGroup* g, int rank);
void local_group_detach(LocalGroup* g, int rank);

// One collective of party `rank` on `st`: recv = op over the parties' send buffers
// (count elements of 8 bytes for SumU64 / XorU64, 1 byte for SumI8).  in-place
// (send == recv) is allowed.  Blocks the calling host thread until every party
// has entered the same collective.  Returns 0 on success, 1 on a mismatch of
// count / op between parties (the group is then broken), 2 on timeout, 3 on a
// CUDA error, 4 if the group is broken.
int local_group_allreduce(LocalGroup* g, int rank, const void* send, void* recv, size_t count, RedOp op,
                          cudaStream_t st);

// out[i] = XOR_{q < P} gathered[q * n + i] (the local half of the NCCL XOR reveal).
cudaError_t launch_xor_gathered(const uint64_t* gathered, int P, int64_t n, uint64_t* out, cudaStream_t st);

}  // namespace mpc
