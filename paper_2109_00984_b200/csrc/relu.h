// relu.h — ReLU path kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "elementwise.h"

namespace mpc {

// All P (<= 8) parties on one device: out = ReLU shares of x ([P][n]); sign_out (optional,
// [P][n]) = arithmetic shares of [x < 0].  relu_id < 2^32 selects every stream of the path.
cudaError_t launch_relu_all(const KeySet& kp, uint64_t kttp, uint64_t id, int P, const uint64_t* x, uint64_t* out,
                            uint64_t* sign_out, int64_t n, cudaStream_t st);

}  // namespace mpc
