// beaver_elementwise.h — elementwise Beaver multiplication / square kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mpc {

// TTP triple (square = false: a, b, c) or Beaver pair (square = true: a, b = a^2; c unused)
// for parties [out_lo, out_hi), buffers [out_hi - out_lo][n].
cudaError_t launch_ttp_elementwise(bool square, uint64_t key, uint64_t id, int P, int out_lo, int out_hi,
                                   uint64_t* a, uint64_t* b, uint64_t* c, int64_t n, cudaStream_t st);
// All P parties on this device ([P][n] buffers): eps (and delta) revealed as local sums, then every z_p;
// bits > 0: per-share truncation (P <= 2).  square: y and c unused.
cudaError_t launch_beaver_elementwise_all(bool square, const uint64_t* x, const uint64_t* y, const uint64_t* a,
                                          const uint64_t* b, const uint64_t* c, uint64_t* z, int P, int64_t n,
                                          int bits, cudaStream_t st);
// One party after the reveal: ed = [eps | delta] (square: eps), party0 adds the public term.
cudaError_t launch_beaver_elementwise_finish(bool square, const uint64_t* ed, const uint64_t* a, const uint64_t* b,
                                             const uint64_t* c, uint64_t* z, int64_t n, int party0, int bits,
                                             cudaStream_t st);

}  // namespace mpc
