// relu.h — ReLU path kernels (internal).
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "elementwise.h"

namespace mpc {

// All P (<= 8) parties on one device: out = ReLU shares of x ([P][n]); sign_out (optional,
// [P][n]) = arithmetic shares of [x < 0].  relu_id < 2^32 selects every stream of the path.
cudaError_t launch_relu_all(const KeySet& kp, uint64_t kttp, uint64_t id, int P, const uint64_t* x, uint64_t* out,
                            uint64_t* sign_out, int64_t n, cudaStream_t st);

// ---- one party per context (reveals over the transport) ----
// The A2B adder tree (R24): node [lo, hi) of height H = ceil(log2(hi - lo)) adds
// the values of its children [lo, mid) and [mid, hi), mid = lo + 2^(H-1); its
// value replaces V[lo].  Nodes of one height run together, 7 rounds per height.
struct ReluNode { uint64_t add_id; int lo, mid; };
constexpr int kReluMaxNodes = 8;                  // P <= 16
// nodes_by_height[h - 1] = the adders of height h, h = 1..ceil(log2 P); add ids as the fused kernel's
void relu_tree_nodes(int P, uint64_t relu_id, std::vector<std::vector<ReluNode>>& nodes_by_height);

struct ReluAdderArgs {
    uint64_t kttp;
    int P, p, nnodes;
    ReluNode node[kReluMaxNodes];
    uint64_t* V;          // [P][n] binary shares held by party p (leaf values / node outputs)
    uint64_t* G;          // [nnodes][n] generate, party p's binary share
    uint64_t* Pr;         // [nnodes][n] propagate
    uint64_t* ED;         // [4][nnodes][n]: e, d of gate 0, e, d of gate 1 (revealed in place)
    int64_t n;
};
// V[Q] = <[x]_Q>_p for Q < P (binary PRZS of every party's arithmetic share; x = [x]_p).
cudaError_t launch_relu_leaf(const KeySet& kp, int P, int p, uint64_t relu_id, const uint64_t* x, uint64_t* V,
                             int64_t n, cudaStream_t st);
// Step l = 0..7 of the adders of one height: finish AND level l-1 from the
// revealed ED (l >= 1), then mask AND level l into ED (l <= 6), or write the
// sum into V[lo] (l = 7).  Reveal after step l: 2*nnodes*n words for l = 0, 6,
// 4*nnodes*n for l = 1..5.
cudaError_t launch_relu_adder_step(const ReluAdderArgs& a, int l, cudaStream_t st);
// Alg. 2 step 1: zbits = packed (sign(<x>_p) ^ <r>_p); word w holds element pairs
// 32w..32w+31 (bit t: element 2(32w+t), bit 32+t: element 2(32w+t)+1);
// relu_zbits_words(n) words.
int64_t relu_zbits_words(int64_t n);
cudaError_t launch_relu_b2a_mask(uint64_t kttp, int P, int p, uint64_t relu_id, const uint64_t* xb, uint64_t* zbits,
                                 int64_t n, cudaStream_t st);
// Alg. 2 step 2 from the revealed zbits: [x < 0]_p, then the multiplication's
// mask ed = [x_p - a_p | (1 - [x < 0])_p - b_p] ([2][n]); sign_out optional.
cudaError_t launch_relu_b2a_mul_mask(uint64_t kttp, int P, int p, uint64_t relu_id, const uint64_t* zbits,
                                     const uint64_t* x, uint64_t* ed, uint64_t* sign_out, int64_t n, cudaStream_t st);
// out_p = c_p + eps b_p + a_p delta + [p = 0] eps delta from the revealed ed.
cudaError_t launch_relu_mul_finish(uint64_t kttp, int P, int p, uint64_t relu_id, const uint64_t* ed, uint64_t* out,
                                   int64_t n, cudaStream_t st);

}  // namespace mpc
