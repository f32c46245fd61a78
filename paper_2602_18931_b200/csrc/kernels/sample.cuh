// K4R — speculative rejection sampling over the target's verify rows (extension: the reference
// is greedy-only, so this path is "parity unpinned" by it and checked against the
// plain-C restatement oracle/restate.c or_model_rejection_verify, which follows the same rule
// in the same fp64 summation order).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "wanspec_b200.h"

namespace wsb {

// One CTA per request over its k+1 bf16 logits rows (row i predicts position base + i):
//   target distribution of row i: p(x) = exp(x*tau - max)/Z in fp64 (tau = inv_temp); with
//     top_p < 1, the nucleus N = {x : key(x) >= t*}, t* = the largest 16-bit order key of the
//     bf16 logits whose tail mass sum_{key >= t*} p >= top_p (ties at the threshold value are
//     all kept), and p'(x) = p(x) / mass(N) on N, 0 elsewhere; forced[row] >= 0 replaces the
//     row by a point mass (the past-the-end EOS rule, oracle.hpp:88-102);
//   for i < k: (w0..w3) = Philox4x32-10(counter = (request lo, request hi, step, i), key = seed),
//     u = unit(w0, w1); accept c_i iff u * q_i < p'_i(c_i), q_i = the draft's probability of c_i
//     (the controller's tree node); on reject, bonus ~ residual r(x) = max(0, p'_i(x) - d_i(x))
//     with d_i(c_i) = q_i and d_i(x) = (1 - q_i)/(V - 1) elsewhere (the draft distribution
//     completed uniformly), inverse CDF in ascending id order at u2 = unit(w2, w3);
//   all k accepted: bonus ~ p'_k at row k's u2;
//   final_entropy = the untruncated entropy (nats) of the bonus row (entropy_of, oracle.hpp:21-33).
// Every sum is fp64 in a fixed order: per-thread contiguous id chunks of ceil(V / 512), summed
// sequentially, then a fixed pairwise tree over the 512 partials (prefixes: sequential over
// chunks) — deterministic and batch-invariant.
constexpr int kSampleThreads = 512;

void verify_rejection_bf16(const void* logits, std::uint32_t n_req, std::uint32_t k, std::uint32_t vocab,
                           std::uint32_t ld, float inv_temp, float top_p, const std::uint32_t* cand,
                           const double* cand_prob, std::uint64_t seed, const std::uint64_t* request,
                           const std::uint32_t* step, const std::int32_t* forced, ws_verify_out* out,
                           cudaStream_t stream);

}  // namespace wsb
