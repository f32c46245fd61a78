#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "wanspec_b200.h"

namespace wsb {

// Per-row softmax statistics in the log2 domain: p(x) = 2^(x*cl - m2) / Z with cl = inv_temp*log2(e).
struct RowStats {
  float m2;  // max(x) * cl
  float z;   // sum 2^(x*cl - m2)
  float cl;  // inv_temp * log2(e)
  float h;   // entropy (nats)
};

// Vocab tile per warp: fixed (not derived from the row count) so a row's statistics are
// bit-identical at any batch size (batch invariance) — tiles = ceil(V / kRowTile).
constexpr std::uint32_t kRowTile = 8192;

std::size_t rowstats_workspace_bytes(std::uint32_t rows, std::uint32_t vocab, std::uint32_t n_req);

// K3: fused softmax + entropy + top-2 over bf16 logits rows (+ optional K4 greedy verify
// epilogue when cand != nullptr: rows are n_req groups of k+1, run_target_step semantics on
// the argmaxes). `workspace` must be zero-initialised once (counters self-reset).
// forced (optional, device, per row): >= 0 overrides the row with a fully confident prediction
// of that token (prob 1, entropy 0) — the past-the-end EOS rule of SequenceTrace
// (oracle.hpp:88-102, :118) applied to model rows that predict positions >= sequence_length-1.
void row_stats_bf16(const void* logits, std::uint32_t rows, std::uint32_t vocab, std::uint32_t ld, float inv_temp,
                    ws_pred* out_pred, RowStats* out_stats, void* workspace, std::uint32_t n_req, std::uint32_t k,
                    const std::uint32_t* cand, ws_verify_out* verify_out, cudaStream_t stream,
                    const std::int32_t* forced = nullptr);

}  // namespace wsb
