// ws_ctx: one GPU's hot-path state (tiny-pair tables + lanes, optional real-model pair).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "kernels/k9_oracle.cuh"
#include "model/model_backend.hpp"

struct ws_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  wsb::DevTables tables;
  std::vector<std::unique_ptr<wsb::OracleLane>> lanes;
  std::unique_ptr<wsb::ModelPair> models;
  // real-model protocol threads' backends (streams, workspaces), kept across runs
  std::vector<std::unique_ptr<wsb::ModelBackend_Llama>> model_lanes;
  // per-call model boundary (ws_model_open / _verify / _draft): its own streams and workspaces
  std::unique_ptr<wsb::ModelBackend_Llama> call_backend;
  std::uint32_t call_k = 0;
  // model-step statistics of this context's last ws_run_model_sim (ws_model_stats)
  struct ModelStats {
    double target_ms = 0, draft_ms = 0;
    std::uint64_t target_rows = 0, draft_rows = 0, target_forwards = 0, draft_forwards = 0;
    std::uint64_t target_out_rows = 0, draft_out_rows = 0;
    double prefill_target_ms = 0, prefill_draft_ms = 0;
    std::uint64_t prefill_rows = 0, prefill_forwards = 0;
    std::uint64_t verify_kv_pos = 0, verify_attn_pairs = 0, draft_kv_pos = 0, draft_attn_pairs = 0;
    std::uint64_t prefill_kv_pos = 0, prefill_attn_pairs = 0;
  } last_stats;

  wsb::OracleLane& lane(std::size_t i) {
    while (lanes.size() <= i) lanes.emplace_back(new wsb::OracleLane(&tables, device));
    return *lanes[i];
  }
};

namespace wsb {
int ops_guarded_rc(const char* what, const std::exception& e);
// Shared by capi.cpp / capi_model.cpp: SimConfig validation + conversion and the shard runner.
SimCfg sim_cfg_from_abi(const ws_sim_cfg& c);
void run_shard(const ws_sim_cfg* c, const SimCfg& cfg, ModelBackend& backend, ws_run_out* out, int device);
// One protocol thread per backend, each over a contiguous range of the shard's requests.
void run_shard_threads(const ws_sim_cfg* c, const SimCfg& cfg, const std::vector<ModelBackend*>& backends,
                       ws_run_out* out, int device);
}  // namespace wsb
