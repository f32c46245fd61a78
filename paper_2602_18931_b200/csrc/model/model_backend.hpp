// Real-model backend for the batched driver (BASELINE config 3): the controller's verify runs
// the target model (Llama-3.1-8B shape), the worker's draft rollout and the controller's local
// draft/catch-up run the draft model (Llama-3.2-1B shape). Each batched round becomes one
// target forward over every pending verify row and one draft forward over every pending draft
// row, followed by the fused K3/K4 epilogues.
//
// KV caches are content-addressed, like the protocol itself (controller.hpp:145-156): per
// request a linear target cache and a linear controller-draft cache checked by longest common
// prefix, and for the worker a linear committed prefix plus a token trie of speculative nodes
// (the device mirror of the worker's SpecTree). A job feeds exactly the context tokens whose KV
// is missing; accepted speculative KV migrates into the prefix on commit (slot copies).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../host/driver.hpp"
#include "llama.hpp"

namespace wsb {

struct ModelPairCfg {
  std::string target = "llama3-8b";
  std::string draft = "llama3.2-1b";
  std::uint64_t seed = 1;
  std::uint32_t prompt_len = 128;
  std::uint32_t max_requests = 256;
  std::uint32_t max_ctx = 256;     // prompt + generated + k + 2
  std::uint32_t trie_slots = 512;  // speculative-node KV slots per request (worker)
  float plant_target = 16.f;       // planted shared bigram bias (logit units)
  float plant_draft = 16.f;
  float draft_plant_rate = 0.8f;   // fraction of input tokens whose plant the draft also sees
  int draft_device = -1;           // split placement: the draft model on another GPU (-1: same)
  int tp = 1;                      // target tensor-parallel ranks (GPUs device .. device + tp - 1)
};

class ModelPair;

class ModelBackend_Llama : public ModelBackend {
 public:
  ModelBackend_Llama(ModelPair* pair, std::uint32_t seq_len, TokenId eos, std::uint32_t k);
  ~ModelBackend_Llama() override;
  void run_round(const RoundJobs& jobs, RoundResults& res, int verify_mode, std::uint64_t sample_seed) override;
  bool wants_context() const override { return true; }
  // lane 0 = target stream (verify), lanes 1..n = draft streams (worker + controller drafts)
  bool has_lanes() const override { return true; }
  int n_lanes() const override;
  std::size_t submit(int lane, const RoundJobs& jobs, int verify_mode, std::uint64_t sample_seed) override;
  int wait_any(std::uint32_t busy) override;
  int poll_any(std::uint32_t busy) override;
  void complete(int lane, RoundResults& res) override;
  KernelProfiler& profiler(int lane);  // lane 0: target forwards; lanes 1..n: draft forwards
  // After complete(0): the per-row predictions (top-2 + entropy, K3) of the last verify batch,
  // n_rows = verify jobs x (k + 1), request-major (the per-call boundary's rows export).
  void verify_rows(ws_pred* host, std::size_t n_rows);
  // New run on the same pair (the caller reset the per-request caches): run parameters, zeroed
  // counters; streams, workspaces and device buffers are kept.
  void reset_run(std::uint32_t seq_len, TokenId eos, std::uint32_t k);
  // WS_VERIFY_REJECTION on the model path (K4R): the target's softmax temperature and nucleus
  void set_sampling(float temperature, float top_p) {
    inv_temp_ = temperature > 0.f ? 1.f / temperature : 1.f;
    top_p_ = top_p > 0.f && top_p < 1.f ? top_p : 1.f;
  }
  double target_ms = 0, draft_ms = 0;
  std::uint64_t target_rows = 0, draft_rows_fed = 0, target_forwards = 0, draft_forwards = 0;
  std::uint64_t target_out_rows = 0, draft_out_rows = 0;  // rows through the LM head + K3
  std::uint64_t target_kv_pos() const;  // attention work of this backend's forwards (since reset_run)
  std::uint64_t target_attn_pairs() const;
  std::uint64_t draft_kv_pos() const;
  std::uint64_t draft_attn_pairs() const;
  std::uint64_t rows_by_kind[3] = {0, 0, 0}, jobs_by_kind[3] = {0, 0, 0};  // JobKind
  double host_submit_ms[2] = {0, 0}, host_wait_ms = 0;  // host time in submit (per lane) / wait_any

 private:
  void fill_ctx(const RoundJobs& jobs, std::uint32_t r, const JobCtx& c);
  std::size_t verify_take(const RoundJobs& jobs);  // padding-aware batch trim (lanes driver)
  void submit_verify(const RoundJobs& jobs, std::size_t nv);
  void submit_draft(int lane, const RoundJobs& jobs);
  void submit_draft_sub(int lane, struct DraftSub& sub, const RoundJobs& jobs);
  cudaStream_t draft_stream(int lane) const;
  ModelPair* p_;
  std::uint32_t L_;
  TokenId eos_;
  std::uint32_t k_;
  std::uint64_t draft_batch_ = 0;
  int verify_mode_ = WS_VERIFY_GREEDY;
  std::uint64_t sample_seed_ = 0;
  float inv_temp_ = 1.f, top_p_ = 1.f;
  struct Lanes;
  std::unique_ptr<Lanes> ln_;
};

// Owns both models, their KV caches and the per-request cache state on one device.
class ModelPair {
 public:
  ModelPair(const ModelPairCfg& cfg, int device);
  ~ModelPair();
  void reset_requests();  // forget all cached KV state (new run)
  // Late PDL trigger policy for a run over n_local requests (see model_backend.cu)
  void set_pdl_late_for(std::uint32_t n_local);
  void evict(std::uint32_t r);  // forget request r's cached KV (target, controller draft, worker)
  // Prompt prefill (its own phase, before the first verify / draft): the KV of prompt positions
  // [0, P-1) of each listed request is written for the target (verify cache), and once for the
  // draft model into the worker's committed prefix, then copied into the controller's draft
  // cache. Every later verify forward then feeds exactly k+1 rows (the last prompt token + the
  // k candidates), so verify forwards and prefill forwards are timed as separate units.
  struct PrefillStats {
    double target_ms = 0, draft_ms = 0;
    std::uint64_t rows = 0, target_forwards = 0, draft_forwards = 0, launches = 0, h2d = 0;
    std::uint64_t kv_pos = 0, attn_pairs = 0;  // target side
  };
  PrefillStats prefill_prompts(const std::uint32_t* reqs, std::size_t n);
  // Teacher-forced trace export: for requests [first, first + n), the target's
  // greedy continuation of the prompt for `length` positions; at every position the target's
  // and the draft's top-2 / entropy on the same (committed) context. out: n * length records,
  // request-major. Overwrites the requests' KV (the caches are reset).
  void export_trace(std::uint32_t first, std::uint32_t n, std::uint32_t length, ws_token_record* out);
  const ModelPairCfg& cfg() const { return cfg_; }
  LlamaModel& target() { return *target_; }
  LlamaModel& draft() { return *draft_; }
  // Draft replicas (a tensor-parallel target spreads the draft model over its ranks: request r's
  // draft jobs always run on replica r % n, whose KV holds its caches)
  int draft_replicas() const { return static_cast<int>(draft_reps_.size()); }
  LlamaModel& draft(int rep) { return rep == 0 ? *draft_ : *draft_reps_[static_cast<std::size_t>(rep)]; }
  int draft_device(int rep) const { return rep_devices_[static_cast<std::size_t>(rep)]; }
  int replica_of(std::uint32_t request) const { return static_cast<int>(request % draft_reps_.size()); }
  const std::vector<TokenId>& prompt(std::uint32_t r);
  std::int32_t plant(TokenId t, bool draft) const;
  int device() const { return device_; }  // the target model's GPU
  int draft_device() const { return draft_device_; }
  int max_rows() const { return max_rows_; }

  struct Impl;
  std::unique_ptr<Impl> impl;

 private:
  ModelPairCfg cfg_;
  int device_;
  std::unique_ptr<LlamaModel> target_, draft_;
  std::vector<std::unique_ptr<LlamaModel>> draft_reps_;  // [0] empty (draft_ is replica 0)
  std::vector<int> rep_devices_;
  std::vector<std::vector<TokenId>> prompts_;
  int max_rows_ = 0;
  int draft_device_ = 0;
};

}  // namespace wsb
