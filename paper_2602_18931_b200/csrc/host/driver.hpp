// Batched deterministic event driver. Each request is the reference's RequestSim
// (sim.hpp:166-416) restated: virtual clock, rtt/2 FIFO-clamped frames, model steps occupying
// their device for t_target / t_draft, identical tie-breaking. The difference is the model-call
// seam (sim.hpp:294-318): a step's inputs are captured when it is LAUNCHED (as the runtime does,
// runtime.hpp:336) and registered as a job; a request advances until its next event is a
// completion whose job has not run yet, then every pending job of every request runs in one
// batched GPU round, and all requests continue. Per-request decisions are therefore identical
// to the sequential reference while each GPU launch covers the whole shard.
#pragma once

#include "common.hpp"
#include "protocol.hpp"
#include "wanspec_b200.h"

#include <cstdint>
#include <random>
#include <string>
#include <vector>

namespace wsb {

// SimConfig (sim.hpp:28-80) + the extension's verify mode.
struct SimCfg {
  bool baseline = false;
  int verify = WS_VERIFY_GREEDY;
  SimTime rtt = 0, jitter = 0, r_estimate = -1, t_target = 23400, t_draft = 7500;
  std::uint32_t k = 2, b = 2, s = 4, catchup_batch_limit = 32;
  double theta = 0.5, phi = 0.5;
  std::size_t max_nodes = 64;
  bool wait_backstop = false;
  std::uint64_t sample_seed = 0;
  std::uint64_t oracle_seed = 1;
  TokenId eos = 32767;
  // wall-clock mode (host/wallclock.hpp): real time, GPU completions, injected RTT queues
  bool wallclock = false;
  std::string decision_log;  // NDJSON decision log path ("" = none; one file per protocol thread)

  ControllerCfg controller_cfg() const;  // sim.hpp:54-68
  WorkerCfg worker_cfg() const;          // sim.hpp:70-79
};

// Job / result records are the C ABI's (include/wanspec_b200.h) so the K9 kernel, the
// callback seam and the driver share one layout: a verify job is a batched run_target_step
// (oracle.hpp:127-139), a draft job a draft_prediction row (oracle.hpp:96-98).
using VerifyJob = ws_verify_job;
using DraftJob = ws_draft_job;
using VerifyOut = ws_verify_out;

// Context of a job for context-dependent (real) models: tokens ctx_tokens[off, off+len) are the
// model input after the prompt (committed tokens, then the speculative path for drafts);
// the first n_committed of them are committed.
enum JobKind : std::uint32_t { kJobVerify = 0, kJobCtrlDraft = 1, kJobWorkerDraft = 2 };
struct JobCtx {
  std::uint32_t off, len, n_committed, kind;
};

struct RoundJobs {
  std::vector<VerifyJob> verify;
  std::vector<TokenId> cands;
  std::vector<double> cand_probs;  // (want_ctx) the draft probability of each candidate (tree node)
  std::vector<DraftJob> draft;
  bool want_ctx = false;  // set by backends that need contexts (real models)
  std::vector<JobCtx> verify_ctx, draft_ctx;
  std::vector<TokenId> ctx_tokens;
  void clear() {
    verify.clear();
    cands.clear();
    cand_probs.clear();
    draft.clear();
    verify_ctx.clear();
    draft_ctx.clear();
    ctx_tokens.clear();
  }
};
struct RoundResults {
  std::vector<VerifyOut> verify;
  std::vector<ws_pred> draft;
};

struct BackendStats {
  std::uint64_t rounds = 0, launches = 0, verify_rows = 0, draft_rows = 0, h2d = 0, d2h = 0;
  double kernel_ms = 0.0;
};

// The GPU side of one protocol thread. run_round must fill res.verify / res.draft in job order.
//
// Backends may also expose two asynchronous lanes (lane 0: verify jobs on the target device,
// lane 1: draft jobs on the draft device — the reference's two devices, ControllerDevices in
// controller.hpp). The driver then runs continuous batching: a lane that goes idle takes every
// job pending at that moment, and a request resumes as soon as the results it waits on are
// back, so the target and draft forwards overlap instead of meeting at a round barrier.
// Per-request results are unchanged (each job's inputs are captured at launch and the kernels
// are batch-invariant).
class ModelBackend {
 public:
  virtual ~ModelBackend() = default;
  virtual void run_round(const RoundJobs& jobs, RoundResults& res, int verify_mode,
                         std::uint64_t sample_seed) = 0;
  virtual bool wants_context() const { return false; }
  virtual bool has_lanes() const { return false; }
  virtual int n_lanes() const { return 2; }  // lane 0: verify; lanes 1..n-1: draft
  // lane 0 reads jobs.verify/cands/verify_ctx, lane 1 jobs.draft/draft_ctx (+ ctx_tokens);
  // `jobs` must stay alive and unchanged until complete(lane). Returns how many of the lane's
  // jobs (a prefix) it took; the driver keeps the rest pending for the lane's next batch (a
  // backend may trim a batch to a tile-friendly size).
  virtual std::size_t submit(int lane, const RoundJobs& jobs, int verify_mode, std::uint64_t sample_seed);
  virtual int wait_any(std::uint32_t busy_lanes);      // blocks until a busy lane (bit) is done
  virtual int poll_any(std::uint32_t busy_lanes) { return wait_any(busy_lanes); }  // -1: none done yet
  virtual void complete(int lane, RoundResults& res);  // fills res.verify (lane 0) / res.draft
  BackendStats stats;
};

struct RequestOutput {
  ws_request_metrics metrics{};
  std::vector<TokenId> ctrl;
  std::vector<TokenId> wrk;
  std::vector<ws_step_log> steps;
};

// Runs the listed requests (global indices; table block = index) to completion through
// `backend`, one batched round at a time. Throws ConfigError / std::logic_error like the
// reference (sim.hpp:198, :200).
void run_requests(const SimCfg& cfg, const std::uint32_t* requests, std::size_t n,
                  ModelBackend& backend, RequestOutput* outs, bool log_steps);

}  // namespace wsb
