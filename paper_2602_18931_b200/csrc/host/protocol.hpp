// Controller (Algorithm 1) and worker (Algorithm 2) state machines: the reference's
// controller/worker interface (controller.hpp, worker.hpp) restated over the flat SpecTree.
// Pure state machines: the driver owns the clock, launches model steps on the GPU and folds
// the results back through apply_*.
#pragma once

#include "common.hpp"
#include "spectree.hpp"

#include <cstdint>
#include <vector>

namespace wsb {

// controller.hpp:21-40
struct ControllerCfg {
  std::uint32_t k = 2;
  SimTime rtt_estimate = 0;
  double phi = 0.5;
  SimTime t_target = 23400;
  SimTime t_draft = 7500;
  std::uint32_t catchup_batch_limit = 32;
  std::size_t max_nodes = 64;
  TokenId eos = 32767;
  bool wait_backstop = false;
  void validate() const;
};

// controller.hpp:42-51
struct ControllerCounters {
  std::uint64_t target_steps = 0;
  std::uint64_t local_draft_steps = 0;
  std::uint64_t catchup_batches = 0;
  std::uint64_t draft_passes = 0;
  std::uint64_t sync_stalls = 0;
  std::uint64_t entropy_resets = 0;
  std::uint64_t stale_specs_dropped = 0;
  std::uint64_t stale_local_drafts = 0;
};

// controller.hpp:53-78
struct ControllerState {
  SpecTree tree;
  std::vector<TokenId> committed;
  bool finished = false;
  SimTime t_update = 0;
  std::vector<TokenId> draft_context;
  SimTime wait_since = -1;
  std::uint64_t request_id = 0;
  ControllerCounters counters;
  void reset(std::uint64_t request, SimTime now, std::size_t max_nodes);
};

// controller.hpp:93-103 — the verify job the target GPU runs.
struct StepTarget {
  std::uint64_t base = 0;
  std::vector<NodeId> ids;
  std::vector<TokenId> tokens;
};

// controller.hpp:105-115; catchup_plan (:83-91) kept as (lag, limit): passes = ceil(lag/limit),
// at least one.
struct StepDraftLocal {
  NodeId leaf = kRootId;
  std::uint64_t anchor = 0;
  std::uint64_t lag = 0;
  std::uint32_t limit = 32;
  std::vector<TokenId> context;
  std::uint64_t passes() const { return lag == 0 ? 1 : (lag + limit - 1) / limit; }
};

enum class ActionKind { step_target, step_draft_local, wait, finish };

// controller.hpp:117-126
struct ControllerAction {
  ActionKind kind = ActionKind::wait;
  StepTarget target;
  StepDraftLocal local;
  SimTime wait_until = 0;
  bool has_backstop = false;
  SimTime backstop_at = 0;
  std::uint64_t final_length = 0;
};

// controller.hpp:132-137
struct ControllerDevices {
  bool target_busy = false;
  bool draft_busy = false;
  bool any_busy() const { return target_busy || draft_busy; }
};

// controller.hpp:167-230. `inbox` is consumed (messages may be moved from).
void controller_poll(ControllerState& st, const ControllerCfg& cfg, SimTime now,
                     std::vector<Message>& inbox, ControllerDevices devices, ControllerAction& out);

// controller.hpp:235-266. Appends the Validation (and Eos) messages to `out`.
void apply_target_result(ControllerState& st, const ControllerCfg& cfg, const Validation& result,
                         SimTime now, std::vector<Message>& out);

// controller.hpp:273-288
void apply_local_draft(ControllerState& st, const ControllerCfg& cfg, const StepDraftLocal& plan,
                       const Pred& prediction);

// worker.hpp:20-33
struct WorkerCfg {
  std::uint32_t b = 2;
  double theta = 0.5;
  std::uint32_t s = 4;
  SimTime t_draft = 7500;
  std::size_t max_nodes = 64;
  TokenId eos = 32767;
  void validate() const;
};

// worker.hpp:35-41
struct WorkerCounters {
  std::uint64_t draft_steps = 0;
  std::uint64_t speculations_sent = 0;
  std::uint64_t prunes_applied = 0;
  std::uint64_t branches = 0;
  std::uint64_t stale_outputs_dropped = 0;
};

// worker.hpp:43-58
struct WorkerState {
  SpecTree tree;
  std::vector<TokenId> committed;
  bool finished = false;
  std::uint64_t request_id = 0;
  WorkerCounters counters;
  void reset(std::uint64_t request, std::size_t max_nodes);
};

// worker.hpp:60-66
struct DraftLeaf {
  NodeId id = kRootId;
  std::uint64_t anchor = 0;
};

// worker.hpp:75-97: returns false (WorkerFinish) or fills `leaves` (StepDraft).
bool worker_poll(WorkerState& st, const WorkerCfg& cfg, std::vector<Message>& inbox,
                 std::vector<DraftLeaf>& leaves);

// worker.hpp:110-141 — the entropy-triggered branch policy (θ, b). preds[i] is the draft
// prediction for leaves[i].
void apply_draft_output(WorkerState& st, const WorkerCfg& cfg, const std::vector<DraftLeaf>& leaves,
                        const Pred* preds, std::vector<Message>& out);

// oracle.hpp:356-363
inline void commit_tokens(std::vector<TokenId>& committed, bool& finished, const Validation& v,
                          TokenId eos) {
  const std::size_t n = v.accepted.size() + 1;
  for (std::size_t i = 0; i < n; ++i) {
    if (finished) return;
    const TokenId t = i < v.accepted.size() ? v.accepted[i] : v.bonus;
    committed.push_back(t);
    if (t == eos) finished = true;
  }
}

}  // namespace wsb
