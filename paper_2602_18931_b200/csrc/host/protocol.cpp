// Controller / worker state machines; each function cites the reference lines it restates.
#include "protocol.hpp"

#include <utility>

namespace wsb {

// controller.hpp:32-39
void ControllerCfg::validate() const {
  if (k < 1) throw ConfigError("controller: k must be >= 1");
  if (rtt_estimate < 0) throw ConfigError("controller: R must be >= 0");
  if (t_target <= 0 || t_draft <= 0) throw ConfigError("controller: step durations must be > 0");
  if (catchup_batch_limit < 1) throw ConfigError("controller: catchup_batch_limit must be >= 1");
}

// controller.hpp:67-75
void ControllerState::reset(std::uint64_t request, SimTime now, std::size_t max_nodes) {
  tree.reset(max_nodes);
  committed.clear();
  finished = false;
  t_update = now;
  draft_context.clear();
  wait_since = -1;
  request_id = request;
  counters = ControllerCounters{};
}

namespace {

// controller.hpp:145-156 — content-addressed anchor resolution.
bool resolve_speculation(const SpecTree& tree, const std::vector<TokenId>& committed,
                         const Message& s, NodeId* parent) {
  const std::uint64_t here = tree.committed_len();
  if (s.base > here) return false;
  const std::uint64_t overlap = here - s.base;
  if (s.path.size() < overlap) return false;
  for (std::uint64_t i = 0; i < overlap; ++i)
    if (s.path[i] != committed[s.base + i]) return false;
  return tree.resolve_path(s.path.data() + overlap, s.path.size() - overlap, parent);
}

// controller.hpp:194-209 (plan_local) with catchup_plan (:83-91) folded into (lag, limit).
void plan_local(ControllerState& st, const ControllerCfg& cfg, ControllerAction& out) {
  st.wait_since = -1;
  NodeId leaf;
  st.tree.frontier(1, &leaf);
  StepDraftLocal& plan = out.local;
  plan.leaf = leaf;
  plan.anchor = st.tree.extension_position(leaf);
  plan.context = st.committed;
  static thread_local std::vector<TokenId> path;
  st.tree.path_tokens(leaf, path);
  plan.context.insert(plan.context.end(), path.begin(), path.end());
  std::size_t lcp = 0;
  while (lcp < plan.context.size() && lcp < st.draft_context.size() &&
         plan.context[lcp] == st.draft_context[lcp])
    ++lcp;
  plan.lag = plan.context.size() - lcp;
  plan.limit = cfg.catchup_batch_limit;
  out.kind = ActionKind::step_draft_local;
}

}  // namespace

// controller.hpp:167-230
void controller_poll(ControllerState& st, const ControllerCfg& cfg, SimTime now,
                     std::vector<Message>& inbox, ControllerDevices devices, ControllerAction& out) {
  for (Message& m : inbox) {
    if (m.kind != MsgKind::speculation || st.finished || m.request_id != st.request_id) continue;
    NodeId parent;
    if (!resolve_speculation(st.tree, st.committed, m, &parent)) {
      ++st.counters.stale_specs_dropped;
      continue;
    }
    if (!st.tree.append(parent, m.cands, m.n_cands, Origin::worker)) ++st.counters.stale_specs_dropped;
  }
  out.has_backstop = false;

  if (st.finished) {
    st.wait_since = -1;
    out.kind = ActionKind::finish;
    out.final_length = st.committed.size();
    return;
  }

  if (!devices.target_busy) {
    out.target.ids.resize(cfg.k);
    out.target.tokens.resize(cfg.k);
    if (st.tree.best_path(cfg.k, out.target.ids.data(), out.target.tokens.data())) {
      st.wait_since = -1;
      out.kind = ActionKind::step_target;
      out.target.base = st.tree.committed_len();
      return;
    }
  }

  if (!devices.draft_busy && st.tree.depth() < cfg.k && sat_add(st.t_update, cfg.rtt_estimate) > now) {
    plan_local(st, cfg, out);
    return;
  }

  out.kind = ActionKind::wait;
  out.wait_until = sat_add(st.t_update, cfg.rtt_estimate);
  if (devices.any_busy()) {
    st.wait_since = -1;  // a step is running: progress, not a stall
    return;
  }
  if (st.wait_since < 0) st.wait_since = now;
  if (cfg.wait_backstop && cfg.rtt_estimate > 0) {
    // 3 * R wraps like the reference's signed product for R = kInfiniteTime.
    const SimTime three_r = static_cast<SimTime>(3ull * static_cast<std::uint64_t>(cfg.rtt_estimate));
    const SimTime deadline = sat_add(st.wait_since, three_r);
    if (now >= deadline) {
      plan_local(st, cfg, out);
      return;
    }
    out.has_backstop = true;
    out.backstop_at = deadline;
  }
}

// controller.hpp:235-266
void apply_target_result(ControllerState& st, const ControllerCfg& cfg, const Validation& result,
                         SimTime now, std::vector<Message>& out) {
  const std::uint64_t base = st.tree.committed_len();
  commit_tokens(st.committed, st.finished, result, cfg.eos);
  st.tree.prune(result);

  ++st.counters.target_steps;
  if (result.length() < cfg.k + 1) {  // resync-on-mismatch
    st.t_update = now;
    ++st.counters.sync_stalls;
  } else if (result.final_entropy > cfg.phi) {  // φ staleness clock
    st.t_update = now;
    ++st.counters.entropy_resets;
  }

  Message v;
  v.request_id = st.request_id;
  v.kind = MsgKind::validation;
  v.base = base;
  v.result = result;
  out.push_back(std::move(v));
  if (st.finished) {
    Message e;
    e.request_id = st.request_id;
    e.kind = MsgKind::eos;
    e.final_length = st.committed.size();
    out.push_back(std::move(e));
  }
}

// controller.hpp:273-288
void apply_local_draft(ControllerState& st, const ControllerCfg&, const StepDraftLocal& plan,
                       const Pred& prediction) {
  ++st.counters.local_draft_steps;
  st.counters.catchup_batches += plan.passes() - 1;
  st.counters.draft_passes += plan.passes();
  st.draft_context = plan.context;
  const bool leaf_live = plan.leaf == kRootId ? true : st.tree.contains(plan.leaf);
  if (!leaf_live || st.tree.extension_position(plan.leaf) != plan.anchor) {
    ++st.counters.stale_local_drafts;
    return;
  }
  CandIn c{prediction.id[0], prediction.prob[0], prediction.entropy};
  st.tree.append(plan.leaf, &c, 1, Origin::controller);
}

// worker.hpp:28-32
void WorkerCfg::validate() const {
  if (b < 1 || b > 2) throw ConfigError("worker: b must be 1 or 2");
  if (s < 1) throw ConfigError("worker: s must be >= 1");
  if (t_draft <= 0) throw ConfigError("worker: t_draft must be > 0");
}

// worker.hpp:52-57
void WorkerState::reset(std::uint64_t request, std::size_t max_nodes) {
  tree.reset(max_nodes);
  committed.clear();
  finished = false;
  request_id = request;
  counters = WorkerCounters{};
}

// worker.hpp:75-97
bool worker_poll(WorkerState& st, const WorkerCfg& cfg, std::vector<Message>& inbox,
                 std::vector<DraftLeaf>& leaves) {
  for (const Message& m : inbox) {
    if (m.request_id != st.request_id) continue;
    if (m.kind == MsgKind::validation) {
      if (m.base != st.tree.committed_len()) continue;  // duplicate or out of date
      commit_tokens(st.committed, st.finished, m.result, cfg.eos);
      st.tree.prune(m.result);
      ++st.counters.prunes_applied;
    } else if (m.kind == MsgKind::eos) {
      st.finished = true;
    }
  }
  if (st.finished) return false;
  NodeId ids[64];
  std::vector<NodeId> big;
  NodeId* dst = ids;
  if (cfg.s > 64) {
    big.resize(cfg.s);
    dst = big.data();
  }
  const std::size_t n = st.tree.frontier(cfg.s, dst);
  leaves.resize(n);
  for (std::size_t i = 0; i < n; ++i) leaves[i] = DraftLeaf{dst[i], st.tree.extension_position(dst[i])};
  return true;
}

// worker.hpp:110-141
void apply_draft_output(WorkerState& st, const WorkerCfg& cfg, const std::vector<DraftLeaf>& leaves,
                        const Pred* preds, std::vector<Message>& out) {
  ++st.counters.draft_steps;
  for (std::size_t i = 0; i < leaves.size(); ++i) {
    const DraftLeaf& o = leaves[i];
    if (o.id != kRootId && !st.tree.contains(o.id)) {
      ++st.counters.stale_outputs_dropped;
      continue;
    }
    const Pred& p = preds[i];
    Message m;
    m.request_id = st.request_id;
    m.kind = MsgKind::speculation;
    m.cands[0] = CandIn{p.id[0], p.prob[0], p.entropy};
    m.n_cands = 1;
    if (cfg.b >= 2 && p.entropy >= cfg.theta && p.n >= 2) {  // branch gate worker.hpp:122-125
      m.cands[1] = CandIn{p.id[1], p.prob[1], p.entropy};
      m.n_cands = 2;
      ++st.counters.branches;
    }
    m.base = st.tree.committed_len();
    st.tree.path_tokens(o.id, m.path);
    if (!st.tree.append(o.id, m.cands, m.n_cands, Origin::worker)) {
      ++st.counters.stale_outputs_dropped;
      continue;
    }
    out.push_back(std::move(m));
    ++st.counters.speculations_sent;
  }
}

}  // namespace wsb
