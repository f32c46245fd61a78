// Wall-clock driver (see wallclock.hpp).
#include "wallclock.hpp"

#include "wire.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <deque>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace wsb {

namespace {

using Clock = std::chrono::steady_clock;

// net.hpp:149-163 — receiver-side delay, FIFO-clamped; jitter draws as rng.hpp:44-48.
struct LatencyEmulator {
  SimTime one_way = 0, jitter = 0, last_visible = 0;
  std::mt19937_64 rng;
  SimTime visible_at(SimTime sent) {
    SimTime d = one_way;
    if (jitter > 0) {
      const std::uint64_t n = static_cast<std::uint64_t>(2 * jitter + 1);
      d += static_cast<SimTime>(rng() % n) - jitter;
    }
    if (d < 0) d = 0;
    const SimTime v = std::max(sent + d, last_visible);
    last_visible = v;
    return v;
  }
};

// A message in flight: its wire frame (host/wire.hpp, the reference's encoding) and the
// instant it becomes visible at the receiver.
struct Frame {
  SimTime visible = 0;
  std::vector<std::uint8_t> bytes;
};

// ---- decision-log NDJSON (read back by oracle/ref_shim.cpp ref_replay_model_log) ----
void put_ids(std::string& s, const std::vector<TokenId>& v) {
  s += '[';
  for (std::size_t i = 0; i < v.size(); ++i) {
    if (i) s += ',';
    s += std::to_string(v[i]);
  }
  s += ']';
}
void put_num(std::string& s, double x) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", x);
  s += b;
}
void put_msg(std::string& s, const Message& m) {
  s += "{\"kind\":" + std::to_string(static_cast<int>(m.kind)) + ",\"seq\":" + std::to_string(m.seq_no) +
       ",\"base\":" + std::to_string(m.base);
  if (m.kind == MsgKind::speculation) {
    s += ",\"path\":";
    put_ids(s, m.path);
    s += ",\"cands\":[";
    for (std::uint32_t j = 0; j < m.n_cands; ++j) {
      if (j) s += ',';
      s += "[" + std::to_string(m.cands[j].token) + ",";
      put_num(s, m.cands[j].prob);
      s += ",";
      put_num(s, m.cands[j].entropy);
      s += "]";
    }
    s += "]";
  } else if (m.kind == MsgKind::validation) {
    s += ",\"accepted\":";
    put_ids(s, m.result.accepted);
    s += ",\"bonus\":" + std::to_string(m.result.bonus) + ",\"h\":";
    put_num(s, m.result.final_entropy);
  } else if (m.kind == MsgKind::eos) {
    s += ",\"final_length\":" + std::to_string(m.final_length);
  }
  s += "}";
}

class WallRequest {
 public:
  WallRequest(const SimCfg& cfg, std::uint32_t request)
      : cfg_(cfg), ccfg_(cfg.controller_cfg()), wcfg_(cfg.worker_cfg()), request_(request) {
    const std::uint64_t seed = cfg.oracle_seed ^ (0x9e3779b97f4a7c15ULL * (static_cast<std::uint64_t>(request) + 1));
    to_ctrl_emu_ = LatencyEmulator{cfg.rtt / 2, cfg.jitter, 0, std::mt19937_64(seed ^ 0xCCULL)};
    to_wrk_emu_ = LatencyEmulator{cfg.rtt / 2, cfg.jitter, 0, std::mt19937_64(seed ^ 0x77ULL)};
  }

  void start(SimTime now) {
    start_ = now;
    ctrl_.reset(request_, now, cfg_.max_nodes);
    wrk_.reset(request_, cfg_.max_nodes);
    if (!cfg_.baseline) {  // the handshake: the worker joins half an RTT in (sim.hpp:183-190)
      Message hello;
      hello.request_id = request_;
      hello.kind = MsgKind::hello;
      send_to_worker(std::move(hello), now);
    }
    dirty_ = true;
  }

  bool finished() const { return ctrl_.finished && !devices_.any_busy(); }
  std::uint32_t request() const { return request_; }

  // Earliest future instant this request needs a turn without a GPU completion (frames).
  SimTime next_wake() const {
    SimTime t = kInfiniteTime;
    if (!to_ctrl_.empty()) t = std::min(t, to_ctrl_.front().visible);
    if (!to_wrk_.empty() && !wrk_busy_ && !wrk_done_) t = std::min(t, to_wrk_.front().visible);
    if (backstop_at_ >= 0 && !devices_.any_busy()) t = std::min(t, backstop_at_);
    return t;
  }

  // One controller turn and one worker turn at `now`; launches go to the pending batches.
  void turn(SimTime now, RoundJobs& vjobs, RoundJobs& djobs, std::vector<std::pair<WallRequest*, int>>& vslots,
            std::vector<std::pair<WallRequest*, int>>& dslots, std::string* log, std::uint64_t& turns) {
    // frames that became visible
    std::vector<Message> new_ctrl;
    while (!to_ctrl_.empty() && to_ctrl_.front().visible <= now) {
      const std::vector<std::uint8_t>& b = to_ctrl_.front().bytes;
      rd_ctrl_.feed(b.data(), b.size());  // the receiver's frame reader (FIFO seq check)
      to_ctrl_.pop_front();
      Message m;
      while (rd_ctrl_.next(m)) new_ctrl.push_back(std::move(m));
    }
    while (!to_wrk_.empty() && to_wrk_.front().visible <= now) {
      const std::vector<std::uint8_t>& b = to_wrk_.front().bytes;
      rd_wrk_.feed(b.data(), b.size());
      to_wrk_.pop_front();
      Message m;
      if (!rd_wrk_.next(m)) continue;
      if (m.kind == MsgKind::hello)
        worker_started_ = true;
      else
        inbox_wrk_.push_back(std::move(m));
      wrk_dirty_ = true;
    }
    const bool backstop_due = backstop_at_ >= 0 && now >= backstop_at_;
    if (backstop_due) backstop_at_ = -1;
    if (!new_ctrl.empty() || target_ready_ || local_ready_ || dirty_ || backstop_due) ctrl_turn(now, new_ctrl, vjobs, djobs, vslots, dslots, log, turns);
    if (!cfg_.baseline && worker_started_ && !wrk_busy_ && !wrk_done_ && (wrk_dirty_ || worker_ready_))
      worker_turn(now, djobs, dslots);
  }

  void deliver_verify(const ws_verify_out& o, SimTime now) {
    target_res_.accepted.assign(target_.tokens.begin(), target_.tokens.begin() + o.accepted);
    target_res_.bonus = o.bonus;
    target_res_.final_entropy = o.final_entropy;
    target_ready_ = true;
    (void)now;
  }
  void deliver_local(const ws_pred& p) {
    local_pred_ = to_pred(p);
    local_ready_ = true;
  }
  void deliver_worker(int i, const ws_pred& p) {
    worker_preds_[static_cast<std::size_t>(i)] = to_pred(p);
    if (++worker_delivered_ == worker_leaves_.size()) worker_ready_ = true;
  }

  void collect(RequestOutput& out) const {
    ws_request_metrics& m = out.metrics;
    m.latency = finish_time_ - start_;
    m.tokens_committed = ctrl_.committed.size();
    m.target_steps = ctrl_.counters.target_steps;
    m.ctrl_draft_passes = ctrl_.counters.draft_passes;
    m.ctrl_local_draft_steps = ctrl_.counters.local_draft_steps;
    m.ctrl_catchup_batches = ctrl_.counters.catchup_batches;
    m.worker_draft_steps = wrk_.counters.draft_steps;
    m.sync_stalls = ctrl_.counters.sync_stalls;
    m.entropy_resets = ctrl_.counters.entropy_resets;
    m.stale_specs = ctrl_.counters.stale_specs_dropped;
    out.ctrl = ctrl_.committed;
    out.wrk = wrk_.committed;
    out.steps = steps_;
  }

 private:
  static Pred to_pred(const ws_pred& p) {
    Pred q;
    q.n = p.n;
    q.id[0] = p.id[0];
    q.id[1] = p.id[1];
    q.prob[0] = p.prob[0];
    q.prob[1] = p.prob[1];
    q.entropy = p.entropy;
    return q;
  }

  void send_to_worker(Message&& m, SimTime now) {
    if (cfg_.baseline) return;
    m.seq_no = ++seq_to_worker_;
    Frame f{to_wrk_emu_.visible_at(now), {}};
    wire_encode(m, f.bytes);
    to_wrk_.push_back(std::move(f));
  }
  void send_to_ctrl(Message&& m, SimTime now) {
    m.seq_no = ++seq_to_ctrl_;
    Frame f{to_ctrl_emu_.visible_at(now), {}};
    wire_encode(m, f.bytes);
    to_ctrl_.push_back(std::move(f));
  }

  // serve_controller's loop body (runtime.hpp:262-335) for one wake-up
  void ctrl_turn(SimTime now, std::vector<Message>& frames, RoundJobs& vjobs, RoundJobs& djobs,
                 std::vector<std::pair<WallRequest*, int>>& vslots,
                 std::vector<std::pair<WallRequest*, int>>& dslots, std::string* log, std::uint64_t& turns) {
    dirty_ = false;
    ++turns;
    std::string rec;
    if (log) {
      rec = "{\"r\":" + std::to_string(request_) + ",\"now\":" + std::to_string(now);
      if (first_turn_) rec += ",\"start\":" + std::to_string(start_);
      rec += ",\"frames\":[";
      for (std::size_t i = 0; i < frames.size(); ++i) {
        if (i) rec += ',';
        put_msg(rec, frames[i]);
      }
      rec += "]";
    }
    first_turn_ = false;
    for (Message& m : frames) inbox_ctrl_.push_back(std::move(m));
    std::vector<Message> out;
    if (target_ready_) {
      target_ready_ = false;
      devices_.target_busy = false;
      if (log) {
        rec += ",\"target\":{\"base\":" + std::to_string(target_.base) + ",\"tokens\":";
        put_ids(rec, target_.tokens);
        rec += ",\"accepted\":" + std::to_string(target_res_.accepted.size()) +
               ",\"bonus\":" + std::to_string(target_res_.bonus) + ",\"h\":";
        put_num(rec, target_res_.final_entropy);
        rec += "}";
      }
      const bool was = ctrl_.finished;
      out.clear();
      apply_target_result(ctrl_, ccfg_, target_res_, now, out);
      for (Message& m : out) send_to_worker(std::move(m), now);
      if (!was && ctrl_.finished) finish_time_ = now;
      log_step(now);
    }
    if (local_ready_) {
      local_ready_ = false;
      devices_.draft_busy = false;
      if (log) {
        rec += ",\"local\":{\"anchor\":" + std::to_string(local_.anchor) + ",\"context\":";
        put_ids(rec, local_.context);
        rec += ",\"pred\":{\"n\":" + std::to_string(local_pred_.n) + ",\"id\":[" + std::to_string(local_pred_.id[0]) +
               "," + std::to_string(local_pred_.id[1]) + "],\"prob\":[";
        put_num(rec, local_pred_.prob[0]);
        rec += ",";
        put_num(rec, local_pred_.prob[1]);
        rec += "],\"h\":";
        put_num(rec, local_pred_.entropy);
        rec += "}}";
      }
      apply_local_draft(ctrl_, ccfg_, local_, local_pred_);
    }
    if (log) rec += ",\"t_update\":" + std::to_string(ctrl_.t_update);
    std::string launches;
    if (!ctrl_.finished) {
      ControllerAction act;
      for (;;) {
        controller_poll(ctrl_, ccfg_, now, inbox_ctrl_, devices_, act);
        inbox_ctrl_.clear();
        if (act.kind == ActionKind::step_target) {
          devices_.target_busy = true;
          target_ = act.target;
          VerifyJob j;
          j.seq = request_;
          j.k = static_cast<std::uint32_t>(target_.tokens.size());
          j.base = target_.base;
          j.request = request_;
          j.step = static_cast<std::uint32_t>(ctrl_.counters.target_steps);
          j.cand_off = static_cast<std::uint32_t>(vjobs.cands.size());
          vjobs.cands.insert(vjobs.cands.end(), target_.tokens.begin(), target_.tokens.end());
          vjobs.verify.push_back(j);
          if (vjobs.want_ctx) {
            for (NodeId id : target_.ids) vjobs.cand_probs.push_back(ctrl_.tree.node(id).prob);
            vjobs.verify_ctx.push_back(JobCtx{static_cast<std::uint32_t>(vjobs.ctx_tokens.size()),
                                              static_cast<std::uint32_t>(ctrl_.committed.size()),
                                              static_cast<std::uint32_t>(ctrl_.committed.size()), kJobVerify});
            vjobs.ctx_tokens.insert(vjobs.ctx_tokens.end(), ctrl_.committed.begin(), ctrl_.committed.end());
          }
          vslots.push_back({this, 0});
          if (log) {
            launches += launches.empty() ? "" : ",";
            launches += "{\"target\":{\"base\":" + std::to_string(target_.base) + ",\"tokens\":";
            put_ids(launches, target_.tokens);
            launches += "}}";
          }
          continue;
        }
        if (act.kind == ActionKind::step_draft_local) {
          devices_.draft_busy = true;
          local_ = act.local;
          djobs.draft.push_back(DraftJob{request_, 0, local_.anchor});
          if (djobs.want_ctx) {
            djobs.draft_ctx.push_back(JobCtx{static_cast<std::uint32_t>(djobs.ctx_tokens.size()),
                                             static_cast<std::uint32_t>(local_.context.size()),
                                             static_cast<std::uint32_t>(ctrl_.committed.size()), kJobCtrlDraft});
            djobs.ctx_tokens.insert(djobs.ctx_tokens.end(), local_.context.begin(), local_.context.end());
          }
          dslots.push_back({this, -1});
          if (log) {
            launches += launches.empty() ? "" : ",";
            launches += "{\"local\":{\"anchor\":" + std::to_string(local_.anchor) + ",\"context\":";
            put_ids(launches, local_.context);
            launches += "}}";
          }
          continue;
        }
        if (act.kind == ActionKind::wait && act.has_backstop) backstop_at_ = act.backstop_at;
        break;
      }
    }
    if (log) {
      rec += ",\"launch\":[" + launches + "]}\n";
      *log += rec;
    }
  }

  // serve_worker's loop body (runtime.hpp:174-199): fold finished draft outputs, then draft the
  // next frontier at once (the worker free-runs)
  void worker_turn(SimTime now, RoundJobs& djobs, std::vector<std::pair<WallRequest*, int>>& dslots) {
    wrk_dirty_ = false;
    if (worker_ready_) {
      worker_ready_ = false;
      std::vector<Message> out;
      apply_draft_output(wrk_, wcfg_, worker_leaves_, worker_preds_.data(), out);
      for (Message& m : out) send_to_ctrl(std::move(m), now);
    }
    if (!worker_poll(wrk_, wcfg_, inbox_wrk_, worker_leaves_)) {
      wrk_done_ = true;
      inbox_wrk_.clear();
      return;
    }
    inbox_wrk_.clear();
    wrk_busy_ = true;
    worker_preds_.assign(worker_leaves_.size(), Pred{});
    worker_delivered_ = 0;
    for (std::size_t i = 0; i < worker_leaves_.size(); ++i) {
      djobs.draft.push_back(DraftJob{request_, 0, worker_leaves_[i].anchor});
      if (djobs.want_ctx) {
        wrk_.tree.path_tokens(worker_leaves_[i].id, path_tmp_);
        djobs.draft_ctx.push_back(JobCtx{static_cast<std::uint32_t>(djobs.ctx_tokens.size()),
                                         static_cast<std::uint32_t>(wrk_.committed.size() + path_tmp_.size()),
                                         static_cast<std::uint32_t>(wrk_.committed.size()), kJobWorkerDraft});
        djobs.ctx_tokens.insert(djobs.ctx_tokens.end(), wrk_.committed.begin(), wrk_.committed.end());
        djobs.ctx_tokens.insert(djobs.ctx_tokens.end(), path_tmp_.begin(), path_tmp_.end());
      }
      dslots.push_back({this, static_cast<int>(i)});
    }
    if (worker_leaves_.empty()) wrk_busy_ = false;
  }

 public:
  void worker_results_in() { wrk_busy_ = false; }

 private:
  void log_step(SimTime now) {
    ws_step_log s{};
    s.request = request_;
    s.step = static_cast<std::uint32_t>(ctrl_.counters.target_steps - 1);
    s.base = target_.base;
    s.accepted = static_cast<std::uint32_t>(target_res_.accepted.size());
    s.bonus = target_res_.bonus;
    s.final_entropy = target_res_.final_entropy;
    s.time = now;
    if (target_res_.length() < ccfg_.k + 1)
      s.flags = WS_STEP_SYNC_STALL;
    else if (target_res_.final_entropy > ccfg_.phi)
      s.flags = WS_STEP_ENTROPY_RESET;
    steps_.push_back(s);
  }

  const SimCfg& cfg_;
  ControllerCfg ccfg_;
  WorkerCfg wcfg_;
  std::uint32_t request_;
  ControllerState ctrl_;
  WorkerState wrk_;
  ControllerDevices devices_;
  std::deque<Frame> to_ctrl_, to_wrk_;
  FrameReader rd_ctrl_, rd_wrk_;
  LatencyEmulator to_ctrl_emu_, to_wrk_emu_;
  std::uint64_t seq_to_ctrl_ = 0, seq_to_worker_ = 0;
  std::vector<Message> inbox_ctrl_, inbox_wrk_;
  StepTarget target_;
  Validation target_res_;
  StepDraftLocal local_;
  Pred local_pred_;
  std::vector<DraftLeaf> worker_leaves_;
  std::vector<Pred> worker_preds_;
  std::size_t worker_delivered_ = 0;
  std::vector<TokenId> path_tmp_;
  std::vector<ws_step_log> steps_;
  SimTime start_ = 0, finish_time_ = 0, backstop_at_ = -1;
  bool target_ready_ = false, local_ready_ = false, worker_ready_ = false;
  bool worker_started_ = false, wrk_busy_ = false, wrk_done_ = false;
  bool dirty_ = false, wrk_dirty_ = false, first_turn_ = true;
};

}  // namespace

void run_requests_wallclock(const SimCfg& cfg, const std::uint32_t* requests, std::size_t n, ModelBackend& backend,
                            RequestOutput* outs, const std::string& log_path, WallclockStats* stats) {
  if (!backend.has_lanes()) throw ConfigError("wall-clock mode needs a backend with asynchronous lanes");
  const int n_lanes = std::max(2, backend.n_lanes());
  std::vector<std::unique_ptr<WallRequest>> reqs;
  for (std::size_t i = 0; i < n; ++i) reqs.emplace_back(new WallRequest(cfg, requests[i]));
  RoundJobs pend_v, pend_d;
  std::vector<RoundJobs> fly(n_lanes);
  pend_v.want_ctx = pend_d.want_ctx = backend.wants_context();
  for (RoundJobs& f : fly) f.want_ctx = backend.wants_context();
  std::vector<std::pair<WallRequest*, int>> vslots, dslots;
  std::vector<std::vector<std::pair<WallRequest*, int>>> slots_fly(n_lanes);
  RoundResults res;
  std::string log_buf, *log = log_path.empty() ? nullptr : &log_buf;
  std::uint64_t turns = 0;
  std::uint32_t busy = 0;
  const auto t0 = Clock::now();
  auto now_us = [&] {
    return static_cast<SimTime>(std::chrono::duration_cast<std::chrono::microseconds>(Clock::now() - t0).count());
  };
  for (auto& r : reqs) r->start(0);
  std::vector<char> done(n, 0);
  std::size_t live = n;
  while (live > 0) {
    SimTime now = now_us();
    // fold every completed GPU step (its results are visible now)
    for (;;) {
      const int lane = busy ? backend.poll_any(busy) : -1;
      if (lane < 0) break;
      backend.complete(lane, res);
      busy &= ~(1u << lane);
      auto& sl = slots_fly[lane];
      for (std::size_t j = 0; j < sl.size(); ++j) {
        WallRequest* r = sl[j].first;
        if (lane == 0)
          r->deliver_verify(res.verify[j], now);
        else if (sl[j].second < 0)
          r->deliver_local(res.draft[j]);
        else
          r->deliver_worker(sl[j].second, res.draft[j]);
      }
      if (lane != 0)
        for (std::size_t j = 0; j < sl.size(); ++j)
          if (sl[j].second >= 0) sl[j].first->worker_results_in();
      sl.clear();
    }
    now = now_us();
    for (std::size_t i = 0; i < n; ++i) {
      if (done[i]) continue;
      reqs[i]->turn(now, pend_v, pend_d, vslots, dslots, log, turns);
      if (reqs[i]->finished()) {
        done[i] = 1;
        --live;
      }
    }
    // launch on idle lanes: every pending job (continuous batching)
    for (int lane = 1; lane < n_lanes && !pend_d.draft.empty(); ++lane) {
      if (busy & (1u << lane)) continue;
      std::swap(pend_d, fly[lane]);
      std::swap(dslots, slots_fly[lane]);
      pend_d.clear();
      dslots.clear();
      const std::size_t took = backend.submit(lane, fly[lane], cfg.verify, cfg.sample_seed);
      if (took != fly[lane].draft.size()) throw std::logic_error("wall-clock: draft batch trimmed");
      busy |= 1u << lane;
    }
    if (!(busy & 1u) && !pend_v.verify.empty()) {
      std::swap(pend_v, fly[0]);
      std::swap(vslots, slots_fly[0]);
      pend_v.clear();
      vslots.clear();
      const std::size_t took = backend.submit(0, fly[0], cfg.verify, cfg.sample_seed);
      if (took != fly[0].verify.size()) throw std::logic_error("wall-clock: verify batch trimmed");
      busy |= 1u;
    }
    if (live == 0) break;
    // sleep until the next frame becomes visible, or poll the GPU lanes
    SimTime wake = kInfiniteTime;
    for (std::size_t i = 0; i < n; ++i)
      if (!done[i]) wake = std::min(wake, reqs[i]->next_wake());
    const SimTime t = now_us();
    if (busy) {
      if (wake > t) std::this_thread::sleep_for(std::chrono::microseconds(std::min<SimTime>(wake - t, 20)));
    } else if (wake == kInfiniteTime) {
      throw std::logic_error("wall-clock: requests blocked with nothing in flight");
    } else if (wake > t) {
      std::this_thread::sleep_for(std::chrono::microseconds(std::min<SimTime>(wake - t, 1000)));
    }
  }
  while (busy) {  // in-flight worker drafts of finished requests
    const int lane = backend.wait_any(busy);
    backend.complete(lane, res);
    busy &= ~(1u << lane);
  }
  for (std::size_t i = 0; i < n; ++i) reqs[i]->collect(outs[i]);
  if (stats) {
    stats->wall_ms = static_cast<double>(now_us()) / 1e3;
    stats->turns = turns;
  }
  if (log) {
    std::FILE* f = std::fopen(log_path.c_str(), "w");
    if (!f) throw ConfigError("wall-clock: cannot write the decision log " + log_path);
    std::fwrite(log_buf.data(), 1, log_buf.size(), f);
    std::fclose(f);
  }
}

}  // namespace wsb
