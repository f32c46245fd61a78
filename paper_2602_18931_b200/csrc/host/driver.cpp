// Batched event driver; RequestRun restates RequestSim (sim.hpp:166-416) with the model-call
// seam turned into launch-time jobs (see driver.hpp).
#include "driver.hpp"
#include "wallclock.hpp"

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <unordered_map>
#include <queue>
#include <stdexcept>
#include <utility>

namespace wsb {

ControllerCfg SimCfg::controller_cfg() const {
  ControllerCfg c;
  c.k = k;
  c.rtt_estimate = baseline ? kInfiniteTime : (r_estimate < 0 ? rtt : r_estimate);
  c.phi = phi;
  c.t_target = t_target;
  c.t_draft = t_draft;
  c.catchup_batch_limit = catchup_batch_limit;
  c.max_nodes = max_nodes;
  c.eos = eos;
  c.wait_backstop = wait_backstop;
  return c;
}

WorkerCfg SimCfg::worker_cfg() const {
  WorkerCfg w;
  w.b = b;
  w.theta = theta;
  w.s = s;
  w.t_draft = t_draft;
  w.max_nodes = max_nodes;
  w.eos = eos;
  return w;
}

namespace {

// rng.hpp:20-34 (Lemire) and :44-48 over std::mt19937_64 — jitter draws only.
std::uint64_t uniform_below(std::mt19937_64& rng, std::uint64_t n) {
  std::uint64_t x = rng();
  unsigned __int128 m = static_cast<unsigned __int128>(x) * n;
  auto lo = static_cast<std::uint64_t>(m);
  if (lo < n) {
    const std::uint64_t threshold = (0 - n) % n;
    while (lo < threshold) {
      x = rng();
      m = static_cast<unsigned __int128>(x) * n;
      lo = static_cast<std::uint64_t>(m);
    }
  }
  return static_cast<std::uint64_t>(m >> 64);
}
std::int64_t uniform_jitter(std::mt19937_64& rng, std::int64_t spread) {
  if (spread <= 0) return 0;
  return static_cast<std::int64_t>(uniform_below(rng, static_cast<std::uint64_t>(2 * spread + 1))) - spread;
}

constexpr std::uint64_t kMaxEvents = 10'000'000;  // sim.hpp:220

enum class EvKind : std::uint8_t {
  frame_to_ctrl, frame_to_worker, target_done, ctrl_draft_done, worker_draft_done, wait_expiry
};

struct Event {
  SimTime time;
  std::uint64_t tie;
  EvKind kind;
  std::uint32_t msg;  // frame pool index
};
struct EventAfter {  // sim.hpp:234-239
  bool operator()(const Event& a, const Event& b) const {
    if (a.time != b.time) return a.time > b.time;
    return a.tie > b.tie;
  }
};

class RequestRun {
 public:
  RequestRun(const SimCfg& cfg, std::uint32_t request, bool log_steps)
      : cfg_(cfg),
        ccfg_(cfg.controller_cfg()),
        wcfg_(cfg.worker_cfg()),
        request_id_(request),
        jitter_rng_(cfg.oracle_seed ^ (0x9e3779b97f4a7c15ULL * (static_cast<std::uint64_t>(request) + 1))),
        log_steps_(log_steps) {
    ctrl_.reset(request, 0, cfg.max_nodes);
    wrk_.reset(request, cfg.max_nodes);
  }

  enum class Status { blocked, done };

  // Advances the virtual clock until the next event is a model completion whose job has not
  // been executed yet (jobs for everything launched are appended to `jobs`), or until done.
  Status advance(RoundJobs& vjobs, RoundJobs& djobs) {
    jobs_v_ = &vjobs;
    jobs_d_ = &djobs;
    if (!started_) {
      started_ = true;
      if (!cfg_.baseline) {  // sim.hpp:183-190: Hello starts the worker at rtt/2
        Message hello;
        hello.request_id = request_id_;
        hello.kind = MsgKind::hello;
        send_to_worker(std::move(hello), 0);
      }
      pump();
    }
    while (!done() && !queue_.empty()) {
      const Event& top = queue_.top();
      if (!ready(top.kind)) return Status::blocked;
      Event ev = queue_.top();
      queue_.pop();
      if (ev.time < now_) throw std::logic_error("sim: event scheduled in the past");
      now_ = ev.time;
      handle(ev);
      pump();
      if (++processed_ > kMaxEvents) throw std::logic_error("sim: event budget exceeded");
    }
    if (!ctrl_.finished) throw std::logic_error("sim: request did not finish");
    return Status::done;
  }

  // Result delivery from the batched round.
  void deliver_verify(const VerifyOut& r) {
    Validation& v = target_result_;
    v.accepted.assign(target_.tokens.begin(), target_.tokens.begin() + r.accepted);
    v.bonus = r.bonus;
    v.final_entropy = r.final_entropy;
    target_ready_ = true;
  }
  void deliver_local(const ws_pred& p) {
    local_result_ = to_pred(p);
    local_ready_ = true;
  }
  void deliver_worker(std::size_t i, const ws_pred& p) {
    worker_results_[i] = to_pred(p);
    if (++worker_delivered_ == worker_leaves_.size()) worker_ready_ = true;
  }

  void collect(RequestOutput& out) {
    ws_request_metrics& m = out.metrics;  // sim.hpp:202-213
    m.latency = finish_time_;
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
    out.steps = std::move(steps_);
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

  bool ready(EvKind k) const {
    switch (k) {
      case EvKind::target_done: return target_ready_;
      case EvKind::ctrl_draft_done: return local_ready_;
      case EvKind::worker_draft_done: return worker_ready_;
      default: return true;
    }
  }

  bool done() const { return ctrl_.finished && (cfg_.baseline || wrk_.finished); }  // sim.hpp:241-244

  void schedule(SimTime t, EvKind kind, std::uint32_t msg = 0) {
    queue_.push(Event{t, next_tie_++, kind, msg});
  }

  std::uint32_t park(Message&& m) {
    std::uint32_t idx;
    if (!pool_free_.empty()) {
      idx = pool_free_.back();
      pool_free_.pop_back();
      pool_[idx] = std::move(m);
    } else {
      idx = static_cast<std::uint32_t>(pool_.size());
      pool_.push_back(std::move(m));
    }
    return idx;
  }

  SimTime frame_delay() {  // sim.hpp:258-262
    SimTime d = cfg_.rtt / 2;
    if (cfg_.jitter > 0) d += uniform_jitter(jitter_rng_, cfg_.jitter);
    return d < 0 ? 0 : d;
  }

  void send_to_worker(Message&& m, SimTime now) {  // sim.hpp:264-273
    if (cfg_.baseline) return;
    m.seq_no = ++seq_to_worker_;
    SimTime t = std::max(now + frame_delay(), last_to_worker_);
    last_to_worker_ = t;
    schedule(t, EvKind::frame_to_worker, park(std::move(m)));
  }

  void send_to_ctrl(Message&& m, SimTime now) {  // sim.hpp:275-283
    m.seq_no = ++seq_to_ctrl_;
    SimTime t = std::max(now + frame_delay(), last_to_ctrl_);
    last_to_ctrl_ = t;
    schedule(t, EvKind::frame_to_ctrl, park(std::move(m)));
  }

  void handle(const Event& ev) {  // sim.hpp:285-322
    switch (ev.kind) {
      case EvKind::frame_to_ctrl:
        inbox_ctrl_.push_back(std::move(pool_[ev.msg]));
        pool_free_.push_back(ev.msg);
        break;
      case EvKind::frame_to_worker:
        if (pool_[ev.msg].kind == MsgKind::hello) worker_started_ = true;
        inbox_wrk_.push_back(std::move(pool_[ev.msg]));
        pool_free_.push_back(ev.msg);
        break;
      case EvKind::target_done: {
        devices_.target_busy = false;
        target_ready_ = false;
        const bool was_finished = ctrl_.finished;
        outbox_.clear();
        apply_target_result(ctrl_, ccfg_, target_result_, now_, outbox_);
        if (log_steps_) {
          ws_step_log s{};
          s.request = static_cast<std::uint32_t>(request_id_);
          s.step = static_cast<std::uint32_t>(ctrl_.counters.target_steps - 1);
          s.base = target_.base;
          s.accepted = static_cast<std::uint32_t>(target_result_.accepted.size());
          s.bonus = target_result_.bonus;
          s.final_entropy = target_result_.final_entropy;
          s.time = now_;
          if (target_result_.length() < ccfg_.k + 1)
            s.flags = WS_STEP_SYNC_STALL;
          else if (target_result_.final_entropy > ccfg_.phi)
            s.flags = WS_STEP_ENTROPY_RESET;
          steps_.push_back(s);
        }
        if (!was_finished && ctrl_.finished) finish_time_ = now_;
        for (Message& m : outbox_) send_to_worker(std::move(m), now_);
        break;
      }
      case EvKind::ctrl_draft_done:
        devices_.draft_busy = false;
        local_ready_ = false;
        apply_local_draft(ctrl_, ccfg_, local_, local_result_);
        break;
      case EvKind::worker_draft_done:
        wrk_busy_ = false;
        worker_ready_ = false;
        outbox_.clear();
        apply_draft_output(wrk_, wcfg_, worker_leaves_, worker_results_.data(), outbox_);
        for (Message& m : outbox_) send_to_ctrl(std::move(m), now_);
        break;
      case EvKind::wait_expiry:
        break;
    }
  }

  void pump() {  // sim.hpp:324-333
    bool progressed = true;
    while (progressed) {
      progressed = false;
      if (!ctrl_.finished) progressed |= poll_controller();
      if (!cfg_.baseline && worker_started_ && !wrk_busy_ && !wrk_.finished)
        progressed |= poll_worker();
    }
  }

  bool poll_controller() {  // sim.hpp:337-375
    bool launched = false;
    while (!(devices_.target_busy && devices_.draft_busy)) {
      inbox_tmp_.clear();
      std::swap(inbox_tmp_, inbox_ctrl_);
      controller_poll(ctrl_, ccfg_, now_, inbox_tmp_, devices_, action_);
      if (action_.kind == ActionKind::step_target) {
        devices_.target_busy = true;
        std::swap(target_, action_.target);
        // launch: register the verify job (inputs captured now, runtime.hpp:336)
        VerifyJob j;
        j.seq = static_cast<std::uint32_t>(request_id_);
        j.k = static_cast<std::uint32_t>(target_.tokens.size());
        j.base = target_.base;
        j.request = request_id_;
        j.step = static_cast<std::uint32_t>(ctrl_.counters.target_steps);
        RoundJobs& jv = *jobs_v_;
        j.cand_off = static_cast<std::uint32_t>(jv.cands.size());
        jv.cands.insert(jv.cands.end(), target_.tokens.begin(), target_.tokens.end());
        jv.verify.push_back(j);
        if (jv.want_ctx) {  // committed output (stable until this verify folds)
          for (NodeId id : target_.ids) jv.cand_probs.push_back(ctrl_.tree.node(id).prob);
          jv.verify_ctx.push_back(JobCtx{static_cast<std::uint32_t>(jv.ctx_tokens.size()),
                                         static_cast<std::uint32_t>(ctrl_.committed.size()),
                                         static_cast<std::uint32_t>(ctrl_.committed.size()), kJobVerify});
          jv.ctx_tokens.insert(jv.ctx_tokens.end(), ctrl_.committed.begin(), ctrl_.committed.end());
        }
        verify_slots_->push_back(this);
        target_ready_ = false;
        schedule(now_ + ccfg_.t_target, EvKind::target_done);
        launched = true;
        continue;
      }
      if (action_.kind == ActionKind::step_draft_local) {
        devices_.draft_busy = true;
        std::swap(local_, action_.local);
        RoundJobs& jd = *jobs_d_;
        jd.draft.push_back(DraftJob{static_cast<std::uint32_t>(request_id_), 0, local_.anchor});
        draft_slots_->push_back({this, kLocalSlot});
        if (jd.want_ctx) {  // plan.context = committed + leaf path (controller.hpp:200-201)
          jd.draft_ctx.push_back(JobCtx{static_cast<std::uint32_t>(jd.ctx_tokens.size()),
                                        static_cast<std::uint32_t>(local_.context.size()),
                                        static_cast<std::uint32_t>(ctrl_.committed.size()), kJobCtrlDraft});
          jd.ctx_tokens.insert(jd.ctx_tokens.end(), local_.context.begin(), local_.context.end());
        }
        local_ready_ = false;
        schedule(now_ + static_cast<SimTime>(local_.passes()) * ccfg_.t_draft, EvKind::ctrl_draft_done);
        launched = true;
        continue;
      }
      if (action_.kind == ActionKind::wait && action_.has_backstop &&
          action_.backstop_at != armed_backstop_) {
        armed_backstop_ = action_.backstop_at;
        schedule(action_.backstop_at, EvKind::wait_expiry);
      }
      break;  // Wait or Finish
    }
    return launched;
  }

  bool poll_worker() {  // sim.hpp:377-391
    inbox_tmp_.clear();
    std::swap(inbox_tmp_, inbox_wrk_);
    if (!worker_poll(wrk_, wcfg_, inbox_tmp_, worker_leaves_)) return false;  // WorkerFinish
    wrk_busy_ = true;
    worker_results_.resize(worker_leaves_.size());
    worker_delivered_ = 0;
    RoundJobs& jd = *jobs_d_;
    for (std::size_t i = 0; i < worker_leaves_.size(); ++i) {
      jd.draft.push_back(DraftJob{static_cast<std::uint32_t>(request_id_), 0, worker_leaves_[i].anchor});
      draft_slots_->push_back({this, static_cast<std::uint32_t>(i)});
      if (jd.want_ctx) {  // worker committed + path_tokens(leaf)
        wrk_.tree.path_tokens(worker_leaves_[i].id, path_tmp_);
        jd.draft_ctx.push_back(JobCtx{static_cast<std::uint32_t>(jd.ctx_tokens.size()),
                                      static_cast<std::uint32_t>(wrk_.committed.size() + path_tmp_.size()),
                                      static_cast<std::uint32_t>(wrk_.committed.size()), kJobWorkerDraft});
        jd.ctx_tokens.insert(jd.ctx_tokens.end(), wrk_.committed.begin(), wrk_.committed.end());
        jd.ctx_tokens.insert(jd.ctx_tokens.end(), path_tmp_.begin(), path_tmp_.end());
      }
    }
    worker_ready_ = worker_leaves_.empty();
    schedule(now_ + wcfg_.t_draft, EvKind::worker_draft_done);
    return true;
  }

 public:
  static constexpr std::uint32_t kLocalSlot = 0xFFFFFFFFu;
  struct DraftSlot {
    RequestRun* run;
    std::uint32_t which;
  };
  std::vector<RequestRun*>* verify_slots_ = nullptr;
  std::vector<DraftSlot>* draft_slots_ = nullptr;

 private:
  const SimCfg& cfg_;
  ControllerCfg ccfg_;
  WorkerCfg wcfg_;
  ControllerState ctrl_;
  WorkerState wrk_;
  std::uint64_t request_id_;
  std::mt19937_64 jitter_rng_;
  bool log_steps_;
  RoundJobs* jobs_v_ = nullptr;  // where launched verify jobs are registered
  RoundJobs* jobs_d_ = nullptr;  // ... draft jobs (the same object in lockstep mode)

  std::priority_queue<Event, std::vector<Event>, EventAfter> queue_;
  std::vector<Message> pool_;
  std::vector<std::uint32_t> pool_free_;
  std::uint64_t next_tie_ = 0;
  SimTime now_ = 0;
  SimTime finish_time_ = 0;
  ControllerDevices devices_;
  bool wrk_busy_ = false;
  bool worker_started_ = false;
  bool started_ = false;
  SimTime armed_backstop_ = -1;
  std::vector<Message> inbox_ctrl_, inbox_wrk_, inbox_tmp_, outbox_;
  std::uint64_t seq_to_worker_ = 0, seq_to_ctrl_ = 0;
  SimTime last_to_worker_ = 0, last_to_ctrl_ = 0;
  std::uint64_t processed_ = 0;
  ControllerAction action_;

  // in-flight model steps (one per device, ControllerDevices + wrk_busy_)
  StepTarget target_;
  Validation target_result_;
  bool target_ready_ = false;
  StepDraftLocal local_;
  Pred local_result_;
  bool local_ready_ = false;
  std::vector<DraftLeaf> worker_leaves_;
  std::vector<Pred> worker_results_;
  std::size_t worker_delivered_ = 0;
  bool worker_ready_ = false;

  std::vector<ws_step_log> steps_;
  std::vector<TokenId> path_tmp_;
};

// A backend took only jobs [0, took) of a lane batch: the rest go back to the (empty) pending
// list in order — they lead the lane's next batch, so nothing is deferred twice in a row.
void requeue_verify(RoundJobs& fly, std::vector<RequestRun*>& fly_slots, std::size_t took, RoundJobs& pend,
                    std::vector<RequestRun*>& pend_slots) {
  for (std::size_t j = took; j < fly.verify.size(); ++j) {
    VerifyJob v = fly.verify[j];
    const std::uint32_t off = v.cand_off;
    v.cand_off = static_cast<std::uint32_t>(pend.cands.size());
    pend.cands.insert(pend.cands.end(), fly.cands.begin() + off, fly.cands.begin() + off + v.k);
    pend.verify.push_back(v);
    if (fly.want_ctx) {
      pend.cand_probs.insert(pend.cand_probs.end(), fly.cand_probs.begin() + off, fly.cand_probs.begin() + off + v.k);
      JobCtx c = fly.verify_ctx[j];
      const std::uint32_t o = c.off;
      c.off = static_cast<std::uint32_t>(pend.ctx_tokens.size());
      pend.ctx_tokens.insert(pend.ctx_tokens.end(), fly.ctx_tokens.begin() + o, fly.ctx_tokens.begin() + o + c.len);
      pend.verify_ctx.push_back(c);
    }
    pend_slots.push_back(fly_slots[j]);
  }
  fly.verify.resize(took);
  if (fly.want_ctx) fly.verify_ctx.resize(took);
  fly_slots.resize(took);
}

void requeue_draft(RoundJobs& fly, std::vector<RequestRun::DraftSlot>& fly_slots, std::size_t took, RoundJobs& pend,
                   std::vector<RequestRun::DraftSlot>& pend_slots) {
  for (std::size_t j = took; j < fly.draft.size(); ++j) {
    pend.draft.push_back(fly.draft[j]);
    if (fly.want_ctx) {
      JobCtx c = fly.draft_ctx[j];
      const std::uint32_t o = c.off;
      c.off = static_cast<std::uint32_t>(pend.ctx_tokens.size());
      pend.ctx_tokens.insert(pend.ctx_tokens.end(), fly.ctx_tokens.begin() + o, fly.ctx_tokens.begin() + o + c.len);
      pend.draft_ctx.push_back(c);
    }
    pend_slots.push_back(fly_slots[j]);
  }
  fly.draft.resize(took);
  if (fly.want_ctx) fly.draft_ctx.resize(took);
  fly_slots.resize(took);
}

// Continuous batching over the backend's lanes (see ModelBackend): lane 0 takes verify jobs,
// lanes 1..n-1 take draft jobs — with several draft lanes the next draft batch is planned and
// launched while the previous one still runs, so the critical draft path never waits on the
// host.
void run_requests_lanes(const SimCfg& cfg, const std::uint32_t* requests, std::size_t n, ModelBackend& backend,
                        RequestOutput* outs, bool log_steps) {
  const int n_lanes = std::max(2, backend.n_lanes());
  std::vector<std::unique_ptr<RequestRun>> runs;
  runs.reserve(n);
  std::vector<RequestRun*> vslots, vslots_fly;
  std::vector<RequestRun::DraftSlot> dslots;
  std::vector<std::vector<RequestRun::DraftSlot>> dslots_fly(n_lanes);
  for (std::size_t i = 0; i < n; ++i) {
    runs.emplace_back(new RequestRun(cfg, requests[i], log_steps));
    runs.back()->verify_slots_ = &vslots;
    runs.back()->draft_slots_ = &dslots;
  }
  std::unordered_map<const RequestRun*, std::size_t> index;
  for (std::size_t i = 0; i < n; ++i) index[runs[i].get()] = i;
  RoundJobs pend_v, pend_d;
  std::vector<RoundJobs> fly(n_lanes);
  pend_v.want_ctx = pend_d.want_ctx = backend.wants_context();
  for (RoundJobs& f : fly) f.want_ctx = backend.wants_context();
  RoundResults res;
  std::vector<std::size_t> ready(n);
  for (std::size_t i = 0; i < n; ++i) ready[i] = i;
  std::vector<char> queued(n, 0);
  std::size_t live = n;
  std::uint32_t busy = 0;  // bit per lane
  auto wake = [&](RequestRun* r) {
    const std::size_t i = index[r];
    if (!queued[i]) {
      queued[i] = 1;
      ready.push_back(i);
    }
  };
  while (live > 0) {
    for (std::size_t i : ready) {
      queued[i] = 0;
      if (runs[i] && runs[i]->advance(pend_v, pend_d) == RequestRun::Status::done) {
        runs[i]->collect(outs[i]);
        runs[i].reset();
        --live;
      }
    }
    ready.clear();
    if (live == 0) break;
    for (int lane = 1; lane < n_lanes && !pend_d.draft.empty(); ++lane) {
      if (busy & (1u << lane)) continue;
      std::swap(pend_d, fly[lane]);
      std::swap(dslots, dslots_fly[lane]);
      pend_d.clear();
      dslots.clear();
      const std::size_t took = backend.submit(lane, fly[lane], cfg.verify, cfg.sample_seed);
      if (took < fly[lane].draft.size()) requeue_draft(fly[lane], dslots_fly[lane], took, pend_d, dslots);
      busy |= 1u << lane;
    }
    // Verify batching: a verify batch of fewer than vmin jobs waits while a draft batch is in
    // flight (it joins the jobs that arrive meanwhile). Config 3 on one B200: 128 → 71 verify
    // forwards per run at the same rows, +3% tokens/s (profiles/r01_driver_policy.md).
    // WS_VERIFY_MIN overrides (0: submit whenever the verify lane is idle).
    static const std::size_t vmin = [] {
      const char* e = std::getenv("WS_VERIFY_MIN");
      return e ? static_cast<std::size_t>(std::atoi(e)) : std::size_t{32};
    }();
    if (!(busy & 1u) && !pend_v.verify.empty() && (pend_v.verify.size() >= vmin || !(busy & ~1u))) {
      std::swap(pend_v, fly[0]);
      std::swap(vslots, vslots_fly);
      pend_v.clear();
      vslots.clear();
      const std::size_t took = backend.submit(0, fly[0], cfg.verify, cfg.sample_seed);
      if (took < fly[0].verify.size()) requeue_verify(fly[0], vslots_fly, took, pend_v, vslots);
      busy |= 1u;
    }
    if (!busy) throw std::logic_error("driver: requests blocked with no pending model step");
    const int lane = backend.wait_any(busy);
    backend.complete(lane, res);
    busy &= ~(1u << lane);
    if (lane == 0) {
      for (std::size_t j = 0; j < vslots_fly.size(); ++j) {
        vslots_fly[j]->deliver_verify(res.verify[j]);
        wake(vslots_fly[j]);
      }
    } else {
      for (std::size_t j = 0; j < dslots_fly[lane].size(); ++j) {
        const auto& s = dslots_fly[lane][j];
        if (s.which == RequestRun::kLocalSlot)
          s.run->deliver_local(res.draft[j]);
        else
          s.run->deliver_worker(s.which, res.draft[j]);
        wake(s.run);
      }
    }
  }
}

}  // namespace

std::size_t ModelBackend::submit(int, const RoundJobs&, int, std::uint64_t) {
  throw std::logic_error("backend has no asynchronous lanes");
}
int ModelBackend::wait_any(std::uint32_t) { throw std::logic_error("backend has no asynchronous lanes"); }
void ModelBackend::complete(int, RoundResults&) { throw std::logic_error("backend has no asynchronous lanes"); }

void run_requests(const SimCfg& cfg, const std::uint32_t* requests, std::size_t n,
                  ModelBackend& backend, RequestOutput* outs, bool log_steps) {
  if (cfg.wallclock) {
    run_requests_wallclock(cfg, requests, n, backend, outs, cfg.decision_log, nullptr);
    return;
  }
  static const bool lockstep = std::getenv("WS_LOCKSTEP") != nullptr;  // A/B switch for the bench
  if (backend.has_lanes() && !lockstep) {
    run_requests_lanes(cfg, requests, n, backend, outs, log_steps);
    return;
  }
  std::vector<std::unique_ptr<RequestRun>> runs;
  runs.reserve(n);
  std::vector<RequestRun*> verify_slots;
  std::vector<RequestRun::DraftSlot> draft_slots;
  for (std::size_t i = 0; i < n; ++i) {
    runs.emplace_back(new RequestRun(cfg, requests[i], log_steps));
    runs.back()->verify_slots_ = &verify_slots;
    runs.back()->draft_slots_ = &draft_slots;
  }
  std::vector<std::size_t> active(n);
  for (std::size_t i = 0; i < n; ++i) active[i] = i;
  RoundJobs jobs;
  jobs.want_ctx = backend.wants_context();
  RoundResults res;
  while (!active.empty()) {
    jobs.clear();
    verify_slots.clear();
    draft_slots.clear();
    std::size_t w = 0;
    for (std::size_t a = 0; a < active.size(); ++a) {
      const std::size_t i = active[a];
      if (runs[i]->advance(jobs, jobs) == RequestRun::Status::done) {
        runs[i]->collect(outs[i]);
        runs[i].reset();
      } else {
        active[w++] = i;
      }
    }
    active.resize(w);
    if (active.empty()) break;
    if (jobs.verify.empty() && jobs.draft.empty())
      throw std::logic_error("driver: requests blocked with no pending model step");
    backend.run_round(jobs, res, cfg.verify, cfg.sample_seed);
    for (std::size_t j = 0; j < verify_slots.size(); ++j) verify_slots[j]->deliver_verify(res.verify[j]);
    for (std::size_t j = 0; j < draft_slots.size(); ++j) {
      const auto& s = draft_slots[j];
      if (s.which == RequestRun::kLocalSlot)
        s.run->deliver_local(res.draft[j]);
      else
        s.run->deliver_worker(s.which, res.draft[j]);
    }
  }
}

}  // namespace wsb
