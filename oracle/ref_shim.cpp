// ORACLE — TEST INFRASTRUCTURE ONLY. Compiles the UNMODIFIED reference headers where they
// lie (/root/reference/proj/include/wanspec, via -I) into oracle/_ref/libwanspec_ref.so with
// a C ABI, so tests and bench.py's reference arm can run the reference's own
// run_sim_full / RequestSim (sim.hpp:166-442), run_target_step (oracle.hpp:127-139),
// Oracle synthesis (oracle.hpp:262-352) and entropy_of (oracle.hpp:21-33).
//
// The only interposition is at the model-call seam the reference itself names
// (SURVEY §8b): `run_target_step` at sim.hpp:297 is routed through hooked_target_step, which
// (a) logs each verify step for per-step parity and (b) in WS_VERIFY_REJECTION mode replaces
// the greedy rule by the restated rejection rule (oracle/restate.c) — the reference state
// machines, scheduler and tree stay byte-for-byte the reference's.
#include "wanspec/controller.hpp"
#include "wanspec/oracle.hpp"
#include "wanspec/worker.hpp"

#include <span>

namespace wanspec {
ValidationResult hooked_target_step(const SequenceTrace& trace, std::uint64_t base,
                                    std::span<const TokenId> candidates);
// Model mode (ref_run_sim_models): the fold-back calls at the same seam (sim.hpp:299, :306,
// :315) receive the state the real-model calls need — the controller's committed tokens, the
// local-draft plan's context, the worker tree's leaf paths — and replace the oracle's
// predictions by the caller's model before delegating to the reference's own functions.
std::vector<Message> hooked_apply_target_result(ControllerState& st, const ControllerConfig& cfg,
                                                const ValidationResult& result, SimTime now);
void hooked_apply_local_draft(ControllerState& st, const ControllerConfig& cfg, const StepDraftLocal& plan,
                              const Prediction& prediction);
std::vector<Message> hooked_apply_draft_output(WorkerState& st, const WorkerConfig& cfg,
                                               std::span<const LeafOutput> outputs);
}  // namespace wanspec
#define run_target_step hooked_target_step
#define apply_target_result hooked_apply_target_result
#define apply_local_draft hooked_apply_local_draft
#define apply_draft_output hooked_apply_draft_output
#include "wanspec/sim.hpp"
#undef run_target_step
#undef apply_target_result
#undef apply_local_draft
#undef apply_draft_output

#include "wanspec/experiment.hpp"  // after sim.hpp: its model seams stay the hooked ones (inert here)

extern "C" {
#include "restate.h"
}

#include <atomic>
#include <fstream>
#include <optional>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

namespace {

// Model callbacks of ref_run_sim_models (the caller's GPU models behind the C ABI's per-call
// boundary): the context is the tokens after the prompt — committed, then the speculative path.
typedef int (*ref_verify_fn)(void* user, std::uint32_t request, const std::uint32_t* committed, std::uint32_t n,
                             const std::uint32_t* cand, std::uint32_t k, ws_verify_out* out);
typedef int (*ref_draft_fn)(void* user, std::uint32_t request, std::uint32_t kind, const std::uint32_t* context,
                            std::uint32_t len, std::uint32_t n_committed, ws_pred* out);

struct HookCtx {
  const ws_sim_cfg* cfg = nullptr;
  std::uint64_t request = 0;
  std::uint32_t step = 0;
  std::vector<ws_step_log>* log = nullptr;
  // model mode
  ref_verify_fn verify = nullptr;
  ref_draft_fn draft = nullptr;
  void* user = nullptr;
  std::vector<wanspec::TokenId> cands;  // the pending target step's candidates (sim.hpp:297)
  std::uint64_t base = 0;
};
thread_local HookCtx g_hook;

wanspec::Prediction from_pred(const ws_pred& p) {
  wanspec::Prediction out;
  for (std::uint32_t j = 0; j < p.n && j < 2; ++j) out.top_candidates.push_back({p.id[j], p.prob[j]});
  out.entropy = p.entropy;
  return out;
}

void to_pred(const wanspec::Prediction& p, ws_pred* out) {
  std::memset(out, 0, sizeof(*out));
  out->n = static_cast<std::uint32_t>(p.top_candidates.size() > 2 ? 2 : p.top_candidates.size());
  for (std::uint32_t j = 0; j < out->n; ++j) {
    out->id[j] = p.top_candidates[j].id;
    out->prob[j] = p.top_candidates[j].prob;
  }
  out->entropy = p.entropy;
}

void to_record(const wanspec::TokenRecord& r, ws_token_record* o) {
  std::memset(o, 0, sizeof(*o));
  o->target_token = r.target_token;
  o->target_top2 = r.target_prediction.top_candidates.at(1).id;
  o->target_p1 = r.target_prediction.top_candidates.at(0).prob;
  o->target_p2 = r.target_prediction.top_candidates.at(1).prob;
  o->target_entropy = r.target_prediction.entropy;
  o->draft_top1 = r.draft_prediction.top_candidates.at(0).id;
  o->draft_top2 = r.draft_prediction.top_candidates.at(1).id;
  o->draft_p1 = r.draft_prediction.top_candidates.at(0).prob;
  o->draft_p2 = r.draft_prediction.top_candidates.at(1).prob;
  o->draft_entropy = r.draft_prediction.entropy;
}

// When set (ref_set_trace_path), runs use the reference's trace oracle on that NDJSON file
// (OracleKind::trace, oracle.hpp:258-290) instead of the stochastic tiny pair.
std::string g_trace_path;

wanspec::SimConfig to_sim(const ws_sim_cfg* c) {
  wanspec::SimConfig s;
  s.mode = c->mode == WS_MODE_BASELINE ? wanspec::SimMode::baseline : wanspec::SimMode::wanspec;
  s.rtt = c->rtt;
  s.jitter = c->jitter;
  s.r_estimate = c->r_estimate;
  s.t_target = c->t_target;
  s.t_draft = c->t_draft;
  s.k = c->k;
  s.b = c->b;
  s.s = c->s;
  s.theta = c->theta;
  s.phi = c->phi;
  s.catchup_batch_limit = c->catchup_batch_limit;
  s.max_nodes = c->max_nodes;
  s.wait_backstop = c->wait_backstop != 0;
  s.num_requests = c->num_requests;
  s.oracle.seed = c->oracle.seed;
  s.oracle.vocab_size = c->oracle.vocab_size;
  s.oracle.eos_id = c->oracle.eos_id;
  s.oracle.match_prob = c->oracle.match_prob;
  s.oracle.entropy_low = c->oracle.entropy_low;
  s.oracle.entropy_high = c->oracle.entropy_high;
  s.oracle.second_correct_prob = c->oracle.second_correct_prob;
  s.oracle.sequence_length = c->oracle.sequence_length;
  return s;
}

void set_err(char* err, std::size_t n, const char* msg) {
  if (err && n) {
    std::strncpy(err, msg, n - 1);
    err[n - 1] = 0;
  }
}

}  // namespace

namespace wanspec {
// The seam: sim.hpp:296-297 calls this at target_done.
ValidationResult hooked_target_step(const SequenceTrace& trace, std::uint64_t base,
                                    std::span<const TokenId> candidates) {
  ValidationResult v;
  const ws_sim_cfg* cfg = g_hook.cfg;
  if (cfg && cfg->verify == WS_VERIFY_REJECTION) {
    std::vector<ws_token_record> recs(trace.length());
    for (std::size_t i = 0; i < trace.length(); ++i) to_record(trace.records()[i], &recs[i]);
    std::uint32_t a = 0, bonus = 0;
    double h = 0.0;
    or_rejection_verify(recs.data(), static_cast<std::uint32_t>(recs.size()), trace.eos(),
                        cfg->oracle.vocab_size, cfg->sample_seed, g_hook.request, g_hook.step,
                        base, candidates.data(), static_cast<std::uint32_t>(candidates.size()),
                        &a, &bonus, &h);
    v.accepted.assign(candidates.begin(), candidates.begin() + a);
    v.bonus_token = bonus;
    v.final_entropy = h;
  } else {
    v = run_target_step(trace, base, candidates);  // the reference's own (oracle.hpp:127)
  }
  if (g_hook.verify) {  // model mode: the result is computed in hooked_apply_target_result
    g_hook.cands.assign(candidates.begin(), candidates.end());
    g_hook.base = base;
    return v;
  }
  if (g_hook.log && cfg) {
    ws_step_log s{};
    s.request = static_cast<std::uint32_t>(g_hook.request);
    s.step = g_hook.step;
    s.base = base;
    s.accepted = static_cast<std::uint32_t>(v.accepted.size());
    s.bonus = v.bonus_token;
    s.final_entropy = v.final_entropy;
    s.time = -1;
    // controller.hpp:246-252
    if (v.length() < cfg->k + 1)
      s.flags = WS_STEP_SYNC_STALL;
    else if (v.final_entropy > cfg->phi)
      s.flags = WS_STEP_ENTROPY_RESET;
    g_hook.log->push_back(s);
  }
  ++g_hook.step;
  return v;
}

namespace {
void log_step(const ValidationResult& v, std::uint64_t base) {
  const ws_sim_cfg* cfg = g_hook.cfg;
  if (!g_hook.log || !cfg) return;
  ws_step_log s{};
  s.request = static_cast<std::uint32_t>(g_hook.request);
  s.step = g_hook.step;
  s.base = base;
  s.accepted = static_cast<std::uint32_t>(v.accepted.size());
  s.bonus = v.bonus_token;
  s.final_entropy = v.final_entropy;
  s.time = -1;
  if (v.length() < cfg->k + 1)
    s.flags = WS_STEP_SYNC_STALL;
  else if (v.final_entropy > cfg->phi)
    s.flags = WS_STEP_ENTROPY_RESET;
  g_hook.log->push_back(s);
}
}  // namespace

std::vector<Message> hooked_apply_target_result(ControllerState& st, const ControllerConfig& cfg,
                                                const ValidationResult& result, SimTime now) {
  if (!g_hook.verify) return apply_target_result(st, cfg, result, now);
  // the model's run_target_step over committed[0, base) + the candidates captured at sim.hpp:297
  if (st.committed.size() != g_hook.base) throw std::logic_error("model seam: committed length != base");
  ws_verify_out o{};
  const auto k = static_cast<std::uint32_t>(g_hook.cands.size());
  if (g_hook.verify(g_hook.user, static_cast<std::uint32_t>(g_hook.request), st.committed.data(),
                    static_cast<std::uint32_t>(st.committed.size()), g_hook.cands.data(), k, &o) != 0)
    throw std::runtime_error("model seam: verify callback failed");
  ValidationResult v;
  v.accepted.assign(g_hook.cands.begin(), g_hook.cands.begin() + o.accepted);
  v.bonus_token = o.bonus;
  v.final_entropy = o.final_entropy;
  log_step(v, g_hook.base);
  ++g_hook.step;
  return apply_target_result(st, cfg, v, now);
}

void hooked_apply_local_draft(ControllerState& st, const ControllerConfig& cfg, const StepDraftLocal& plan,
                              const Prediction& prediction) {
  if (!g_hook.draft) return apply_local_draft(st, cfg, plan, prediction);
  ws_pred p{};
  if (g_hook.draft(g_hook.user, static_cast<std::uint32_t>(g_hook.request), WS_JOB_CTRL_DRAFT, plan.context.data(),
                   static_cast<std::uint32_t>(plan.context.size()), static_cast<std::uint32_t>(st.committed.size()),
                   &p) != 0)
    throw std::runtime_error("model seam: draft callback failed");
  apply_local_draft(st, cfg, plan, from_pred(p));
}

std::vector<Message> hooked_apply_draft_output(WorkerState& st, const WorkerConfig& cfg,
                                               std::span<const LeafOutput> outputs) {
  if (!g_hook.draft) return apply_draft_output(st, cfg, outputs);
  std::vector<LeafOutput> mine(outputs.begin(), outputs.end());
  std::vector<TokenId> ctx;
  for (LeafOutput& o : mine) {
    if (o.leaf != kRootId && !st.tree.contains(o.leaf)) continue;  // dropped by the fold anyway
    ctx = st.committed;
    const std::vector<TokenId> path = st.tree.path_tokens(o.leaf);
    ctx.insert(ctx.end(), path.begin(), path.end());
    ws_pred p{};
    if (g_hook.draft(g_hook.user, static_cast<std::uint32_t>(g_hook.request), WS_JOB_WORKER_DRAFT, ctx.data(),
                     static_cast<std::uint32_t>(ctx.size()), static_cast<std::uint32_t>(st.committed.size()), &p) != 0)
      throw std::runtime_error("model seam: draft callback failed");
    o.prediction = from_pred(p);
  }
  return apply_draft_output(st, cfg, std::span<const LeafOutput>(mine));
}

}  // namespace wanspec

extern "C" {

// The reference's own RequestSim (sim.hpp:166-416) for requests [first, first + local) of cfg,
// one at a time (sim.hpp:433), with its three model calls answered by the caller's models
// through the callbacks (the drop-in at the reference's seam). Outputs as
// ref_run_sim. Traces are still dealt from the tiny oracle (they fix sequence lengths only;
// every prediction the state machines see comes from the callbacks).
int ref_run_sim_models(const ws_sim_cfg* c, ref_verify_fn verify, ref_draft_fn draft, void* user, ws_run_out* out,
                       char* err, std::size_t errlen);

static ref_verify_fn g_verify_cb = nullptr;
static ref_draft_fn g_draft_cb = nullptr;
static void* g_cb_user = nullptr;

int ref_run_sim(const ws_sim_cfg* c, int threads, ws_run_out* out, char* err, std::size_t errlen);

int ref_run_sim_models(const ws_sim_cfg* c, ref_verify_fn verify, ref_draft_fn draft, void* user, ws_run_out* out,
                       char* err, std::size_t errlen) {
  if (!verify || !draft) {
    set_err(err, errlen, "ref_run_sim_models: null callback");
    return WS_EARG;
  }
  g_verify_cb = verify;
  g_draft_cb = draft;
  g_cb_user = user;
  const int rc = ref_run_sim(c, 1, out, err, errlen);  // callbacks are not thread-safe: one thread
  g_verify_cb = nullptr;
  g_draft_cb = nullptr;
  g_cb_user = nullptr;
  return rc;
}

// run_sim_full (sim.hpp:429-442): traces dealt in request order from one Oracle, then each
// request runs the reference RequestSim. threads > 1 partitions the shard's requests over a
// thread pool (the same independence run_sim_full relies on).
int ref_run_sim(const ws_sim_cfg* c, int threads, ws_run_out* out, char* err, std::size_t errlen) {
  try {
    wanspec::SimConfig cfg = to_sim(c);
    if (!g_trace_path.empty()) {
      cfg.oracle.kind = wanspec::OracleKind::trace;
      cfg.oracle.trace_path = g_trace_path;
    }
    cfg.validate();
    if (c->first_request >= c->num_requests) throw wanspec::ConfigError("shard out of range");
    std::uint32_t local = c->local_requests ? c->local_requests : c->num_requests - c->first_request;
    if (c->first_request + local > c->num_requests) throw wanspec::ConfigError("shard out of range");
    wanspec::Oracle oracle = wanspec::Oracle::open(cfg.oracle);
    std::vector<wanspec::SequenceTrace> traces;
    traces.reserve(c->first_request + local);
    for (std::uint32_t r = 0; r < c->first_request + local; ++r) traces.push_back(oracle.next_sequence());

    std::vector<wanspec::RequestMetrics> metrics(local);
    std::vector<std::vector<wanspec::TokenId>> couts(local), wouts(local);
    std::vector<std::vector<ws_step_log>> logs(local);
    std::vector<std::string> errors(local);
    std::atomic<std::uint32_t> next{0};
    auto work = [&] {
      for (std::uint32_t i = next.fetch_add(1); i < local; i = next.fetch_add(1)) {
        std::uint32_t r = c->first_request + i;
        g_hook.cfg = c;
        g_hook.request = r;
        g_hook.step = 0;
        g_hook.log = out && out->steps ? &logs[i] : nullptr;
        g_hook.verify = g_verify_cb;
        g_hook.draft = g_draft_cb;
        g_hook.user = g_cb_user;
        try {
          wanspec::detail::RequestSim sim(cfg, traces[r], r,
                                          cfg.oracle.seed ^ (0x9e3779b97f4a7c15ULL * (r + 1)));
          metrics[i] = sim.run();
          couts[i] = sim.controller_output();
          wouts[i] = sim.worker_output();
        } catch (const std::exception& e) {
          errors[i] = e.what();
        }
        g_hook = HookCtx{};
      }
    };
    int nt = threads < 1 ? 1 : threads;
    if (nt == 1) {
      work();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < nt; ++t) pool.emplace_back(work);
      for (auto& t : pool) t.join();
    }
    for (std::uint32_t i = 0; i < local; ++i)
      if (!errors[i].empty()) {
        set_err(err, errlen, errors[i].c_str());
        return WS_ELOGIC;
      }
    if (out) {
      std::uint64_t ns = 0;
      for (std::uint32_t i = 0; i < local; ++i) {
        const auto& m = metrics[i];
        if (out->metrics)
          out->metrics[i] = ws_request_metrics{m.latency, m.tokens_committed, m.target_steps,
                                               m.ctrl_draft_passes, m.ctrl_local_draft_steps,
                                               m.ctrl_catchup_batches, m.worker_draft_steps,
                                               m.sync_stalls, m.entropy_resets, m.stale_specs};
        auto put = [&](const std::vector<wanspec::TokenId>& v, std::uint32_t* toks,
                       std::uint32_t* lens) {
          if (!lens) return;
          lens[i] = static_cast<std::uint32_t>(v.size());
          if (toks)
            for (std::size_t j = 0; j < v.size() && j < out->max_len; ++j)
              toks[static_cast<std::size_t>(i) * out->max_len + j] = v[j];
        };
        put(couts[i], out->ctrl_tokens, out->ctrl_len);
        put(wouts[i], out->wrk_tokens, out->wrk_len);
        for (const auto& s : logs[i]) {
          if (out->steps && ns < out->max_steps) out->steps[ns] = s;
          ++ns;
        }
      }
      out->n_steps = ns;
    }
    return WS_OK;
  } catch (const wanspec::ConfigError& e) {
    set_err(err, errlen, e.what());
    return WS_ECONFIG;
  } catch (const wanspec::ProtocolError& e) {
    set_err(err, errlen, e.what());
    return WS_EPROTO;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return WS_ELOGIC;
  }
}

// Replays a wall-clock decision log (ws_run_model_wallclock, host/wallclock.hpp: one NDJSON
// line per controller turn) through the REFERENCE's controller state machine, the way
// replay_decision_log (runtime.hpp:404-454) replays a runtime recording: the same fold-in order
// and clock readings, with the logged model results standing in for the oracle (real models
// cannot be recomputed). Every step the reference launches must equal the logged launch (base +
// candidate tokens, local-draft anchor + context), and t_update after every turn must match;
// out receives the replayed committed streams and metrics of requests [first, first + local).
// Returns WS_OK, or WS_EPROTO with the first divergence in err.
int ref_replay_model_log(const ws_sim_cfg* c, const char* path, ws_run_out* out, std::uint64_t* turns, char* err,
                         std::size_t errlen) {
  try {
    wanspec::SimConfig cfg = to_sim(c);
    wanspec::ControllerConfig ccfg = cfg.controller_config();
    const std::uint32_t local = c->local_requests ? c->local_requests : c->num_requests - c->first_request;
    struct St {
      wanspec::ControllerState st;
      wanspec::ControllerDevices dev;
      std::vector<wanspec::Message> inbox;
      std::optional<wanspec::StepTarget> target;
      std::optional<wanspec::StepDraftLocal> plan;
      bool started = false;
      explicit St(std::size_t mn) : st(mn) {}
    };
    std::vector<St> rs;
    rs.reserve(local);
    for (std::uint32_t i = 0; i < local; ++i) rs.emplace_back(cfg.max_nodes);
    std::ifstream f(path);
    if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    std::string line;
    std::uint64_t n = 0;
    auto fail = [&](const std::string& what) {
      throw wanspec::ProtocolError("turn " + std::to_string(n) + ": " + what);
    };
    while (std::getline(f, line)) {
      if (line.empty()) continue;
      const nlohmann::json j = nlohmann::json::parse(line);
      const std::uint32_t r = j.at("r").get<std::uint32_t>();
      if (r < c->first_request || r >= c->first_request + local) fail("request outside the shard");
      St& q = rs[r - c->first_request];
      const wanspec::SimTime now = j.at("now").get<wanspec::SimTime>();
      if (j.contains("start")) {
        q.st.reset(r, j.at("start").get<wanspec::SimTime>(), cfg.max_nodes);
        q.dev = {};
        q.inbox.clear();
        q.started = true;
      }
      if (!q.started) fail("turn before the request start");
      for (const auto& fr : j.at("frames")) {
        wanspec::Message m;
        m.request_id = r;
        m.seq_no = fr.at("seq").get<std::uint64_t>();
        if (fr.at("kind").get<int>() != 2) fail("controller frame is not a speculation");
        wanspec::SpeculationMsg sm;
        sm.base = fr.at("base").get<std::uint64_t>();
        sm.path = fr.at("path").get<std::vector<wanspec::TokenId>>();
        for (const auto& cd : fr.at("cands"))
          sm.candidates.push_back({cd.at(0).get<wanspec::TokenId>(), cd.at(1).get<double>(), cd.at(2).get<double>()});
        m.body = std::move(sm);
        q.inbox.push_back(std::move(m));
      }
      if (j.contains("target")) {
        const auto& t = j.at("target");
        q.dev.target_busy = false;
        if (!q.target || q.target->base != t.at("base").get<std::uint64_t>() ||
            q.target->tokens() != t.at("tokens").get<std::vector<wanspec::TokenId>>())
          fail("target completion does not match the step the reference launched");
        const auto tokens = q.target->tokens();
        wanspec::ValidationResult v;
        const std::size_t a = t.at("accepted").get<std::size_t>();
        v.accepted.assign(tokens.begin(), tokens.begin() + a);
        v.bonus_token = t.at("bonus").get<wanspec::TokenId>();
        v.final_entropy = t.at("h").get<double>();
        wanspec::apply_target_result(q.st, ccfg, v, now);
        q.target.reset();
      }
      if (j.contains("local")) {
        const auto& l = j.at("local");
        q.dev.draft_busy = false;
        if (!q.plan || q.plan->anchor != l.at("anchor").get<std::uint64_t>() ||
            q.plan->context != l.at("context").get<std::vector<wanspec::TokenId>>())
          fail("local-draft completion does not match the plan the reference launched");
        const auto& pj = l.at("pred");
        wanspec::Prediction p;
        const std::uint32_t np = pj.at("n").get<std::uint32_t>();
        for (std::uint32_t i = 0; i < np && i < 2; ++i)
          p.top_candidates.push_back({pj.at("id").at(i).get<wanspec::TokenId>(), pj.at("prob").at(i).get<double>()});
        p.entropy = pj.at("h").get<double>();
        wanspec::apply_local_draft(q.st, ccfg, *q.plan, p);
        q.plan.reset();
      }
      if (q.st.t_update != j.at("t_update").get<wanspec::SimTime>()) fail("t_update differs");
      std::vector<nlohmann::json> launched;
      if (!q.st.finished) {
        for (;;) {
          wanspec::ControllerAction act = wanspec::controller_poll(q.st, ccfg, now, q.inbox, q.dev);
          q.inbox.clear();
          if (auto* t = std::get_if<wanspec::StepTarget>(&act)) {
            q.dev.target_busy = true;
            launched.push_back({{"target", {{"base", t->base}, {"tokens", t->tokens()}}}});
            q.target = std::move(*t);
          } else if (auto* d = std::get_if<wanspec::StepDraftLocal>(&act)) {
            q.dev.draft_busy = true;
            launched.push_back({{"local", {{"anchor", d->anchor}, {"context", d->context}}}});
            q.plan = std::move(*d);
          } else {
            break;
          }
        }
      }
      if (nlohmann::json(launched) != j.at("launch")) fail("launch decisions differ: " + nlohmann::json(launched).dump());
      ++n;
    }
    if (turns) *turns = n;
    if (out) {
      for (std::uint32_t i = 0; i < local; ++i) {
        const auto& st = rs[i].st;
        if (out->metrics) {
          ws_request_metrics m{};
          m.tokens_committed = st.committed.size();
          m.target_steps = st.counters.target_steps;
          m.ctrl_draft_passes = st.counters.draft_passes;
          m.ctrl_local_draft_steps = st.counters.local_draft_steps;
          m.ctrl_catchup_batches = st.counters.catchup_batches;
          m.sync_stalls = st.counters.sync_stalls;
          m.entropy_resets = st.counters.entropy_resets;
          m.stale_specs = st.counters.stale_specs_dropped;
          out->metrics[i] = m;
        }
        if (out->ctrl_len) {
          out->ctrl_len[i] = static_cast<std::uint32_t>(st.committed.size());
          if (out->ctrl_tokens)
            for (std::size_t t = 0; t < st.committed.size() && t < out->max_len; ++t)
              out->ctrl_tokens[static_cast<std::size_t>(i) * out->max_len + t] = st.committed[t];
        }
      }
    }
    return WS_OK;
  } catch (const wanspec::ProtocolError& e) {
    set_err(err, errlen, e.what());
    return WS_EPROTO;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return WS_ELOGIC;
  }
}

// The reference's experiment front-end end to end (experiment.hpp): parse_experiment on `text`,
// run_experiment with `seed` as the effective seed, and its three renderings.
int ref_experiment(const char* text, std::uint64_t seed, char* csv, std::size_t csv_len, char* per_seed,
                   std::size_t ps_len, char* manifest, std::size_t m_len, char* err, std::size_t errlen) {
  try {
    wanspec::ExperimentConfig cfg = wanspec::parse_experiment(text);
    wanspec::ExperimentResult r = wanspec::run_experiment(cfg, seed, 1);
    const std::string a = wanspec::render_csv(r), b = wanspec::render_per_seed_csv(r),
                      c = wanspec::render_manifest(r);
    if (a.size() >= csv_len || b.size() >= ps_len || c.size() >= m_len) throw std::runtime_error("buffer too small");
    std::memcpy(csv, a.c_str(), a.size() + 1);
    std::memcpy(per_seed, b.c_str(), b.size() + 1);
    std::memcpy(manifest, c.c_str(), c.size() + 1);
    return WS_OK;
  } catch (const wanspec::ParseError& e) {
    set_err(err, errlen, e.what());
    return WS_EPARSE;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return WS_ECONFIG;
  }
}

// The reference's wire codec (wire.hpp:149-280) over the flat ws_wire_msg.
int ref_wire_encode(const ws_wire_msg* m, std::uint8_t* out, std::size_t cap, std::size_t* len) {
  wanspec::Message msg;
  msg.request_id = m->request_id;
  msg.seq_no = m->seq_no;
  switch (m->kind) {
    case WS_MSG_HELLO: msg.body = wanspec::HelloMsg{m->config_digest}; break;
    case WS_MSG_SPECULATION: {
      wanspec::SpeculationMsg sm;
      sm.base = m->base;
      sm.path.assign(m->path, m->path + m->n_path);
      for (std::uint32_t i = 0; i < m->n_cands; ++i)
        sm.candidates.push_back({m->cand_token[i], m->cand_prob[i], m->cand_entropy[i]});
      msg.body = std::move(sm);
      break;
    }
    case WS_MSG_VALIDATION: {
      wanspec::ValidationMsg v;
      v.base = m->base;
      v.result.accepted.assign(m->accepted, m->accepted + m->n_accepted);
      v.result.bonus_token = m->bonus;
      v.result.final_entropy = m->final_entropy;
      msg.body = std::move(v);
      break;
    }
    case WS_MSG_EOS: msg.body = wanspec::EosMsg{m->final_length}; break;
    default: msg.body = wanspec::ByeMsg{}; break;
  }
  const std::vector<std::uint8_t> f = wanspec::encode(msg);
  if (f.size() > cap) return WS_EARG;
  std::memcpy(out, f.data(), f.size());
  *len = f.size();
  return WS_OK;
}

// decode_frame (wire.hpp:198-280): WS_OK / WS_WIRE_NEED_MORE / WS_EPROTO (+ message in err).
int ref_wire_decode(const std::uint8_t* bytes, std::size_t n, ws_wire_msg* out, std::size_t* consumed, char* err,
                    std::size_t errlen) {
  const wanspec::Decoded d = wanspec::decode_frame(std::span<const std::uint8_t>(bytes, n));
  if (d.status == wanspec::DecodeStatus::need_more) return WS_WIRE_NEED_MORE;
  if (d.status == wanspec::DecodeStatus::error) {
    set_err(err, errlen, ("wire: " + d.error).c_str());
    return WS_EPROTO;
  }
  std::memset(out, 0, sizeof(*out));
  const wanspec::Message& m = d.message;
  out->kind = static_cast<std::uint32_t>(m.kind());
  out->request_id = m.request_id;
  out->seq_no = m.seq_no;
  if (const auto* h = std::get_if<wanspec::HelloMsg>(&m.body)) out->config_digest = h->config_digest;
  if (const auto* sm = std::get_if<wanspec::SpeculationMsg>(&m.body)) {
    out->base = sm->base;
    out->n_path = static_cast<std::uint32_t>(sm->path.size());
    std::copy(sm->path.begin(), sm->path.end(), out->path);
    out->n_cands = static_cast<std::uint32_t>(sm->candidates.size());
    for (std::size_t i = 0; i < sm->candidates.size() && i < 2; ++i) {
      out->cand_token[i] = sm->candidates[i].token;
      out->cand_prob[i] = sm->candidates[i].prob;
      out->cand_entropy[i] = sm->candidates[i].entropy;
    }
  }
  if (const auto* v = std::get_if<wanspec::ValidationMsg>(&m.body)) {
    out->base = v->base;
    out->n_accepted = static_cast<std::uint32_t>(v->result.accepted.size());
    std::copy(v->result.accepted.begin(), v->result.accepted.end(), out->accepted);
    out->bonus = v->result.bonus_token;
    out->final_entropy = v->result.final_entropy;
  }
  if (const auto* e = std::get_if<wanspec::EosMsg>(&m.body)) out->final_length = e->final_length;
  *consumed = d.consumed;
  return WS_OK;
}

// Trace oracle selection for ref_run_sim / ref_trace_deal (nullptr or "" = stochastic).
void ref_set_trace_path(const char* path) { g_trace_path = path ? path : ""; }

// The reference's trace oracle over `path` (validation, seeded shuffle, oracle.hpp:183-290):
// the first n dealt sequences as records, n * max_len, positions past a sequence's length left
// zero; lens[s] = its stored length.
int ref_trace_deal(const ws_oracle_cfg* c, const char* path, std::uint32_t n, std::uint32_t max_len,
                   ws_token_record* out, std::uint32_t* lens, char* err, std::size_t errlen) {
  try {
    wanspec::OracleConfig oc;
    oc.kind = wanspec::OracleKind::trace;
    oc.trace_path = path;
    oc.seed = c->seed;
    oc.vocab_size = c->vocab_size;
    oc.eos_id = c->eos_id;
    oc.sequence_length = c->sequence_length;
    wanspec::Oracle o = wanspec::Oracle::open(oc);
    for (std::uint32_t s = 0; s < n; ++s) {
      wanspec::SequenceTrace t = o.next_sequence();
      if (t.length() > max_len) throw wanspec::ConfigError("trace sequence longer than max_len");
      lens[s] = static_cast<std::uint32_t>(t.length());
      for (std::size_t i = 0; i < t.length(); ++i)
        to_record(t.records()[i], &out[static_cast<std::size_t>(s) * max_len + i]);
    }
    return WS_OK;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return WS_ECONFIG;
  }
}

// Oracle::open + next_sequence × n (oracle.hpp:264-290).
int ref_oracle_synth(const ws_oracle_cfg* c, std::uint32_t n_seq, ws_token_record* out) {
  try {
    wanspec::OracleConfig oc;
    oc.seed = c->seed;
    oc.vocab_size = c->vocab_size;
    oc.eos_id = c->eos_id;
    oc.match_prob = c->match_prob;
    oc.entropy_low = c->entropy_low;
    oc.entropy_high = c->entropy_high;
    oc.second_correct_prob = c->second_correct_prob;
    oc.sequence_length = c->sequence_length;
    wanspec::Oracle o = wanspec::Oracle::open(oc);
    for (std::uint32_t s = 0; s < n_seq; ++s) {
      wanspec::SequenceTrace t = o.next_sequence();
      for (std::size_t i = 0; i < t.length(); ++i)
        to_record(t.records()[i], &out[static_cast<std::size_t>(s) * c->sequence_length + i]);
    }
    return WS_OK;
  } catch (const wanspec::ConfigError&) {
    return WS_ECONFIG;
  }
}

static wanspec::SequenceTrace trace_from(const ws_token_record* recs, std::uint32_t len,
                                         std::uint32_t eos) {
  std::vector<wanspec::TokenRecord> v(len);
  for (std::uint32_t i = 0; i < len; ++i) {
    const ws_token_record& r = recs[i];
    v[i].position = i;
    v[i].target_token = r.target_token;
    v[i].target_prediction.top_candidates = {{r.target_token, r.target_p1}, {r.target_top2, r.target_p2}};
    v[i].target_prediction.entropy = r.target_entropy;
    v[i].draft_prediction.top_candidates = {{r.draft_top1, r.draft_p1}, {r.draft_top2, r.draft_p2}};
    v[i].draft_prediction.entropy = r.draft_entropy;
  }
  return wanspec::SequenceTrace(std::move(v), eos);
}

// run_target_step (oracle.hpp:127-139), called directly (not through the hook).
int ref_target_step(const ws_token_record* recs, std::uint32_t len, std::uint32_t eos,
                    std::uint64_t base, const std::uint32_t* cand, std::uint32_t k,
                    std::uint32_t* acc, std::uint32_t* bonus, double* h) {
  wanspec::SequenceTrace t = trace_from(recs, len, eos);
  wanspec::ValidationResult v =
      wanspec::run_target_step(t, base, std::span<const wanspec::TokenId>(cand, k));
  *acc = static_cast<std::uint32_t>(v.accepted.size());
  *bonus = v.bonus_token;
  *h = v.final_entropy;
  return WS_OK;
}

// SequenceTrace::draft_prediction (oracle.hpp:96-98).
int ref_draft_prediction(const ws_token_record* recs, std::uint32_t len, std::uint32_t eos,
                         std::uint64_t pos, ws_pred* out) {
  wanspec::SequenceTrace t = trace_from(recs, len, eos);
  to_pred(t.draft_prediction(pos), out);
  return WS_OK;
}

// entropy_of (oracle.hpp:21-33); WS_EARG where the reference throws invalid_argument.
int ref_entropy_of(const double* p, std::size_t n, double* out) {
  try {
    *out = wanspec::entropy_of(std::span<const double>(p, n));
    return WS_OK;
  } catch (const std::invalid_argument&) {
    return WS_EARG;
  }
}

}  // extern "C"
