// C ABI of the real-model path (include/wanspec_b200.h "real-model pair").
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "context.hpp"
#include "kernels/cuda_check.hpp"
#include "model/llama.hpp"
#include "model/model_backend.hpp"
#include "wanspec_b200.h"

struct ws_model {
  std::unique_ptr<wsb::LlamaModel> m;
  int device = 0;
};

namespace {
template <class F>
int guard(const char* what, F&& f) {
  try {
    f();
    return WS_OK;
  } catch (const std::exception& e) {
    return wsb::ops_guarded_rc(what, e);
  }
}
}  // namespace

extern "C" {

int ws_model_load(ws_ctx* ctx, const ws_model_cfg* c) { return ws_model_load_split(ctx, c, -1); }

int ws_model_load_split(ws_ctx* ctx, const ws_model_cfg* c, int draft_device) {
  return guard("ws_model_load_split", [&] {
    if (!ctx || !c || !c->target || !c->draft) throw std::invalid_argument("null argument");
    wsb::ModelPairCfg m;
    m.target = c->target;
    m.draft = c->draft;
    m.seed = c->seed;
    if (c->prompt_len) m.prompt_len = c->prompt_len;
    if (c->max_requests) m.max_requests = c->max_requests;
    if (c->max_ctx) m.max_ctx = c->max_ctx;
    if (c->trie_slots) m.trie_slots = c->trie_slots;
    m.plant_target = c->plant_target;
    m.plant_draft = c->plant_draft;
    m.draft_plant_rate = c->draft_plant_rate;
    m.draft_device = draft_device;
    m.tp = c->tp > 1 ? static_cast<int>(c->tp) : 1;
    if (m.prompt_len < 1) throw wsb::ConfigError("prompt_len must be >= 1");
    if (draft_device >= 0) {
      int n = 0;
      WS_CUDA(cudaGetDeviceCount(&n));
      if (draft_device >= n) throw wsb::ConfigError("draft_device out of range");
    }
    WS_CUDA(cudaSetDevice(ctx->device));
    ctx->model_lanes.clear();
    ctx->call_backend.reset();
    ctx->models.reset();
    ctx->models.reset(new wsb::ModelPair(m, ctx->device));
  });
}

namespace {
void run_model(ws_ctx* ctx, const ws_sim_cfg* c, ws_run_out* out, bool wallclock, const char* log_path);
}

int ws_run_model_sim(ws_ctx* ctx, const ws_sim_cfg* c, ws_run_out* out) {
  return guard("ws_run_model_sim", [&] { run_model(ctx, c, out, false, nullptr); });
}

int ws_run_model_wallclock(ws_ctx* ctx, const ws_sim_cfg* c, ws_run_out* out, const char* decision_log) {
  return guard("ws_run_model_wallclock", [&] { run_model(ctx, c, out, true, decision_log); });
}

}  // extern "C"

namespace {
void run_model(ws_ctx* ctx, const ws_sim_cfg* c, ws_run_out* out, bool wallclock, const char* log_path) {
  {
    if (!ctx || !c) throw std::invalid_argument("null argument");
    if (!ctx->models) throw wsb::ConfigError("no model loaded (ws_model_load)");
    wsb::SimCfg cfg = wsb::sim_cfg_from_abi(*c);
    cfg.wallclock = wallclock;
    if (log_path) cfg.decision_log = log_path;
    if (wallclock && c->host_threads > 1 && log_path && *log_path)
      throw wsb::ConfigError("wall-clock decision log: one protocol thread only");
    wsb::ModelPair& mp = *ctx->models;
    const auto& mc = mp.cfg();
    if (c->oracle.vocab_size != static_cast<std::uint32_t>(mp.target().shape().vocab))
      throw wsb::ConfigError("oracle.vocab_size must equal the model vocabulary");
    if (c->num_requests > mc.max_requests) throw wsb::ConfigError("num_requests exceeds the loaded max_requests");
    if (mc.prompt_len + c->oracle.sequence_length + c->k + 2 > mc.max_ctx)
      throw wsb::ConfigError("prompt + sequence_length + k exceeds max_ctx");
    WS_CUDA(cudaSetDevice(ctx->device));
    mp.reset_requests();
    // prompt prefill: its own phase before the protocol starts (every verify then feeds k+1 rows)
    const std::uint32_t first = c->first_request;
    const std::uint32_t n_local = c->local_requests ? c->local_requests : c->num_requests - c->first_request;
    mp.set_pdl_late_for(n_local);
    std::vector<std::uint32_t> reqs(n_local);
    for (std::uint32_t i = 0; i < n_local; ++i) reqs[i] = first + i;
    const wsb::ModelPair::PrefillStats pre = mp.prefill_prompts(reqs.data(), reqs.size());
    const bool prof = std::getenv("WS_PROFILE") != nullptr;
    // host_threads protocol threads, each with its own backend (streams, workspaces) over a
    // contiguous range of the shard's requests: small per-thread batches still keep the GPU
    // busy because the threads' forwards run concurrently.
    const std::uint32_t local = c->local_requests ? c->local_requests : c->num_requests - c->first_request;
    const std::uint32_t threads = std::min(std::max<std::uint32_t>(1, c->host_threads), local);
    auto& owned = ctx->model_lanes;  // created once per thread index, reused across runs
    while (owned.size() < threads)
      owned.emplace_back(new wsb::ModelBackend_Llama(&mp, c->oracle.sequence_length, c->oracle.eos_id, c->k));
    std::vector<wsb::ModelBackend*> backends;
    std::vector<wsb::ModelBackend_Llama*> used;
    for (std::uint32_t t = 0; t < threads; ++t) {
      owned[t]->reset_run(c->oracle.sequence_length, c->oracle.eos_id, c->k);
      owned[t]->set_sampling(c->temperature, c->top_p);
      for (int lane = 0; lane < owned[t]->n_lanes(); ++lane) owned[t]->profiler(lane).enable(prof);
      backends.push_back(owned[t].get());
      used.push_back(owned[t].get());
    }
    wsb::run_shard_threads(c, cfg, backends, out, ctx->device);
    if (prof) {
      for (int which = 0; which < 2; ++which) {
        double ms[wsb::KernelProfiler::kClasses] = {};
        unsigned long long cnt[wsb::KernelProfiler::kClasses] = {};
        for (auto* bk : used)
          for (int lane = which; lane < (which == 0 ? 1 : bk->n_lanes()); ++lane) {
            wsb::KernelProfiler& p = bk->profiler(lane);
            p.collect();
            for (int k = 0; k < wsb::KernelProfiler::kClasses; ++k) {
              ms[k] += p.ms[k];
              cnt[k] += p.count[k];
              p.ms[k] = 0;
              p.count[k] = 0;
            }
          }
        std::fprintf(stderr, "[ws-profile] {\"model\": \"%s\"", which == 0 ? "target" : "draft");
        for (int k = 0; k < wsb::KernelProfiler::kClasses; ++k)
          std::fprintf(stderr, ", \"%s\": [%.3f, %llu]", wsb::KernelProfiler::name(k), ms[k], cnt[k]);
        std::fprintf(stderr, "}\n");
      }
    }
    ws_ctx::ModelStats st;
    std::uint64_t rows_kind[3] = {0, 0, 0}, jobs_kind[3] = {0, 0, 0};
    for (auto* bk : used) {
      st.target_ms += bk->target_ms;
      st.draft_ms += bk->draft_ms;
      st.target_rows += bk->target_rows;
      st.draft_rows += bk->draft_rows_fed;
      st.target_forwards += bk->target_forwards;
      st.draft_forwards += bk->draft_forwards;
      st.target_out_rows += bk->target_out_rows;
      st.draft_out_rows += bk->draft_out_rows;
      st.verify_kv_pos += bk->target_kv_pos();
      st.verify_attn_pairs += bk->target_attn_pairs();
      st.draft_kv_pos += bk->draft_kv_pos();
      st.draft_attn_pairs += bk->draft_attn_pairs();
      for (int k = 0; k < 3; ++k) {
        rows_kind[k] += bk->rows_by_kind[k];
        jobs_kind[k] += bk->jobs_by_kind[k];
      }
    }
    st.prefill_target_ms = pre.target_ms;
    st.prefill_draft_ms = pre.draft_ms;
    st.prefill_rows = pre.rows;
    st.prefill_forwards = pre.target_forwards;
    st.prefill_kv_pos = pre.kv_pos;
    st.prefill_attn_pairs = pre.attn_pairs;
    ctx->last_stats = st;
    if (out) {
      out->gpu_launches += pre.launches;
      out->h2d_bytes += pre.h2d;
      out->kernel_ms += pre.target_ms + pre.draft_ms;
    }
    if (std::getenv("WS_DEBUG_ROWS")) {
      std::fprintf(stderr,
                   "[ws] target rows %llu in %llu fwd (%.1f ms) | draft rows ctrl %llu / %llu jobs, worker %llu / "
                   "%llu jobs in %llu fwd (%.1f ms)\n",
                   (unsigned long long)st.target_rows, (unsigned long long)st.target_forwards, st.target_ms,
                   (unsigned long long)rows_kind[1], (unsigned long long)jobs_kind[1],
                   (unsigned long long)rows_kind[2], (unsigned long long)jobs_kind[2],
                   (unsigned long long)st.draft_forwards, st.draft_ms);
      for (auto* bk : used)
        std::fprintf(stderr, "[ws] host ms: submit verify %.1f, submit draft %.1f, wait %.1f\n", bk->host_submit_ms[0],
                     bk->host_submit_ms[1], bk->host_wait_ms);
    }
  }
}
}  // namespace

extern "C" {

int ws_model_export_trace(ws_ctx* ctx, uint32_t first_request, uint32_t n, uint32_t length, ws_token_record* out) {
  return guard("ws_model_export_trace", [&] {
    if (!ctx || !out) throw std::invalid_argument("null argument");
    if (!ctx->models) throw wsb::ConfigError("no model loaded (ws_model_load)");
    wsb::DeviceGuard dg(ctx->device);
    ctx->models->export_trace(first_request, n, length, out);
  });
}

int ws_model_stats(ws_ctx* ctx, double* target_ms, double* draft_ms, uint64_t* target_rows, uint64_t* draft_rows,
                   uint64_t* target_forwards, uint64_t* draft_forwards) {
  if (!ctx) return WS_EARG;
  const ws_ctx::ModelStats& g_last = ctx->last_stats;
  if (target_ms) *target_ms = g_last.target_ms;
  if (draft_ms) *draft_ms = g_last.draft_ms;
  if (target_rows) *target_rows = g_last.target_rows;
  if (draft_rows) *draft_rows = g_last.draft_rows;
  if (target_forwards) *target_forwards = g_last.target_forwards;
  if (draft_forwards) *draft_forwards = g_last.draft_forwards;
  return WS_OK;
}

int ws_model_open(ws_ctx* ctx, uint32_t k, uint32_t sequence_length, uint32_t eos_id) {
  return guard("ws_model_open", [&] {
    if (!ctx) throw std::invalid_argument("null argument");
    if (!ctx->models) throw wsb::ConfigError("no model loaded (ws_model_load)");
    if (k < 1 || sequence_length < 1) throw wsb::ConfigError("k and sequence_length must be >= 1");
    wsb::DeviceGuard dg(ctx->device);
    wsb::ModelPair& mp = *ctx->models;
    if (mp.cfg().prompt_len + sequence_length + k + 2 > mp.cfg().max_ctx)
      throw wsb::ConfigError("prompt + sequence_length + k exceeds max_ctx");
    mp.reset_requests();
    if (!ctx->call_backend) ctx->call_backend.reset(new wsb::ModelBackend_Llama(&mp, sequence_length, eos_id, k));
    ctx->call_backend->reset_run(sequence_length, eos_id, k);
    ctx->call_k = k;
  });
}

int ws_model_prefill(ws_ctx* ctx, uint32_t n, const uint32_t* requests) {
  return guard("ws_model_prefill", [&] {
    if (!ctx || (n && !requests)) throw std::invalid_argument("null argument");
    if (!ctx->call_backend) throw wsb::ConfigError("no per-call session (ws_model_open)");
    for (uint32_t i = 0; i < n; ++i)
      if (requests[i] >= ctx->models->cfg().max_requests) throw std::invalid_argument("request out of range");
    wsb::DeviceGuard dg(ctx->device);
    ctx->models->prefill_prompts(requests, n);
  });
}

namespace {
// One lane's batch through the per-call backend: submit (until every job is taken), wait, fold.
void call_lane(ws_ctx* ctx, int lane, wsb::RoundJobs& jobs, wsb::RoundResults& res) {
  wsb::ModelBackend_Llama& bk = *ctx->call_backend;
  const std::size_t took = bk.submit(lane, jobs, WS_VERIFY_GREEDY, 0);
  const std::size_t n = lane == 0 ? jobs.verify.size() : jobs.draft.size();
  if (took != n) throw std::logic_error("per-call batch was trimmed (unset WS_VERIFY_TRIM)");
  while (bk.wait_any(1u << lane) != lane) {
  }
  bk.complete(lane, res);
}

void check_jobs(ws_ctx* ctx, uint32_t n, const ws_model_job* jobs, const uint32_t* tokens, bool verify) {
  if (!ctx || (n && (!jobs || !tokens))) throw std::invalid_argument("null argument");
  if (!ctx->call_backend) throw wsb::ConfigError("no per-call session (ws_model_open)");
  for (uint32_t j = 0; j < n; ++j) {
    const ws_model_job& q = jobs[j];
    if (q.request >= ctx->models->cfg().max_requests) throw std::invalid_argument("request out of range");
    if (verify ? (q.kind != WS_JOB_VERIFY || q.len != q.n_committed)
               : (q.kind != WS_JOB_CTRL_DRAFT && q.kind != WS_JOB_WORKER_DRAFT) || q.n_committed > q.len)
      throw std::invalid_argument("bad job kind / lengths");
  }
}

void fill_tokens(wsb::RoundJobs& r, uint32_t n, const ws_model_job* jobs, const uint32_t* tokens) {
  std::uint64_t end = 0;
  for (uint32_t j = 0; j < n; ++j) end = std::max<std::uint64_t>(end, jobs[j].off + jobs[j].len);
  r.ctx_tokens.assign(tokens, tokens + end);
}
}  // namespace

int ws_model_verify(ws_ctx* ctx, uint32_t n, const ws_model_job* jobs, const uint32_t* tokens, const uint32_t* cand,
                    ws_verify_out* out, ws_pred* rows_opt) {
  return guard("ws_model_verify", [&] {
    check_jobs(ctx, n, jobs, tokens, true);
    if (n && (!cand || !out)) throw std::invalid_argument("null argument");
    if (!n) return;
    wsb::DeviceGuard dg(ctx->device);
    const uint32_t k = ctx->call_k;
    wsb::RoundJobs r;
    r.want_ctx = true;
    fill_tokens(r, n, jobs, tokens);
    for (uint32_t j = 0; j < n; ++j) {
      const ws_model_job& q = jobs[j];
      r.verify.push_back(ws_verify_job{q.request, k, q.n_committed, q.request, 0, j * k});
      r.verify_ctx.push_back(wsb::JobCtx{static_cast<std::uint32_t>(q.off), q.len, q.n_committed, wsb::kJobVerify});
    }
    r.cands.assign(cand, cand + static_cast<std::size_t>(n) * k);
    wsb::RoundResults res;
    call_lane(ctx, 0, r, res);
    std::memcpy(out, res.verify.data(), n * sizeof(ws_verify_out));
    if (rows_opt) ctx->call_backend->verify_rows(rows_opt, static_cast<std::size_t>(n) * (k + 1));
  });
}

int ws_model_draft(ws_ctx* ctx, uint32_t n, const ws_model_job* jobs, const uint32_t* tokens, ws_pred* out) {
  return guard("ws_model_draft", [&] {
    check_jobs(ctx, n, jobs, tokens, false);
    if (n && !out) throw std::invalid_argument("null argument");
    if (!n) return;
    wsb::DeviceGuard dg(ctx->device);
    wsb::RoundJobs r;
    r.want_ctx = true;
    fill_tokens(r, n, jobs, tokens);
    for (uint32_t j = 0; j < n; ++j) {
      const ws_model_job& q = jobs[j];
      r.draft.push_back(ws_draft_job{q.request, 0, q.len});
      r.draft_ctx.push_back(wsb::JobCtx{static_cast<std::uint32_t>(q.off), q.len, q.n_committed, q.kind});
    }
    wsb::RoundResults res;
    call_lane(ctx, 1, r, res);
    std::memcpy(out, res.draft.data(), n * sizeof(ws_pred));
  });
}

int ws_model_evict(ws_ctx* ctx, uint32_t request) {
  return guard("ws_model_evict", [&] {
    if (!ctx) throw std::invalid_argument("null argument");
    if (!ctx->models) throw wsb::ConfigError("no model loaded (ws_model_load)");
    ctx->models->evict(request);
  });
}

int ws_model_run_stats(ws_ctx* ctx, ws_run_stats* o) {
  return guard("ws_model_run_stats", [&] {
    if (!ctx || !o) throw std::invalid_argument("null argument");
    const ws_ctx::ModelStats& s = ctx->last_stats;
    o->verify_ms = s.target_ms;
    o->draft_ms = s.draft_ms;
    o->prefill_target_ms = s.prefill_target_ms;
    o->prefill_draft_ms = s.prefill_draft_ms;
    o->verify_rows = s.target_rows;
    o->verify_out_rows = s.target_out_rows;
    o->verify_forwards = s.target_forwards;
    o->draft_rows = s.draft_rows;
    o->draft_out_rows = s.draft_out_rows;
    o->draft_forwards = s.draft_forwards;
    o->prefill_rows = s.prefill_rows;
    o->prefill_forwards = s.prefill_forwards;
    o->verify_kv_pos = s.verify_kv_pos;
    o->verify_attn_pairs = s.verify_attn_pairs;
    o->draft_kv_pos = s.draft_kv_pos;
    o->draft_attn_pairs = s.draft_attn_pairs;
    o->prefill_kv_pos = s.prefill_kv_pos;
    o->prefill_attn_pairs = s.prefill_attn_pairs;
  });
}

int ws_model_create_tp(const char* shape, uint64_t seed, int64_t n_slots, int max_rows, int device, int tp,
                       ws_model** out) {
  return guard("ws_model_create", [&] {
    if (!shape || !out || n_slots <= 0) throw std::invalid_argument("bad argument");
    auto h = std::make_unique<ws_model>();
    h->device = device;
    h->m.reset(new wsb::LlamaModel(wsb::shape_by_name(shape), seed, n_slots, max_rows > 0 ? max_rows : 64, device,
                                   tp > 1 ? tp : 1));
    *out = h.release();
  });
}

int ws_model_create(const char* shape, uint64_t seed, int64_t n_slots, int max_rows, int device, ws_model** out) {
  return ws_model_create_tp(shape, seed, n_slots, max_rows, device, 1, out);
}

int ws_model_destroy(ws_model* m) {
  delete m;
  return WS_OK;
}

int ws_model_copy_weight(ws_model* m, const char* which, int layer, void* dst, int64_t numel) {
  return guard("ws_model_copy_weight", [&] {
    std::int64_t n = 0;
    void* src = m->m->weight(which, layer, &n);
    if (n != numel) throw std::invalid_argument("numel mismatch: expected " + std::to_string(n));
    WS_CUDA(cudaMemcpy(dst, src, static_cast<std::size_t>(n) * 2, cudaMemcpyDeviceToDevice));
  });
}

int ws_model_forward(ws_model* m, int n_rows, const int32_t* tok, const int32_t* pos, const int32_t* slot,
                     int n_groups, const int32_t* groups, int n_extra, const int32_t* extra,
                     const uint64_t* row_mask, int n_out, const int32_t* out_rows, void* logits_out, void* stream) {
  return guard("ws_model_forward", [&] {
    if (!m || n_rows <= 0 || !tok || !pos || !slot || !groups || n_groups <= 0) throw std::invalid_argument("bad argument");
    WS_CUDA(cudaSetDevice(m->device));
    wsb::ForwardBatch b;
    b.tok.assign(tok, tok + n_rows);
    b.pos.assign(pos, pos + n_rows);
    b.slot.assign(slot, slot + n_rows);
    for (int g = 0; g < n_groups; ++g) {
      const int32_t* q = groups + 7 * g;
      if (q[6] && q[5] > 64) throw std::invalid_argument("masked group with more than 64 extras");
      b.groups.push_back(wsb::AttnGroup{q[0], q[1], q[2], q[3], q[4], q[5], q[6] ? 1 : 0, 0});
    }
    b.row_mask.assign(n_rows, 0ull);
    if (row_mask)
      for (int i = 0; i < n_rows; ++i) b.row_mask[i] = row_mask[i];
    if (n_extra > 0) b.extra.assign(extra, extra + n_extra);
    if (n_out > 0) b.out_rows.assign(out_rows, out_rows + n_out);
    for (int i = 0; i < n_rows; ++i)
      if (slot[i] < 0 || slot[i] >= m->m->n_slots()) throw std::invalid_argument("slot out of range");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    m->m->forward(b, 0.f, st);
    if (n_out > 0 && logits_out)
      WS_CUDA(cudaMemcpyAsync(logits_out, m->m->logits(),
                              static_cast<std::size_t>(n_out) * m->m->shape().vocab * 2, cudaMemcpyDeviceToDevice, st));
    WS_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
