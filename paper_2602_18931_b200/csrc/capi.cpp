// C ABI (include/wanspec_b200.h). Exceptions never cross the boundary: every entry point maps
// the reference's error classes (types.hpp:35-45, sim.hpp:198/:200) onto WS_E* codes and keeps
// the message in a thread-local buffer (ws_last_error).
#include "wanspec_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "host/driver.hpp"
#include "host/tinypair.hpp"
#include "kernels/cuda_check.hpp"
#include "kernels/k9_oracle.cuh"

#include "context.hpp"
#include "host/wire.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    g_err.clear();
    f();
    return WS_OK;
  } catch (const wsb::ConfigError& e) {
    g_err = e.what();
    return WS_ECONFIG;
  } catch (const wsb::ProtocolError& e) {
    g_err = e.what();
    return WS_EPROTO;
  } catch (const wsb::CudaError& e) {
    g_err = e.what();
    return WS_ECUDA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return WS_EARG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return WS_ELOGIC;
  }
}

void need(bool cond, const char* what) {
  if (!cond) throw std::invalid_argument(what);
}

// SimConfig::validate (sim.hpp:46-52) + conversion.
wsb::SimCfg to_cfg(const ws_sim_cfg& c) {
  if (c.rtt < 0 || c.jitter < 0) throw wsb::ConfigError("sim: delays must be >= 0");
  if (c.num_requests < 1) throw wsb::ConfigError("sim: num_requests must be >= 1");
  if (c.verify != WS_VERIFY_GREEDY && c.verify != WS_VERIFY_REJECTION)
    throw wsb::ConfigError("sim: unknown verify mode");
  wsb::SimCfg s;
  s.baseline = c.mode == WS_MODE_BASELINE;
  s.verify = c.verify;
  s.rtt = c.rtt;
  s.jitter = c.jitter;
  s.r_estimate = c.r_estimate;
  s.t_target = c.t_target;
  s.t_draft = c.t_draft;
  s.k = c.k;
  s.b = c.b;
  s.s = c.s;
  s.catchup_batch_limit = c.catchup_batch_limit;
  s.theta = c.theta;
  s.phi = c.phi;
  s.max_nodes = c.max_nodes;
  s.wait_backstop = c.wait_backstop != 0;
  s.sample_seed = c.sample_seed;
  s.oracle_seed = c.oracle.seed;
  s.eos = c.oracle.eos_id;
  s.controller_cfg().validate();
  s.worker_cfg().validate();
  wsb::validate_oracle(c.oracle);
  return s;
}

// Runs the shard of `c` through the batched driver, one ModelBackend per protocol thread, and
// writes RunOutputs (sim.hpp:420-427) into `out`.
template <class LaneOf>
void execute(const ws_sim_cfg* c, const wsb::SimCfg& cfg, std::uint32_t threads, LaneOf&& lane_of,
             ws_run_out* out, int device) {
  const std::uint32_t local = c->local_requests ? c->local_requests : c->num_requests - c->first_request;
  std::vector<std::uint32_t> reqs(local);
  for (std::uint32_t i = 0; i < local; ++i) reqs[i] = c->first_request + i;
  std::vector<wsb::RequestOutput> outs(local);
  const bool log_steps = out && out->steps;
  threads = std::min(std::max<std::uint32_t>(1, threads), local);
  for (std::uint32_t t = 0; t < threads; ++t) lane_of(t).stats = wsb::BackendStats{};
  // Contiguous chunks of requests per protocol thread; each thread owns one lane (stream).
  std::vector<std::string> errs(threads);
  std::vector<int> codes(threads, WS_OK);
  auto work = [&](std::uint32_t t) {
    const std::uint32_t lo = static_cast<std::uint32_t>((static_cast<std::uint64_t>(local) * t) / threads);
    const std::uint32_t hi = static_cast<std::uint32_t>((static_cast<std::uint64_t>(local) * (t + 1)) / threads);
    codes[t] = guarded([&] {
      if (device >= 0) WS_CUDA(cudaSetDevice(device));
      wsb::run_requests(cfg, reqs.data() + lo, hi - lo, lane_of(t), outs.data() + lo, log_steps);
    });
    errs[t] = g_err;
  };
  if (threads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (std::uint32_t t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  for (std::uint32_t t = 0; t < threads; ++t)
    if (codes[t] != WS_OK) {
      if (codes[t] == WS_ECUDA) throw wsb::CudaError(errs[t]);
      if (codes[t] == WS_ECONFIG) throw wsb::ConfigError(errs[t]);
      if (codes[t] == WS_EARG) throw std::invalid_argument(errs[t]);
      throw std::logic_error(errs[t]);
    }
  if (!out) return;
  std::uint64_t ns = 0;
  for (std::uint32_t i = 0; i < local; ++i) {
    const wsb::RequestOutput& o = outs[i];
    if (out->metrics) out->metrics[i] = o.metrics;
    auto put = [&](const std::vector<wsb::TokenId>& v, std::uint32_t* toks, std::uint32_t* lens) {
      if (!lens) return;
      lens[i] = static_cast<std::uint32_t>(v.size());
      if (!toks) return;
      if (v.size() > out->max_len) throw std::invalid_argument("ws_run_sim: max_len too small");
      std::memcpy(toks + static_cast<std::size_t>(i) * out->max_len, v.data(), v.size() * sizeof(std::uint32_t));
    };
    put(o.ctrl, out->ctrl_tokens, out->ctrl_len);
    put(o.wrk, out->wrk_tokens, out->wrk_len);
    for (const ws_step_log& s : o.steps) {
      if (out->steps && ns < out->max_steps) out->steps[ns] = s;
      ++ns;
    }
  }
  out->n_steps = ns;
  out->rounds = out->gpu_launches = out->verify_rows = out->draft_rows = 0;
  out->h2d_bytes = out->d2h_bytes = 0;
  out->kernel_ms = 0.0;
  for (std::uint32_t t = 0; t < threads; ++t) {
    const wsb::BackendStats& s = lane_of(t).stats;
    out->rounds += s.rounds;
    out->gpu_launches += s.launches;
    out->verify_rows += s.verify_rows;
    out->draft_rows += s.draft_rows;
    out->h2d_bytes += s.h2d;
    out->d2h_bytes += s.d2h;
    out->kernel_ms += s.kernel_ms;
  }
}

void check_shard(const ws_sim_cfg* c) {
  if (c->first_request >= c->num_requests) throw wsb::ConfigError("sim: shard out of range");
  const std::uint32_t local = c->local_requests ? c->local_requests : c->num_requests - c->first_request;
  if (static_cast<std::uint64_t>(c->first_request) + local > c->num_requests)
    throw wsb::ConfigError("sim: shard out of range");
}

void run_resident(ws_ctx* ctx, const ws_sim_cfg* c, ws_run_out* out) {
  need(ctx && c, "ws_run_sim: null argument");
  const wsb::SimCfg cfg = to_cfg(*c);
  check_shard(c);
  const std::uint32_t local = c->local_requests ? c->local_requests : c->num_requests - c->first_request;
  if (!ctx->tables.block || ctx->tables.n_seq < c->first_request + local ||
      ctx->tables.seq_len != c->oracle.sequence_length || ctx->tables.eos != c->oracle.eos_id ||
      ctx->tables.vocab != c->oracle.vocab_size)
    throw wsb::ConfigError("sim: resident oracle tables do not match the config");
  WS_CUDA(cudaSetDevice(ctx->device));
  const std::uint32_t threads = std::min(std::max<std::uint32_t>(1, c->host_threads), local);
  for (std::uint32_t t = 0; t < threads; ++t) ctx->lane(t);  // create lanes before threads start
  execute(c, cfg, threads, [&](std::uint32_t t) -> wsb::ModelBackend& { return *ctx->lanes[t]; }, out,
          ctx->device);
}

// The host-logic seam: the round is delegated to a caller-supplied function.
class CallbackBackend : public wsb::ModelBackend {
 public:
  CallbackBackend(ws_model_round_fn fn, void* user)
      : fn_(fn), user_(user), lanes_(std::getenv("WS_EMULATE_LANES") != nullptr) {}
  void run_round(const wsb::RoundJobs& jobs, wsb::RoundResults& res, int mode, std::uint64_t seed) override {
    res.verify.resize(jobs.verify.size());
    res.draft.resize(jobs.draft.size());
    const int rc = fn_(user_, static_cast<std::uint32_t>(jobs.verify.size()), jobs.verify.data(), jobs.cands.data(),
                       static_cast<std::uint32_t>(jobs.draft.size()), jobs.draft.data(), res.verify.data(),
                       res.draft.data(), mode, seed);
    if (rc != 0) throw std::logic_error("model round callback failed");
    stats.rounds += 1;
    stats.verify_rows += jobs.verify.size();
    stats.draft_rows += jobs.draft.size();
  }

  // WS_EMULATE_LANES=1: the lanes continuous-batching driver (verify + two draft lanes) over the callback (CPU tests
  // of the lanes driver); completions are returned in a scrambled but seeded order, and every
  // batch of more than one job is cut in half (the rest stays pending — partial takes).
  bool has_lanes() const override { return lanes_; }
  std::size_t submit(int lane, const wsb::RoundJobs& jobs, int mode, std::uint64_t seed) override {
    wsb::RoundJobs one;
    const std::size_t n = lane == 0 ? jobs.verify.size() : jobs.draft.size();
    const std::size_t take = n > 1 ? (n + 1) / 2 : n;
    if (lane == 0) {
      one.verify.assign(jobs.verify.begin(), jobs.verify.begin() + take);
      one.cands = jobs.cands;
    } else {
      one.draft.assign(jobs.draft.begin(), jobs.draft.begin() + take);
    }
    run_round(one, done_[lane], mode, seed);
    return take;
  }
  int n_lanes() const override { return 3; }  // verify + two draft lanes
  int wait_any(std::uint32_t busy) override {
    int lanes[3], n = 0;
    for (int l = 0; l < 3; ++l)
      if (busy & (1u << l)) lanes[n++] = l;
    rng_ ^= rng_ << 13;
    rng_ ^= rng_ >> 7;
    rng_ ^= rng_ << 17;
    return lanes[rng_ % static_cast<std::uint64_t>(n)];
  }
  void complete(int lane, wsb::RoundResults& res) override {
    if (lane == 0)
      res.verify.swap(done_[0].verify);
    else
      res.draft.swap(done_[lane].draft);
  }

 private:
  ws_model_round_fn fn_;
  void* user_;
  bool lanes_;
  wsb::RoundResults done_[3];
  std::uint64_t rng_ = 0x9E3779B97F4A7C15ULL;
};

}  // namespace

namespace wsb {
// Error mapping shared with capi_ops.cpp (device-pointer entry points).
int ops_guarded_rc(const char* what, const std::exception& e) {
  g_err = std::string(what) + ": " + e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return WS_ECONFIG;
  if (dynamic_cast<const CudaError*>(&e)) return WS_ECUDA;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return WS_EARG;
  return WS_ELOGIC;
}
SimCfg sim_cfg_from_abi(const ws_sim_cfg& c) {
  SimCfg s = to_cfg(c);
  check_shard(&c);
  return s;
}
void run_shard(const ws_sim_cfg* c, const SimCfg& cfg, ModelBackend& backend, ws_run_out* out, int device) {
  execute(c, cfg, 1, [&](std::uint32_t) -> ModelBackend& { return backend; }, out, device);
}
void run_shard_threads(const ws_sim_cfg* c, const SimCfg& cfg, const std::vector<ModelBackend*>& backends,
                       ws_run_out* out, int device) {
  execute(c, cfg, static_cast<std::uint32_t>(backends.size()),
          [&](std::uint32_t t) -> ModelBackend& { return *backends[t]; }, out, device);
}
}  // namespace wsb

extern "C" {

int ws_abi_version(void) { return WS_ABI_VERSION; }

int ws_wire_encode(const ws_wire_msg* m, uint8_t* out, size_t cap, size_t* len) {
  return guarded([&] {
    need(m && out && len, "ws_wire_encode: null argument");
    if (m->kind < WS_MSG_HELLO || m->kind > WS_MSG_BYE) throw std::invalid_argument("ws_wire_encode: bad kind");
    if (m->n_path > WS_WIRE_MAX_PATH || m->n_cands > 2 || m->n_accepted > WS_WIRE_MAX_ACCEPTED)
      throw std::invalid_argument("ws_wire_encode: field count out of range");
    wsb::Message msg;
    msg.kind = static_cast<wsb::MsgKind>(m->kind);
    msg.request_id = m->request_id;
    msg.seq_no = m->seq_no;
    msg.base = m->base;
    msg.config_digest = m->config_digest;
    msg.final_length = m->final_length;
    msg.path.assign(m->path, m->path + m->n_path);
    msg.n_cands = m->n_cands;
    for (uint32_t i = 0; i < m->n_cands; ++i) msg.cands[i] = wsb::CandIn{m->cand_token[i], m->cand_prob[i], m->cand_entropy[i]};
    msg.result.accepted.assign(m->accepted, m->accepted + m->n_accepted);
    msg.result.bonus = m->bonus;
    msg.result.final_entropy = m->final_entropy;
    std::vector<std::uint8_t> buf;
    wsb::wire_encode(msg, buf);
    if (buf.size() > cap) throw std::invalid_argument("ws_wire_encode: output buffer too small");
    std::memcpy(out, buf.data(), buf.size());
    *len = buf.size();
  });
}

int ws_wire_decode(const uint8_t* bytes, size_t n, ws_wire_msg* out, size_t* consumed) {
  bool more = false;
  const int rc = guarded([&] {
    need((bytes || n == 0) && out && consumed, "ws_wire_decode: null argument");
    const wsb::Decoded d = wsb::wire_decode_frame(bytes, n);
    if (d.status == wsb::DecodeStatus::need_more) {
      more = true;
      *consumed = 0;
      return;
    }
    if (d.status == wsb::DecodeStatus::error) throw wsb::ProtocolError("wire: " + d.error);
    const wsb::Message& m = d.message;
    if (m.path.size() > WS_WIRE_MAX_PATH) throw wsb::ProtocolError("wire: path longer than WS_WIRE_MAX_PATH");
    std::memset(out, 0, sizeof(*out));
    out->kind = static_cast<uint32_t>(m.kind);
    out->request_id = m.request_id;
    out->seq_no = m.seq_no;
    out->base = m.base;
    out->config_digest = m.config_digest;
    out->final_length = m.final_length;
    out->n_path = static_cast<uint32_t>(m.path.size());
    std::copy(m.path.begin(), m.path.end(), out->path);
    out->n_cands = m.n_cands;
    for (uint32_t i = 0; i < m.n_cands; ++i) {
      out->cand_token[i] = m.cands[i].token;
      out->cand_prob[i] = m.cands[i].prob;
      out->cand_entropy[i] = m.cands[i].entropy;
    }
    out->n_accepted = static_cast<uint32_t>(m.result.accepted.size());
    std::copy(m.result.accepted.begin(), m.result.accepted.end(), out->accepted);
    out->bonus = m.result.bonus;
    out->final_entropy = m.result.final_entropy;
    *consumed = d.consumed;
  });
  return rc == WS_OK && more ? WS_WIRE_NEED_MORE : rc;
}

const char* ws_last_error(void) { return g_err.c_str(); }

int ws_device_count(int* out) {
  return guarded([&] {
    need(out != nullptr, "ws_device_count: null");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *out = n;
  });
}

int ws_create(int device, ws_ctx** out) {
  return guarded([&] {
    need(out != nullptr, "ws_create: null");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw wsb::CudaError("ws_create: no CUDA device (the hot path has no CPU fallback)");
    }
    if (device < 0 || device >= n) throw std::invalid_argument("ws_create: device out of range");
    WS_CUDA(cudaSetDevice(device));
    auto ctx = std::make_unique<ws_ctx>();
    ctx->device = device;
    WS_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    *out = ctx.release();
  });
}

int ws_destroy(ws_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    ctx->lanes.clear();
    wsb::free_tables(ctx->tables);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int ws_oracle_synth(const ws_oracle_cfg* cfg, uint32_t n_seq, ws_token_record* out) {
  return guarded([&] {
    need(cfg && out, "ws_oracle_synth: null argument");
    wsb::synth_tiny_pair(*cfg, n_seq, out);
  });
}

int ws_load_oracle(ws_ctx* ctx, uint32_t n_seq, uint32_t seq_len, uint32_t vocab_size, uint32_t eos_id,
                   const ws_token_record* records) {
  return guarded([&] {
    need(ctx && records && n_seq > 0 && seq_len > 0, "ws_load_oracle: bad argument");
    if (eos_id >= vocab_size) throw wsb::ConfigError("oracle: eos_id must be < vocab_size");
    WS_CUDA(cudaSetDevice(ctx->device));
    wsb::upload_tables(ctx->tables, n_seq, seq_len, vocab_size, eos_id, records, ctx->stream);
  });
}

static void single_round(ws_ctx* ctx, wsb::RoundJobs& jobs, wsb::RoundResults& res, int mode,
                         std::uint64_t seed) {
  need(ctx != nullptr, "null context");
  if (!ctx->tables.block) throw wsb::ConfigError("oracle tables not loaded");
  WS_CUDA(cudaSetDevice(ctx->device));
  ctx->lane(0).run_round(jobs, res, mode, seed);
}

static void verify_impl(ws_ctx* ctx, uint32_t n, uint32_t k, int mode, std::uint64_t seed, const uint32_t* seq,
                        const uint64_t* request, const uint32_t* step, const uint64_t* base, const uint32_t* cand,
                        uint32_t* acc, uint32_t* bonus, double* h) {
  need(seq && base && (cand || k == 0) && acc && bonus && h, "ws_verify: null argument");
  wsb::RoundJobs jobs;
  for (uint32_t j = 0; j < n; ++j) {
    if (seq[j] >= ctx->tables.n_seq) throw std::invalid_argument("ws_verify: seq out of range");
    wsb::VerifyJob v{seq[j], k, base[j], request ? request[j] : 0, step ? step[j] : 0,
                     static_cast<uint32_t>(jobs.cands.size())};
    jobs.cands.insert(jobs.cands.end(), cand + static_cast<std::size_t>(j) * k, cand + static_cast<std::size_t>(j + 1) * k);
    jobs.verify.push_back(v);
  }
  if (n == 0) return;
  wsb::RoundResults res;
  single_round(ctx, jobs, res, mode, seed);
  for (uint32_t j = 0; j < n; ++j) {
    acc[j] = res.verify[j].accepted;
    bonus[j] = res.verify[j].bonus;
    h[j] = res.verify[j].final_entropy;
  }
}

int ws_verify(ws_ctx* ctx, uint32_t n, uint32_t k, const uint32_t* seq, const uint64_t* base, const uint32_t* cand,
              uint32_t* acc_len, uint32_t* bonus, double* final_entropy) {
  return guarded([&] {
    need(ctx != nullptr, "ws_verify: null context");
    verify_impl(ctx, n, k, WS_VERIFY_GREEDY, 0, seq, nullptr, nullptr, base, cand, acc_len, bonus, final_entropy);
  });
}

int ws_verify_rejection(ws_ctx* ctx, uint32_t n, uint32_t k, uint64_t sample_seed, const uint32_t* seq,
                        const uint64_t* request, const uint32_t* step, const uint64_t* base, const uint32_t* cand,
                        uint32_t* acc_len, uint32_t* bonus, double* final_entropy) {
  return guarded([&] {
    need(ctx && request && step, "ws_verify_rejection: null argument");
    verify_impl(ctx, n, k, WS_VERIFY_REJECTION, sample_seed, seq, request, step, base, cand, acc_len, bonus,
                final_entropy);
  });
}

int ws_draft(ws_ctx* ctx, uint32_t n, const uint32_t* seq, const uint64_t* pos, ws_pred* out) {
  return guarded([&] {
    need(ctx && seq && pos && out, "ws_draft: null argument");
    if (n == 0) return;
    wsb::RoundJobs jobs;
    for (uint32_t j = 0; j < n; ++j) {
      if (seq[j] >= ctx->tables.n_seq) throw std::invalid_argument("ws_draft: seq out of range");
      jobs.draft.push_back(wsb::DraftJob{seq[j], 0, pos[j]});
    }
    wsb::RoundResults res;
    single_round(ctx, jobs, res, WS_VERIFY_GREEDY, 0);
    std::memcpy(out, res.draft.data(), n * sizeof(ws_pred));
  });
}

int ws_run_sim_resident(ws_ctx* ctx, const ws_sim_cfg* cfg, ws_run_out* out) {
  return guarded([&] { run_resident(ctx, cfg, out); });
}

int ws_run_sim(ws_ctx* ctx, const ws_sim_cfg* cfg, ws_run_out* out) {
  return guarded([&] {
    need(ctx && cfg, "ws_run_sim: null argument");
    wsb::validate_oracle(cfg->oracle);
    std::vector<ws_token_record> recs(static_cast<std::size_t>(cfg->num_requests) * cfg->oracle.sequence_length);
    wsb::synth_tiny_pair(cfg->oracle, cfg->num_requests, recs.data());
    WS_CUDA(cudaSetDevice(ctx->device));
    const std::size_t up = wsb::upload_tables(ctx->tables, cfg->num_requests, cfg->oracle.sequence_length,
                                              cfg->oracle.vocab_size, cfg->oracle.eos_id, recs.data(), ctx->stream);
    run_resident(ctx, cfg, out);
    if (out) out->h2d_bytes += up;
  });
}

int ws_run_sim_with_model(const ws_sim_cfg* cfg, ws_model_round_fn fn, void* user, ws_run_out* out) {
  return guarded([&] {
    need(cfg && fn, "ws_run_sim_with_model: null argument");
    const wsb::SimCfg c = to_cfg(*cfg);
    check_shard(cfg);
    CallbackBackend backend(fn, user);
    execute(cfg, c, 1, [&](std::uint32_t) -> wsb::ModelBackend& { return backend; }, out, -1);
  });
}

}  // extern "C"
