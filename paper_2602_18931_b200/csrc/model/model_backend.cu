// Real-model backend (see model_backend.hpp).
#include "model_backend.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <chrono>
#include <thread>

#include "../kernels/cuda_check.hpp"
#include "../kernels/rowstats.cuh"
#include "../kernels/sample.cuh"

#include <nvtx3/nvToolsExt.h>

namespace wsb {

namespace {

std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct LinearCache {
  std::vector<TokenId> valid;  // tokens whose KV is valid at positions [0, size)
};

struct TrieNode {
  TokenId tok = 0;
  std::int32_t slot = -1;
  std::int32_t parent = -1;  // -1 = trie root (position == prefix length)
  std::vector<std::int32_t> kids;
};

// Worker draft KV: committed prefix (linear) + content trie of speculative nodes.
struct TreeCache {
  std::vector<TokenId> prefix;
  std::vector<TrieNode> nodes;
  std::vector<std::int32_t> root_kids;
  std::vector<std::int32_t> free_nodes;
  std::vector<std::int32_t> free_slots;
  bool init = false;

  void reset(std::int32_t slot0, std::int32_t n) {
    prefix.clear();
    nodes.clear();
    root_kids.clear();
    free_nodes.clear();
    free_slots.clear();
    for (std::int32_t i = n - 1; i >= 0; --i) free_slots.push_back(slot0 + i);
    init = true;
  }
  const std::vector<std::int32_t>& kids_of(std::int32_t n) const { return n < 0 ? root_kids : nodes[n].kids; }
  std::int32_t find(std::int32_t parent, TokenId t) const {
    for (std::int32_t c : kids_of(parent))
      if (nodes[c].tok == t) return c;
    return -2;
  }
  void free_subtree(std::int32_t n) {
    std::vector<std::int32_t> st{n};
    while (!st.empty()) {
      const std::int32_t x = st.back();
      st.pop_back();
      for (std::int32_t c : nodes[x].kids) st.push_back(c);
      nodes[x].kids.clear();
      free_slots.push_back(nodes[x].slot);
      nodes[x].slot = -1;
      free_nodes.push_back(x);
    }
  }
  void drop_all() {
    for (std::int32_t c : root_kids) free_subtree(c);
    root_kids.clear();
  }
  std::int32_t add(std::int32_t parent, TokenId t) {
    std::int32_t id;
    if (!free_nodes.empty()) {
      id = free_nodes.back();
      free_nodes.pop_back();
    } else {
      id = static_cast<std::int32_t>(nodes.size());
      nodes.emplace_back();
    }
    TrieNode& n = nodes[id];
    n.tok = t;
    n.parent = parent;
    n.kids.clear();
    n.slot = free_slots.back();
    free_slots.pop_back();
    (parent < 0 ? root_kids : nodes[parent].kids).push_back(id);
    return id;
  }
  // The chain root→n has migrated into the prefix: n's children become the new root
  // children; the chain and every side branch are freed (their KV was copied or is stale).
  void reroot_at(std::int32_t n) {
    std::vector<std::int32_t> keep = nodes[n].kids;
    nodes[n].kids.clear();
    for (std::int32_t c : keep) nodes[c].parent = -1;
    std::vector<std::int32_t> old_root = root_kids;
    root_kids.clear();
    for (std::int32_t c : old_root) free_subtree(c);
    root_kids = keep;
  }
  std::uint64_t last_alloc_round = ~0ull;
};

}  // namespace

struct ModelPair::Impl {
  std::vector<LinearCache> tgt, ctrl;
  std::vector<TreeCache> wrk;
  // prefill phase: one stream + workspace per model, created on first use
  struct Side {
    int dev = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    std::unique_ptr<ForwardWorkspace> ws;
  };
  std::vector<Side> pre;  // [0] target, [1 + rep] draft replica rep
  ~Impl() {
    for (Side& sd : pre) {
      if (!sd.st) continue;
      cudaSetDevice(sd.dev);
      sd.ws.reset();
      cudaEventDestroy(sd.e0);
      cudaEventDestroy(sd.e1);
      cudaStreamDestroy(sd.st);
    }
  }
};

// One draft lane: its stream, forward workspace, K3/K4 buffers and pinned results. Several
// draft lanes let the host plan and launch the next draft batch while the previous one runs
// (every actor has at most one draft job set in flight, so lanes never touch the same KV).
struct DraftSub {  // one draft replica's share of a draft batch
  int rep = 0;
  std::vector<std::uint32_t> idx;  // the batch's job indices this replica runs
  int device = 0;
  cudaStream_t st = nullptr;
  std::unique_ptr<ForwardWorkspace> ws;
  ws_pred* d_pred = nullptr;
  void* d_ws = nullptr;
  ws_pred* h_pred = nullptr;
  std::size_t cap = 0;
  ForwardBatch b;
  std::vector<std::int32_t> job_out, copy_src, copy_dst;  // job_out: output row, -1 forced EOS
  std::uint32_t nd = 0;
  bool ran = false;
  cudaEvent_t e_start = nullptr, e_end = nullptr, done = nullptr;
  ~DraftSub() {
    cudaSetDevice(device);
    if (d_pred) cudaFree(d_pred);
    if (d_ws) cudaFree(d_ws);
    if (h_pred) cudaFreeHost(h_pred);
    for (cudaEvent_t e : {e_start, e_end, done})
      if (e) cudaEventDestroy(e);
    ws.reset();
    if (st) cudaStreamDestroy(st);
  }
};

// One draft lane: a sub-lane per draft replica; the lane completes when every sub-lane has.
struct DraftLane {
  std::vector<std::unique_ptr<DraftSub>> sub;
  std::uint32_t nd = 0;
  cudaEvent_t done = nullptr;  // on sub[0]'s device, after every sub-lane's work
  ~DraftLane() {
    if (done) {
      cudaSetDevice(sub[0]->device);
      cudaEventDestroy(done);
    }
    sub.clear();
  }
};

// One protocol thread's GPU state: the verify lane's stream, forward workspace, K3/K4
// buffers, pinned staging and results, plus its draft lanes. Several backends share one
// ModelPair (weights, KV pools, per-request caches) and serve disjoint request ranges
// concurrently.
struct ModelBackend_Llama::Lanes {
  int device = 0;    // verify lane (target model)
  int device_d = 0;  // draft lanes (the same GPU, or another under split placement)
  cudaStream_t st_t = nullptr;  // verify (target) stream
  std::unique_ptr<ForwardWorkspace> ws_t;
  std::vector<std::unique_ptr<DraftLane>> dl;  // lanes 1..n
  // verify lane
  ws_pred* d_pred = nullptr;
  ws_verify_out* d_vout = nullptr;
  std::uint32_t* d_cands = nullptr;
  std::int32_t* d_forced = nullptr;
  double* d_cprob = nullptr;           // K4R inputs: candidate draft probabilities,
  std::uint64_t* d_req = nullptr;      // per-job request ids (Philox counter words)
  std::uint32_t* d_step = nullptr;     // and per-request verify step indices
  void* d_ws = nullptr;
  unsigned char* h_stage = nullptr;
  ws_verify_out* h_vout = nullptr;
  std::size_t cap_v = 0;
  ForwardBatch tb;
  std::vector<TokenId> ctx;
  std::vector<std::int32_t> forced;
  std::uint32_t nv = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr, done = nullptr;  // done: after the verify D2H
  ~Lanes() {
    dl.clear();
    cudaSetDevice(device);
    for (void* q : {static_cast<void*>(d_pred), static_cast<void*>(d_vout), static_cast<void*>(d_cands),
                    static_cast<void*>(d_forced), static_cast<void*>(d_cprob), static_cast<void*>(d_req),
                    static_cast<void*>(d_step), d_ws})
      if (q) cudaFree(q);
    for (void* q : {static_cast<void*>(h_stage), static_cast<void*>(h_vout)})
      if (q) cudaFreeHost(q);
    for (cudaEvent_t e : {e0, e1, done})
      if (e) cudaEventDestroy(e);
    ws_t.reset();
    if (st_t) cudaStreamDestroy(st_t);
  }
};

ModelPair::ModelPair(const ModelPairCfg& cfg, int device) : cfg_(cfg), device_(device), impl(new Impl) {
  WS_CUDA(cudaSetDevice(device));
  const LlamaShape ts = shape_by_name(cfg.target), ds = shape_by_name(cfg.draft);
  if (ts.vocab != ds.vocab) throw ConfigError("target and draft vocabularies differ");
  const std::int64_t R = cfg.max_requests, C = cfg.max_ctx;
  max_rows_ = static_cast<int>(std::min<std::int64_t>(R * 20, 8192));
  draft_device_ = cfg.draft_device >= 0 ? cfg.draft_device : device;
  target_.reset(new LlamaModel(ts, cfg.seed * 2 + 1, R * C, max_rows_, device, cfg.tp));
  draft_.reset(new LlamaModel(ds, cfg.seed * 2 + 2, R * (2 * C + cfg.trie_slots), max_rows_, draft_device_));
  draft_reps_.emplace_back();
  rep_devices_.push_back(draft_device_);
  // a tensor-parallel target with no explicit draft GPU: one draft replica per rank (the same
  // weights), each serving the requests r with r % tp == its index — the draft work is spread
  // over the ranks instead of skewing one of them
  if (cfg.tp > 1 && cfg.draft_device < 0)
    for (int g = 1; g < cfg.tp; ++g) {
      draft_reps_.emplace_back(
          new LlamaModel(ds, cfg.seed * 2 + 2, R * (2 * C + cfg.trie_slots), max_rows_, device + g));
      rep_devices_.push_back(device + g);
    }
  WS_CUDA(cudaSetDevice(device));
  prompts_.resize(cfg.max_requests);
  if (const char* e = std::getenv("WS_TARGET_CTAS")) target_->set_max_ctas(std::atoi(e));
  if (const char* e = std::getenv("WS_DRAFT_CTAS")) draft_->set_max_ctas(std::atoi(e));
  reset_requests();
}

// Late PDL trigger: a model's GEMMs let the next kernel of its chain launch once their last
// accumulator is ready, so its prologue and weight prefetch overlap the epilogue on the SMs that
// free up — at the price of dependents parked on those SMs, which the other lane's kernels then
// cannot use. Measured on config 3 (profiles/r02_pdl_late.md): for the draft model, +3.9 % at
// 64 requests per GPU (the draft chain is the critical path), -0.5 % at 128 and neutral at 256
// (the verify lane loses what the draft lane gains); for both models, -1 % at 256. Default: the
// draft model's GEMMs at <= 96 requests per GPU. WS_PDL_LATE = 0 | 1 | draft | target forces.
void ModelPair::set_pdl_late_for(std::uint32_t n_local) {
  const char* e = std::getenv("WS_PDL_LATE");
  const std::string v = e ? e : (n_local <= 96 ? "draft" : "0");
  target_->set_pdl_late(v == "1" || v == "target");
  for (int r = 0; r < draft_replicas(); ++r) draft(r).set_pdl_late(v == "1" || v == "draft");
}

ModelPair::~ModelPair() {
  cudaSetDevice(device_);
  target_.reset();
  draft_.reset();
}

void ModelPair::reset_requests() {
  impl->tgt.assign(cfg_.max_requests, LinearCache{});
  impl->ctrl.assign(cfg_.max_requests, LinearCache{});
  impl->wrk.assign(cfg_.max_requests, TreeCache{});
}

ModelPair::PrefillStats ModelPair::prefill_prompts(const std::uint32_t* reqs, std::size_t n) {
  PrefillStats out;
  const std::int32_t P = static_cast<std::int32_t>(cfg_.prompt_len);
  if (n == 0 || P < 2) return out;
  const std::int32_t MC = static_cast<std::int32_t>(cfg_.max_ctx);
  const std::int32_t S = 2 * MC + static_cast<std::int32_t>(cfg_.trie_slots);
  constexpr std::int32_t kMaxRows = 8192;  // rows per prefill forward (the GEMMs' efficient regime)
  const std::size_t per = static_cast<std::size_t>(std::max(1, kMaxRows / (P - 1)));
  const int n_sides = 1 + draft_replicas();
  if (impl->pre.size() < static_cast<std::size_t>(n_sides)) impl->pre.resize(n_sides);
  for (int side = 0; side < n_sides; ++side) {
    Impl::Side& sd = impl->pre[side];
    const int rep = side - 1;
    LlamaModel& m = side == 0 ? *target_ : draft(rep);
    const int dev = side == 0 ? device_ : draft_device(rep);
    DeviceGuard dg(dev);
    if (!sd.st) {
      sd.dev = dev;
      WS_CUDA(cudaStreamCreateWithFlags(&sd.st, cudaStreamNonBlocking));
      WS_CUDA(cudaEventCreate(&sd.e0));
      WS_CUDA(cudaEventCreate(&sd.e1));
      sd.ws = m.make_workspace(64);
    }
    // this side's requests: all (target), or those served by the draft replica
    std::vector<std::uint32_t> mine;
    for (std::size_t i = 0; i < n; ++i)
      if (side == 0 || replica_of(reqs[i]) == rep) mine.push_back(reqs[i]);
    WS_CUDA(cudaEventRecord(sd.e0, sd.st));
    const std::size_t h2d0 = sd.ws->h2d;
    const std::uint64_t kv0 = sd.ws->kv_pos, ap0 = sd.ws->attn_pairs;
    ForwardBatch b;
    std::vector<std::int32_t> src, dst;
    for (std::size_t i0 = 0; i0 < mine.size(); i0 += per) {
      b.clear();
      for (std::size_t i = i0; i < std::min(mine.size(), i0 + per); ++i) {
        const std::uint32_t r = mine[i];
        const std::vector<TokenId>& pr = prompt(r);
        // target: the linear verify cache; draft: the worker's committed prefix region
        const std::int32_t base = side == 0 ? static_cast<std::int32_t>(r) * MC : static_cast<std::int32_t>(r) * S + MC;
        const std::int32_t row0 = static_cast<std::int32_t>(b.tok.size());
        const std::int32_t eoff = static_cast<std::int32_t>(b.extra.size());
        for (std::int32_t p = 0; p < P - 1; ++p) {
          b.tok.push_back(static_cast<std::int32_t>(pr[p]));
          b.pos.push_back(p);
          b.slot.push_back(base + p);
          b.extra.push_back(base + p);
          if (side > 0) {
            src.push_back(base + p);
            dst.push_back(static_cast<std::int32_t>(r) * S + p);  // the controller's draft cache
          }
        }
        b.groups.push_back(AttnGroup{row0, P - 1, base, 0, eoff, P - 1});
      }
      b.row_mask.assign(b.tok.size(), 0ull);
      b.prefill = true;
      nvtxRangePushA(side == 0 ? "ws.prefill.target" : "ws.prefill.draft");
      m.forward(b, 0.f, sd.st, *sd.ws);  // no output rows: KV only, no LM head
      nvtxRangePop();
      out.rows += side == 0 ? b.tok.size() : 0;
      (side == 0 ? out.target_forwards : out.draft_forwards) += 1;
      out.launches += 1 + 4ull * m.shape().layers;
    }
    if (side > 0 && !src.empty()) {
      m.copy_slots(src, dst, sd.st, *sd.ws);
      out.launches += 1;
    }
    WS_CUDA(cudaEventRecord(sd.e1, sd.st));
    out.h2d += sd.ws->h2d - h2d0;
    if (side == 0) {
      out.kv_pos += sd.ws->kv_pos - kv0;
      out.attn_pairs += sd.ws->attn_pairs - ap0;
    }
  }
  float draft_max = 0.f;
  for (int side = 0; side < n_sides; ++side) {
    Impl::Side& sd = impl->pre[side];
    DeviceGuard dg(sd.dev);
    WS_CUDA(cudaEventSynchronize(sd.e1));
    float ms = 0.f;
    WS_CUDA(cudaEventElapsedTime(&ms, sd.e0, sd.e1));
    if (side == 0)
      out.target_ms += ms;
    else
      draft_max = std::max(draft_max, ms);  // the replicas prefill concurrently
  }
  out.draft_ms += draft_max;
  for (std::size_t i = 0; i < n; ++i) {
    const std::uint32_t r = reqs[i];
    const std::vector<TokenId>& pr = prompt(r);
    const std::vector<TokenId> head(pr.begin(), pr.begin() + (P - 1));
    impl->tgt[r].valid = head;
    impl->ctrl[r].valid = head;
    TreeCache& t = impl->wrk[r];
    t.reset(static_cast<std::int32_t>(r) * S + 2 * MC, static_cast<std::int32_t>(cfg_.trie_slots));
    t.prefix = head;
  }
  return out;
}

void ModelPair::evict(std::uint32_t r) {
  if (r >= cfg_.max_requests) throw ConfigError("evict: request index exceeds max_requests");
  impl->tgt[r] = LinearCache{};
  impl->ctrl[r] = LinearCache{};
  impl->wrk[r] = TreeCache{};
}

void ModelPair::export_trace(std::uint32_t first, std::uint32_t n, std::uint32_t length, ws_token_record* out) {
  if (first + n > cfg_.max_requests) throw ConfigError("export_trace: requests exceed max_requests");
  if (cfg_.prompt_len + length > cfg_.max_ctx) throw ConfigError("export_trace: prompt + length exceeds max_ctx");
  if (n == 0 || length == 0) return;
  const std::int32_t P = static_cast<std::int32_t>(cfg_.prompt_len), MC = static_cast<std::int32_t>(cfg_.max_ctx);
  const std::int32_t S = 2 * MC + static_cast<std::int32_t>(cfg_.trie_slots);
  const std::uint32_t V = static_cast<std::uint32_t>(target_->shape().vocab);
  reset_requests();
  struct Side {
    LlamaModel* m;
    int dev;
    bool draft;
    std::int32_t stride;
    cudaStream_t st = nullptr;
    std::unique_ptr<ForwardWorkspace> ws;
    ws_pred* d_pred = nullptr;
    void* d_rs = nullptr;
    std::vector<ws_pred> h;
  } sides[2] = {{target_.get(), device_, false, MC}, {draft_.get(), draft_device_, true, S}};
  const std::uint32_t rows_max = n * static_cast<std::uint32_t>(P);
  for (Side& sd : sides) {
    DeviceGuard dg(sd.dev);
    WS_CUDA(cudaStreamCreateWithFlags(&sd.st, cudaStreamNonBlocking));
    sd.ws = sd.m->make_workspace(static_cast<int>(rows_max));
    WS_CUDA(cudaMalloc(&sd.d_pred, n * sizeof(ws_pred)));
    const std::size_t wb = rowstats_workspace_bytes(n, V, 0);
    WS_CUDA(cudaMalloc(&sd.d_rs, wb));
    WS_CUDA(cudaMemset(sd.d_rs, 0, wb));
    sd.h.resize(n);
  }
  // The prompt head [0, P-1) as in a model run: one prompt-prefill forward (KV only, the
  // prefill kind of ForwardBatch), so every position's KV comes from the same kind of forward
  // as in ModelPair::prefill_prompts + the verify / draft forwards.
  if (P > 1) {
    for (Side& sd : sides) {
      DeviceGuard dg(sd.dev);
      ForwardBatch b;
      for (std::uint32_t j = 0; j < n; ++j) {
        const std::uint32_t r = first + j;
        const std::vector<TokenId>& pr = prompt(r);
        const std::int32_t base = static_cast<std::int32_t>(r) * sd.stride;
        const std::int32_t row0 = static_cast<std::int32_t>(b.tok.size());
        const std::int32_t eoff = static_cast<std::int32_t>(b.extra.size());
        for (std::int32_t p = 0; p < P - 1; ++p) {
          b.tok.push_back(static_cast<std::int32_t>(pr[p]));
          b.pos.push_back(p);
          b.slot.push_back(base + p);
          b.extra.push_back(base + p);
        }
        b.groups.push_back(AttnGroup{row0, P - 1, base, 0, eoff, P - 1});
      }
      b.row_mask.assign(b.tok.size(), 0ull);
      b.prefill = true;
      sd.m->forward(b, 0.f, sd.st, *sd.ws);
    }
  }
  std::vector<TokenId> last(n);  // the token fed at each step (prompt tail, then greedy)
  for (std::uint32_t i = 0; i < length; ++i) {
    for (Side& sd : sides) {
      DeviceGuard dg(sd.dev);
      ForwardBatch b;
      for (std::uint32_t j = 0; j < n; ++j) {
        const std::uint32_t r = first + j;
        const std::vector<TokenId>& pr = prompt(r);
        const std::int32_t base = static_cast<std::int32_t>(r) * sd.stride;
        const std::int32_t row0 = static_cast<std::int32_t>(b.tok.size());
        const std::int32_t eoff = static_cast<std::int32_t>(b.extra.size());
        // step 0 feeds the last prompt token (position P - 1) over the prefilled head; step i
        // feeds the greedy token of position P + i - 1
        const std::int32_t p0 = P - 1 + static_cast<std::int32_t>(i);
        const TokenId t = i == 0 ? pr[P - 1] : last[j];
        b.tok.push_back(static_cast<std::int32_t>(t));
        b.pos.push_back(p0);
        b.slot.push_back(base + p0);
        b.extra.push_back(base + p0);
        b.groups.push_back(AttnGroup{row0, 1, base, p0, eoff, 1});
        b.out_rows.push_back(static_cast<std::int32_t>(b.tok.size()) - 1);
        b.plant.push_back(plant(static_cast<TokenId>(b.tok.back()), sd.draft));
      }
      b.row_mask.assign(b.tok.size(), 0ull);
      sd.m->forward(b, sd.draft ? cfg_.plant_draft : cfg_.plant_target, sd.st, *sd.ws);
      row_stats_bf16(sd.ws->logits, n, V, V, 1.0f, sd.d_pred, nullptr, sd.d_rs, 0, 0, nullptr, nullptr, sd.st,
                     nullptr);
      WS_CUDA(cudaMemcpyAsync(sd.h.data(), sd.d_pred, n * sizeof(ws_pred), cudaMemcpyDeviceToHost, sd.st));
    }
    for (Side& sd : sides) {
      DeviceGuard dg(sd.dev);
      WS_CUDA(cudaStreamSynchronize(sd.st));
    }
    for (std::uint32_t j = 0; j < n; ++j) {
      const ws_pred& t = sides[0].h[j];
      const ws_pred& d = sides[1].h[j];
      ws_token_record& rec = out[static_cast<std::size_t>(j) * length + i];
      rec.target_token = t.id[0];
      rec.target_top2 = t.id[1];
      rec.target_p1 = t.prob[0];
      rec.target_p2 = t.n > 1 ? t.prob[1] : 0.0;
      rec.target_entropy = t.entropy;
      rec.draft_top1 = d.id[0];
      rec.draft_top2 = d.id[1];
      rec.draft_p1 = d.prob[0];
      rec.draft_p2 = d.n > 1 ? d.prob[1] : 0.0;
      rec.draft_entropy = d.entropy;
      last[j] = t.id[0];  // teacher forcing along the target's greedy path
    }
  }
  for (Side& sd : sides) {
    DeviceGuard dg(sd.dev);
    sd.ws.reset();
    cudaFree(sd.d_pred);
    cudaFree(sd.d_rs);
    cudaStreamDestroy(sd.st);
  }
  reset_requests();  // the requests' KV regions were overwritten
}

const std::vector<TokenId>& ModelPair::prompt(std::uint32_t r) {
  if (r >= prompts_.size()) throw ConfigError("request index exceeds max_requests");
  std::vector<TokenId>& p = prompts_[r];
  if (p.empty()) {
    std::mt19937_64 g(cfg_.seed ^ (0x51ed270b27a3c6f1ULL * (r + 1)));
    const std::uint32_t V = static_cast<std::uint32_t>(target_->shape().vocab);
    p.resize(cfg_.prompt_len);
    for (auto& t : p) t = static_cast<TokenId>(g() % (V - 256));  // stay clear of special ids
  }
  return p;
}

std::int32_t ModelPair::plant(TokenId t, bool is_draft) const {
  const std::uint32_t V = static_cast<std::uint32_t>(target_->shape().vocab);
  if (is_draft) {
    const std::uint64_t h2 = splitmix64(t ^ 0xD1B54A32D192ED03ULL ^ cfg_.seed);
    if (static_cast<double>(h2 % 1000000) >= cfg_.draft_plant_rate * 1e6) return -1;
  }
  return static_cast<std::int32_t>(splitmix64(t ^ 0xA0761D6478BD642FULL ^ cfg_.seed) % (V - 256));
}

ModelBackend_Llama::ModelBackend_Llama(ModelPair* pair, std::uint32_t seq_len, TokenId eos, std::uint32_t k)
    : p_(pair), L_(seq_len), eos_(eos), k_(k), ln_(new Lanes) {
  Lanes& L = *ln_;
  L.device = pair->device();
  L.device_d = pair->draft_device();
  WS_CUDA(cudaSetDevice(L.device));
  // The draft lane is the critical path of the continuous-batching loop (requests mostly wait
  // on draft results), so its stream gets the higher scheduling priority; the verify lane's
  // large GEMMs fill the SMs it leaves idle. WS_DRAFT_PRIO=0 gives both lanes equal priority.
  int prio_lo = 0, prio_hi = 0;
  WS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  const char* dp = std::getenv("WS_DRAFT_PRIO");
  const bool draft_first = !(dp && (dp[0] == '0' || dp[0] == '-'));
  const bool target_first = dp && dp[0] == '-';  // WS_DRAFT_PRIO=-1: the verify lane first
  WS_CUDA(cudaStreamCreateWithPriority(&L.st_t, cudaStreamNonBlocking, target_first ? prio_hi : prio_lo));
  WS_CUDA(cudaEventCreate(&L.e0));
  WS_CUDA(cudaEventCreate(&L.e1));
  WS_CUDA(cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming));
  // workspaces grow to the batch sizes actually seen (a cap of max_rows each would be GBs of
  // logits per protocol thread)
  L.ws_t = pair->target().make_workspace(64);
  // WS_DRAFT_LANES: draft lanes per protocol thread (default 1)
  int n_draft = 1;
  if (const char* e = std::getenv("WS_DRAFT_LANES")) n_draft = std::max(1, std::min(8, std::atoi(e)));
  for (int i = 0; i < n_draft; ++i) {
    std::unique_ptr<DraftLane> g(new DraftLane);
    for (int rep = 0; rep < pair->draft_replicas(); ++rep) {
      std::unique_ptr<DraftSub> d(new DraftSub);
      d->rep = rep;
      d->device = pair->draft_device(rep);
      WS_CUDA(cudaSetDevice(d->device));
      WS_CUDA(cudaStreamCreateWithPriority(&d->st, cudaStreamNonBlocking, draft_first ? prio_hi : prio_lo));
      WS_CUDA(cudaEventCreate(&d->e_start));
      WS_CUDA(cudaEventCreate(&d->e_end));
      WS_CUDA(cudaEventCreateWithFlags(&d->done, cudaEventDisableTiming));
      d->ws = pair->draft(rep).make_workspace(64);
      g->sub.push_back(std::move(d));
    }
    WS_CUDA(cudaSetDevice(g->sub[0]->device));
    WS_CUDA(cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming));
    L.dl.push_back(std::move(g));
  }
  WS_CUDA(cudaSetDevice(L.device));
}
ModelBackend_Llama::~ModelBackend_Llama() = default;

void ModelBackend_Llama::reset_run(std::uint32_t seq_len, TokenId eos, std::uint32_t k) {
  L_ = seq_len;
  eos_ = eos;
  if (k != k_) ln_->cap_v = 0;  // candidate staging is sized by k: regrow on the next batch
  k_ = k;
  stats = BackendStats{};
  target_ms = draft_ms = 0;
  target_rows = draft_rows_fed = target_forwards = draft_forwards = 0;
  target_out_rows = draft_out_rows = 0;
  ln_->ws_t->kv_pos = ln_->ws_t->attn_pairs = 0;
  for (auto& g : ln_->dl)
    for (auto& d : g->sub) d->ws->kv_pos = d->ws->attn_pairs = 0;
  for (int i = 0; i < 3; ++i) rows_by_kind[i] = jobs_by_kind[i] = 0;
  host_submit_ms[0] = host_submit_ms[1] = host_wait_ms = 0;
}

std::uint64_t ModelBackend_Llama::target_kv_pos() const { return ln_->ws_t->kv_pos; }
std::uint64_t ModelBackend_Llama::target_attn_pairs() const { return ln_->ws_t->attn_pairs; }
std::uint64_t ModelBackend_Llama::draft_kv_pos() const {
  std::uint64_t n = 0;
  for (const auto& g : ln_->dl)
    for (const auto& d : g->sub) n += d->ws->kv_pos;
  return n;
}
std::uint64_t ModelBackend_Llama::draft_attn_pairs() const {
  std::uint64_t n = 0;
  for (const auto& g : ln_->dl)
    for (const auto& d : g->sub) n += d->ws->attn_pairs;
  return n;
}

int ModelBackend_Llama::n_lanes() const { return 1 + static_cast<int>(ln_->dl.size()); }

KernelProfiler& ModelBackend_Llama::profiler(int lane) {
  return lane == 0 ? ln_->ws_t->prof : ln_->dl.at(lane - 1)->sub[0]->ws->prof;
}

namespace {
// Row at context position pos predicts committed index pos + 1 - P; past the generation cap
// that prediction is a forced EOS (oracle.hpp:88-102).
inline std::int32_t forced_at(std::int32_t pos, std::int32_t P, std::uint32_t L, TokenId eos) {
  return (pos + 1 - P) >= static_cast<std::int32_t>(L) - 1 ? static_cast<std::int32_t>(eos) : -1;
}
}  // namespace

void ModelBackend_Llama::fill_ctx(const RoundJobs& jobs, std::uint32_t r, const JobCtx& c) {
  ModelPair::Impl& I = *p_->impl;
  Lanes& L = *ln_;
  const std::vector<TokenId>& prompt = p_->prompt(r);
  L.ctx.assign(prompt.begin(), prompt.end());
  L.ctx.insert(L.ctx.end(), jobs.ctx_tokens.begin() + c.off, jobs.ctx_tokens.begin() + c.off + c.len);
}

// Lane 0: one target forward over every pending verify row, then the fused K3/K4 greedy
// verify epilogue; verify outs land in pinned memory.
// Padding-aware trim of a verify batch: the GEMMs tile rows by 256 (CTA pairs), so a batch a
// few rows past a multiple of 256 pays a whole extra row block in every projection. When the
// overflow is at most kSlack rows, the trailing jobs are left for the lane's next batch (they
// lead it). Rows per job = the context tokens missing from its cache (a read-only LCP pass).
// Off by default (WS_VERIFY_TRIM=1 enables): measured on config 3 it turns 129 verify forwards
// into 150 smaller ones at the same step time (2.70 s both ways).
std::size_t ModelBackend_Llama::verify_take(const RoundJobs& jobs) {
  static const bool on = [] {
    const char* e = std::getenv("WS_VERIFY_TRIM");
    return e && e[0] == '1';
  }();
  const std::size_t nv = jobs.verify.size();
  if (!on || nv < 2) return nv;
  constexpr std::size_t kUnit = 256, kSlack = 64;
  ModelPair::Impl& I = *p_->impl;
  Lanes& L = *ln_;
  const std::int32_t P = static_cast<std::int32_t>(p_->cfg().prompt_len);
  std::vector<std::size_t> rows(nv);
  std::size_t total = 0;
  for (std::size_t j = 0; j < nv; ++j) {
    const VerifyJob& vj = jobs.verify[j];
    const JobCtx& c = jobs.verify_ctx[j];
    const std::uint32_t r = static_cast<std::uint32_t>(vj.request);
    const std::vector<TokenId>& prompt = p_->prompt(r);
    const std::int32_t n_ctx = P + static_cast<std::int32_t>(c.len) + static_cast<std::int32_t>(vj.k);
    const std::int32_t first = n_ctx - static_cast<std::int32_t>(k_) - 1;
    const std::vector<TokenId>& valid = I.tgt[r].valid;
    std::int32_t lcp = 0;
    auto tok_at = [&](std::int32_t p) -> TokenId {
      return p < P ? prompt[p] : jobs.ctx_tokens[c.off + (p - P)];
    };
    while (lcp < first && lcp < static_cast<std::int32_t>(valid.size()) && valid[lcp] == tok_at(lcp)) ++lcp;
    rows[j] = static_cast<std::size_t>(n_ctx - lcp);
    total += rows[j];
  }
  const std::size_t over = total % kUnit;
  if (total <= kUnit || over == 0 || over > kSlack) return nv;
  const std::size_t cap = total - over;
  std::size_t acc = 0, take = 0;
  while (take < nv && acc + rows[take] <= cap) acc += rows[take++];
  return std::max<std::size_t>(1, take);
}

void ModelBackend_Llama::submit_verify(const RoundJobs& jobs, std::size_t nv_take) {
  ModelPair::Impl& I = *p_->impl;
  Lanes& L = *ln_;
  DeviceGuard dg(L.device);
  const ModelPairCfg& cfg = p_->cfg();
  cudaStream_t st = L.st_t;
  const std::int32_t P = static_cast<std::int32_t>(cfg.prompt_len);
  const std::int32_t MC = static_cast<std::int32_t>(cfg.max_ctx);
  const std::int32_t V = p_->target().shape().vocab;
  const std::uint32_t nv = static_cast<std::uint32_t>(nv_take);
  L.nv = nv;
  if (!nv) return;
  const std::size_t need = static_cast<std::size_t>(nv) * (k_ + 1) + 16;
  if (need > L.cap_v) {  // the lane is idle here (the driver submits only to idle lanes)
    for (void* q : {static_cast<void*>(L.d_pred), static_cast<void*>(L.d_vout), static_cast<void*>(L.d_cands),
                    static_cast<void*>(L.d_forced), static_cast<void*>(L.d_cprob), static_cast<void*>(L.d_req),
                    static_cast<void*>(L.d_step), L.d_ws})
      if (q) cudaFree(q);
    for (void* q : {static_cast<void*>(L.h_stage), static_cast<void*>(L.h_vout)})
      if (q) cudaFreeHost(q);
    L.cap_v = need * 2;
    WS_CUDA(cudaMalloc(&L.d_pred, L.cap_v * sizeof(ws_pred)));
    WS_CUDA(cudaMalloc(&L.d_vout, L.cap_v * sizeof(ws_verify_out)));
    WS_CUDA(cudaMalloc(&L.d_cands, L.cap_v * k_ * 4 + 64));
    WS_CUDA(cudaMalloc(&L.d_forced, L.cap_v * 4));
    WS_CUDA(cudaMalloc(&L.d_cprob, L.cap_v * k_ * sizeof(double) + 64));
    WS_CUDA(cudaMalloc(&L.d_req, L.cap_v * sizeof(std::uint64_t)));
    WS_CUDA(cudaMalloc(&L.d_step, L.cap_v * sizeof(std::uint32_t)));
    const std::size_t wsb_ = rowstats_workspace_bytes(static_cast<std::uint32_t>(L.cap_v), V,
                                                      static_cast<std::uint32_t>(L.cap_v));
    WS_CUDA(cudaMalloc(&L.d_ws, wsb_));
    WS_CUDA(cudaMemset(L.d_ws, 0, wsb_));
    WS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&L.h_vout), L.cap_v * sizeof(ws_verify_out),
                          cudaHostAllocDefault));
    // staging: cands (k u32) + forced ((k+1) i32) + cand probs (k f64) + request (u64) + step (u32) per job
    WS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&L.h_stage), L.cap_v * (k_ * 16 + 24) + 256, cudaHostAllocDefault));
  }
  ForwardBatch& b = L.tb;
  b.clear();
  L.forced.assign(static_cast<std::size_t>(nv) * (k_ + 1), -1);
  std::uint32_t* hc = reinterpret_cast<std::uint32_t*>(L.h_stage);
  for (std::uint32_t j = 0; j < nv; ++j) {
    const VerifyJob& vj = jobs.verify[j];
    const std::uint32_t r = static_cast<std::uint32_t>(vj.request);
    fill_ctx(jobs, r, jobs.verify_ctx[j]);
    L.ctx.insert(L.ctx.end(), jobs.cands.begin() + vj.cand_off, jobs.cands.begin() + vj.cand_off + vj.k);
    const std::int32_t n_ctx = static_cast<std::int32_t>(L.ctx.size());
    const std::int32_t first = n_ctx - static_cast<std::int32_t>(k_) - 1;  // = P + base - 1
    if (n_ctx > MC) throw ConfigError("model path: verify context " + std::to_string(n_ctx) + " exceeds max_ctx");
    LinearCache& c = I.tgt[r];
    std::int32_t lcp = 0;
    while (lcp < first && lcp < static_cast<std::int32_t>(c.valid.size()) && c.valid[lcp] == L.ctx[lcp]) ++lcp;
    const std::int32_t base_slot = static_cast<std::int32_t>(r) * MC;
    const std::int32_t row0 = static_cast<std::int32_t>(b.tok.size());
    const std::int32_t eoff = static_cast<std::int32_t>(b.extra.size());
    for (std::int32_t p = lcp; p < n_ctx; ++p) {
      b.tok.push_back(static_cast<std::int32_t>(L.ctx[p]));
      b.pos.push_back(p);
      b.slot.push_back(base_slot + p);
      b.extra.push_back(base_slot + p);
    }
    b.groups.push_back(AttnGroup{row0, n_ctx - lcp, base_slot, lcp, eoff, n_ctx - lcp});
    b.row_mask.resize(b.tok.size(), 0ull);
    for (std::int32_t p = first; p < n_ctx; ++p) {
      b.out_rows.push_back(row0 + p - lcp);
      b.plant.push_back(p_->plant(L.ctx[p], false));
      L.forced[j * (k_ + 1) + (p - first)] = forced_at(p, P, L_, eos_);
    }
    c.valid.assign(L.ctx.begin(), L.ctx.end());
    std::memcpy(hc + j * k_, jobs.cands.data() + vj.cand_off, k_ * 4);
  }
  std::memcpy(hc + nv * k_, L.forced.data(), L.forced.size() * 4);
  WS_CUDA(cudaMemcpyAsync(L.d_cands, hc, nv * k_ * 4, cudaMemcpyHostToDevice, st));
  WS_CUDA(cudaMemcpyAsync(L.d_forced, hc + nv * k_, L.forced.size() * 4, cudaMemcpyHostToDevice, st));
  const bool rejection = verify_mode_ == WS_VERIFY_REJECTION;
  if (rejection) {  // K4R inputs, staged after the candidates and forced rows
    if (jobs.cand_probs.size() < jobs.cands.size()) throw std::logic_error("model path: candidate probabilities missing");
    unsigned char* h = reinterpret_cast<unsigned char*>(hc + nv * k_ + L.forced.size());
    h = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(h) + 7) & ~std::uintptr_t(7));
    double* hp = reinterpret_cast<double*>(h);
    std::uint64_t* hr = reinterpret_cast<std::uint64_t*>(hp + static_cast<std::size_t>(nv) * k_);
    std::uint32_t* hs = reinterpret_cast<std::uint32_t*>(hr + nv);
    for (std::uint32_t j = 0; j < nv; ++j) {
      const VerifyJob& vj = jobs.verify[j];
      std::memcpy(hp + static_cast<std::size_t>(j) * k_, jobs.cand_probs.data() + vj.cand_off, k_ * sizeof(double));
      hr[j] = vj.request;
      hs[j] = vj.step;
    }
    WS_CUDA(cudaMemcpyAsync(L.d_cprob, hp, static_cast<std::size_t>(nv) * k_ * sizeof(double), cudaMemcpyHostToDevice, st));
    WS_CUDA(cudaMemcpyAsync(L.d_req, hr, nv * sizeof(std::uint64_t), cudaMemcpyHostToDevice, st));
    WS_CUDA(cudaMemcpyAsync(L.d_step, hs, nv * sizeof(std::uint32_t), cudaMemcpyHostToDevice, st));
    stats.h2d += static_cast<std::size_t>(nv) * (k_ * 8 + 12);
  }
  WS_CUDA(cudaEventRecord(L.e0, st));
  // NVTX: one range per verify / draft forward submission (SURVEY §5 tracing; host ranges that
  // nsys / ncu correlate with the launches they enclose)
  nvtxRangePushA("ws.verify");
  p_->target().forward(b, cfg.plant_target, st, *L.ws_t);
  if (rejection)
    verify_rejection_bf16(L.ws_t->logits, nv, k_, V, V, inv_temp_, top_p_, L.d_cands, L.d_cprob, sample_seed_,
                          L.d_req, L.d_step, L.d_forced, L.d_vout, st);
  else
    row_stats_bf16(L.ws_t->logits, nv * (k_ + 1), V, V, 1.0f, L.d_pred, nullptr, L.d_ws, nv, k_, L.d_cands,
                   L.d_vout, st, L.d_forced);
  nvtxRangePop();
  WS_CUDA(cudaEventRecord(L.e1, st));
  WS_CUDA(cudaMemcpyAsync(L.h_vout, L.d_vout, nv * sizeof(ws_verify_out), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaEventRecord(L.done, st));
  target_rows += b.tok.size();
  target_out_rows += b.out_rows.size();
  target_forwards += 1;
  stats.launches += 1 + 8ull * p_->target().shape().layers + 4;
  stats.h2d += nv * k_ * 4 + L.forced.size() * 4;
  stats.d2h += nv * sizeof(ws_verify_out);
  stats.verify_rows += nv;
}

// Lanes 1..n: one draft forward over every pending draft job (worker leaves as shared-prefix
// tree groups, controller local drafts / catch-up as causal groups), then K3/K4 row statistics.
void ModelBackend_Llama::submit_draft(int lane, const RoundJobs& jobs) {
  DraftLane& G = *ln_->dl.at(lane - 1);
  G.nd = static_cast<std::uint32_t>(jobs.draft.size());
  for (auto& d : G.sub) {
    d->idx.clear();
    d->nd = 0;
    d->ran = false;
  }
  if (!G.nd) return;
  ++draft_batch_;
  for (std::uint32_t j = 0; j < G.nd; ++j) G.sub[p_->replica_of(jobs.draft[j].seq)]->idx.push_back(j);
  for (auto& d : G.sub)
    if (!d->idx.empty()) submit_draft_sub(lane, *d, jobs);
  for (auto& d : G.sub)
    if (d->ran) {  // one logical draft forward (its replicas' shares run concurrently)
      draft_forwards += 1;
      break;
    }
  // the lane's completion: sub-lane 0's stream after every other sub-lane's work
  DraftSub& s0 = *G.sub[0];
  DeviceGuard dg(s0.device);
  for (std::size_t i = 1; i < G.sub.size(); ++i)
    if (!G.sub[i]->idx.empty()) WS_CUDA(cudaStreamWaitEvent(s0.st, G.sub[i]->done, 0));
  WS_CUDA(cudaEventRecord(G.done, draft_stream(lane)));
}

void ModelBackend_Llama::submit_draft_sub(int lane, DraftSub& D, const RoundJobs& jobs) {
  ModelPair::Impl& I = *p_->impl;
  Lanes& L = *ln_;
  DeviceGuard dg(D.device);
  LlamaModel& dm = p_->draft(D.rep);
  const ModelPairCfg& cfg = p_->cfg();
  const std::int32_t P = static_cast<std::int32_t>(cfg.prompt_len);
  const std::int32_t MC = static_cast<std::int32_t>(cfg.max_ctx);
  const std::int32_t V = dm.shape().vocab;
  const std::uint32_t nd = static_cast<std::uint32_t>(D.idx.size());
  D.nd = nd;
  const std::size_t need = static_cast<std::size_t>(nd) + 16;
  if (need > D.cap) {  // the lane is idle here (the driver submits only to idle lanes)
    if (D.d_pred) cudaFree(D.d_pred);
    if (D.d_ws) cudaFree(D.d_ws);
    if (D.h_pred) cudaFreeHost(D.h_pred);
    D.cap = need * 2;
    const std::size_t wsb_ = rowstats_workspace_bytes(static_cast<std::uint32_t>(D.cap), V, 0);
    WS_CUDA(cudaMalloc(&D.d_ws, wsb_));
    WS_CUDA(cudaMemset(D.d_ws, 0, wsb_));
    WS_CUDA(cudaMalloc(&D.d_pred, D.cap * sizeof(ws_pred)));
    WS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&D.h_pred), D.cap * sizeof(ws_pred), cudaHostAllocDefault));
  }
  ForwardBatch& b = D.b;
  b.clear();
  D.job_out.assign(nd, -1);
  D.copy_src.clear();
  D.copy_dst.clear();
  // the open shared-prefix tree group of one request's worker leaves (masked attention group)
  struct TreeGroup {
    bool active = false;
    std::uint32_t req = 0;
    std::int32_t row0 = 0, n_rows = 0, prefix_slot = 0, prefix_len = 0;
    std::vector<std::int32_t> slots;
    int index_of(std::int32_t s) {
      for (std::size_t i = 0; i < slots.size(); ++i)
        if (slots[i] == s) return static_cast<int>(i);
      slots.push_back(s);
      return static_cast<int>(slots.size()) - 1;
    }
  } wg;
  std::vector<std::int32_t> anc, row_slots;
  auto flush_wg = [&] {
    if (!wg.active) return;
    const std::int32_t eo = static_cast<std::int32_t>(b.extra.size());
    b.extra.insert(b.extra.end(), wg.slots.begin(), wg.slots.end());
    b.groups.push_back(AttnGroup{wg.row0, wg.n_rows, wg.prefix_slot, wg.prefix_len, eo,
                                 static_cast<std::int32_t>(wg.slots.size()), 1, 0});
    wg.active = false;
  };
  const std::int32_t S = 2 * MC + static_cast<std::int32_t>(cfg.trie_slots);
  for (std::uint32_t j = 0; j < nd; ++j) {
    const DraftJob& dj = jobs.draft[D.idx[j]];
    const JobCtx& jc = jobs.draft_ctx[D.idx[j]];
    const std::uint32_t r = dj.seq;
    fill_ctx(jobs, r, jc);
    const std::int32_t n_ctx = static_cast<std::int32_t>(L.ctx.size());
    if (forced_at(n_ctx - 1, P, L_, eos_) >= 0) {
      // Past the generation cap the prediction is a confident EOS whatever the context
      // (oracle.hpp:88-102): no forward, no KV (every descendant is forced too).
      D.job_out[j] = -1;
      continue;
    }
    if (n_ctx > MC)
      throw ConfigError("model path: draft context " + std::to_string(n_ctx) + " exceeds max_ctx (kind " +
                        std::to_string(jc.kind) + ", committed " + std::to_string(jc.n_committed) + ", len " +
                        std::to_string(jc.len) + ")");
    if (jc.kind == kJobCtrlDraft) flush_wg();
    const std::int32_t row0 = static_cast<std::int32_t>(b.tok.size());
    const std::int32_t eoff = static_cast<std::int32_t>(b.extra.size());
    if (jc.kind == kJobCtrlDraft) {  // controller local draft + catch-up prefill (controller.hpp:194-208)
      LinearCache& c = I.ctrl[r];
      std::int32_t lcp = 0;
      while (lcp < n_ctx - 1 && lcp < static_cast<std::int32_t>(c.valid.size()) && c.valid[lcp] == L.ctx[lcp]) ++lcp;
      const std::int32_t base_slot = static_cast<std::int32_t>(r) * S;
      for (std::int32_t p = lcp; p < n_ctx; ++p) {
        b.tok.push_back(static_cast<std::int32_t>(L.ctx[p]));
        b.pos.push_back(p);
        b.slot.push_back(base_slot + p);
        b.extra.push_back(base_slot + p);
      }
      b.groups.push_back(AttnGroup{row0, n_ctx - lcp, base_slot, lcp, eoff, n_ctx - lcp});
      c.valid.assign(L.ctx.begin(), L.ctx.end());
    } else {  // worker leaf: committed prefix + trie
      TreeCache& t = I.wrk[r];
      const std::int32_t pre_base = static_cast<std::int32_t>(r) * S + MC;
      if (!t.init) t.reset(static_cast<std::int32_t>(r) * S + 2 * MC, static_cast<std::int32_t>(cfg.trie_slots));
      const std::int32_t n_comm = P + static_cast<std::int32_t>(jc.n_committed);
      // prefix must agree with the context (committed is append-only; defensive check)
      std::int32_t pl = static_cast<std::int32_t>(t.prefix.size());
      std::int32_t agree = 0;
      while (agree < pl && agree < n_comm && t.prefix[agree] == L.ctx[agree]) ++agree;
      if (agree < pl) {
        t.prefix.resize(agree);
        t.drop_all();
        pl = agree;
      }
      // migrate speculative nodes that became committed into the prefix
      std::int32_t cur = -1;
      while (pl < n_comm) {
        const std::int32_t c = t.find(cur, L.ctx[pl]);
        if (c < 0) break;
        D.copy_src.push_back(t.nodes[c].slot);
        D.copy_dst.push_back(pre_base + pl);
        t.prefix.push_back(L.ctx[pl]);
        ++pl;
        cur = c;
      }
      if (cur >= 0) t.reroot_at(cur);  // copies are queued before this batch's forward
      if (pl < n_comm) t.drop_all();   // committed diverged from every cached branch
      // node-slot pressure: stale branches are dropped (never within a batch that already
      // allocated for this request — those slots are written by this batch's forward)
      if (static_cast<std::int32_t>(t.free_slots.size()) < n_ctx - n_comm + 2) {
        if (t.last_alloc_round == draft_batch_) throw std::logic_error("model path: worker trie slots exhausted");
        t.drop_all();
      }
      // Rows: committed tokens missing from the prefix, else the unmatched tail of the
      // speculative path; the last token is always fed (its logits are the output).
      //   prefix_len_g = pl           (committed rows follow)
      //                = n_ctx - 1    (root job, everything cached: re-feed the last token)
      //                = n_comm       (leaf job: matched trie ancestors, then the leaf)
      const std::int32_t prefix_len_g = pl < n_comm ? pl : (n_ctx == n_comm ? n_ctx - 1 : n_comm);
      std::int32_t q = prefix_len_g;
      std::int32_t node = -1;
      anc.clear();
      const bool leaf_job = q == n_comm && n_ctx > n_comm;
      if (leaf_job) {
        while (q < n_ctx - 1) {
          const std::int32_t c = t.find(node, L.ctx[q]);
          if (c < 0) break;
          anc.push_back(t.nodes[c].slot);
          node = c;
          ++q;
        }
      }
      const std::int32_t rows = n_ctx - q;
      row_slots.clear();
      for (std::int32_t p = q; p < n_ctx; ++p) {
        std::int32_t slot;
        if (p < n_comm) {
          slot = pre_base + p;
        } else {
          std::int32_t c = t.find(node, L.ctx[p]);
          if (c < 0) {
            c = t.add(node, L.ctx[p]);
            t.last_alloc_round = draft_batch_;
          }
          slot = t.nodes[c].slot;
          node = c;
        }
        b.tok.push_back(static_cast<std::int32_t>(L.ctx[p]));
        b.pos.push_back(p);
        b.slot.push_back(slot);
        row_slots.push_back(slot);
      }
      for (std::int32_t p = pl; p < std::min(n_comm, n_ctx); ++p) t.prefix.push_back(L.ctx[p]);
      if (!leaf_job || anc.size() + row_slots.size() > 64) {
        // root / catch-up job: its own causal group
        flush_wg();
        const std::int32_t eo = static_cast<std::int32_t>(b.extra.size());
        b.extra.insert(b.extra.end(), anc.begin(), anc.end());
        b.extra.insert(b.extra.end(), row_slots.begin(), row_slots.end());
        b.row_mask.resize(b.tok.size(), 0ull);
        b.groups.push_back(AttnGroup{row0, rows, pre_base, prefix_len_g, eo,
                                     static_cast<std::int32_t>(b.extra.size()) - eo});
      } else {
        // leaf job: joins the request's shared-prefix tree group (one pass over the prefix
        // for all of the request's leaves); each row sees its ancestor chain + itself
        if (wg.active && (wg.req != r || wg.slots.size() + anc.size() + row_slots.size() > 64)) flush_wg();
        if (!wg.active) {
          wg.active = true;
          wg.req = r;
          wg.row0 = row0;
          wg.n_rows = 0;
          wg.prefix_slot = pre_base;
          wg.prefix_len = n_comm;
          wg.slots.clear();
        }
        unsigned long long mask = 0ull;
        for (std::int32_t s : anc) mask |= 1ull << wg.index_of(s);
        for (std::int32_t s : row_slots) {
          mask |= 1ull << wg.index_of(s);
          b.row_mask.push_back(mask);
        }
        wg.n_rows += rows;
      }
    }
    if (jc.kind == kJobCtrlDraft) b.row_mask.resize(b.tok.size(), 0ull);
    const std::int32_t last = static_cast<std::int32_t>(b.tok.size()) - 1;
    rows_by_kind[jc.kind] += static_cast<std::uint64_t>(last + 1 - row0);
    jobs_by_kind[jc.kind] += 1;
    D.job_out[j] = static_cast<std::int32_t>(b.out_rows.size());
    b.out_rows.push_back(last);
    b.plant.push_back(p_->plant(L.ctx[n_ctx - 1], true));
  }
  flush_wg();
  if (b.row_mask.size() != b.tok.size()) throw std::logic_error("model path: row mask bookkeeping");
  const std::uint32_t n_out = static_cast<std::uint32_t>(b.out_rows.size());
  cudaStream_t sd = D.rep == 0 ? draft_stream(lane) : D.st;
  if (n_out) {
    dm.copy_slots(D.copy_src, D.copy_dst, sd, *D.ws);
    WS_CUDA(cudaEventRecord(D.e_start, sd));
    nvtxRangePushA("ws.draft");
    dm.forward(b, cfg.plant_draft, sd, *D.ws);
    row_stats_bf16(D.ws->logits, n_out, V, V, 1.0f, D.d_pred, nullptr, D.d_ws, 0, 0, nullptr, nullptr, sd,
                   nullptr);
    nvtxRangePop();
    WS_CUDA(cudaEventRecord(D.e_end, sd));
    WS_CUDA(cudaMemcpyAsync(D.h_pred, D.d_pred, n_out * sizeof(ws_pred), cudaMemcpyDeviceToHost, sd));
    D.ran = true;
    draft_rows_fed += b.tok.size();
    draft_out_rows += n_out;
    stats.launches += 1 + 8ull * dm.shape().layers + 4 + (D.copy_src.empty() ? 0 : 1);
    stats.d2h += n_out * sizeof(ws_pred);
  }
  WS_CUDA(cudaEventRecord(D.done, sd));
  stats.draft_rows += nd;
}

cudaStream_t ModelBackend_Llama::draft_stream(int lane) const {
  // WS_SERIAL=1 serialises every forward on one stream (clean per-kernel profiles); default
  // overlaps the lanes
  static const bool serial = std::getenv("WS_SERIAL") != nullptr;
  const DraftSub& s0 = *ln_->dl.at(lane - 1)->sub[0];
  return serial && s0.device == ln_->device ? ln_->st_t : s0.st;
}

std::size_t ModelBackend_Llama::submit(int lane, const RoundJobs& jobs, int verify_mode, std::uint64_t sample_seed) {
  if (verify_mode != WS_VERIFY_GREEDY && verify_mode != WS_VERIFY_REJECTION)
    throw ConfigError("model path: unknown verify mode");
  verify_mode_ = verify_mode;
  sample_seed_ = sample_seed;
  stats.rounds += 1;
  const auto t0 = std::chrono::steady_clock::now();
  std::size_t took;
  if (lane == 0) {
    took = verify_take(jobs);
    submit_verify(jobs, took);
  } else {
    submit_draft(lane, jobs);
    took = jobs.draft.size();
  }
  host_submit_ms[lane == 0 ? 0 : 1] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return took;
}

int ModelBackend_Llama::wait_any(std::uint32_t busy) {
  Lanes& L = *ln_;
  const int n = n_lanes();
  const auto t0 = std::chrono::steady_clock::now();
  struct Acc {
    double& ms;
    std::chrono::steady_clock::time_point t0;
    ~Acc() { ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
  } acc{host_wait_ms, t0};
  for (;;) {
    for (int lane = 0; lane < n; ++lane) {
      if (!(busy & (1u << lane))) continue;
      // each event is queried with its own GPU current (split placement: two devices)
      DeviceGuard dg(lane == 0 ? L.device : L.dl[lane - 1]->sub[0]->device);
      const cudaError_t e = cudaEventQuery(lane == 0 ? L.done : L.dl[lane - 1]->done);
      if (e == cudaSuccess) return lane;
      if (e != cudaErrorNotReady) WS_CUDA(e);
    }
    std::this_thread::yield();
  }
}

void ModelBackend_Llama::verify_rows(ws_pred* host, std::size_t n_rows) {
  Lanes& L = *ln_;
  if (n_rows > static_cast<std::size_t>(L.nv) * (k_ + 1)) throw std::invalid_argument("verify_rows: too many rows");
  if (!n_rows) return;
  DeviceGuard dg(L.device);
  WS_CUDA(cudaMemcpy(host, L.d_pred, n_rows * sizeof(ws_pred), cudaMemcpyDeviceToHost));
}

int ModelBackend_Llama::poll_any(std::uint32_t busy) {
  Lanes& L = *ln_;
  for (int lane = 0; lane < n_lanes(); ++lane) {
    if (!(busy & (1u << lane))) continue;
    DeviceGuard dg(lane == 0 ? L.device : L.dl[lane - 1]->sub[0]->device);
    const cudaError_t e = cudaEventQuery(lane == 0 ? L.done : L.dl[lane - 1]->done);
    if (e == cudaSuccess) return lane;
    if (e != cudaErrorNotReady) WS_CUDA(e);
  }
  return -1;
}

void ModelBackend_Llama::complete(int lane, RoundResults& res) {
  Lanes& L = *ln_;
  DeviceGuard dg(lane == 0 ? L.device : L.dl.at(lane - 1)->sub[0]->device);
  float ms = 0.f;
  if (lane == 0) {
    res.verify.resize(L.nv);
    if (!L.nv) return;
    WS_CUDA(cudaEventSynchronize(L.done));
    std::memcpy(res.verify.data(), L.h_vout, L.nv * sizeof(ws_verify_out));
    WS_CUDA(cudaEventElapsedTime(&ms, L.e0, L.e1));
    target_ms += ms;
  } else {
    DraftLane& G = *L.dl.at(lane - 1);
    res.draft.resize(G.nd);
    if (!G.nd) return;
    WS_CUDA(cudaEventSynchronize(G.done));
    float lane_ms = 0.f;  // the sub-lanes run concurrently: the unit's time is the longest
    for (auto& dp : G.sub) {
      DraftSub& D = *dp;
      for (std::uint32_t t = 0; t < D.nd; ++t) {
        const std::uint32_t j = D.idx[t];
        if (D.job_out[t] >= 0) {
          res.draft[j] = D.h_pred[D.job_out[t]];
        } else {
          ws_pred e{};
          e.n = 1;
          e.id[0] = eos_;
          e.prob[0] = 1.0;
          res.draft[j] = e;
        }
      }
      if (D.ran) {
        DeviceGuard dd(D.device);
        WS_CUDA(cudaEventElapsedTime(&ms, D.e_start, D.e_end));
        lane_ms = std::max(lane_ms, ms);
      }
    }
    draft_ms += lane_ms;
  }
  stats.kernel_ms = target_ms + draft_ms;
}

// Lockstep round (WS_LOCKSTEP=1): both lanes, then both results.
void ModelBackend_Llama::run_round(const RoundJobs& jobs, RoundResults& res, int verify_mode,
                                   std::uint64_t sample_seed) {
  verify_mode_ = verify_mode;
  sample_seed_ = sample_seed;
  stats.rounds += 1;
  submit_verify(jobs, jobs.verify.size());  // lockstep rounds take every job
  submit_draft(1, jobs);
  complete(0, res);
  complete(1, res);
}

}  // namespace wsb
