// Batched Llama forward (see llama.hpp).
#include "llama.hpp"

#include <chrono>

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "../kernels/cuda_check.hpp"
#include "../kernels/gemm_tc.cuh"
#include "llama_tp.hpp"

namespace wsb {

std::int64_t LlamaShape::params_mm() const {
  const std::int64_t per = static_cast<std::int64_t>(qkv_dim()) * d + static_cast<std::int64_t>(d) * n_q * hd +
                           3ll * ffn * d;
  return per * layers + static_cast<std::int64_t>(vocab) * d;
}

LlamaShape shape_by_name(const std::string& name) {
  // "<shape>:L<n>" — the named shape truncated to its first n layers (real-shape parity tests)
  if (const std::size_t c = name.find(":L"); c != std::string::npos) {
    LlamaShape s = shape_by_name(name.substr(0, c));
    const int n = std::atoi(name.c_str() + c + 2);
    if (n < 1 || n > s.layers) throw ConfigError("bad layer truncation: " + name);
    s.layers = n;
    s.name = name;
    return s;
  }
  // Llama-3.1-8B / Llama-3.2-1B / Llama-3.1-70B hyper-parameters (BASELINE configs 3 and 5).
  if (name == "llama3-8b") return LlamaShape{name, 32, 4096, 32, 8, 128, 14336, 128256, 1e-5f, 500000.f, 8.f, false};
  if (name == "llama3.2-1b") return LlamaShape{name, 16, 2048, 32, 8, 64, 8192, 128256, 1e-5f, 500000.f, 32.f, true};
  if (name == "llama3-70b") return LlamaShape{name, 80, 8192, 64, 8, 128, 28672, 128256, 1e-5f, 500000.f, 8.f, false};
  if (name == "tiny") return LlamaShape{name, 2, 256, 4, 2, 64, 512, 1000, 1e-5f, 10000.f, 0.f, false};
  if (name == "tiny-draft") return LlamaShape{name, 1, 256, 4, 2, 64, 512, 1000, 1e-5f, 10000.f, 0.f, true};
  if (name == "tiny128") return LlamaShape{name, 2, 512, 4, 1, 128, 1024, 2000, 1e-5f, 500000.f, 8.f, false};
  throw ConfigError("unknown model shape: " + name);
}

namespace {

// HF Llama-3 rope scaling (low/high freq factors 1/4, original context 8192).
std::vector<float> llama3_inv_freq(const LlamaShape& s) {
  std::vector<float> f(s.hd / 2);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < s.hd / 2; ++i) {
    double inv = 1.0 / std::pow(static_cast<double>(s.rope_theta), (2.0 * i) / s.hd);
    if (s.rope_factor > 0.f) {
      const double factor = s.rope_factor, lo = 1.0, hi = 4.0, old_ctx = 8192.0;
      const double wavelen = 2 * pi / inv;
      const double lo_wl = old_ctx / lo, hi_wl = old_ctx / hi;
      if (wavelen > lo_wl) {
        inv = inv / factor;
      } else if (wavelen >= hi_wl) {
        const double smooth = (old_ctx / wavelen - lo) / (hi - lo);
        inv = (1 - smooth) * inv / factor + smooth * inv;
      }
    }
    f[i] = static_cast<float>(inv);
  }
  return f;
}

std::size_t al(std::size_t x) { return (x + 255) & ~static_cast<std::size_t>(255); }

}  // namespace

LlamaModel::LlamaModel(const LlamaShape& s, std::uint64_t seed, std::int64_t n_slots, int max_rows, int device, int tp)
    : s_(s), device_(device), n_slots_(n_slots), tp_(tp < 1 ? 1 : tp) {
  WS_CUDA(cudaSetDevice(device));
  if (s.d % 64 || s.ffn % 64 || (s.n_q * s.hd) % 64) throw ConfigError("model dims must be multiples of 64");
  if (s.n_q % s.n_kv) throw ConfigError("n_q must be a multiple of n_kv");
  if (tp_ > 1) {  // weights, KV pools and activations live in the per-rank shards
    init_tp(seed, max_rows);
    return;
  }
  // ---- weights in one block ----
  const std::size_t d = s.d, V = s.vocab;
  std::vector<std::pair<void**, std::size_t>> tensors;
  attn_norm_.resize(s.layers);
  wqkv_.resize(s.layers);
  wo_.resize(s.layers);
  mlp_norm_.resize(s.layers);
  wgu_.resize(s.layers);
  wdown_.resize(s.layers);
  std::size_t total = 0;
  auto reserve = [&](std::size_t elems) {
    const std::size_t off = total;
    total += al(elems * 2);
    return off;
  };
  struct Item {
    void** dst;
    std::size_t off, n;
    float std_, mean;
  };
  std::vector<Item> items;
  items.push_back({&embed_, reserve(V * d), V * d, 0.02f, 0.f});
  for (int l = 0; l < s.layers; ++l) {
    items.push_back({&attn_norm_[l], reserve(d), d, 0.f, 1.f});
    items.push_back({&wqkv_[l], reserve(static_cast<std::size_t>(s.qkv_dim()) * d), static_cast<std::size_t>(s.qkv_dim()) * d, 0.02f, 0.f});
    items.push_back({&wo_[l], reserve(d * s.n_q * s.hd), d * s.n_q * s.hd, 0.02f, 0.f});
    items.push_back({&mlp_norm_[l], reserve(d), d, 0.f, 1.f});
    items.push_back({&wgu_[l], reserve(2 * static_cast<std::size_t>(s.ffn) * d), 2 * static_cast<std::size_t>(s.ffn) * d, 0.02f, 0.f});
    items.push_back({&wdown_[l], reserve(d * s.ffn), d * s.ffn, 0.02f, 0.f});
  }
  items.push_back({&final_norm_, reserve(d), d, 0.f, 1.f});
  if (!s.tied) items.push_back({&lm_head_, reserve(V * d), V * d, 0.02f, 0.f});
  WS_CUDA(cudaMalloc(&weight_block_, total));
  std::uint32_t sid = 1;
  for (const Item& it : items) {
    *it.dst = static_cast<unsigned char*>(weight_block_) + it.off;
    fill_normal_bf16(*it.dst, static_cast<std::int64_t>(it.n), seed, sid++, it.std_, it.mean, nullptr);
  }
  if (s.tied) lm_head_ = embed_;
  // RMSNorm weights are folded into the projections they feed (the GEMMs apply only the
  // per-row rsqrt scale, gemm_tc.cuh NormEpi); the norm tensors stay for reference/tests.
  for (int l = 0; l < s.layers; ++l) {
    fold_norm_weight(wqkv_[l], s.qkv_dim(), s.d, attn_norm_[l], nullptr);
    fold_norm_weight(wgu_[l], 2 * static_cast<std::int64_t>(s.ffn), s.d, mlp_norm_[l], nullptr);
  }
  const std::vector<float> inv = llama3_inv_freq(s);
  WS_CUDA(cudaMalloc(&inv_freq_, inv.size() * sizeof(float)));
  WS_CUDA(cudaMemcpy(inv_freq_, inv.data(), inv.size() * sizeof(float), cudaMemcpyHostToDevice));
  {  // cos/sin table [kMaxPos][hd/2] in fp64 → fp32 (the fused QKV epilogue reads it)
    std::vector<float2> cs(static_cast<std::size_t>(kMaxPos) * (s.hd / 2));
    for (int p = 0; p < kMaxPos; ++p)
      for (int i = 0; i < s.hd / 2; ++i) {
        const double a = static_cast<double>(p) * static_cast<double>(inv[i]);
        cs[static_cast<std::size_t>(p) * (s.hd / 2) + i] = make_float2(static_cast<float>(std::cos(a)),
                                                                       static_cast<float>(std::sin(a)));
      }
    WS_CUDA(cudaMalloc(reinterpret_cast<void**>(&rope_cs_), cs.size() * sizeof(float2)));
    WS_CUDA(cudaMemcpy(rope_cs_, cs.data(), cs.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }
  // ---- KV pools ----
  const std::size_t pool = static_cast<std::size_t>(s.layers) * n_slots * s.n_kv * s.hd * 2;
  WS_CUDA(cudaMalloc(&k_pool_, pool));
  WS_CUDA(cudaMalloc(&v_pool_, pool));
  WS_CUDA(cudaMemset(k_pool_, 0, pool));
  WS_CUDA(cudaMemset(v_pool_, 0, pool));
  ws0_ = make_workspace(max_rows);
  if (std::getenv("WS_PROFILE_MODEL")) ws0_->prof.enable(true);  // per-class times (probes)
  WS_CUDA(cudaDeviceSynchronize());
}

std::unique_ptr<ForwardWorkspace> LlamaModel::make_workspace(int max_rows) const {
  WS_CUDA(cudaSetDevice(device_));
  std::unique_ptr<ForwardWorkspace> ws(new ForwardWorkspace(device_));
  ensure_rows(*ws, max_rows, max_rows);
  // split-K partials (row-sliced beyond 4096 rows; WS_GEMM_WS_ROWS shrinks it for the slicing tests)
  const char* wr = std::getenv("WS_GEMM_WS_ROWS");
  ws->gemm_ws_bytes = gemm_workspace_bytes(wr ? std::max(1, std::atoi(wr)) : 4096);
  WS_CUDA(cudaMalloc(&ws->gemm_ws, ws->gemm_ws_bytes));
  WS_CUDA(cudaMemset(ws->gemm_ws, 0, ws->gemm_ws_bytes));
  return ws;
}

ForwardWorkspace::~ForwardWorkspace() {
  cudaSetDevice(device);
  for (void* p : {static_cast<void*>(x), xb, static_cast<void*>(ss), qkv, q, attn, h, logits, xo,
                  static_cast<void*>(d_meta), gemm_ws})
    if (p) cudaFree(p);
  if (h_meta) cudaFreeHost(h_meta);
  if (meta_ev) cudaEventDestroy(meta_ev);
}

LlamaModel::~LlamaModel() {
  cudaSetDevice(device_);
  if (ws0_ && ws0_->prof.on()) {  // WS_PROFILE_MODEL: the own workspace's per-class device time
    KernelProfiler& p = ws0_->prof;
    p.collect();
    std::fprintf(stderr, "[ws-profile] {\"model\": \"%s\"", s_.name.c_str());
    for (int k = 0; k < KernelProfiler::kClasses; ++k)
      std::fprintf(stderr, ", \"%s\": [%.3f, %llu]", KernelProfiler::name(k), p.ms[k],
                   static_cast<unsigned long long>(p.count[k]));
    std::fprintf(stderr, "}\n");
  }
  if (ws0_ && ws0_->host_fwd && std::getenv("WS_PROFILE_HOST"))
    std::fprintf(stderr, "[ws-host] {\"model\": \"%s\", \"forwards\": %llu, \"host_ms_per_forward\": %.4f}\n",
                 s_.name.c_str(), static_cast<unsigned long long>(ws0_->host_fwd), ws0_->host_ms / ws0_->host_fwd);
  if (rope_cs_) cudaFree(rope_cs_);
  ws0_.reset();
  for (void* p : {weight_block_, static_cast<void*>(inv_freq_), k_pool_, v_pool_})
    if (p) cudaFree(p);
}

void LlamaModel::ensure_rows(ForwardWorkspace& ws, int rows, int out_rows) const {
  if (tp_ > 1) return ensure_tp(ws, rows, out_rows);
  if (rows <= ws.cap_rows && out_rows <= ws.cap_out) return;
  rows = std::max(rows, ws.cap_rows);
  out_rows = std::max(out_rows, ws.cap_out);
  for (void* p : {static_cast<void*>(ws.x), ws.xb, static_cast<void*>(ws.ss), ws.qkv, ws.q, ws.attn, ws.h, ws.logits,
                  ws.xo})
    if (p) cudaFree(p);
  const std::size_t R = rows, O = out_rows;
  WS_CUDA(cudaMalloc(reinterpret_cast<void**>(&ws.x), R * s_.d * 4));
  WS_CUDA(cudaMalloc(&ws.xb, R * s_.d * 2));
  WS_CUDA(cudaMalloc(reinterpret_cast<void**>(&ws.ss), R * (s_.d / 32) * 4));
  WS_CUDA(cudaMalloc(&ws.qkv, R * s_.qkv_dim() * 2));
  WS_CUDA(cudaMalloc(&ws.q, R * s_.n_q * s_.hd * 2));
  WS_CUDA(cudaMalloc(&ws.attn, R * s_.n_q * s_.hd * 2));
  WS_CUDA(cudaMalloc(&ws.h, R * s_.ffn * 2));
  WS_CUDA(cudaMalloc(&ws.xo, O * s_.d * 2));
  WS_CUDA(cudaMalloc(&ws.logits, O * static_cast<std::size_t>(s_.vocab) * 2));
  ws.cap_rows = rows;
  ws.cap_out = out_rows;
}

void* LlamaModel::weight(const std::string& w, int l, std::int64_t* numel) {
  const std::int64_t d = s_.d;
  auto ret = [&](void* p, std::int64_t n) {
    if (numel) *numel = n;
    return p;
  };
  if (w == "embed") return ret(embed_, d * s_.vocab);
  if (w == "lm_head") return ret(lm_head_, d * s_.vocab);
  if (w == "final_norm") return ret(final_norm_, d);
  // the last forward's activations in the model's own workspace (stage-wise parity tests):
  // ws_x = fp32 residual [cap_rows][d] (numel counted in bf16 units); ws_q / ws_attn / ws_h =
  // the last layer's rotated q, attention output and SwiGLU output (bf16)
  if (w == "ws_x") return ret(ws0_->x, 2ll * ws0_->cap_rows * d);
  if (w == "ws_attn") return ret(ws0_->attn, static_cast<std::int64_t>(ws0_->cap_rows) * s_.n_q * s_.hd);
  if (w == "ws_h") return ret(ws0_->h, static_cast<std::int64_t>(ws0_->cap_rows) * s_.ffn);
  if (w == "ws_q") return ret(ws0_->q, static_cast<std::int64_t>(ws0_->cap_rows) * s_.n_q * s_.hd);
  if (w == "ws_xo") return ret(ws0_->xo, static_cast<std::int64_t>(ws0_->cap_out) * d);
  // the KV pools [layer][slot][n_kv][hd] (tests read back what the QKV epilogue stored)
  if (w == "k_pool" || w == "v_pool")
    return ret(w == "k_pool" ? k_pool_ : v_pool_, static_cast<std::int64_t>(s_.layers) * n_slots_ * s_.n_kv * s_.hd);
  if (l < 0 || l >= s_.layers) throw std::invalid_argument("layer out of range");
  if (w == "attn_norm") return ret(attn_norm_[l], d);
  if (w == "mlp_norm") return ret(mlp_norm_[l], d);
  if (w == "wqkv") return ret(wqkv_[l], d * s_.qkv_dim());
  if (w == "wo") return ret(wo_[l], d * s_.n_q * s_.hd);
  if (w == "wgu") return ret(wgu_[l], d * 2 * s_.ffn);
  if (w == "wdown") return ret(wdown_[l], d * s_.ffn);
  throw std::invalid_argument("unknown weight " + w);
}

void LlamaModel::copy_slots(const std::vector<std::int32_t>& src, const std::vector<std::int32_t>& dst,
                            cudaStream_t st, ForwardWorkspace& ws) {
  if (src.empty()) return;
  unsigned char*& d_meta_ = ws.d_meta;
  unsigned char*& h_meta_ = ws.h_meta;
  std::size_t& cap_meta_ = ws.cap_meta;
  std::size_t& h2d_ = ws.h2d;
  const std::size_t n = src.size();
  const std::size_t need = 2 * n * 4;
  if (need > cap_meta_) {
    if (d_meta_) cudaFree(d_meta_);
    if (h_meta_) cudaFreeHost(h_meta_);
    cap_meta_ = std::max(need, 2 * cap_meta_);
    WS_CUDA(cudaMalloc(&d_meta_, cap_meta_));
    WS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_meta_), cap_meta_, cudaHostAllocDefault));
  }
  WS_CUDA(cudaStreamSynchronize(st));  // staging reuse
  std::memcpy(h_meta_, src.data(), n * 4);
  std::memcpy(h_meta_ + n * 4, dst.data(), n * 4);
  WS_CUDA(cudaMemcpyAsync(d_meta_, h_meta_, need, cudaMemcpyHostToDevice, st));
  h2d_ += need;
  wsb::copy_slots(k_pool_, v_pool_, reinterpret_cast<std::int32_t*>(d_meta_),
                  reinterpret_cast<std::int32_t*>(d_meta_ + n * 4), static_cast<int>(n), s_.layers,
                  n_slots_ * s_.n_kv * s_.hd, s_.n_kv * s_.hd, st);
  WS_CUDA(cudaStreamSynchronize(st));
}

MetaLayout LlamaModel::pack_meta(const ForwardBatch& b, ForwardWorkspace& ws, cudaStream_t st) const {
  const int n = static_cast<int>(b.tok.size());
  const int n_out = static_cast<int>(b.out_rows.size());
  // ---- one packed H2D for all metadata ----
  // attention entries: one per CTA pass of attention_vectors_per_cta query vectors (a catch-up
  // group larger than that becomes several entries; pad = its first vector)
  const int G = s_.n_q / s_.n_kv;
  const int vpc = attention_vectors_per_cta(s_.hd);
  ws.grp_sorted.clear();
  for (const AttnGroup& g : b.groups) {
    ws.kv_pos += static_cast<std::uint64_t>(g.prefix_len + g.extra_len);
    ws.attn_pairs += static_cast<std::uint64_t>(g.n_rows) * (g.prefix_len + g.extra_len);
  }
  for (const AttnGroup& g : b.groups)
    for (int v0 = 0; v0 < g.n_rows * G; v0 += vpc) {
      AttnGroup e = g;
      e.pad = v0;
      ws.grp_sorted.push_back(e);
    }
  const std::size_t s_tok = al(n * 4), s_grp = al(ws.grp_sorted.size() * sizeof(AttnGroup)), s_ext = al(b.extra.size() * 4 + 4),
                    s_out = al(n_out * 4 + 4);
  const std::size_t s_msk = al(b.row_mask.size() * 8 + 8);
  const std::size_t need = 3 * s_tok + s_grp + s_ext + 2 * s_out + s_msk;
  // the previous forward's metadata copy out of the pinned staging has retired (only that copy —
  // not the whole previous forward, so the host can queue this forward while that one runs;
  // the device block d_meta is overwritten in stream order after the previous forward's kernels)
  if (ws.meta_pending) WS_CUDA(cudaEventSynchronize(ws.meta_ev));
  ws.meta_pending = false;
  if (need > ws.cap_meta) {
    WS_CUDA(cudaStreamSynchronize(st));  // d_meta may still be read by the previous forward
    if (ws.d_meta) cudaFree(ws.d_meta);
    if (ws.h_meta) cudaFreeHost(ws.h_meta);
    ws.cap_meta = std::max(need, 2 * ws.cap_meta);
    WS_CUDA(cudaMalloc(&ws.d_meta, ws.cap_meta));
    WS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ws.h_meta), ws.cap_meta, cudaHostAllocDefault));
  }
  std::size_t o = 0;
  auto put = [&](const void* src, std::size_t bytes, std::size_t slot_bytes) {
    if (bytes) std::memcpy(ws.h_meta + o, src, bytes);
    const std::size_t at = o;
    o += slot_bytes;
    return at;
  };
  const std::size_t o_tok = put(b.tok.data(), n * 4, s_tok);
  const std::size_t o_pos = put(b.pos.data(), n * 4, s_tok);
  const std::size_t o_slot = put(b.slot.data(), n * 4, s_tok);
  const std::size_t o_grp = put(ws.grp_sorted.data(), ws.grp_sorted.size() * sizeof(AttnGroup), s_grp);
  const std::size_t o_ext = put(b.extra.data(), b.extra.size() * 4, s_ext);
  const std::size_t o_out = put(b.out_rows.data(), n_out * 4, s_out);
  const std::size_t o_pl = put(b.plant.data(), b.plant.size() * 4, s_out);
  const std::size_t o_msk = put(b.row_mask.data(), b.row_mask.size() * 8, s_msk);
  WS_CUDA(cudaMemcpyAsync(ws.d_meta, ws.h_meta, o, cudaMemcpyHostToDevice, st));
  if (!ws.meta_ev) WS_CUDA(cudaEventCreateWithFlags(&ws.meta_ev, cudaEventDisableTiming));
  WS_CUDA(cudaEventRecord(ws.meta_ev, st));
  ws.meta_pending = true;
  ws.h2d += o;
  MetaLayout ml;
  ml.tok = o_tok;
  ml.pos = o_pos;
  ml.slot = o_slot;
  ml.grp = o_grp;
  ml.ext = o_ext;
  ml.out = o_out;
  ml.pl = o_pl;
  ml.msk = o_msk;
  ml.bytes = o;
  ml.n_entries = static_cast<int>(ws.grp_sorted.size());
  return ml;
}

// WS_PREFILL_CHUNKS=1 (A/B): prompt-prefill forwards use the shapes' canonical chunks too
static bool prefill_one_chunk() {
  static const bool one = [] {
    const char* e = std::getenv("WS_PREFILL_CHUNKS");
    return !(e && e[0] == '1');
  }();
  return one;
}

void LlamaModel::forward(const ForwardBatch& b, float plant, cudaStream_t st, ForwardWorkspace& ws) {
  const int n = static_cast<int>(b.tok.size());
  const int n_out = static_cast<int>(b.out_rows.size());
  if (n == 0) return;
  if (b.pos.size() != b.tok.size() || b.slot.size() != b.tok.size()) throw std::invalid_argument("forward: ragged rows");
  for (std::int32_t p : b.pos)
    if (p < 0 || p >= kMaxPos) throw std::invalid_argument("forward: position out of the RoPE table range");
  if (tp_ > 1) return forward_tp(b, plant, st, ws);
  struct HostClock {  // the forward's host enqueue time (returns when the last kernel is queued)
    ForwardWorkspace& w;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    ~HostClock() {
      w.host_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      ++w.host_fwd;
    }
  } host_clock{ws};
  ensure_rows(ws, n, n_out);
  float* const x_ = ws.x;
  void* const xb_ = ws.xb;
  float* const ss_ = ws.ss;
  void* const q_ = ws.q;
  void* const attn_ = ws.attn;
  void* const h_ = ws.h;
  void* const logits_ = ws.logits;
  void* const xo_ = ws.xo;
  unsigned char*& d_meta_ = ws.d_meta;
  unsigned char*& h_meta_ = ws.h_meta;
  std::size_t& cap_meta_ = ws.cap_meta;
  std::size_t& h2d_ = ws.h2d;
  std::vector<AttnGroup>& grp_sorted_ = ws.grp_sorted;
  KernelProfiler& prof_ = ws.prof;
  const int cap_rows_ = ws.cap_rows;
  void* const gemm_ws_ = ws.gemm_ws;
  const std::size_t gemm_ws_bytes_ = ws.gemm_ws_bytes;
  const MetaLayout ml = pack_meta(b, ws, st);
  const std::size_t o_tok = ml.tok, o_pos = ml.pos, o_slot = ml.slot, o_grp = ml.grp, o_ext = ml.ext, o_out = ml.out,
                    o_pl = ml.pl, o_msk = ml.msk;
  auto I = [&](std::size_t off) { return reinterpret_cast<const std::int32_t*>(d_meta_ + off); };

  const int d = s_.d, qd = s_.n_q * s_.hd;
  auto with_ws = [&](GemmArgs g) {
    g.ws = gemm_ws_;
    g.ws_bytes = gemm_ws_bytes_;
    g.max_ctas = max_ctas_;
    g.pdl_late = pdl_late_ ? 1 : 0;
    if (b.prefill && prefill_one_chunk()) g.chunks_ = 1;
    return g;
  };
  const std::int64_t layer_stride = n_slots_ * s_.n_kv * s_.hd;
  const AttnShape ash{s_.n_q, s_.n_kv, s_.hd, s_.n_kv * s_.hd, 1.0f / std::sqrt(static_cast<float>(s_.hd))};
  prof_.begin(st);
  // Fused RMSNorm: the embedding and every residual update (O / down epilogues) also emit the
  // bf16 row and its chunk statistics; the normed projections (QKV, gate/up) scale their
  // accumulator rows by rsqrt(mean(x^2) + eps) — no separate norm kernels inside the stack.
  NormEpi produce, consume;
  produce.xb = xb_;
  produce.ld_xb = d;
  produce.ss = ss_;
  produce.ld_ss = cap_rows_;
  consume.ss_in = ss_;
  consume.ld_ss = cap_rows_;
  consume.eps = s_.eps;
  embed_rows(embed_, I(o_tok), n, d, x_, xb_, ss_, cap_rows_, st);
  prof_.mark(KernelProfiler::kEmbed, st);
  for (int l = 0; l < s_.layers; ++l) {
    __nv_bfloat16* kp = static_cast<__nv_bfloat16*>(k_pool_) + l * layer_stride;
    __nv_bfloat16* vp = static_cast<__nv_bfloat16*>(v_pool_) + l * layer_stride;
    // QKV projection (attention norm fused) with RoPE + KV append fused into the epilogue
    GemmArgs qa{xb_, wqkv_[l], nullptr, n, s_.qkv_dim(), d, d, d, s_.qkv_dim(), kEpiQKVRope, 0};
    qa.rope = RopeEpi{I(o_pos), I(o_slot), rope_cs_, q_, kp, vp, s_.n_q, s_.n_kv, s_.hd};
    qa.norm = consume;
    gemm_tn(with_ws(qa), st);
    prof_.mark(KernelProfiler::kQKV, st);
    attention(q_, kp, vp, reinterpret_cast<const AttnGroup*>(d_meta_ + o_grp), static_cast<int>(grp_sorted_.size()),
              I(o_ext), reinterpret_cast<const unsigned long long*>(d_meta_ + o_msk), ash, attn_, st);
    prof_.mark(KernelProfiler::kAttn, st);
    GemmArgs oa{attn_, wo_[l], x_, n, d, qd, qd, qd, d, kEpiAddF32, 0};
    oa.norm = produce;
    gemm_tn(with_ws(oa), st);
    prof_.mark(KernelProfiler::kO, st);
    GemmArgs ga{xb_, wgu_[l], h_, n, 2 * s_.ffn, d, d, d, s_.ffn, kEpiSwiGLU, 0};
    ga.norm = consume;
    gemm_tn(with_ws(ga), st);
    prof_.mark(KernelProfiler::kGateUp, st);
    GemmArgs da{h_, wdown_[l], x_, n, d, s_.ffn, s_.ffn, s_.ffn, d, kEpiAddF32, 0};
    if (l + 1 < s_.layers) da.norm = produce;
    gemm_tn(with_ws(da), st);
    prof_.mark(KernelProfiler::kDown, st);
  }
  if (n_out == 0) return;
  rmsnorm_rows(x_, d, I(o_out), final_norm_, s_.eps, n_out, d, xo_, d, st);
  prof_.mark(KernelProfiler::kNorm, st);
  gemm_tn(with_ws(GemmArgs{xo_, lm_head_, logits_, n_out, s_.vocab, d, d, d, s_.vocab, kEpiBF16, 0}), st);
  prof_.mark(KernelProfiler::kLMHead, st);
  if (plant > 0.f && !b.plant.empty()) plant_bias(logits_, s_.vocab, I(o_pl), plant, n_out, st);
  prof_.mark(KernelProfiler::kPlant, st);
}

// ---- KernelProfiler ----
void KernelProfiler::enable(bool on) {
  on_ = on;
}
void KernelProfiler::begin(cudaStream_t st) {
  if (!on_) return;
  collect();
  if (!start_) WS_CUDA(cudaEventCreate(&start_));
  WS_CUDA(cudaEventRecord(start_, st));
  used_ = 0;
  marks_.clear();
}
void KernelProfiler::mark(int cls, cudaStream_t st) {
  if (!on_) return;
  if (used_ == pool_.size()) {
    cudaEvent_t e;
    WS_CUDA(cudaEventCreate(&e));
    pool_.push_back(e);
  }
  WS_CUDA(cudaEventRecord(pool_[used_], st));
  marks_.emplace_back(cls, pool_[used_]);
  ++used_;
}
void KernelProfiler::collect() {
  if (!on_ || marks_.empty()) return;
  WS_CUDA(cudaEventSynchronize(marks_.back().second));
  cudaEvent_t prev = start_;
  for (const auto& [cls, e] : marks_) {
    float t = 0.f;
    WS_CUDA(cudaEventElapsedTime(&t, prev, e));
    ms[cls] += t;
    count[cls] += 1;
    prev = e;
  }
  marks_.clear();
}
const char* KernelProfiler::name(int cls) {
  static const char* n[] = {"embed", "rmsnorm", "gemm_qkv", "rope_kv_append", "attention", "gemm_o_add",
                            "gemm_gate_up_swiglu", "gemm_down_add", "gemm_lm_head", "plant_bias", "tp_allreduce"};
  return cls >= 0 && cls < kClasses ? n[cls] : "?";
}

}  // namespace wsb
