// Tensor-parallel Llama target (BASELINE config 5: the Llama-3.1-70B shape over the GPUs of one
// box). One host thread per rank submits that rank's stream; rank 0 is the caller's GPU and
// stream, ranks 1.. the next GPUs. Per layer and rank:
//   QKV GEMM (local heads; fused norm, RoPE, KV append into the rank's KV pool)
//   -> attention over the local heads (K2)
//   -> O GEMM: fp32 partial of the row-parallel projection
//   -> tp_allreduce_residual (kernels/tp.cu): partials summed over NVLink in rank order, fused
//      with the residual add and the fused-RMSNorm producer outputs, broadcast to every replica
//   -> gate/up GEMM (local ffn slice, fused norm + SwiGLU) -> down GEMM partial -> all-reduce.
// The LM head is vocabulary-parallel: rank g writes its column slice straight into rank 0's
// logits through a peer pointer, then K3/K4 run once on rank 0. Shard g's weights are the exact
// slices of the single-GPU model's weights (same Philox streams, fill_normal_bf16_2d), so a TP
// run and a one-GPU run of the same seed evaluate the same model.
#include "llama_tp.hpp"

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>

#include "../kernels/cuda_check.hpp"
#include "../kernels/gemm_tc.cuh"
#include "../kernels/tp.cuh"

namespace wsb {

namespace {
std::size_t al256(std::size_t x) { return (x + 255) & ~static_cast<std::size_t>(255); }

void enable_peers(int dev0, int tp) {
  for (int i = 0; i < tp; ++i)
    for (int j = 0; j < tp; ++j) {
      if (i == j) continue;
      int can = 0;
      WS_CUDA(cudaDeviceCanAccessPeer(&can, dev0 + i, dev0 + j));
      if (!can) throw ConfigError("tensor parallel: GPUs " + std::to_string(dev0 + i) + " and " +
                                  std::to_string(dev0 + j) + " have no peer access");
      WS_CUDA(cudaSetDevice(dev0 + i));
      const cudaError_t e = cudaDeviceEnablePeerAccess(dev0 + j, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else
        WS_CUDA(e);
    }
}
}  // namespace

LlamaModel::TPShard::~TPShard() {
  cudaSetDevice(device);
  for (void* p : {block, static_cast<void*>(rope_cs), k_pool, v_pool})
    if (p) cudaFree(p);
}

TPActs::~TPActs() {
  for (Rank& q : r) {
    cudaSetDevice(q.device);
    for (void* p : {static_cast<void*>(q.x), q.xb, static_cast<void*>(q.ss), static_cast<void*>(q.part), q.q, q.attn,
                    q.h, q.xo, static_cast<void*>(q.d_meta), static_cast<void*>(q.flags),
                    static_cast<void*>(q.counter), q.gemm_ws})
      if (p) cudaFree(p);
    if (q.ev) cudaEventDestroy(q.ev);
    if (&q != &r[0] && q.st) cudaStreamDestroy(q.st);
  }
  if (ev_in && !r.empty()) {
    cudaSetDevice(r[0].device);
    cudaEventDestroy(ev_in);
  }
}

void LlamaModel::init_tp(std::uint64_t seed, int max_rows) {
  const LlamaShape& s = s_;
  const int P = tp_;
  if (P > kMaxTP) throw ConfigError("tensor parallel: at most 8 ranks");
  int n_dev = 0;
  WS_CUDA(cudaGetDeviceCount(&n_dev));
  if (device_ + P > n_dev) throw ConfigError("tensor parallel: needs " + std::to_string(P) + " GPUs from device " +
                                             std::to_string(device_));
  if (s.n_q % P || s.n_kv % P || s.ffn % (16 * P) || s.vocab % P || (s.vocab / P) % 8)
    throw ConfigError("tensor parallel: heads / ffn / vocabulary not divisible by the rank count");
  enable_peers(device_, P);
  const std::int64_t d = s.d, hd = s.hd, L = s.layers;
  const int nq_l = s.n_q / P, nkv_l = s.n_kv / P, ffn_l = s.ffn / P, vs = s.vocab / P;
  // the single-GPU model's Philox stream ids (LlamaModel ctor: embed, 6 per layer, final norm, head)
  auto sid_layer = [](int l, int k) { return static_cast<std::uint32_t>(2 + 6 * l + k); };
  const std::uint32_t sid_final = static_cast<std::uint32_t>(2 + 6 * L), sid_head = sid_final + 1;
  // RoPE table (as the single-GPU model)
  std::vector<float> inv(s.hd / 2);
  {
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < s.hd / 2; ++i) {
      double f = 1.0 / std::pow(static_cast<double>(s.rope_theta), (2.0 * i) / s.hd);
      if (s.rope_factor > 0.f) {
        const double factor = s.rope_factor, lo = 1.0, hi = 4.0, old_ctx = 8192.0;
        const double wl = 2 * pi / f;
        if (wl > old_ctx / lo)
          f = f / factor;
        else if (wl >= old_ctx / hi) {
          const double sm = (old_ctx / wl - lo) / (hi - lo);
          f = (1 - sm) * f / factor + sm * f;
        }
      }
      inv[i] = static_cast<float>(f);
    }
  }
  std::vector<float2> cs(static_cast<std::size_t>(kMaxPos) * (s.hd / 2));
  for (int p = 0; p < kMaxPos; ++p)
    for (int i = 0; i < s.hd / 2; ++i) {
      const double a = static_cast<double>(p) * static_cast<double>(inv[i]);
      cs[static_cast<std::size_t>(p) * (s.hd / 2) + i] =
          make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
    }
  for (int g = 0; g < P; ++g) {
    std::unique_ptr<TPShard> sh(new TPShard);
    sh->rank = g;
    sh->device = device_ + g;
    sh->nq = nq_l;
    sh->nkv = nkv_l;
    sh->ffn = ffn_l;
    sh->v0 = g * vs;
    sh->vs = vs;
    WS_CUDA(cudaSetDevice(sh->device));
    const std::int64_t qkv_l = static_cast<std::int64_t>(nq_l + 2 * nkv_l) * hd;
    std::size_t total = 0;
    auto take = [&](std::int64_t elems) {
      const std::size_t o = total;
      total += al256(static_cast<std::size_t>(elems) * 2);
      return o;
    };
    const std::size_t o_emb = take(static_cast<std::int64_t>(s.vocab) * d);
    const std::size_t o_head = s.tied ? 0 : take(static_cast<std::int64_t>(vs) * d);
    const std::size_t o_fn = take(d);
    std::vector<std::size_t> o_an(L), o_qkv(L), o_wo(L), o_mn(L), o_gu(L), o_dn(L);
    for (int l = 0; l < L; ++l) {
      o_an[l] = take(d);
      o_qkv[l] = take(qkv_l * d);
      o_wo[l] = take(d * nq_l * hd);
      o_mn[l] = take(d);
      o_gu[l] = take(2ll * ffn_l * d);
      o_dn[l] = take(d * ffn_l);
    }
    WS_CUDA(cudaMalloc(&sh->block, total));
    auto at = [&](std::size_t o) { return static_cast<void*>(static_cast<unsigned char*>(sh->block) + o); };
    sh->embed = at(o_emb);
    fill_normal_bf16(sh->embed, static_cast<std::int64_t>(s.vocab) * d, seed, 1, 0.02f, 0.f, nullptr);
    if (s.tied) {
      sh->lm_head = static_cast<__nv_bfloat16*>(sh->embed) + static_cast<std::size_t>(sh->v0) * d;
    } else {
      sh->lm_head = at(o_head);
      fill_normal_bf16_2d(sh->lm_head, vs, d, d, sh->v0, 0, seed, sid_head, 0.02f, 0.f, nullptr);
    }
    sh->final_norm = at(o_fn);
    fill_normal_bf16(sh->final_norm, d, seed, sid_final, 0.f, 1.f, nullptr);
    for (int l = 0; l < L; ++l) {
      sh->attn_norm.push_back(at(o_an[l]));
      fill_normal_bf16(sh->attn_norm[l], d, seed, sid_layer(l, 0), 0.f, 1.f, nullptr);
      // [q heads | k heads | v heads] of the rank: three row ranges of the full projection
      void* w = at(o_qkv[l]);
      sh->wqkv.push_back(w);
      const std::int64_t rows_q = nq_l * hd, rows_kv = nkv_l * hd;
      __nv_bfloat16* wb = static_cast<__nv_bfloat16*>(w);
      fill_normal_bf16_2d(wb, rows_q, d, d, g * rows_q, 0, seed, sid_layer(l, 1), 0.02f, 0.f, nullptr);
      fill_normal_bf16_2d(wb + rows_q * d, rows_kv, d, d, s.n_q * hd + g * rows_kv, 0, seed, sid_layer(l, 1), 0.02f,
                          0.f, nullptr);
      fill_normal_bf16_2d(wb + (rows_q + rows_kv) * d, rows_kv, d, d, (s.n_q + s.n_kv) * hd + g * rows_kv, 0, seed,
                          sid_layer(l, 1), 0.02f, 0.f, nullptr);
      // O: the rank's input columns of every output row
      sh->wo.push_back(at(o_wo[l]));
      fill_normal_bf16_2d(sh->wo[l], d, nq_l * hd, static_cast<std::int64_t>(s.n_q) * hd, 0, g * nq_l * hd, seed,
                          sid_layer(l, 2), 0.02f, 0.f, nullptr);
      sh->mlp_norm.push_back(at(o_mn[l]));
      fill_normal_bf16(sh->mlp_norm[l], d, seed, sid_layer(l, 3), 0.f, 1.f, nullptr);
      // gate/up interleaved in 16-row blocks: the rank's features are a contiguous row range
      sh->wgu.push_back(at(o_gu[l]));
      fill_normal_bf16_2d(sh->wgu[l], 2ll * ffn_l, d, d, 2ll * g * ffn_l, 0, seed, sid_layer(l, 4), 0.02f, 0.f,
                          nullptr);
      sh->wdown.push_back(at(o_dn[l]));
      fill_normal_bf16_2d(sh->wdown[l], d, ffn_l, s.ffn, 0, static_cast<std::int64_t>(g) * ffn_l, seed,
                          sid_layer(l, 5), 0.02f, 0.f, nullptr);
      fold_norm_weight(sh->wqkv[l], qkv_l, s.d, sh->attn_norm[l], nullptr);
      fold_norm_weight(sh->wgu[l], 2ll * ffn_l, s.d, sh->mlp_norm[l], nullptr);
    }
    WS_CUDA(cudaMalloc(reinterpret_cast<void**>(&sh->rope_cs), cs.size() * sizeof(float2)));
    WS_CUDA(cudaMemcpy(sh->rope_cs, cs.data(), cs.size() * sizeof(float2), cudaMemcpyHostToDevice));
    const std::size_t pool = static_cast<std::size_t>(L) * n_slots_ * nkv_l * hd * 2;
    WS_CUDA(cudaMalloc(&sh->k_pool, pool));
    WS_CUDA(cudaMalloc(&sh->v_pool, pool));
    WS_CUDA(cudaMemset(sh->k_pool, 0, pool));
    WS_CUDA(cudaMemset(sh->v_pool, 0, pool));
    WS_CUDA(cudaDeviceSynchronize());
    shards_.push_back(std::move(sh));
  }
  WS_CUDA(cudaSetDevice(device_));
  ws0_ = make_workspace(max_rows);
}

void LlamaModel::ensure_tp(ForwardWorkspace& ws, int rows, int out_rows) const {
  const int P = tp_;
  if (!ws.tp) {
    ws.tp.reset(new TPActs);
    ws.tp->r.resize(P);
    for (int g = 0; g < P; ++g) {
      TPActs::Rank& q = ws.tp->r[g];
      q.device = device_ + g;
      WS_CUDA(cudaSetDevice(q.device));
      if (g > 0) WS_CUDA(cudaStreamCreateWithFlags(&q.st, cudaStreamNonBlocking));
      WS_CUDA(cudaEventCreateWithFlags(&q.ev, cudaEventDisableTiming));
      WS_CUDA(cudaMalloc(&q.flags, 2 * kMaxTP * sizeof(unsigned long long)));
      WS_CUDA(cudaMemset(q.flags, 0, 2 * kMaxTP * sizeof(unsigned long long)));
      WS_CUDA(cudaMalloc(&q.counter, sizeof(unsigned int)));
      WS_CUDA(cudaMemset(q.counter, 0, sizeof(unsigned int)));
    }
    WS_CUDA(cudaSetDevice(device_));
    WS_CUDA(cudaEventCreateWithFlags(&ws.tp->ev_in, cudaEventDisableTiming));
  }
  TPActs& A = *ws.tp;
  if (out_rows > ws.cap_out) {  // rank 0's full logits (every rank writes its vocabulary slice)
    WS_CUDA(cudaSetDevice(device_));
    if (ws.logits) cudaFree(ws.logits);
    ws.cap_out = std::max(out_rows, 2 * ws.cap_out);
    WS_CUDA(cudaMalloc(&ws.logits, static_cast<std::size_t>(ws.cap_out) * s_.vocab * 2));
  }
  if (rows <= A.cap && out_rows <= A.cap_out) {
    ws.cap_rows = A.cap;
    return;
  }
  const int cap = std::max(rows, A.cap), cap_out = std::max(out_rows, A.cap_out);
  const std::size_t d = s_.d;
  for (int g = 0; g < P; ++g) {
    TPActs::Rank& q = A.r[g];
    const TPShard& sh = *shards_[g];
    WS_CUDA(cudaSetDevice(q.device));
    if (q.st) WS_CUDA(cudaStreamSynchronize(q.st));
    for (void* p : {static_cast<void*>(q.x), q.xb, static_cast<void*>(q.ss), static_cast<void*>(q.part), q.q, q.attn,
                    q.h, q.xo})
      if (p) cudaFree(p);
    WS_CUDA(cudaMalloc(reinterpret_cast<void**>(&q.x), static_cast<std::size_t>(cap) * d * 4));
    WS_CUDA(cudaMalloc(&q.xb, static_cast<std::size_t>(cap) * d * 2));
    WS_CUDA(cudaMalloc(reinterpret_cast<void**>(&q.ss), static_cast<std::size_t>(cap) * (d / 32) * 4));
    WS_CUDA(cudaMalloc(reinterpret_cast<void**>(&q.part), static_cast<std::size_t>(cap) * d * 4));
    WS_CUDA(cudaMalloc(&q.q, static_cast<std::size_t>(cap) * sh.nq * s_.hd * 2));
    WS_CUDA(cudaMalloc(&q.attn, static_cast<std::size_t>(cap) * sh.nq * s_.hd * 2));
    WS_CUDA(cudaMalloc(&q.h, static_cast<std::size_t>(cap) * sh.ffn * 2));
    WS_CUDA(cudaMalloc(&q.xo, static_cast<std::size_t>(std::max(1, cap_out)) * d * 2));
  }
  WS_CUDA(cudaSetDevice(device_));
  A.cap = cap;
  A.cap_out = cap_out;
  ws.cap_rows = cap;
}

void LlamaModel::forward_tp(const ForwardBatch& b, float plant, cudaStream_t st, ForwardWorkspace& ws) {
  const int n = static_cast<int>(b.tok.size());
  const int n_out = static_cast<int>(b.out_rows.size());
  const int P = tp_;
  ensure_tp(ws, n, n_out);
  TPActs& A = *ws.tp;
  A.r[0].st = st;
  for (int g = 0; g < P; ++g) {  // every rank's previous forward retired (staging and peer buffers)
    DeviceGuard dg(A.r[g].device);
    WS_CUDA(cudaStreamSynchronize(A.r[g].st));
  }
  const MetaLayout ml = pack_meta(b, ws, st);  // rank 0's copy (and the host staging)
  for (int g = 1; g < P; ++g) {
    TPActs::Rank& q = A.r[g];
    DeviceGuard dg(q.device);
    if (ml.bytes > q.cap_meta) {
      if (q.d_meta) cudaFree(q.d_meta);
      q.cap_meta = std::max(ml.bytes, 2 * q.cap_meta);
      WS_CUDA(cudaMalloc(&q.d_meta, q.cap_meta));
    }
    WS_CUDA(cudaMemcpyAsync(q.d_meta, ws.h_meta, ml.bytes, cudaMemcpyHostToDevice, q.st));
    ws.h2d += ml.bytes;
  }
  {
    DeviceGuard dg(device_);
    WS_CUDA(cudaEventRecord(A.ev_in, st));
  }
  for (int g = 1; g < P; ++g) {
    DeviceGuard dg(A.r[g].device);
    WS_CUDA(cudaStreamWaitEvent(A.r[g].st, A.ev_in, 0));
  }
  auto meta = [&](int g) { return g == 0 ? ws.d_meta : A.r[g].d_meta; };
  auto I = [&](int g, std::size_t off) { return reinterpret_cast<const std::int32_t*>(meta(g) + off); };
  const int d = s_.d, hd = s_.hd, cap = A.cap;
  TPPeers peers;
  peers.tp = P;
  for (int g = 0; g < P; ++g) {
    peers.part[g] = A.r[g].part;
    peers.x[g] = A.r[g].x;
    peers.xb[g] = A.r[g].xb;
    peers.ss[g] = A.r[g].ss;
    peers.flag_a[g] = A.r[g].flags;
    peers.flag_b[g] = A.r[g].flags + kMaxTP;
  }
  const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
  const unsigned long long epoch0 = A.epoch;
  A.epoch += 2ull * s_.layers;  // two all-reduces per layer, the same epochs on every rank
  // One host thread per rank submits that rank's whole layer stack (no device switching, a
  // quarter of the launch latency each); the ranks meet only in the device-side all-reduces.
  auto run_rank = [&](int g) {
    const TPShard& sh = *shards_[g];
    TPActs::Rank& q = A.r[g];
    DeviceGuard dg(q.device);
    TPPeers pg = peers;
    pg.counter = q.counter;
    const std::int64_t layer_stride = n_slots_ * sh.nkv * hd;
    const int qkv_n = (sh.nq + 2 * sh.nkv) * hd, qd = sh.nq * hd;
    NormEpi consume;
    consume.ss_in = q.ss;
    consume.ld_ss = cap;
    consume.eps = s_.eps;
    NormEpi store;
    store.store_only = 1;  // the row-parallel partial overwrites its buffer
    KernelProfiler* prof = g == 0 && ws.prof.on() ? &ws.prof : nullptr;  // rank 0's stream only
    if (prof) prof->begin(q.st);
    embed_rows(sh.embed, I(g, ml.tok), n, d, q.x, q.xb, q.ss, cap, q.st);
    if (prof) prof->mark(KernelProfiler::kEmbed, q.st);
    for (int l = 0; l < s_.layers; ++l) {
      __nv_bfloat16* kp = static_cast<__nv_bfloat16*>(sh.k_pool) + l * layer_stride;
      __nv_bfloat16* vp = static_cast<__nv_bfloat16*>(sh.v_pool) + l * layer_stride;
      GemmArgs qa{q.xb, sh.wqkv[l], nullptr, n, qkv_n, d, d, d, qkv_n, kEpiQKVRope, 0};
      qa.rope = RopeEpi{I(g, ml.pos), I(g, ml.slot), sh.rope_cs, q.q, kp, vp, sh.nq, sh.nkv, hd};
      qa.norm = consume;
      qa.max_ctas = max_ctas_;
      gemm_tn(qa, q.st);
      if (prof) prof->mark(KernelProfiler::kQKV, q.st);
      attention(q.q, kp, vp, reinterpret_cast<const AttnGroup*>(meta(g) + ml.grp), ml.n_entries, I(g, ml.ext),
                reinterpret_cast<const unsigned long long*>(meta(g) + ml.msk),
                AttnShape{sh.nq, sh.nkv, hd, sh.nkv * hd, scale}, q.attn, q.st);
      if (prof) prof->mark(KernelProfiler::kAttn, q.st);
      GemmArgs oa{q.attn, sh.wo[l], q.part, n, d, qd, qd, qd, d, kEpiAddF32, 0};
      oa.norm = store;
      oa.max_ctas = max_ctas_;
      gemm_tn(oa, q.st);
      if (prof) prof->mark(KernelProfiler::kO, q.st);
      tp_allreduce_residual(pg, g, n, d, cap, epoch0 + 2ull * l + 1, false, q.st);
      if (prof) prof->mark(KernelProfiler::kAllReduce, q.st);
      GemmArgs ga{q.xb, sh.wgu[l], q.h, n, 2 * sh.ffn, d, d, d, sh.ffn, kEpiSwiGLU, 0};
      ga.norm = consume;
      ga.max_ctas = max_ctas_;
      gemm_tn(ga, q.st);
      if (prof) prof->mark(KernelProfiler::kGateUp, q.st);
      GemmArgs da{q.h, sh.wdown[l], q.part, n, d, sh.ffn, sh.ffn, sh.ffn, d, kEpiAddF32, 0};
      da.norm = store;
      da.max_ctas = max_ctas_;
      gemm_tn(da, q.st);
      if (prof) prof->mark(KernelProfiler::kDown, q.st);
      tp_allreduce_residual(pg, g, n, d, cap, epoch0 + 2ull * l + 2, l + 1 == s_.layers, q.st);
      if (prof) prof->mark(KernelProfiler::kAllReduce, q.st);
    }
    if (n_out > 0) {
      rmsnorm_rows(q.x, d, I(g, ml.out), sh.final_norm, s_.eps, n_out, d, q.xo, d, q.st);
      // the rank's vocabulary slice, written into rank 0's logits (peer stores for g > 0)
      void* out = static_cast<__nv_bfloat16*>(ws.logits) + sh.v0;
      GemmArgs ha{q.xo, sh.lm_head, out, n_out, sh.vs, d, d, d, s_.vocab, kEpiBF16, 0};
      ha.max_ctas = max_ctas_;
      gemm_tn(ha, q.st);
      if (prof) prof->mark(KernelProfiler::kLMHead, q.st);
    }
    if (g > 0) WS_CUDA(cudaEventRecord(q.ev, q.st));
  };
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(P);
  for (int g = 1; g < P; ++g)
    th.emplace_back([&, g] {
      try {
        run_rank(g);
      } catch (...) {
        err[g] = std::current_exception();
      }
    });
  try {
    run_rank(0);
  } catch (...) {
    err[0] = std::current_exception();
  }
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  DeviceGuard dg(device_);  // rank 0's stream (the caller's) covers every rank's work
  for (int g = 1; g < P; ++g) WS_CUDA(cudaStreamWaitEvent(st, A.r[g].ev, 0));
  if (n_out > 0 && plant > 0.f && !b.plant.empty()) plant_bias(ws.logits, s_.vocab, I(0, ml.pl), plant, n_out, st);
}

}  // namespace wsb
