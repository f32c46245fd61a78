// Llama-architecture forward for the verify (target) and draft models, batched over rows from
// many requests, on the sm_100a kernels (K1 GEMM, K2 attention, K6 plumbing, K3/K4 epilogues).
// Random-init bf16 weights of the named shapes (BASELINE config 3): weights are seeded
// N(0, 0.02) from Philox, norm weights 1. The residual stream is fp32.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../kernels/llama_ops.cuh"

namespace wsb {

struct LlamaShape {
  std::string name;
  int layers, d, n_q, n_kv, hd, ffn, vocab;
  float eps = 1e-5f;
  float rope_theta = 500000.f;
  float rope_factor = 8.f;  // llama3 scaling (0 = none)
  bool tied = false;
  std::int64_t params_mm() const;  // matmul parameters (incl. LM head)
  int qkv_dim() const { return (n_q + 2 * n_kv) * hd; }
};

LlamaShape shape_by_name(const std::string& name);  // "llama3-8b", "llama3.2-1b", "tiny"

// One batched forward: rows with (token, position, own KV slot), attention groups over the
// slot pool, and the list of rows whose logits are wanted.
struct ForwardBatch {
  std::vector<std::int32_t> tok, pos, slot;
  std::vector<AttnGroup> groups;
  std::vector<std::int32_t> extra;
  std::vector<std::int32_t> out_rows;
  std::vector<std::int32_t> plant;  // per output row: planted token (or -1)
  std::vector<unsigned long long> row_mask;  // per row (only read for masked groups)
  // A prompt-prefill forward (ModelPair::prefill_prompts, and the prompt step of export_trace):
  // its GEMMs keep one canonical K chunk. Every position's KV is computed by the same kind of
  // forward in every run (the prompt [0, P-1) by prefill forwards, later positions by verify /
  // draft forwards), so each kind only has to be batch-invariant on its own — and the 8 128-row
  // prefill batches keep their widest tiles (profiles/r02_gemm_chunks.md).
  bool prefill = false;
  void clear() {
    prefill = false;
    row_mask.clear();
    tok.clear();
    pos.clear();
    slot.clear();
    groups.clear();
    extra.clear();
    out_rows.clear();
    plant.clear();
  }
};

// Per-kernel-class device time of the forward, from CUDA events recorded between launches on
// the model's stream (enabled by WS_PROFILE=1; used for the time-share tables in profiles/).
class KernelProfiler {
 public:
  enum Cls { kEmbed, kNorm, kQKV, kRope, kAttn, kO, kGateUp, kDown, kLMHead, kPlant, kAllReduce, kClasses };
  void enable(bool on);
  bool on() const { return on_; }
  void begin(cudaStream_t st);
  void mark(int cls, cudaStream_t st);
  void collect();  // folds completed marks into ms/count (blocks on the last mark)
  static const char* name(int cls);
  double ms[kClasses] = {};
  std::uint64_t count[kClasses] = {};

 private:
  bool on_ = false;
  cudaEvent_t start_ = nullptr;
  std::vector<cudaEvent_t> pool_;
  std::size_t used_ = 0;
  std::vector<std::pair<int, cudaEvent_t>> marks_;
};

// Activation state of one caller's forwards: several callers (protocol threads, each with its
// own streams) run forwards of the same model concurrently — weights and KV pools are shared,
// these buffers are not.
// Per-rank activation buffers of a tensor-parallel forward (llama_tp.cu): rank 0's live on the
// workspace's device, the others on theirs; all are peer-accessible.
struct TPActs {
  struct Rank {
    int device = 0;
    cudaStream_t st = nullptr;  // rank 0: the caller's stream (not owned)
    cudaEvent_t ev = nullptr;
    float* x = nullptr;         // fp32 residual replica [cap][d]
    void* xb = nullptr;         // bf16 replica [cap][d]
    float* ss = nullptr;        // chunk statistics replica [d/32][cap]
    float* part = nullptr;      // fp32 partial of the row-parallel projections [cap][d]
    void* q = nullptr;          // local heads
    void* attn = nullptr;
    void* h = nullptr;          // local ffn slice
    void* xo = nullptr;         // final-norm rows [cap_out][d]
    unsigned char* d_meta = nullptr;
    std::size_t cap_meta = 0;
    unsigned long long* flags = nullptr;  // [2][kMaxTP] epochs (a: partial ready, b: broadcast done)
    unsigned int* counter = nullptr;
    void* gemm_ws = nullptr;
    std::size_t gemm_ws_bytes = 0;
  };
  std::vector<Rank> r;
  int cap = 0, cap_out = 0;
  unsigned long long epoch = 0;
  cudaEvent_t ev_in = nullptr;  // on the caller's stream: the ranks start after it
  ~TPActs();
};

struct ForwardWorkspace {
  explicit ForwardWorkspace(int dev) : device(dev) {}
  ~ForwardWorkspace();
  ForwardWorkspace(const ForwardWorkspace&) = delete;
  ForwardWorkspace& operator=(const ForwardWorkspace&) = delete;
  int device;
  int cap_rows = 0, cap_out = 0;
  float* x = nullptr;   // fp32 residual stream [rows][d]
  void* xb = nullptr;   // its bf16 copy (A of the normed projections) [rows][d]
  float* ss = nullptr;  // per-32-column-chunk sums of squares (fused RMSNorm), chunk-major
  void* qkv = nullptr;
  void* q = nullptr;
  void* attn = nullptr;
  void* h = nullptr;
  void* logits = nullptr;
  void* xo = nullptr;
  unsigned char* d_meta = nullptr;  // batch metadata (device) + pinned staging
  unsigned char* h_meta = nullptr;
  std::size_t cap_meta = 0;
  cudaEvent_t meta_ev = nullptr;  // recorded after a forward's metadata H2D (staging reuse)
  bool meta_pending = false;
  void* gemm_ws = nullptr;  // split-K workspace (K1)
  std::size_t gemm_ws_bytes = 0;
  std::vector<AttnGroup> grp_sorted;
  std::size_t h2d = 0;
  // algorithmic attention work of the forwards run on this workspace (roofline units):
  // kv_pos = sum over groups of the keys read (prefix + extras), attn_pairs = sum over groups of
  // rows x keys (an upper bound of the visible pairs; causal groups see about half their extras)
  std::uint64_t kv_pos = 0, attn_pairs = 0;
  // host time spent enqueueing forwards (metadata staging + kernel launches; WS_PROFILE_HOST)
  double host_ms = 0.0;
  std::uint64_t host_fwd = 0;
  KernelProfiler prof;
  std::unique_ptr<TPActs> tp;  // tensor-parallel models only
};

// Offsets of one forward's packed metadata block (one H2D per forward and device).
struct MetaLayout {
  std::size_t tok = 0, pos = 0, slot = 0, grp = 0, ext = 0, out = 0, pl = 0, msk = 0, bytes = 0;
  int n_entries = 0;
};

class LlamaModel {
 public:
  KernelProfiler& profiler() { return ws0_->prof; }
  // Cap on the persistent GEMM grids (0 = every SM): leaves SMs to a concurrent forward.
  void set_max_ctas(int n) { max_ctas_ = n; }
  // the GEMMs let the next kernel launch once their last accumulator is ready (see ModelPair)
  void set_pdl_late(bool on) { pdl_late_ = on; }
  // tp > 1: the target split over GPUs device .. device + tp - 1 (tensor parallel, llama_tp.cu)
  LlamaModel(const LlamaShape& shape, std::uint64_t seed, std::int64_t n_slots, int max_rows, int device, int tp = 1);
  int tp() const { return tp_; }
  ~LlamaModel();
  LlamaModel(const LlamaModel&) = delete;
  LlamaModel& operator=(const LlamaModel&) = delete;

  const LlamaShape& shape() const { return s_; }
  std::int64_t n_slots() const { return n_slots_; }

  // Uploads the batch (one H2D of a packed block) and runs the forward; logits of the
  // out_rows (bf16 [n_out, vocab]) land in ws.logits. plant_bias > 0 adds the planted bias.
  void forward(const ForwardBatch& b, float plant_bias, cudaStream_t st, ForwardWorkspace& ws);
  void forward(const ForwardBatch& b, float plant_bias, cudaStream_t st) { forward(b, plant_bias, st, *ws0_); }
  const void* logits() const { return ws0_->logits; }
  std::size_t h2d_bytes() const { return ws0_->h2d; }
  void copy_slots(const std::vector<std::int32_t>& src, const std::vector<std::int32_t>& dst, cudaStream_t st,
                  ForwardWorkspace& ws);
  void copy_slots(const std::vector<std::int32_t>& src, const std::vector<std::int32_t>& dst, cudaStream_t st) {
    copy_slots(src, dst, st, *ws0_);
  }
  std::unique_ptr<ForwardWorkspace> make_workspace(int max_rows) const;

  // weight access for tests: which = "embed","attn_norm","wqkv","wo","mlp_norm","wgu","wdown","final_norm","lm_head"
  void* weight(const std::string& which, int layer, std::int64_t* numel);
  void* k_pool() const { return k_pool_; }
  void* v_pool() const { return v_pool_; }

 private:
  void ensure_rows(ForwardWorkspace& ws, int rows, int out_rows) const;
  MetaLayout pack_meta(const ForwardBatch& b, ForwardWorkspace& ws, cudaStream_t st) const;
  // tensor parallelism (llama_tp.cu)
  struct TPShard;
  void init_tp(std::uint64_t seed, int max_rows);
  void ensure_tp(ForwardWorkspace& ws, int rows, int out_rows) const;
  void forward_tp(const ForwardBatch& b, float plant, cudaStream_t st, ForwardWorkspace& ws);
  int tp_ = 1;
  std::vector<std::unique_ptr<TPShard>> shards_;
  std::unique_ptr<ForwardWorkspace> ws0_;  // the model's own workspace (test / single-caller API)
  int max_ctas_ = 0;
  bool pdl_late_ = false;
  LlamaShape s_;
  int device_;
  std::int64_t n_slots_;
  // weights
  void* embed_ = nullptr;
  void* lm_head_ = nullptr;
  void* final_norm_ = nullptr;
  std::vector<void*> attn_norm_, wqkv_, wo_, mlp_norm_, wgu_, wdown_;
  void* weight_block_ = nullptr;
  float* inv_freq_ = nullptr;
  float2* rope_cs_ = nullptr;  // [kMaxPos][hd/2] cos/sin
  static constexpr int kMaxPos = 4096;
  // KV pools [layer][slot][n_kv][hd]
  void* k_pool_ = nullptr;
  void* v_pool_ = nullptr;
};

}  // namespace wsb
