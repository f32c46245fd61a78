// Model-plumbing kernels of the verify / draft forward.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace wsb {

// A run of consecutive query rows that share one attention context: the first `prefix_len`
// positions live at consecutive pool slots starting at `prefix_slot`; then `extra_len` explicit
// slots (tree ancestors + the rows' own new slots). Row j (0-based in the group) attends to
// the prefix and extra[0 .. extra_len - n_rows + j] (causal within the group).
// masked != 0: row j instead sees the extras whose bits are set in row_mask[row0 + j]
// (extra_len <= 64) — the shared-prefix tree group of one request's draft leaves.
struct AttnGroup {
  std::int32_t row0;
  std::int32_t n_rows;
  std::int32_t prefix_slot;
  std::int32_t prefix_len;
  std::int32_t extra_off;
  std::int32_t extra_len;
  std::int32_t masked = 0;
  std::int32_t pad = 0;
};

struct AttnShape {
  int n_q, n_kv, hd;
  int slot_stride;  // elements between consecutive slots of one layer's pool = n_kv * hd
  float scale;      // 1/sqrt(hd)
};

// x[row, :] = float(emb[tok[row], :]); optionally xb = the bf16 row and ss[c][row] = sum of
// squares of 32-column chunk c (chunk-major; the fused-RMSNorm statistics, gemm_tc.cuh NormEpi).
void embed_rows(const void* emb_bf16, const std::int32_t* tok, int rows, int d, float* x, void* xb_bf16, float* ss,
                int ld_ss, cudaStream_t st);

// W[:, k] *= w[k] (bf16 [rows, cols]): folds an RMSNorm weight into the projection it feeds.
void fold_norm_weight(void* W_bf16, std::int64_t rows, int cols, const void* w_bf16, cudaStream_t st);

// y[r] = bf16(x[idx ? idx[r] : r] * rsqrt(mean(x^2) + eps) * w)   (x fp32, w bf16 [d])
void rmsnorm_rows(const float* x, int ld_x, const std::int32_t* idx, const void* w, float eps, int rows, int d,
                  void* y_bf16, int ld_y, cudaStream_t st);

// qkv bf16 [rows, (nq + 2 nkv) * hd] → q bf16 [rows, nq * hd] rotated; K/V rotated/copied into
// the pools at slot[row] (pool layout [slot][n_kv][hd]). RoPE in the rotate-half convention with
// per-dimension inverse frequencies inv_freq[hd/2] (llama3 scaling precomputed on the host).
void rope_kv_append(const void* qkv, int rows, int nq, int nkv, int hd, const std::int32_t* pos,
                    const std::int32_t* slot, const float* inv_freq, void* q_out, void* k_pool, void* v_pool,
                    cudaStream_t st);

// Grouped attention (causal or masked groups) over the slot pools → out bf16 [rows, nq * hd].
// Each entry is one CTA pass over up to attention_vectors_per_cta(hd) of its group's query
// vectors (n_rows * n_q / n_kv), starting at vector `pad`: a group with more vectors is passed
// as several entries.
int attention_vectors_per_cta(int hd);
void attention(const void* q, const void* k_pool, const void* v_pool, const AttnGroup* entries, int n_entries,
               const std::int32_t* extra_slots, const unsigned long long* row_mask, const AttnShape& shape,
               void* out, cudaStream_t st);

// logits[row, plant[row]] += bias (plant < 0: none) — the planted shared bigram bias.
void plant_bias(void* logits_bf16, int ld, const std::int32_t* plant, float bias, int rows, cudaStream_t st);

// Copies whole-slot K/V (all layers) src→dst: layer stride = n_slots*slot_stride elements.
void copy_slots(void* k_pool, void* v_pool, const std::int32_t* src, const std::int32_t* dst, int n, int layers,
                std::int64_t layer_stride, int slot_stride, cudaStream_t st);

// Deterministic N(0, std) bf16 fill from Philox (seed, stream id); value `one` if std == 0.
void fill_normal_bf16(void* out, std::int64_t n, std::uint64_t seed, std::uint32_t stream_id, float std_, float mean,
                      cudaStream_t st);

}  // namespace wsb
