#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace wsb {

enum GemmEpi : int {
  kEpiBF16 = 0,     // out bf16 [M, ldo] = acc
  kEpiAddF32 = 1,   // out fp32 [M, ldo] += acc   (residual stream)
  kEpiSwiGLU = 2,   // out bf16 [M, ldo] = silu(gate) * up; W rows interleaved in 16-row blocks
  kEpiQKVRope = 3,  // fused QKV epilogue: rotate-half RoPE on q/k, q → q_out, k/v → KV pool slots
};

// Operands of the fused QKV epilogue (row r: position pos[r], KV slot slot[r]; cs = cos/sin
// table [max_pos][hd/2] precomputed on the host in fp64 from the llama3-scaled frequencies).
struct RopeEpi {
  const int* pos = nullptr;
  const int* slot = nullptr;
  const float2* cs = nullptr;
  void* q = nullptr;       // bf16 [M, nq*hd]
  void* k_pool = nullptr;  // bf16 [slot][nkv][hd] (this layer)
  void* v_pool = nullptr;
  int nq = 0, nkv = 0, hd = 0;
};

// Fused RMSNorm plumbing (the norm weight itself is folded into the consuming projection):
//   producer (kEpiAddF32): after out += acc, also xb = bf16(out) and ss[col / 32][row] = the sum
//     of squares of each 32-column chunk of the updated residual row (chunked, so the statistic
//     never depends on the tile width: batch- and tile-invariant);
//   consumer (any epilogue): accumulator row r is scaled by rsqrt(sum_c ss_in[c][r] / K + eps)
//     (fixed summation order) before the epilogue's own op — A is then bf16(x), unnormalised.
struct NormEpi {
  void* xb = nullptr;            // producer: bf16 [M, ld_xb]
  int ld_xb = 0;
  float* ss = nullptr;           // producer: fp32 chunk-major [N / 32][ld_ss] (ld_ss >= M)
  const float* ss_in = nullptr;  // consumer: fp32 chunk-major [K / 32][ld_ss]
  int ld_ss = 0;
  float eps = 0.f;
  int store_only = 0;            // kEpiAddF32: out = acc (no residual read) — TP partials
};

struct GemmArgs {
  const void* A;  // bf16 [M, K], row stride lda
  const void* W;  // bf16 [N, K], row stride ldw
  void* out;
  int M, N, K;
  int lda, ldw, ldo;
  int epi = kEpiBF16;
  int bn = 0;        // 0 = auto (multiple of 32 in [64, 256]; see pick_bn)
  int max_ctas = 0;  // persistent grid cap (0 = one CTA per SM; < 0 = one CTA per tile, not persistent)
  int cta_group = 0; // 0 = auto, 1 = single CTAs, 2 = CTA pairs (256-row tiles, cta_group::2)
  RopeEpi rope{};    // kEpiQKVRope only
  NormEpi norm{};    // fused RMSNorm producer / consumer (optional)
  // Split-K workspace (zero-initialised once; see gemm_workspace_bytes). With ws == nullptr the
  // GEMM never splits; splits = 0 picks the (N, K)-determined count.
  void* ws = nullptr;
  std::size_t ws_bytes = 0;
  int splits = 0;
  int chunks_ = 0;  // canonical K chunks (0 = from (N, K); internal: row slices inherit the parent's)
  int pdl_late = 0;  // 1: dependents may launch once each CTA's last accumulator is ready
};

// C = A · W^T on tcgen05 (sm_100a). Throws on bad shapes / CUDA errors.
void gemm_tn(const GemmArgs& g, cudaStream_t stream);
int pick_bn(int M, int N);
void gemm_debug_trace(unsigned long long* out8);  // WS_GEMM_ABLATE & 8 timeline (diagnostics)
int pick_splits(int N, int K);
// Bytes of a split-K workspace serving GEMMs of up to max_rows rows per launch slice.
std::size_t gemm_workspace_bytes(int max_rows);

}  // namespace wsb
