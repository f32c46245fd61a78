#pragma once

#include <cuda_runtime.h>

namespace wsb {

enum GemmEpi : int {
  kEpiBF16 = 0,    // out bf16 [M, ldo] = acc
  kEpiAddF32 = 1,  // out fp32 [M, ldo] += acc   (residual stream)
  kEpiSwiGLU = 2,  // out bf16 [M, ldo] = silu(gate) * up; W rows interleaved in 32-row blocks
};

struct GemmArgs {
  const void* A;  // bf16 [M, K], row stride lda
  const void* W;  // bf16 [N, K], row stride ldw
  void* out;
  int M, N, K;
  int lda, ldw, ldo;
  int epi = kEpiBF16;
  int bn = 0;        // 0 = auto (64/128/256)
  int max_ctas = 0;  // persistent grid cap (0 = one CTA per SM)
};

// C = A · W^T on tcgen05 (sm_100a). Throws on bad shapes / CUDA errors.
void gemm_tn(const GemmArgs& g, cudaStream_t stream);
int pick_bn(int M, int N);

}  // namespace wsb
