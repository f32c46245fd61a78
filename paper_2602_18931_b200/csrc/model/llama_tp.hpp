// One rank's shard of a tensor-parallel Llama target (see llama_tp.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "llama.hpp"

namespace wsb {

struct LlamaModel::TPShard {
  int rank = 0, device = 0;
  int nq = 0, nkv = 0, ffn = 0;  // local heads / ffn features
  int v0 = 0, vs = 0;            // this rank's vocabulary slice of the LM head
  void* block = nullptr;         // all weights of the shard
  void* embed = nullptr;         // full embedding (every rank gathers its own rows)
  void* lm_head = nullptr;       // rows [v0, v0 + vs) of the LM head
  void* final_norm = nullptr;
  std::vector<void*> attn_norm, wqkv, wo, mlp_norm, wgu, wdown;
  float2* rope_cs = nullptr;
  void* k_pool = nullptr;        // [layer][slot][nkv local][hd]
  void* v_pool = nullptr;
  ~TPShard();
};

}  // namespace wsb
