// Device-pointer entry points of the model-path kernels (include/wanspec_b200.h "ops").
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kernels/cuda_check.hpp"
#include "kernels/gemm_tc.cuh"
#include "kernels/rowstats.cuh"
#include "kernels/sample.cuh"
#include "wanspec_b200.h"

namespace wsb {
int ops_guarded_rc(const char* what, const std::exception& e);
}

namespace {
template <class F>
int op_guarded(const char* what, F&& f) {
  try {
    f();
    return WS_OK;
  } catch (const std::exception& e) {
    return wsb::ops_guarded_rc(what, e);
  }
}
}  // namespace

extern "C" {

int ws_op_gemm_bf16(const void* A, const void* W, void* out, int M, int N, int K, int lda, int ldw, int ldo,
                    int epi, int bn, int splits, void* stream) {
  return op_guarded("ws_op_gemm_bf16", [&] {
    if (!A || !W || !out || M <= 0 || N <= 0 || K <= 0) throw std::invalid_argument("gemm: bad argument");
    if (epi == WS_EPI_BF16 + 3) throw std::invalid_argument("gemm: the QKV epilogue needs the model");
    wsb::GemmArgs g{A, W, out, M, N, K, lda, ldw, ldo, epi, bn};
    if (splits != 1) {  // split-K (0 = the (N, K)-determined count) with a process-wide workspace
      static void* ws = nullptr;
      static std::size_t ws_bytes = 0;
      static std::mutex mu;
      std::lock_guard<std::mutex> lk(mu);
      const std::size_t need = wsb::gemm_workspace_bytes(std::max(M, 512));
      if (need > ws_bytes) {
        if (ws) cudaFree(ws);
        WS_CUDA(cudaMalloc(&ws, need));
        WS_CUDA(cudaMemset(ws, 0, need));
        ws_bytes = need;
      }
      g.ws = ws;
      g.ws_bytes = ws_bytes;
      g.splits = splits;
      wsb::gemm_tn(g, static_cast<cudaStream_t>(stream));
      WS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
      return;
    }
    wsb::gemm_tn(g, static_cast<cudaStream_t>(stream));
  });
}

size_t ws_op_row_stats_workspace_bytes(uint32_t rows, uint32_t vocab, uint32_t n_req) {
  return wsb::rowstats_workspace_bytes(rows, vocab, n_req);
}

int ws_op_row_stats_bf16(const void* logits, uint32_t rows, uint32_t vocab, uint32_t ld, float inv_temp,
                         ws_pred* out, void* stats, void* workspace, void* stream) {
  return op_guarded("ws_op_row_stats_bf16", [&] {
    wsb::row_stats_bf16(logits, rows, vocab, ld, inv_temp, out, static_cast<wsb::RowStats*>(stats), workspace, 0, 0,
                        nullptr, nullptr, static_cast<cudaStream_t>(stream));
  });
}

int ws_op_verify_greedy_bf16(const void* logits, uint32_t n_req, uint32_t k, uint32_t vocab, uint32_t ld,
                             const uint32_t* cand, ws_verify_out* out, ws_pred* rows_out, void* workspace,
                             void* stream) {
  return op_guarded("ws_op_verify_greedy_bf16", [&] {
    if (!rows_out || !cand || !out) throw std::invalid_argument("verify_greedy: null argument");
    wsb::row_stats_bf16(logits, n_req * (k + 1), vocab, ld, 1.0f, rows_out, nullptr, workspace, n_req, k, cand, out,
                        static_cast<cudaStream_t>(stream));
  });
}

int ws_op_verify_rejection_bf16(const void* logits, uint32_t n_req, uint32_t k, uint32_t vocab, uint32_t ld,
                                float inv_temp, float top_p, const uint32_t* cand, const double* cand_prob,
                                uint64_t seed, const uint64_t* request, const uint32_t* step, const int32_t* forced,
                                ws_verify_out* out, void* stream) {
  return op_guarded("ws_op_verify_rejection_bf16", [&] {
    wsb::verify_rejection_bf16(logits, n_req, k, vocab, ld, inv_temp, top_p, cand, cand_prob, seed, request, step,
                               forced, out, static_cast<cudaStream_t>(stream));
  });
}

// Diagnostics (not part of the public header): the K1 timeline recorded under WS_GEMM_ABLATE & 8.
int ws_debug_gemm_trace(unsigned long long* out8) {
  return op_guarded("ws_debug_gemm_trace", [&] {
    if (!out8) throw std::invalid_argument("null argument");
    wsb::gemm_debug_trace(out8);
  });
}

}  // extern "C"
