// Device-pointer entry points of the model-path kernels (include/wanspec_b200.h "ops").
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "kernels/cuda_check.hpp"
#include "kernels/gemm_tc.cuh"
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
                    int epi, int bn, void* stream) {
  return op_guarded("ws_op_gemm_bf16", [&] {
    if (!A || !W || !out || M <= 0 || N <= 0 || K <= 0) throw std::invalid_argument("gemm: bad argument");
    wsb::GemmArgs g{A, W, out, M, N, K, lda, ldw, ldo, epi, bn};
    wsb::gemm_tn(g, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
