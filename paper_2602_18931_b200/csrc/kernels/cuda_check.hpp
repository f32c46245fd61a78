#pragma once

#include <cuda_runtime.h>

#include <string>

#include "../host/common.hpp"

#define WS_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::wsb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_));      \
  } while (0)
