// Tensor parallelism for target shapes split over several GPUs of one box (BASELINE config 5,
// Llama-3.1-70B over NVLink 5 / NVSwitch). Column-parallel QKV and gate/up,
// row-parallel O and down; after each row-parallel projection the ranks' fp32 partials are
// summed by a peer-memory collective fused with the residual update and the fused-RMSNorm
// producer outputs — one kernel per all-reduce, no NCCL call on the path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace wsb {

constexpr int kMaxTP = 8;

// Device pointers of every rank (peer access enabled between all ranks).
struct TPPeers {
  int tp = 1;
  const float* part[kMaxTP];       // each rank's fp32 partial [rows][d] of the projection
  float* x[kMaxTP];                // each rank's fp32 residual replica [rows][d]
  void* xb[kMaxTP];                // bf16 copy replica [rows][d] (A operand of the next GEMM)
  float* ss[kMaxTP];               // chunk sums of squares replica, chunk-major [d/32][ld_ss]
  unsigned long long* flag_a[kMaxTP];  // per rank: tp "partial ready" epochs (written by peers)
  unsigned long long* flag_b[kMaxTP];  // per rank: tp "broadcast done" epochs
  unsigned int* counter;           // this rank's CTA counter (self-resetting)
};

// All-reduce fused with the residual stream update, run by every rank on its own stream right
// after its row-parallel GEMM: rank g owns rows [rows*g/tp, rows*(g+1)/tp); for those rows
//   x = x + ((part_0 + part_1) + ... + part_{tp-1})      (rank order: deterministic, and every
//                                                           rank receives the same bits)
// and writes xb = bf16(x) and the 32-column chunk sums of squares into EVERY rank's replica
// (peer stores over NVLink); with write_x_all the fp32 rows as well (the last layer, whose
// residual the final norm reads on every rank). Epoch flags order the ranks: a rank starts
// reading peer partials once every rank's GEMM finished, and returns once every rank's
// broadcast landed in its replica — the next kernel on each stream sees a complete xb / ss.
void tp_allreduce_residual(const TPPeers& p, int rank, int rows, int d, int ld_ss, unsigned long long epoch,
                           bool write_x_all, cudaStream_t st);

// Rows [row0, row0 + rows) x columns [col0, col0 + cols) of the deterministic N(std, mean) bf16
// fill of a full [*, ld_full] tensor (fill_normal_bf16's values), stored densely [rows][cols]:
// the shards of a weight get exactly the single-GPU weight's values.
void fill_normal_bf16_2d(void* out, std::int64_t rows, std::int64_t cols, std::int64_t ld_full, std::int64_t row0,
                         std::int64_t col0, std::uint64_t seed, std::uint32_t stream_id, float std_, float mean,
                         cudaStream_t st);

}  // namespace wsb
