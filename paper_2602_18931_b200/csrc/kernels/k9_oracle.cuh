// K9: the tiny pair's verify / draft on device-resident TokenRecord tables.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../host/driver.hpp"
#include "wanspec_b200.h"

namespace wsb {

// SoA device tables, [n_seq * seq_len] each (coalesced: one request's consecutive positions
// share sectors, so a k+1-position verify walk touches one or two 32 B sectors per array).
struct DevTables {
  std::uint32_t n_seq = 0, seq_len = 0, vocab = 0, eos = 0;
  std::uint32_t* tgt_tok = nullptr;
  std::uint32_t* tgt_top2 = nullptr;
  double* tgt_p1 = nullptr;
  double* tgt_p2 = nullptr;
  double* tgt_h = nullptr;
  std::uint32_t* dft_top1 = nullptr;
  std::uint32_t* dft_top2 = nullptr;
  double* dft_p1 = nullptr;
  double* dft_p2 = nullptr;
  double* dft_h = nullptr;
  void* block = nullptr;  // single allocation backing all arrays
  std::size_t bytes = 0;
};

// Allocates (or reuses) `t` and uploads AoS records as SoA. Returns H2D bytes.
std::size_t upload_tables(DevTables& t, std::uint32_t n_seq, std::uint32_t seq_len, std::uint32_t vocab,
                          std::uint32_t eos, const ws_token_record* recs, cudaStream_t stream);
void free_tables(DevTables& t);

// One protocol thread's GPU lane: a stream, pinned staging and device job/result buffers.
class OracleLane : public ModelBackend {
 public:
  OracleLane(const DevTables* tables, int device);
  ~OracleLane() override;
  void run_round(const RoundJobs& jobs, RoundResults& res, int verify_mode,
                 std::uint64_t sample_seed) override;
  cudaStream_t stream() const { return stream_; }

 private:
  void reserve(std::size_t in_bytes, std::size_t out_bytes);
  const DevTables* t_;
  int device_;
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  unsigned int* d_blocks_done_ = nullptr;      // last-block detection (device, self-resetting)
  unsigned long long* h_flag_ = nullptr;       // mapped completion flag the host spins on
  unsigned long long* d_flag_ = nullptr;
  unsigned long long round_id_ = 0;
  unsigned char* h_in_ = nullptr;
  unsigned char* h_out_ = nullptr;
  unsigned char* d_in_ = nullptr;
  unsigned char* d_out_ = nullptr;
  std::size_t cap_in_ = 0, cap_out_ = 0;
};

}  // namespace wsb
