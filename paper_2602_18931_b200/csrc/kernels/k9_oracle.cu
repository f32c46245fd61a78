// K9 — batched verify / draft over device-resident tiny-pair tables.
//
// One launch per batched round covers every pending verify job (greedy run_target_step,
// oracle.hpp:127-139, or the Philox rejection extension) and every draft row
// (draft_prediction, oracle.hpp:96-98) of all requests on this protocol thread. The work per
// job is a handful of dependent loads, so the kernel is launch/latency bound; the design goal
// is one launch + one H2D + one D2H per round, not bandwidth.
//
// Rejection arithmetic uses explicit round-to-nearest fp64 intrinsics so no FMA contraction
// can change a rounding: results are bit-identical to oracle/restate.c (-ffp-contract=off).
#include "k9_oracle.cuh"

#include <atomic>
#include <cstdlib>
#include <cstring>

#include "cuda_check.hpp"

namespace wsb {

namespace {

struct DPred {
  std::uint32_t n;
  std::uint32_t id[2];
  double p[2];
};

__device__ __forceinline__ void philox4x32_10(std::uint32_t c[4], std::uint32_t k0, std::uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const std::uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const std::uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const std::uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__device__ __forceinline__ double unit_from_words(std::uint32_t hi, std::uint32_t lo) {
  const std::uint64_t x = (static_cast<std::uint64_t>(hi) << 32) | lo;
  return __dmul_rn(static_cast<double>(x >> 11), 0x1.0p-53);
}

__device__ double tail_per_token(const DPred& p, std::uint32_t vocab) {
  double t = 1.0;
  for (std::uint32_t j = 0; j < p.n; ++j) t = __dsub_rn(t, p.p[j]);
  if (t < 0.0) t = 0.0;
  if (vocab <= p.n) return 0.0;
  return __ddiv_rn(t, static_cast<double>(vocab - p.n));
}

__device__ double completed_prob(const DPred& p, std::uint32_t vocab, std::uint32_t x) {
  for (std::uint32_t j = 0; j < p.n; ++j)
    if (p.id[j] == x) return p.p[j];
  return tail_per_token(p, vocab);
}

// restate.c walk_sample: ascending-id inverse CDF over unlisted runs (mass rho) and listed ids.
__device__ std::uint32_t walk_sample(const std::uint32_t* s, const double* m, int ns, double rho,
                                     std::uint32_t vocab, double u) {
  double z = 0.0;
  std::uint32_t prev = 0;
  for (int j = 0; j < ns; ++j) {
    z = __dadd_rn(z, __dmul_rn(static_cast<double>(s[j] - prev), rho));
    z = __dadd_rn(z, m[j]);
    prev = s[j] + 1;
  }
  z = __dadd_rn(z, __dmul_rn(static_cast<double>(vocab - prev), rho));
  const double target = __dmul_rn(u, z);
  double acc = 0.0;
  prev = 0;
  std::uint32_t last_pos = 0;
  bool have_last = false;
  for (int j = 0; j <= ns; ++j) {
    const std::uint32_t end = j < ns ? s[j] : vocab;
    const std::uint32_t run = end - prev;
    if (run > 0 && rho > 0.0) {
      const double seg = __dmul_rn(static_cast<double>(run), rho);
      if (__dadd_rn(acc, seg) > target) {
        const double off = floor(__ddiv_rn(__dsub_rn(target, acc), rho));
        const std::uint32_t o =
            off < 0.0 ? 0u : (off >= static_cast<double>(run) ? run - 1 : static_cast<std::uint32_t>(off));
        return prev + o;
      }
      acc = __dadd_rn(acc, seg);
      last_pos = end - 1;
      have_last = true;
    }
    if (j < ns) {
      if (m[j] > 0.0) {
        if (__dadd_rn(acc, m[j]) > target) return s[j];
        acc = __dadd_rn(acc, m[j]);
        last_pos = s[j];
        have_last = true;
      }
      prev = s[j] + 1;
    }
  }
  return have_last ? last_pos : 0u;
}

__device__ std::uint32_t sample_residual(const DPred& pt, const DPred* pd, std::uint32_t vocab, double u) {
  std::uint32_t s[4];
  int ns = 0;
  for (int w = 0; w < 2; ++w) {
    const DPred* p = w == 0 ? &pt : pd;
    if (!p) continue;
    for (std::uint32_t j = 0; j < p->n; ++j) {
      const std::uint32_t id = p->id[j];
      bool dup = false;
      for (int q = 0; q < ns; ++q) dup |= s[q] == id;
      if (!dup) s[ns++] = id;
    }
  }
  for (int i = 1; i < ns; ++i)
    for (int j = i; j > 0 && s[j - 1] > s[j]; --j) {
      const std::uint32_t t = s[j];
      s[j] = s[j - 1];
      s[j - 1] = t;
    }
  double m[4];
  const double tt = tail_per_token(pt, vocab);
  if (pd) {
    const double td = tail_per_token(*pd, vocab);
    double zr = 0.0;
    for (int j = 0; j < ns; ++j) {
      const double d = __dsub_rn(completed_prob(pt, vocab, s[j]), completed_prob(*pd, vocab, s[j]));
      m[j] = d > 0.0 ? d : 0.0;
      zr = __dadd_rn(zr, m[j]);
    }
    const double dr = __dsub_rn(tt, td);
    const double rho = dr > 0.0 ? dr : 0.0;
    if (zr > 0.0 || (rho > 0.0 && static_cast<std::uint32_t>(ns) < vocab))
      return walk_sample(s, m, ns, rho, vocab, u);
  }
  for (int j = 0; j < ns; ++j) m[j] = completed_prob(pt, vocab, s[j]);
  return walk_sample(s, m, ns, tt, vocab, u);
}

struct KTables {
  std::uint32_t seq_len, vocab, eos;
  const std::uint32_t *tgt_tok, *tgt_top2, *dft_top1, *dft_top2;
  const double *tgt_p1, *tgt_p2, *tgt_h, *dft_p1, *dft_p2, *dft_h;
};

// oracle.hpp:88-102 lookups (past-end → EOS, probability 1, entropy 0).
__device__ __forceinline__ DPred target_pred(const KTables& t, std::size_t row, std::uint64_t pos) {
  DPred p;
  if (pos < t.seq_len) {
    const std::size_t i = row + pos;
    p.n = 2;
    p.id[0] = t.tgt_tok[i];
    p.id[1] = t.tgt_top2[i];
    p.p[0] = t.tgt_p1[i];
    p.p[1] = t.tgt_p2[i];
  } else {
    p.n = 1;
    p.id[0] = t.eos;
    p.id[1] = 0;
    p.p[0] = 1.0;
    p.p[1] = 0.0;
  }
  return p;
}
__device__ __forceinline__ DPred draft_pred(const KTables& t, std::size_t row, std::uint64_t pos) {
  DPred p;
  if (pos < t.seq_len) {
    const std::size_t i = row + pos;
    p.n = 2;
    p.id[0] = t.dft_top1[i];
    p.id[1] = t.dft_top2[i];
    p.p[0] = t.dft_p1[i];
    p.p[1] = t.dft_p2[i];
  } else {
    p.n = 1;
    p.id[0] = t.eos;
    p.id[1] = 0;
    p.p[0] = 1.0;
    p.p[1] = 0.0;
  }
  return p;
}

__global__ void __launch_bounds__(128) k9_round(KTables t, const VerifyJob* __restrict__ vj, std::uint32_t nv,
                                                const std::uint32_t* __restrict__ cands,
                                                const DraftJob* __restrict__ dj, std::uint32_t nd,
                                                VerifyOut* __restrict__ vo, ws_pred* __restrict__ dout,
                                                int mode, std::uint32_t key0, std::uint32_t key1,
                                                unsigned int* __restrict__ blocks_done,
                                                unsigned long long* round_flag, unsigned long long round_id) {
  const std::uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < nv) {
    const VerifyJob j = vj[g];
    const std::size_t row = static_cast<std::size_t>(j.seq) * t.seq_len;
    const std::uint32_t* c = cands + j.cand_off;
    VerifyOut r;
    if (mode == WS_VERIFY_GREEDY) {
      // run_target_step: accept the longest prefix matching the target tokens; bonus =
      // target token at the first unmatched position; entropy there.
      std::uint64_t pos = j.base;
      std::uint32_t a = 0;
      for (; a < j.k; ++a, ++pos) {
        const std::uint32_t tt = pos < t.seq_len ? t.tgt_tok[row + pos] : t.eos;
        if (c[a] != tt) break;
      }
      r.accepted = a;
      r.bonus = pos < t.seq_len ? t.tgt_tok[row + pos] : t.eos;
      r.final_entropy = pos < t.seq_len ? t.tgt_h[row + pos] : 0.0;
    } else {
      // Rejection extension (restate.c or_rejection_verify).
      r.accepted = j.k;
      r.bonus = 0;
      r.final_entropy = 0.0;
      for (std::uint32_t i = 0; i <= j.k; ++i) {
        const std::uint64_t q = j.base + i;
        const DPred pt = target_pred(t, row, q);
        std::uint32_t w[4] = {static_cast<std::uint32_t>(j.request),
                              static_cast<std::uint32_t>(j.request >> 32), j.step, i};
        philox4x32_10(w, key0, key1);
        const double h = q < t.seq_len ? t.tgt_h[row + q] : 0.0;
        if (i == j.k) {
          r.accepted = j.k;
          r.bonus = sample_residual(pt, nullptr, t.vocab, unit_from_words(w[2], w[3]));
          r.final_entropy = h;
          break;
        }
        const DPred pd = draft_pred(t, row, q);
        const double p_t = completed_prob(pt, t.vocab, c[i]);
        const double p_d = completed_prob(pd, t.vocab, c[i]);
        const double u = unit_from_words(w[0], w[1]);
        if (__dmul_rn(u, p_d) < p_t) continue;
        r.accepted = i;
        r.bonus = sample_residual(pt, &pd, t.vocab, unit_from_words(w[2], w[3]));
        r.final_entropy = h;
        break;
      }
    }
    vo[g] = r;
  } else if (g < nv + nd) {
    const DraftJob j = dj[g - nv];
    const std::size_t row = static_cast<std::size_t>(j.seq) * t.seq_len;
    ws_pred p;
    if (j.pos < t.seq_len) {
      const std::size_t i = row + j.pos;
      p.n = 2;
      p.id[0] = t.dft_top1[i];
      p.id[1] = t.dft_top2[i];
      p.prob[0] = t.dft_p1[i];
      p.prob[1] = t.dft_p2[i];
      p.entropy = t.dft_h[i];
    } else {
      p.n = 1;
      p.id[0] = t.eos;
      p.id[1] = 0;
      p.prob[0] = 1.0;
      p.prob[1] = 0.0;
      p.entropy = 0.0;
    }
    p.pad = 0;
    dout[g - nv] = p;
  }
  // Completion without a driver call: every block's results are system-visible before it
  // counts itself; the last block publishes the round id to the mapped flag the host spins on.
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(blocks_done, 1u) == gridDim.x - 1) {
      *blocks_done = 0;
      __threadfence_system();
      *reinterpret_cast<volatile unsigned long long*>(round_flag) = round_id;
    }
  }
}

KTables ktables(const DevTables& t) {
  return KTables{t.seq_len, t.vocab, t.eos, t.tgt_tok, t.tgt_top2, t.dft_top1, t.dft_top2,
                 t.tgt_p1, t.tgt_p2, t.tgt_h, t.dft_p1, t.dft_p2, t.dft_h};
}

inline std::size_t align16(std::size_t x) { return (x + 15) & ~static_cast<std::size_t>(15); }

}  // namespace

std::size_t upload_tables(DevTables& t, std::uint32_t n_seq, std::uint32_t seq_len, std::uint32_t vocab,
                          std::uint32_t eos, const ws_token_record* recs, cudaStream_t stream) {
  const std::size_t n = static_cast<std::size_t>(n_seq) * seq_len;
  const std::size_t a32 = align16(n * 4), a64 = align16(n * 8);
  const std::size_t bytes = 4 * a32 + 6 * a64;
  if (t.bytes < bytes) {
    free_tables(t);
    WS_CUDA(cudaMalloc(&t.block, bytes));
    t.bytes = bytes;
  }
  std::vector<unsigned char> host(bytes);
  unsigned char* p = host.data();
  auto u32 = [&](std::size_t i) { return reinterpret_cast<std::uint32_t*>(p + i * a32); };
  auto f64 = [&](std::size_t i) { return reinterpret_cast<double*>(p + 4 * a32 + i * a64); };
  for (std::size_t i = 0; i < n; ++i) {
    const ws_token_record& r = recs[i];
    u32(0)[i] = r.target_token;
    u32(1)[i] = r.target_top2;
    u32(2)[i] = r.draft_top1;
    u32(3)[i] = r.draft_top2;
    f64(0)[i] = r.target_p1;
    f64(1)[i] = r.target_p2;
    f64(2)[i] = r.target_entropy;
    f64(3)[i] = r.draft_p1;
    f64(4)[i] = r.draft_p2;
    f64(5)[i] = r.draft_entropy;
  }
  WS_CUDA(cudaMemcpyAsync(t.block, host.data(), bytes, cudaMemcpyHostToDevice, stream));
  WS_CUDA(cudaStreamSynchronize(stream));
  unsigned char* d = static_cast<unsigned char*>(t.block);
  t.tgt_tok = reinterpret_cast<std::uint32_t*>(d + 0 * a32);
  t.tgt_top2 = reinterpret_cast<std::uint32_t*>(d + 1 * a32);
  t.dft_top1 = reinterpret_cast<std::uint32_t*>(d + 2 * a32);
  t.dft_top2 = reinterpret_cast<std::uint32_t*>(d + 3 * a32);
  t.tgt_p1 = reinterpret_cast<double*>(d + 4 * a32 + 0 * a64);
  t.tgt_p2 = reinterpret_cast<double*>(d + 4 * a32 + 1 * a64);
  t.tgt_h = reinterpret_cast<double*>(d + 4 * a32 + 2 * a64);
  t.dft_p1 = reinterpret_cast<double*>(d + 4 * a32 + 3 * a64);
  t.dft_p2 = reinterpret_cast<double*>(d + 4 * a32 + 4 * a64);
  t.dft_h = reinterpret_cast<double*>(d + 4 * a32 + 5 * a64);
  t.n_seq = n_seq;
  t.seq_len = seq_len;
  t.vocab = vocab;
  t.eos = eos;
  return bytes;
}

void free_tables(DevTables& t) {
  if (t.block) cudaFree(t.block);
  t = DevTables{};
}

OracleLane::OracleLane(const DevTables* tables, int device) : t_(tables), device_(device) {
  WS_CUDA(cudaSetDevice(device_));
  WS_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  WS_CUDA(cudaEventCreate(&ev0_));
  WS_CUDA(cudaEventCreate(&ev1_));
  WS_CUDA(cudaMalloc(&d_blocks_done_, sizeof(unsigned int)));
  WS_CUDA(cudaMemset(d_blocks_done_, 0, sizeof(unsigned int)));
  WS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_flag_), sizeof(unsigned long long), cudaHostAllocMapped));
  WS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_flag_), h_flag_, 0));
  *h_flag_ = 0;
}

OracleLane::~OracleLane() {
  if (h_in_) cudaFreeHost(h_in_);
  if (h_out_) cudaFreeHost(h_out_);  // d_in_/d_out_ alias these mapped allocations
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  if (d_blocks_done_) cudaFree(d_blocks_done_);
  if (h_flag_) cudaFreeHost(h_flag_);
  if (stream_) cudaStreamDestroy(stream_);
}

// Job and result blocks live in mapped pinned host memory: the round's kernel reads the few KB
// of jobs and writes its results across the bus directly, so a round is one launch + one
// stream sync (no copy-engine round trips, and rounds of different protocol threads overlap).
void OracleLane::reserve(std::size_t in_bytes, std::size_t out_bytes) {
  if (in_bytes > cap_in_) {
    const std::size_t c = std::max(in_bytes, 2 * cap_in_);
    if (h_in_) cudaFreeHost(h_in_);
    WS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_in_), c, cudaHostAllocMapped));
    WS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_in_), h_in_, 0));
    cap_in_ = c;
  }
  if (out_bytes > cap_out_) {
    const std::size_t c = std::max(out_bytes, 2 * cap_out_);
    if (h_out_) cudaFreeHost(h_out_);
    WS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_out_), c, cudaHostAllocMapped));
    WS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_out_), h_out_, 0));
    cap_out_ = c;
  }
}

void OracleLane::run_round(const RoundJobs& jobs, RoundResults& res, int verify_mode,
                           std::uint64_t sample_seed) {
  if (!t_ || !t_->block) throw ConfigError("K9: oracle tables not loaded");
  const std::uint32_t nv = static_cast<std::uint32_t>(jobs.verify.size());
  const std::uint32_t nd = static_cast<std::uint32_t>(jobs.draft.size());
  const std::size_t sv = align16(nv * sizeof(VerifyJob));
  const std::size_t sc = align16(jobs.cands.size() * sizeof(std::uint32_t));
  const std::size_t sd = align16(nd * sizeof(DraftJob));
  const std::size_t ov = align16(nv * sizeof(VerifyOut));
  const std::size_t od = nd * sizeof(ws_pred);
  const std::size_t in_bytes = sv + sc + sd, out_bytes = ov + od;
  reserve(in_bytes + 16, out_bytes + 16);
  std::memcpy(h_in_, jobs.verify.data(), nv * sizeof(VerifyJob));
  std::memcpy(h_in_ + sv, jobs.cands.data(), jobs.cands.size() * sizeof(std::uint32_t));
  std::memcpy(h_in_ + sv + sc, jobs.draft.data(), nd * sizeof(DraftJob));
  const std::uint32_t total = nv + nd;
  const std::uint32_t threads = 128, blocks = std::max<std::uint32_t>(1, (total + threads - 1) / threads);
  // A round is one launch and a spin on the mapped completion flag (no sync call: with several
  // protocol threads per GPU, driver calls serialise on the context). WS_PROFILE adds events.
  static const bool timed = std::getenv("WS_PROFILE") != nullptr;
  if (timed) WS_CUDA(cudaEventRecord(ev0_, stream_));
  const unsigned long long id = ++round_id_;
  k9_round<<<blocks, threads, 0, stream_>>>(
      ktables(*t_), reinterpret_cast<const VerifyJob*>(d_in_), nv,
      reinterpret_cast<const std::uint32_t*>(d_in_ + sv), reinterpret_cast<const DraftJob*>(d_in_ + sv + sc), nd,
      reinterpret_cast<VerifyOut*>(d_out_), reinterpret_cast<ws_pred*>(d_out_ + ov), verify_mode,
      static_cast<std::uint32_t>(sample_seed), static_cast<std::uint32_t>(sample_seed >> 32), d_blocks_done_, d_flag_,
      id);
  WS_CUDA(cudaGetLastError());
  float ms = 0.f;
  if (timed) WS_CUDA(cudaEventRecord(ev1_, stream_));
  for (std::uint64_t spin = 1;; ++spin) {
    if (*reinterpret_cast<volatile unsigned long long*>(h_flag_) == id) break;
    if ((spin & 0xFFFFF) == 0) {  // surface a failed launch instead of spinning forever
      const cudaError_t e = cudaStreamQuery(stream_);
      if (e != cudaSuccess && e != cudaErrorNotReady) WS_CUDA(e);
      if (e == cudaSuccess && *reinterpret_cast<volatile unsigned long long*>(h_flag_) != id)
        throw CudaError("K9: round finished without publishing its completion flag");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  if (timed) {
    WS_CUDA(cudaStreamSynchronize(stream_));
    WS_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
  }
  res.verify.resize(nv);
  res.draft.resize(nd);
  std::memcpy(res.verify.data(), h_out_, nv * sizeof(VerifyOut));
  std::memcpy(res.draft.data(), h_out_ + ov, od);
  stats.rounds += 1;
  stats.launches += 1;
  stats.verify_rows += nv;
  stats.draft_rows += nd;
  stats.h2d += in_bytes;
  stats.d2h += out_bytes;
  stats.kernel_ms += ms;
}

}  // namespace wsb
