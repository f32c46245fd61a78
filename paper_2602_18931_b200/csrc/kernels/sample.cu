// K4R — speculative rejection sampling over the verify rows (see sample.cuh for the rule).
// All fp64 arithmetic that decides an outcome uses explicit _rn intrinsics (no FMA
// contraction), so the host restatement (oracle/restate.c, -ffp-contract=off) performs the same
// operations in the same order; only exp() may differ by an ulp between libdevice and glibc.
#include "sample.cuh"

#include <cuda_bf16.h>

#include <stdexcept>

#include "cuda_check.hpp"
#include "pdl.cuh"

namespace wsb {

namespace {

constexpr int T = kSampleThreads;

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

// order-preserving 16-bit key of a bf16 value (larger value -> larger key)
__device__ __forceinline__ std::uint32_t key16(std::uint16_t b) {
  return (b & 0x8000u) ? (~b & 0xFFFFu) : (b | 0x8000u);
}

// fixed pairwise tree over the T partials (sm[0..T)); every thread returns the total
__device__ double tree_sum(double v, double* sm) {
  sm[threadIdx.x] = v;
  __syncthreads();
  for (int s = T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] = __dadd_rn(sm[threadIdx.x], sm[threadIdx.x + s]);
    __syncthreads();
  }
  const double r = sm[0];
  __syncthreads();
  return r;
}

struct Row {
  const __nv_bfloat16* x;
  std::uint32_t lo, hi;  // this thread's id chunk
  double tau, zmax, Z, S;
  std::int32_t forced;
  std::uint32_t t_star;  // nucleus key threshold (0 = all)
  double M;              // nucleus mass (1 without top-p)
};

__device__ __forceinline__ double zval(const Row& r, std::uint32_t i) {
  return __dmul_rn(static_cast<double>(__bfloat162float(r.x[i])), r.tau);
}
__device__ __forceinline__ std::uint32_t keyat(const Row& r, std::uint32_t i) {
  return key16(__bfloat16_as_ushort(r.x[i]));
}
// p'(i) (the truncated, renormalised target probability)
__device__ __forceinline__ double pprime(const Row& r, std::uint32_t i) {
  if (r.forced >= 0) return static_cast<std::uint32_t>(r.forced) == i ? 1.0 : 0.0;
  if (keyat(r, i) < r.t_star) return 0.0;
  const double p = __ddiv_rn(exp(__dsub_rn(zval(r, i), r.zmax)), r.Z);
  return r.M == 1.0 ? p : __ddiv_rn(p, r.M);
}

__device__ void row_stats(Row& r, std::uint32_t V, float top_p, double* sm, float* smf) {
  if (r.forced >= 0) {
    r.Z = 1.0;
    r.S = 0.0;
    r.zmax = 0.0;
    r.t_star = 0;
    r.M = 1.0;
    return;
  }
  // max of the bf16 values (exact), then Z = sum e, S = sum e (z - zmax) (entropy)
  float mx = -INFINITY;
  for (std::uint32_t i = r.lo; i < r.hi; ++i) mx = fmaxf(mx, __bfloat162float(r.x[i]));
  smf[threadIdx.x] = mx;
  __syncthreads();
  for (int s = T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) smf[threadIdx.x] = fmaxf(smf[threadIdx.x], smf[threadIdx.x + s]);
    __syncthreads();
  }
  r.zmax = __dmul_rn(static_cast<double>(smf[0]), r.tau);
  __syncthreads();
  double z = 0.0, sv = 0.0;
  for (std::uint32_t i = r.lo; i < r.hi; ++i) {
    const double d = __dsub_rn(zval(r, i), r.zmax);
    const double e = exp(d);
    z = __dadd_rn(z, e);
    if (e > 0.0) sv = __dadd_rn(sv, __dmul_rn(e, d));
  }
  r.Z = tree_sum(z, sm);
  r.S = tree_sum(sv, sm);
  r.t_star = 0;
  r.M = 1.0;
  if (top_p < 1.f) {
    const double tp = static_cast<double>(top_p);
    std::uint32_t lo = 0, hi = 65536;
    double m_lo = 1.0;
    while (hi - lo > 1) {
      const std::uint32_t mid = (lo + hi) / 2;
      double part = 0.0;
      for (std::uint32_t i = r.lo; i < r.hi; ++i)
        if (keyat(r, i) >= mid) part = __dadd_rn(part, exp(__dsub_rn(zval(r, i), r.zmax)));
      const double mass = __ddiv_rn(tree_sum(part, sm), r.Z);
      if (mass >= tp) {
        lo = mid;
        m_lo = mass;
      } else {
        hi = mid;
      }
    }
    r.t_star = lo;
    r.M = m_lo;
  }
}

// Inverse-CDF draw in ascending id order from w(x) = max(0, p'(x) - d(x)) (the residual, when
// has_d) or p'(x), u in [0, 1): chunk sums (sequential), a sequential exclusive prefix over the
// chunks (so the chunk intervals [start, start + part) tile [0, R) exactly), the chunk holding
// u*R walked from its start; if rounding leaves the walk empty-handed, the last id with w > 0.
// A zero residual mass falls back to p'.
__device__ std::uint32_t sample_row(const Row& r, std::uint32_t V, bool has_d, std::uint32_t c, double q, double u,
                                    double* scan) {
  __shared__ std::uint32_t pick, lastpos;
  const double tail = V > 1 ? __ddiv_rn(__dsub_rn(1.0, q), static_cast<double>(V - 1)) : 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    const bool resid = has_d && pass == 0;
    auto w = [&](std::uint32_t i) -> double {
      const double p = pprime(r, i);
      if (!resid) return p;
      const double d = __dsub_rn(p, i == c ? q : tail);
      return d > 0.0 ? d : 0.0;
    };
    double part = 0.0;
    for (std::uint32_t i = r.lo; i < r.hi; ++i) part = __dadd_rn(part, w(i));
    scan[threadIdx.x] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double acc = 0.0;
      for (int t = 0; t < T; ++t) {
        const double pt = scan[t];
        scan[t] = acc;
        acc = __dadd_rn(acc, pt);
      }
      scan[T] = acc;
      pick = 0xFFFFFFFFu;
      lastpos = 0;
    }
    __syncthreads();
    const double R = scan[T];
    if (resid && !(R > 0.0)) {  // block-uniform
      __syncthreads();
      continue;
    }
    const double target = __dmul_rn(u, R);
    const double start = scan[threadIdx.x];
    if (part > 0.0) {
      if (target >= start && target < __dadd_rn(start, part)) {
        double acc = start;
        for (std::uint32_t i = r.lo; i < r.hi; ++i) {
          const double v = w(i);
          if (v > 0.0) {
            const double nx = __dadd_rn(acc, v);
            if (nx > target) {
              pick = i;  // at most one chunk holds the target
              break;
            }
            acc = nx;
          }
        }
      }
      std::uint32_t last = r.lo;
      for (std::uint32_t i = r.lo; i < r.hi; ++i)
        if (w(i) > 0.0) last = i;
      atomicMax(&lastpos, last);
    }
    __syncthreads();
    const std::uint32_t res = pick != 0xFFFFFFFFu ? pick : lastpos;
    __syncthreads();
    return res;
  }
  return 0;
}

__global__ void __launch_bounds__(T) verify_rejection_kernel(
    const __nv_bfloat16* __restrict__ logits, std::uint32_t k, std::uint32_t V, std::uint32_t ld, float inv_temp,
    float top_p, const std::uint32_t* __restrict__ cand, const double* __restrict__ cand_prob, std::uint32_t key0,
    std::uint32_t key1, const std::uint64_t* __restrict__ request, const std::uint32_t* __restrict__ step,
    const std::int32_t* __restrict__ forced, ws_verify_out* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  __shared__ double sm[T];
  __shared__ double scan[T + 1];
  __shared__ float smf[T];
  const std::uint32_t j = blockIdx.x;
  const std::uint32_t C = (V + T - 1) / T;
  Row r;
  r.tau = static_cast<double>(inv_temp);
  r.lo = min(V, threadIdx.x * C);
  r.hi = min(V, r.lo + C);
  const std::uint64_t req = request[j];
  for (std::uint32_t i = 0; i <= k; ++i) {
    const std::size_t row = static_cast<std::size_t>(j) * (k + 1) + i;
    r.x = logits + row * ld;
    r.forced = forced ? forced[row] : -1;
    row_stats(r, V, top_p, sm, smf);
    std::uint32_t w[4] = {static_cast<std::uint32_t>(req), static_cast<std::uint32_t>(req >> 32), step[j], i};
    philox4x32_10(w, key0, key1);
    const double u2 = unit_from_words(w[2], w[3]);
    bool reject = false;
    std::uint32_t c = 0;
    double q = 0.0;
    if (i < k) {
      c = cand[static_cast<std::size_t>(j) * k + i];
      q = cand_prob[static_cast<std::size_t>(j) * k + i];
      q = q < 0.0 ? 0.0 : (q > 1.0 ? 1.0 : q);
      const double u = unit_from_words(w[0], w[1]);
      reject = !(__dmul_rn(u, q) < pprime(r, c));
    }
    if (i == k || reject) {
      const std::uint32_t bonus = sample_row(r, V, reject, c, q, u2, scan);
      if (threadIdx.x == 0) {
        ws_verify_out o;
        o.accepted = i;
        o.bonus = bonus;
        o.final_entropy = r.forced >= 0 ? 0.0 : [&] {
          const double h = __dsub_rn(log(r.Z), __ddiv_rn(r.S, r.Z));
          return h < 0.0 ? 0.0 : h;
        }();
        out[j] = o;
      }
      return;
    }
  }
}

}  // namespace

void verify_rejection_bf16(const void* logits, std::uint32_t n_req, std::uint32_t k, std::uint32_t vocab,
                           std::uint32_t ld, float inv_temp, float top_p, const std::uint32_t* cand,
                           const double* cand_prob, std::uint64_t seed, const std::uint64_t* request,
                           const std::uint32_t* step, const std::int32_t* forced, ws_verify_out* out,
                           cudaStream_t stream) {
  if (n_req == 0) return;
  if (!logits || !cand || !cand_prob || !request || !step || !out || vocab == 0 || ld < vocab)
    throw std::invalid_argument("verify_rejection: bad argument");
  if (!(inv_temp > 0.f)) throw std::invalid_argument("verify_rejection: temperature must be > 0");
  if (!(top_p > 0.f)) throw std::invalid_argument("verify_rejection: top_p must be > 0");
  launch_pdl(verify_rejection_kernel, dim3(n_req), dim3(T), 0, stream, 1, static_cast<const __nv_bfloat16*>(logits), k,
             vocab, ld, inv_temp, top_p, cand, cand_prob, static_cast<std::uint32_t>(seed),
             static_cast<std::uint32_t>(seed >> 32), request, step, forced, out);
}

}  // namespace wsb
