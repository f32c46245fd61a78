// K3 — fused vocab-wide softmax + entropy + top-2 over bf16 logits, and the K4 greedy verify
// epilogue fused behind it.
//
// Entropy semantics follow entropy_of (oracle.hpp:21-33): H = -sum p ln p in nats, computed in
// one streaming pass as H = ln Z - S/Z with m = max, Z = sum e^(l-m), S = sum e^(l-m)(l-m)
// (online rescaling when the running max grows), fp32 accumulation. Top-2 follows the
// Prediction tie rule (types.hpp:54-55): descending value, ties to the lower id.
//
// Layout: grid (splits, rows); a CTA streams one fixed 65536-wide vocab chunk of one row with
// 16-byte vector loads (4 in flight per thread), reduces warp → CTA, and the last CTA of a row
// (atomic ticket) merges the chunk partials in chunk order → deterministic and batch-invariant.
// With the verify epilogue enabled, the last row of a request to finish runs run_target_step
// (oracle.hpp:127-139) on the argmaxes: accept while argmax(row i) == cand[i], bonus =
// argmax(row a), final_entropy = H(row a). HBM-bound: rows*V*2 bytes read once.
#include "rowstats.cuh"

#include <cuda_bf16.h>

#include <stdexcept>

#include "cuda_check.hpp"
#include "pdl.cuh"

namespace wsb {

namespace {

constexpr int kThreads = 256;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kFloor = -1.2676506002282294e30f;  // -2^100: exp weight 0, products finite

struct State {
  float m, z, s;  // log2-domain running max, sum, sum e*d
  float v1, v2;   // raw top-2 logits
  std::uint32_t i1, i2;
  float2 z2, s2;  // the vector path's (z, s) as even/odd-element lanes (packed f32x2 math)
};

// The vector path's top-2 is found in two steps. The stream keeps, branch-free, the thread's
// two best 8-element vectors ranked by (vector max desc, vector index asc). A per-element insert
// there would diverge at warp level on almost every vector (profiles/r01_ncu_rowstats.md: 27
// issued instructions per element). Then only those two vectors are rescanned with insert().
// This is exact: the best element lies in the best vector. The second-best element is either in
// that vector too or it is the maximum of its own vector, and then that vector ranks second.
// Ids grow with the vector index inside a thread, so a tie keeps the earlier vector, matching
// the Prediction tie rule (ties to the lower id).
struct Best2 {
  float m1, m2;
  std::uint32_t i1, i2;  // element id of the vector's first lane; kNone if unset
};
constexpr std::uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ void init(State& a) {
  a.m = -INFINITY;
  a.z = 0.f;
  a.s = 0.f;
  a.v1 = a.v2 = -INFINITY;
  a.i1 = a.i2 = 0xFFFFFFFFu;
  a.z2 = a.s2 = make_float2(0.f, 0.f);
}

__device__ __forceinline__ void init(Best2& b) {
  b.m1 = b.m2 = -INFINITY;
  b.i1 = b.i2 = kNone;
}

__device__ __forceinline__ void track(Best2& b, float mx, std::uint32_t id0) {
  const bool p1 = mx > b.m1 || b.i1 == kNone;
  const bool p2 = mx > b.m2 || b.i2 == kNone;
  b.m2 = p1 ? b.m1 : (p2 ? mx : b.m2);
  b.i2 = p1 ? b.i1 : (p2 ? id0 : b.i2);
  b.m1 = p1 ? mx : b.m1;
  b.i1 = p1 ? id0 : b.i1;
}

__device__ __forceinline__ bool better(float v, std::uint32_t i, float w, std::uint32_t j) {
  return v > w || (v == w && i < j);
}

__device__ __forceinline__ void insert(State& a, float v, std::uint32_t i) {
  if (better(v, i, a.v2, a.i2)) {
    if (better(v, i, a.v1, a.i1)) {
      a.v2 = a.v1;
      a.i2 = a.i1;
      a.v1 = v;
      a.i1 = i;
    } else {
      a.v2 = v;
      a.i2 = i;
    }
  }
}

__device__ __forceinline__ void merge(State& a, const State& b) {
  const float m = fmaxf(a.m, b.m);
  float z = 0.f, s = 0.f;
  if (a.z > 0.f) {
    const float f = exp2f(a.m - m);
    z += a.z * f;
    s += f * (a.s + a.z * (a.m - m));
  }
  if (b.z > 0.f) {
    const float f = exp2f(b.m - m);
    z += b.z * f;
    s += f * (b.s + b.z * (b.m - m));
  }
  a.m = m;
  a.z = z;
  a.s = s;
  insert(a, b.v1, b.i1);
  insert(a, b.v2, b.i2);
}

// MUFU.EX2 directly (rel. error ~2^-22): the per-element exponential of the streaming pass.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void absorb8(State& a, Best2& b, const uint4& q, std::uint32_t id0, float cl) {
  // bf16 -> f32 is a 16-bit shift: one integer op per element (low half: shift, high: mask)
  // -inf logits (masked vocabulary) are clamped to -2^100 for the softmax sums: their weight
  // is still exactly 0, but e*d stays 0 instead of 0*(-inf) = NaN (entropy_of's 0 ln 0 = 0,
  // oracle.hpp:21-33). One packed bf16x2 max per two elements; the top-2 rescan reads the raw
  // vector, so a -inf second candidate keeps its value.
  std::uint32_t wd[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&wd[j]);
    h = __hmax2(h, __floats2bfloat162_rn(kFloor, kFloor));
    wd[j] = *reinterpret_cast<const std::uint32_t*>(&h);
  }
  float x[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    x[2 * j] = __uint_as_float(wd[j] << 16);
    x[2 * j + 1] = __uint_as_float(wd[j] & 0xFFFF0000u);
  }
  float mx = x[0];
#pragma unroll
  for (int j = 1; j < 8; ++j) mx = fmaxf(mx, x[j]);
  const float lm = mx * cl;
  if (lm > a.m) {
    if (a.z2.x > 0.f || a.z2.y > 0.f) {
      const float f = exp2f(a.m - lm), dm = a.m - lm;
      const float2 f2 = make_float2(f, f);
      a.s2 = __fmul2_rn(f2, __ffma2_rn(a.z2, make_float2(dm, dm), a.s2));
      a.z2 = __fmul2_rn(a.z2, f2);
    }
    a.m = lm;
  }
  // two elements per packed FFMA2/FADD2 (sm_100): 1.5 instead of 3 FP32 issues per element
  const float2 c2 = make_float2(cl, cl), n2 = make_float2(-a.m, -a.m);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 d = __ffma2_rn(make_float2(x[2 * j], x[2 * j + 1]), c2, n2);
    const float2 e = make_float2(ex2(d.x), ex2(d.y));
    a.z2 = __fadd2_rn(a.z2, e);
    a.s2 = __ffma2_rn(e, d, a.s2);
  }
  track(b, mx, id0);
}

// exact top-2 over one 8-element vector of the row (the rescan of a Best2 entry)
__device__ __forceinline__ void insert8(State& a, const uint4& q, std::uint32_t id0) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = __bfloat1622float2(h[j]);
    insert(a, f.x, id0 + 2 * j);
    insert(a, f.y, id0 + 2 * j + 1);
  }
}

__device__ __forceinline__ void absorb1(State& a, float x, std::uint32_t id, float cl) {
  const float l = fmaxf(x, kFloor) * cl;  // -inf → a finite floor (see absorb8)
  if (l > a.m) {
    if (a.z > 0.f) {
      const float f = exp2f(a.m - l);
      a.s = f * (a.s + a.z * (a.m - l));
      a.z *= f;
    }
    a.m = l;
  }
  const float d = l - a.m;
  const float e = exp2f(d);
  a.z += e;
  a.s = fmaf(e, d, a.s);
  insert(a, x, id);
}

struct Partial {
  float m, z, s, v1, v2;
  std::uint32_t i1, i2, pad;
};

constexpr std::uint32_t kMaxRows = 65535;  // grid.y limit
constexpr std::size_t kTicketBytes = 2 * 65536 * sizeof(std::uint32_t);

__device__ void finalize(const State& a, float cl, std::uint32_t vocab, ws_pred* pred, RowStats* st,
                         std::int32_t forced) {
  if (forced >= 0) {  // past-the-end rule: fully confident prediction, entropy 0
    ws_pred p;
    p.n = 1;
    p.id[0] = static_cast<std::uint32_t>(forced);
    p.id[1] = 0;
    p.pad = 0;
    p.prob[0] = 1.0;
    p.prob[1] = 0.0;
    p.entropy = 0.0;
    *pred = p;
    if (st) *st = RowStats{a.m, a.z, cl, 0.f};
    return;
  }
  const float lnz = logf(a.z);
  float h = lnz - kLn2 * a.s / a.z;
  if (h < 0.f) h = 0.f;
  ws_pred p;
  p.n = vocab >= 2 ? 2u : 1u;
  p.id[0] = a.i1;
  p.id[1] = vocab >= 2 ? a.i2 : 0u;
  p.pad = 0;
  p.prob[0] = static_cast<double>(exp2f(fmaf(a.v1, cl, -a.m)) / a.z);
  p.prob[1] = vocab >= 2 ? static_cast<double>(exp2f(fmaf(a.v2, cl, -a.m)) / a.z) : 0.0;
  p.entropy = static_cast<double>(h);
  *pred = p;
  if (st) *st = RowStats{a.m, a.z, cl, h};
}

__global__ void __launch_bounds__(kThreads) row_stats_kernel(
    const __nv_bfloat16* __restrict__ logits, std::uint32_t vocab, std::uint32_t ld, float cl, bool vec_ok,
    ws_pred* __restrict__ out_pred, RowStats* __restrict__ out_stats, Partial* __restrict__ partials,
    std::uint32_t* __restrict__ row_ticket, std::uint32_t k, const std::uint32_t* __restrict__ cand,
    ws_verify_out* __restrict__ vout, std::uint32_t* __restrict__ req_ticket, const std::int32_t* __restrict__ forced) {
  pdl_trigger();
  pdl_wait();  // inputs come from the previous kernel of the chain
  const std::uint32_t split = blockIdx.x, splits = gridDim.x, row = blockIdx.y;
  const std::uint32_t lo = split * kRowChunk;
  const std::uint32_t hi = min(vocab, lo + kRowChunk);
  const __nv_bfloat16* x = logits + static_cast<std::size_t>(row) * ld;
  State a;
  init(a);
  if (vec_ok) {
    const uint4* v = reinterpret_cast<const uint4*>(x + lo);
    const std::uint32_t nvec = (hi - lo) / 8;
    Best2 best;
    init(best);
    std::uint32_t i = threadIdx.x;
    for (; i + 3 * kThreads < nvec; i += 4 * kThreads) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = __ldcs(v + i + u * kThreads);
      // (loads of the next four issued before these are absorbed measured slower: 62 registers)
#pragma unroll
      for (int u = 0; u < 4; ++u) absorb8(a, best, q[u], lo + 8 * (i + u * kThreads), cl);
    }
    for (; i < nvec; i += kThreads) absorb8(a, best, __ldcs(v + i), lo + 8 * i, cl);
    a.z = a.z2.x + a.z2.y;  // fold the lanes (same running max) before the scalar tail
    a.s = a.s2.x + a.s2.y;
    // rescan the two best vectors (32 B per thread, mostly L2 hits)
    if (best.i1 != kNone) insert8(a, v[(best.i1 - lo) / 8], best.i1);
    if (best.i2 != kNone) insert8(a, v[(best.i2 - lo) / 8], best.i2);
    for (std::uint32_t t = lo + nvec * 8 + threadIdx.x; t < hi; t += kThreads)
      absorb1(a, __bfloat162float(x[t]), t, cl);
  } else {
    for (std::uint32_t t = lo + threadIdx.x; t < hi; t += kThreads) absorb1(a, __bfloat162float(x[t]), t, cl);
  }
  // warp → CTA reduction (fixed order → deterministic): the warp max first, then every lane
  // rescales its (z, s) to it once, so the butterfly levels are plain sums plus the top-2
  // inserts (one exp2 per lane instead of two per level)
  {
    float mw = a.m;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, off));
    if (a.z > 0.f) {
      const float f = exp2f(a.m - mw);
      a.s = f * (a.s + a.z * (a.m - mw));
      a.z *= f;
    }
    a.m = mw;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float z = __shfl_xor_sync(0xffffffffu, a.z, off);
      const float sv = __shfl_xor_sync(0xffffffffu, a.s, off);
      const float v1 = __shfl_xor_sync(0xffffffffu, a.v1, off);
      const float v2 = __shfl_xor_sync(0xffffffffu, a.v2, off);
      const std::uint32_t i1 = __shfl_xor_sync(0xffffffffu, a.i1, off);
      const std::uint32_t i2 = __shfl_xor_sync(0xffffffffu, a.i2, off);
      a.z += z;
      a.s += sv;
      insert(a, v1, i1);
      insert(a, v2, i2);
    }
  }
  __shared__ State warp_states[kThreads / 32];
  __shared__ bool is_last;
  const std::uint32_t w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) warp_states[w] = a;
  __syncthreads();
  if (threadIdx.x != 0) return;
  State r = warp_states[0];
  for (int q = 1; q < kThreads / 32; ++q) merge(r, warp_states[q]);

  if (splits > 1) {
    partials[row * splits + split] = Partial{r.m, r.z, r.s, r.v1, r.v2, r.i1, r.i2, 0};
    __threadfence();
    const std::uint32_t t = atomicAdd(&row_ticket[row], 1u);
    is_last = t == splits - 1;
    if (!is_last) return;
    __threadfence();
    init(r);
    for (std::uint32_t q = 0; q < splits; ++q) {  // chunk order: deterministic
      const Partial* p = &partials[row * splits + q];
      State b;
      b.m = __ldcg(&p->m);
      b.z = __ldcg(&p->z);
      b.s = __ldcg(&p->s);
      b.v1 = __ldcg(&p->v1);
      b.v2 = __ldcg(&p->v2);
      b.i1 = __ldcg(&p->i1);
      b.i2 = __ldcg(&p->i2);
      merge(r, b);
    }
    row_ticket[row] = 0;  // self-reset for the next launch
  }
  finalize(r, cl, vocab, &out_pred[row], out_stats ? &out_stats[row] : nullptr, forced ? forced[row] : -1);

  if (cand) {  // K4 greedy epilogue: the last finished row of the request runs the walk
    const std::uint32_t req = row / (k + 1);
    __threadfence();
    const std::uint32_t t = atomicAdd(&req_ticket[req], 1u);
    if (t != k) return;
    __threadfence();
    req_ticket[req] = 0;
    const ws_pred* rows = out_pred + static_cast<std::size_t>(req) * (k + 1);
    std::uint32_t acc = 0;
    while (acc < k && __ldcg(&rows[acc].id[0]) == cand[static_cast<std::size_t>(req) * k + acc]) ++acc;
    ws_verify_out o;
    o.accepted = acc;
    o.bonus = __ldcg(&rows[acc].id[0]);
    o.final_entropy = __ldcg(&rows[acc].entropy);
    vout[req] = o;
  }
}

}  // namespace

std::size_t rowstats_workspace_bytes(std::uint32_t rows, std::uint32_t vocab, std::uint32_t n_req) {
  const std::uint32_t splits = (vocab + kRowChunk - 1) / kRowChunk;
  (void)n_req;
  return kTicketBytes + static_cast<std::size_t>(rows) * splits * sizeof(Partial) + 64;
}

void row_stats_bf16(const void* logits, std::uint32_t rows, std::uint32_t vocab, std::uint32_t ld, float inv_temp,
                    ws_pred* out_pred, RowStats* out_stats, void* workspace, std::uint32_t n_req, std::uint32_t k,
                    const std::uint32_t* cand, ws_verify_out* verify_out, cudaStream_t stream,
                    const std::int32_t* forced) {
  if (rows == 0) return;
  if (!logits || !out_pred || vocab == 0 || ld < vocab) throw std::invalid_argument("row_stats: bad argument");
  if (!(inv_temp > 0.f)) throw std::invalid_argument("row_stats: temperature must be > 0");
  if (cand && (rows != n_req * (k + 1) || !verify_out)) throw std::invalid_argument("row_stats: verify shape");
  const std::uint32_t splits = (vocab + kRowChunk - 1) / kRowChunk;
  if (splits > 1 || cand) {
    if (!workspace) throw std::invalid_argument("row_stats: workspace required");
  }
  if (rows > kMaxRows || n_req > kMaxRows) throw std::invalid_argument("row_stats: too many rows");
  // Fixed layout whatever the row count: [row tickets | request tickets | partials]. The tickets
  // self-reset, so they must not move between launches of different sizes.
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  std::uint32_t* row_ticket = reinterpret_cast<std::uint32_t*>(ws);
  std::uint32_t* req_ticket = row_ticket + kMaxRows;
  Partial* partials = reinterpret_cast<Partial*>(ws + kTicketBytes);
  const bool vec_ok = (reinterpret_cast<std::uintptr_t>(logits) % 16 == 0) && (ld % 8 == 0);
  dim3 grid(splits, rows);
  launch_pdl(row_stats_kernel, grid, dim3(kThreads), 0, stream, 1, static_cast<const __nv_bfloat16*>(logits), vocab,
             ld, inv_temp * kLog2e, vec_ok, out_pred, out_stats, partials, row_ticket, k, cand, verify_out,
             req_ticket, forced);
}

}  // namespace wsb
