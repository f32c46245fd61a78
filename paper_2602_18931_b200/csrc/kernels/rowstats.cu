// K3 — fused vocab-wide softmax + entropy + top-2 over bf16 logits, and the K4 greedy verify
// epilogue fused behind it.
//
// Entropy semantics follow entropy_of (oracle.hpp:21-33): H = -sum p ln p in nats, computed in
// one streaming pass as H = ln Z - S/Z with m = max, Z = sum e^(l-m), S = sum e^(l-m)(l-m)
// (online rescaling when the running max grows), fp32 accumulation. Top-2 follows the
// Prediction tie rule (types.hpp:54-55): descending value, ties to the lower id.
//
// Layout: a row is cut into fixed 8192-wide tiles (kRowTile). One warp reduces one tile in a
// fixed lane order (lane l streams the tile's 16-byte vectors l, l+32, ...) to a tile partial;
// the last warp to finish a row (atomic ticket) merges the row's tile partials in a fixed tree.
// Neither the tiling nor the trees depend on the row count, so a row's statistics are
// bit-identical at any batch size (batch invariance). Which warp reduces which tile does depend
// on it: the grid is persistent and balanced — every warp takes the same number of consecutive
// tiles (ceil(tiles / resident warps)), so no partial wave of CTAs is left at the end
// (profiles/r02_ncu_k3.md: 64K-chunk CTAs at 535 rows ran 1.45 waves at 46% warps active).
// With the verify epilogue enabled, the last row of a request to finish runs run_target_step
// (oracle.hpp:127-139) on the argmaxes: accept while argmax(row i) == cand[i], bonus =
// argmax(row a), final_entropy = H(row a). HBM-bound: rows*V*2 bytes read once.
#include "rowstats.cuh"

#include <cuda_bf16.h>

#include <atomic>
#include <stdexcept>

#include "cuda_check.hpp"
#include "pdl.cuh"

namespace wsb {

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kFloor = -1.2676506002282294e30f;  // -2^100: exp weight 0, products finite
constexpr std::uint32_t kNone = 0xFFFFFFFFu;

// A (value, id) pair ranked by the Prediction order: value desc, ties to the lower id.
__device__ __forceinline__ bool better(float v, std::uint32_t i, float w, std::uint32_t j) {
  return v > w || (v == w && i < j);
}

// The top-2 of a set, sorted (a1 before a2 in the Prediction order); kNone / -inf when unset.
struct Top2 {
  float v1, v2;
  std::uint32_t i1, i2;
};

__device__ __forceinline__ void init(Top2& t) {
  t.v1 = t.v2 = -INFINITY;
  t.i1 = t.i2 = kNone;
}

// top-2 of the union of two sorted pairs (element ids distinct): commutative, so an xor
// butterfly leaves the same bits in every lane
__device__ __forceinline__ Top2 merge2(const Top2& a, const Top2& b) {
  Top2 r;
  if (better(b.v1, b.i1, a.v1, a.i1)) {
    r.v1 = b.v1;
    r.i1 = b.i1;
    const bool s = better(b.v2, b.i2, a.v1, a.i1);
    r.v2 = s ? b.v2 : a.v1;
    r.i2 = s ? b.i2 : a.i1;
  } else {
    r.v1 = a.v1;
    r.i1 = a.i1;
    const bool s = better(b.v1, b.i1, a.v2, a.i2);
    r.v2 = s ? b.v1 : a.v2;
    r.i2 = s ? b.i1 : a.i2;
  }
  return r;
}

__device__ __forceinline__ void insert(Top2& t, float v, std::uint32_t i) {
  if (better(v, i, t.v2, t.i2)) {
    if (better(v, i, t.v1, t.i1)) {
      t.v2 = t.v1;
      t.i2 = t.i1;
      t.v1 = v;
      t.i1 = i;
    } else {
      t.v2 = v;
      t.i2 = i;
    }
  }
}

__device__ __forceinline__ Top2 shfl_xor(const Top2& t, int off) {
  Top2 r;
  r.v1 = __shfl_xor_sync(0xffffffffu, t.v1, off);
  r.v2 = __shfl_xor_sync(0xffffffffu, t.v2, off);
  r.i1 = __shfl_xor_sync(0xffffffffu, t.i1, off);
  r.i2 = __shfl_xor_sync(0xffffffffu, t.i2, off);
  return r;
}

// Softmax statistics of a set in the log2 domain: m = max(l), z = sum 2^(l-m),
// s = sum 2^(l-m)(l-m). The empty set (m = -inf, z = 0) is merge's exact identity.
struct Stats {
  float m, z, s;
  Top2 t;
};

__device__ __forceinline__ Stats merge(const Stats& a, const Stats& b) {
  Stats r;
  r.m = fmaxf(a.m, b.m);
  float z = 0.f, s = 0.f;
  if (a.z > 0.f) {
    const float f = exp2f(a.m - r.m);
    z += a.z * f;
    s += f * (a.s + a.z * (a.m - r.m));
  }
  if (b.z > 0.f) {
    const float f = exp2f(b.m - r.m);
    z += b.z * f;
    s += f * (b.s + b.z * (b.m - r.m));
  }
  r.z = z;
  r.s = s;
  r.t = merge2(a.t, b.t);
  return r;
}

// One lane's streaming state over its vectors of a tile.
//
// (z, s) are kept relative to a lazy reference m instead of the running max: m only moves when
// a vector's maximum exceeds it by more than kSlack (log2 units), so every term 2^(l-m) stays
// below 2^kSlack and the rescale branch runs about once per lane and tile. (Re-referencing at
// every new running max made some lane of the warp take the branch on ~87% of the vectors —
// 75 issued instructions per 8 elements, profiles/r02_ncu_k3.md.) Any reference gives the same
// statistics: p = 2^(l-m)/Z and H = log2 Z - S/Z do not depend on it; the row's final
// re-references to the true maximum for RowStats.
//
// The top-2 is found in two steps: the stream keeps, branch-free, the lane's two best 8-element
// vectors ranked by (vector max desc, vector index asc) — a per-element insert would diverge at
// warp level on almost every vector (profiles/r01_ncu_rowstats.md: 27 issued instructions per
// element) — and the warp then rescans only the two best vectors of the whole tile. This is
// exact: the best element lies in the best vector; the second-best element is either in that
// vector too or it is the maximum of its own vector, which then ranks second. Vectors are
// contiguous and ids grow with the vector index, so a tie keeps the earlier vector, matching the
// Prediction tie rule.
constexpr float kSlack = 16.f;
#ifndef WS_K3_SLOTS
#define WS_K3_SLOTS 2
#endif
constexpr int kSlots = WS_K3_SLOTS;  // accumulator slots in use (alternate chunks)

struct Lane {
  float m;        // log2-domain reference of (z, s)
  float thr;      // raw-logit threshold that moves the reference: m / cl + kSlack / cl
  float2 z2[2], s2[2];  // (z, s) as even/odd-element lanes (packed f32x2 math), two slots
                        // (alternate chunks) so consecutive chunks' add chains overlap
  float bm1, bm2;  // the two best chunks' (clamped) maxima and first element ids
  std::uint32_t bi1, bi2;
};

// MUFU.EX2 directly (rel. error ~2^-22): the per-element exponential of the streaming pass.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// A lane's contiguous chunk of 2W = 8 bf16 logits (one 16-byte load).
template <int W>
struct Chunk {
  std::uint32_t w[W];
};

// streaming load (evict-first: read once; the tile's rescan of its two best chunks right after
// is the only re-read)
template <int W>
__device__ __forceinline__ Chunk<W> ld_chunk(const std::uint32_t* p) {
  static_assert(W == 4, "16-byte chunks");
  Chunk<W> c;
  asm volatile("ld.global.cs.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3])
               : "l"(p));
  return c;
}

template <int W, int S>
__device__ __forceinline__ void absorb(Lane& a, const Chunk<W>& q, std::uint32_t id0, float cl, float slack_x) {
  // -inf logits (masked vocabulary) are clamped to -2^100 for the softmax sums: their weight is
  // still exactly 0, but e*d stays 0 instead of 0*(-inf) = NaN (entropy_of's 0 ln 0 = 0,
  // oracle.hpp:21-33). One packed bf16x2 max per two elements; the warp's top-2 rescan reads
  // the raw chunk, so a -inf second candidate keeps its value.
  std::uint32_t wd[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&q.w[j]);
    h = __hmax2(h, __floats2bfloat162_rn(kFloor, kFloor));
    wd[j] = *reinterpret_cast<const std::uint32_t*>(&h);
  }
  // bf16 -> f32 is a 16-bit shift: one integer op per element (low half: shift, high: mask)
  float x[2 * W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    x[2 * j] = __uint_as_float(wd[j] << 16);
    x[2 * j + 1] = __uint_as_float(wd[j] & 0xFFFF0000u);
  }
  // chunk max as a tree (short dependency chain)
  float t[W];
#pragma unroll
  for (int j = 0; j < W; ++j) t[j] = fmaxf(x[2 * j], x[2 * j + 1]);
#pragma unroll
  for (int w = W / 2; w > 0; w /= 2)
#pragma unroll
    for (int j = 0; j < w; ++j) t[j] = fmaxf(t[j], t[j + w]);
  const float mx = t[0];
  if (mx > a.thr) {  // move the reference (rare: the first chunk, then jumps of > kSlack)
    const float lm = mx * cl, dm = a.m - lm, f = exp2f(dm);
    const float2 f2 = make_float2(f, f), d2 = make_float2(dm, dm);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      a.s2[u] = __fmul2_rn(f2, __ffma2_rn(a.z2[u], d2, a.s2[u]));
      a.z2[u] = __fmul2_rn(a.z2[u], f2);
    }
    a.m = lm;
    a.thr = mx + slack_x;
  }
  // branch-free two-best-chunks update
  const bool p1 = mx > a.bm1, p2 = mx > a.bm2;
  a.bm2 = p1 ? a.bm1 : (p2 ? mx : a.bm2);
  a.bi2 = p1 ? a.bi1 : (p2 ? id0 : a.bi2);
  a.bm1 = p1 ? mx : a.bm1;
  a.bi1 = p1 ? id0 : a.bi1;
  // two elements per packed FFMA2/FADD2 (sm_100): 1.5 instead of 3 FP32 issues per element; the
  // chunk's z as a tree, then one add into the slot
  const float2 c2 = make_float2(cl, cl), n2 = make_float2(-a.m, -a.m);
  float2 e[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    const float2 d = __ffma2_rn(make_float2(x[2 * j], x[2 * j + 1]), c2, n2);
    e[j] = make_float2(ex2(d.x), ex2(d.y));
    a.s2[S] = __ffma2_rn(e[j], d, a.s2[S]);
  }
#pragma unroll
  for (int w = W / 2; w > 0; w /= 2)
#pragma unroll
    for (int j = 0; j < w; ++j) e[j] = __fadd2_rn(e[j], e[j + w]);
  a.z2[S] = __fadd2_rn(a.z2[S], e[0]);
}

// one element (scalar path, or a vector row's tail): statistics and an exact top-2 insert
__device__ __forceinline__ void absorb1(float& m, float& z, float& s, Top2& t, float x, std::uint32_t id, float cl) {
  const float l = fmaxf(x, kFloor) * cl;  // -inf → a finite floor (see absorb)
  if (l > m) {
    if (z > 0.f) {
      const float f = exp2f(m - l);
      s = f * (s + z * (m - l));
      z *= f;
    }
    m = l;
  }
  const float d = l - m;
  const float e = exp2f(d);
  z += e;
  s = fmaf(e, d, s);
  insert(t, x, id);
}

struct Partial {
  float m, z, s, v1, v2;
  std::uint32_t i1, i2, pad;
};

constexpr std::uint32_t kMaxRows = 65535;
constexpr std::size_t kTicketBytes = 2 * 65536 * sizeof(std::uint32_t);

__device__ void finalize(const Stats& a, float cl, std::uint32_t vocab, ws_pred* pred, RowStats* st,
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
  p.id[0] = a.t.i1;
  p.id[1] = vocab >= 2 ? a.t.i2 : 0u;
  p.pad = 0;
  p.prob[0] = static_cast<double>(exp2f(fmaf(a.t.v1, cl, -a.m)) / a.z);
  p.prob[1] = vocab >= 2 ? static_cast<double>(exp2f(fmaf(a.t.v2, cl, -a.m)) / a.z) : 0.0;
  p.entropy = static_cast<double>(h);
  *pred = p;
  if (st) *st = RowStats{a.m, a.z, cl, h};
}

// The lane's chunks of a tile (chunks lane, lane+32, ... of 2W elements) in batches of four:
// four loads in flight, then four absorbs alternating the two accumulator slots. (Measured
// against register double-buffering, 32-byte chunks and a per-warp TMA ring of shared-memory
// stages: all slower at the verify batch — profiles/r02_ncu_k3.md; the kernel is bound by
// issue latency at the occupancy its registers allow, not by bytes in flight.)
template <int W>
__device__ __forceinline__ void stream_chunks(Lane& a, const __nv_bfloat16* __restrict__ x, std::uint32_t lo,
                                              std::uint32_t nch, float cl, std::uint32_t lane) {
  constexpr std::uint32_t E = 2 * W;
#ifndef WS_K3_B
#define WS_K3_B 4
#endif
  constexpr int B = WS_K3_B;
  const float slack_x = kSlack / cl;
  const std::uint32_t* base = reinterpret_cast<const std::uint32_t*>(x + lo) + lane * W;
  const int nj = lane < nch ? static_cast<int>((nch - lane + 31) / 32) : 0;
  auto id = [&](int j) { return lo + E * (lane + 32u * static_cast<std::uint32_t>(j)); };
  int j = 0;
  for (; j + B <= nj; j += B) {
    Chunk<W> q[B];
#pragma unroll
    for (int u = 0; u < B; ++u) q[u] = ld_chunk<W>(base + (j + u) * 32 * W);
#pragma unroll
    for (int u = 0; u < B; ++u) {
      if ((u & 1) && kSlots > 1)
        absorb<W, 1>(a, q[u], id(j + u), cl, slack_x);
      else
        absorb<W, 0>(a, q[u], id(j + u), cl, slack_x);
    }
  }
  for (; j < nj; ++j) absorb<W, 0>(a, ld_chunk<W>(base + j * 32 * W), id(j), cl, slack_x);
}

__device__ __forceinline__ void init(Lane& a) {
  a.m = -3.0e38f;  // finite: the first rescale multiplies z = s = 0 by exp2(-huge) = 0
  a.thr = -INFINITY;
  a.z2[0] = a.z2[1] = a.s2[0] = a.s2[1] = make_float2(0.f, 0.f);
  a.bm1 = a.bm2 = -INFINITY;
  a.bi1 = a.bi2 = kNone;
}

// The end of a tile [lo, hi) of row x whose first `streamed` elements went through the lanes'
// chunk streams (state a; E elements per chunk) and whose rest are absorbed element-wise here:
// the warp's statistics, identical in every lane.
template <std::uint32_t E>
__device__ __forceinline__ Stats tile_finish(const Lane& a, const __nv_bfloat16* __restrict__ x, std::uint32_t lo,
                                             std::uint32_t hi, std::uint32_t streamed, float cl, std::uint32_t lane) {
  float m = -INFINITY, z = 0.f, s = 0.f;
  Top2 tail;
  init(tail);
  Top2 cand;
  init(cand);
  if constexpr (E > 0) {
    m = a.bi1 == kNone ? -INFINITY : a.m;
    z = (a.z2[0].x + a.z2[0].y) + (a.z2[1].x + a.z2[1].y);  // fold (same reference) before the tail
    s = (a.s2[0].x + a.s2[0].y) + (a.s2[1].x + a.s2[1].y);
    // the tile's two best chunks (xor butterfly over the lanes' two best)
    Top2 b{a.bm1, a.bm2, a.bi1, a.bi2};
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) b = merge2(b, shfl_xor(b, off));
    // rescan them: lanes [0, E) read the best chunk's elements, [E, 2E) the second's (raw
    // values, L2 hits: this warp streamed them a moment ago)
    const std::uint32_t vid = lane < E ? b.i1 : (lane < 2 * E ? b.i2 : kNone);
    if (vid != kNone) {
      const std::uint32_t i = vid + (lane & (E - 1));
      cand.v1 = __bfloat162float(x[i]);
      cand.i1 = i;
    }
  }
  for (std::uint32_t t = lo + streamed + lane; t < hi; t += 32) absorb1(m, z, s, tail, __bfloat162float(x[t]), t, cl);
  cand = merge2(cand, tail);
  // (m, z, s): the warp max first, then every lane rescales to it once, so the butterfly levels
  // are plain sums (fixed order → deterministic)
  float mw = m;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, off));
  if (z > 0.f) {
    const float f = exp2f(m - mw);
    s = f * (s + z * (m - mw));
    z *= f;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    z += __shfl_xor_sync(0xffffffffu, z, off);
    s += __shfl_xor_sync(0xffffffffu, s, off);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) cand = merge2(cand, shfl_xor(cand, off));
  return Stats{mw, z, s, cand};
}

// Statistics of one tile [lo, hi) of row x (vw: chunk words — 4: 16-byte chunks, 0: element-wise
// for rows that are not 16-byte aligned).
template <int vw>
__device__ __forceinline__ Stats tile_stats(const __nv_bfloat16* __restrict__ x, std::uint32_t lo, std::uint32_t hi,
                                            float cl, std::uint32_t lane) {
  constexpr std::uint32_t E = 2 * vw;
  Lane a;
  init(a);
  std::uint32_t streamed = 0;
  if constexpr (vw != 0) {
    const std::uint32_t nch = (hi - lo) / E;
    stream_chunks<vw>(a, x, lo, nch, cl, lane);
    streamed = nch * E;
  }
  return tile_finish<E>(a, x, lo, hi, streamed, cl, lane);
}

struct RowArgs {
  const __nv_bfloat16* logits;
  std::uint32_t vocab, ld;
  float cl;
  std::uint32_t tiles, items, per_warp;
  ws_pred* out_pred;
  RowStats* out_stats;
  Partial* partials;
  std::uint32_t* row_ticket;
  std::uint32_t k;
  const std::uint32_t* cand;
  ws_verify_out* vout;
  std::uint32_t* req_ticket;
  const std::int32_t* forced;
};

// The warp's tiles of one row form a segment: their partials are published with one fence and
// one ticket add (amortised over the segment); the warp that completes the row's count merges
// all of its tile partials, always in the same fixed tree, finalises the row and, with the
// verify epilogue, walks the request once its last row is done. r: the segment's last tile.
__device__ __forceinline__ void finish_segment(const RowArgs& g, Stats r, std::uint32_t row, std::uint32_t seg_n,
                                               std::uint32_t lane) {
  if (g.tiles > 1) {
    std::uint32_t t = 0;
    if (lane == 0) {
      __threadfence();
      t = atomicAdd(&g.row_ticket[row], seg_n);
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t + seg_n != g.tiles) return;
    __threadfence();
    // lane q merges tiles q, q+32, ... in order, then a fixed xor tree over the lanes
    Stats acc{-INFINITY, 0.f, 0.f, {-INFINITY, -INFINITY, kNone, kNone}};
    for (std::uint32_t q = lane; q < g.tiles; q += 32) {
      const Partial* p = &g.partials[row * g.tiles + q];
      Stats b{__ldcg(&p->m), __ldcg(&p->z), __ldcg(&p->s), {__ldcg(&p->v1), __ldcg(&p->v2), __ldcg(&p->i1),
                                                            __ldcg(&p->i2)}};
      acc = merge(acc, b);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      Stats b{__shfl_xor_sync(0xffffffffu, acc.m, off), __shfl_xor_sync(0xffffffffu, acc.z, off),
              __shfl_xor_sync(0xffffffffu, acc.s, off), shfl_xor(acc.t, off)};
      acc = merge(acc, b);
    }
    r = acc;
    if (lane == 0) g.row_ticket[row] = 0;  // self-reset for the next launch
  }
  if (lane != 0) return;
  {  // re-reference (z, s) from the lazy reference to the row's true maximum (RowStats.m2)
    const float mt = fmaxf(r.t.v1, kFloor) * g.cl;
    if (r.z > 0.f && mt != r.m) {
      const float f = exp2f(r.m - mt);
      r.s = f * (r.s + r.z * (r.m - mt));
      r.z *= f;
      r.m = mt;
    }
  }
  finalize(r, g.cl, g.vocab, &g.out_pred[row], g.out_stats ? &g.out_stats[row] : nullptr,
           g.forced ? g.forced[row] : -1);

  if (g.cand) {  // K4 greedy epilogue: the last finished row of the request runs the walk
    const std::uint32_t req = row / (g.k + 1);
    __threadfence();
    const std::uint32_t t = atomicAdd(&g.req_ticket[req], 1u);
    if (t != g.k) return;
    __threadfence();
    g.req_ticket[req] = 0;
    const ws_pred* rows = g.out_pred + static_cast<std::size_t>(req) * (g.k + 1);
    std::uint32_t acc = 0;
    while (acc < g.k && __ldcg(&rows[acc].id[0]) == g.cand[static_cast<std::size_t>(req) * g.k + acc]) ++acc;
    ws_verify_out o;
    o.accepted = acc;
    o.bonus = __ldcg(&rows[acc].id[0]);
    o.final_entropy = __ldcg(&rows[acc].entropy);
    g.vout[req] = o;
  }
}

// 4 CTAs of 8 warps per SM (<= 64 registers): measured best against 1-3 (profiles/r02_ncu_k3.md)
#ifndef WS_K3_MINB
#define WS_K3_MINB 4
#endif
template <int vw>
__global__ void __launch_bounds__(kThreads, WS_K3_MINB) row_stats_kernel(const __grid_constant__ RowArgs g) {
  pdl_trigger();
  pdl_wait();  // inputs come from the previous kernel of the chain
  const std::uint32_t lane = threadIdx.x & 31;
  const std::uint32_t gw = blockIdx.x * kWarps + threadIdx.x / 32;
  const std::uint32_t first = gw * g.per_warp;
  const std::uint32_t last = min(g.items, first + g.per_warp);
  for (std::uint32_t it = first; it < last;) {
    __syncwarp();  // lane 0 may still be in the previous row's epilogue
    const std::uint32_t row = it / g.tiles;
    const std::uint32_t seg_end = min(last, (row + 1) * g.tiles), seg_n = seg_end - it;
    const __nv_bfloat16* x = g.logits + static_cast<std::size_t>(row) * g.ld;
    Stats r;
    for (; it < seg_end; ++it) {
      const std::uint32_t tile = it - row * g.tiles;
      const std::uint32_t lo = tile * kRowTile, hi = min(g.vocab, lo + kRowTile);
      r = tile_stats<vw>(x, lo, hi, g.cl, lane);
      if (g.tiles > 1 && lane == 0)
        g.partials[row * g.tiles + tile] = Partial{r.m, r.z, r.s, r.t.v1, r.t.v2, r.t.i1, r.t.i2, 0};
    }
    finish_segment(g, r, row, seg_n, lane);
  }
}

// resident warps of a row-stats kernel on a device (cached per device and kernel)
template <typename K>
std::uint32_t resident_warps(K kernel, int threads, std::atomic<int>* cache) {
  int dev = 0;
  WS_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) dev = 0;
  int w = cache[dev].load(std::memory_order_relaxed);
  if (w == 0) {
    int sms = 0, blocks = 0;
    WS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    WS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, threads, 0));
    w = sms * (blocks > 0 ? blocks : 1) * (threads / 32);
    cache[dev].store(w, std::memory_order_relaxed);
  }
  return static_cast<std::uint32_t>(w);
}

// balanced persistent grid: every warp reduces per_warp consecutive tiles
template <typename K>
void launch_balanced(K kernel, int threads, std::atomic<int>* cache, RowArgs g, std::uint32_t rows,
                     cudaStream_t stream) {
  g.items = rows * g.tiles;
  const std::uint32_t slots = resident_warps(kernel, threads, cache);
  g.per_warp = (g.items + slots - 1) / slots;
  const std::uint32_t warps = (g.items + g.per_warp - 1) / g.per_warp;
  const std::uint32_t wpc = static_cast<std::uint32_t>(threads / 32);
  launch_pdl(kernel, dim3((warps + wpc - 1) / wpc), dim3(threads), 0, stream, 1, g);
}

}  // namespace

std::size_t rowstats_workspace_bytes(std::uint32_t rows, std::uint32_t vocab, std::uint32_t n_req) {
  const std::uint32_t tiles = (vocab + kRowTile - 1) / kRowTile;
  (void)n_req;
  return kTicketBytes + static_cast<std::size_t>(rows) * tiles * sizeof(Partial) + 64;
}

void row_stats_bf16(const void* logits, std::uint32_t rows, std::uint32_t vocab, std::uint32_t ld, float inv_temp,
                    ws_pred* out_pred, RowStats* out_stats, void* workspace, std::uint32_t n_req, std::uint32_t k,
                    const std::uint32_t* cand, ws_verify_out* verify_out, cudaStream_t stream,
                    const std::int32_t* forced) {
  if (rows == 0) return;
  if (!logits || !out_pred || vocab == 0 || ld < vocab) throw std::invalid_argument("row_stats: bad argument");
  if (!(inv_temp > 0.f)) throw std::invalid_argument("row_stats: temperature must be > 0");
  if (cand && (rows != n_req * (k + 1) || !verify_out)) throw std::invalid_argument("row_stats: verify shape");
  const std::uint32_t tiles = (vocab + kRowTile - 1) / kRowTile;
  if (tiles > 1 || cand) {
    if (!workspace) throw std::invalid_argument("row_stats: workspace required");
  }
  if (rows > kMaxRows || n_req > kMaxRows) throw std::invalid_argument("row_stats: too many rows");
  if (static_cast<std::uint64_t>(rows) * tiles > 0xFFFFFFFFull) throw std::invalid_argument("row_stats: too large");
  // Fixed layout whatever the row count: [row tickets | request tickets | partials]. The tickets
  // self-reset, so they must not move between launches of different sizes.
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  std::uint32_t* row_ticket = reinterpret_cast<std::uint32_t*>(ws);
  std::uint32_t* req_ticket = row_ticket + kMaxRows;
  Partial* partials = reinterpret_cast<Partial*>(ws + kTicketBytes);
  // 16-byte chunks when every row starts 16-byte aligned, else element-wise
  const bool vec = reinterpret_cast<std::uintptr_t>(logits) % 16 == 0 && ld % 8 == 0;
  RowArgs g{static_cast<const __nv_bfloat16*>(logits), vocab, ld, inv_temp * kLog2e, tiles, 0, 0, out_pred,
            out_stats, partials, row_ticket, k, cand, verify_out, req_ticket, forced};
  static std::atomic<int> c4[64], c0[64];
  if (vec)
    launch_balanced(row_stats_kernel<4>, kThreads, c4, g, rows, stream);
  else
    launch_balanced(row_stats_kernel<0>, kThreads, c0, g, rows, stream);
}

}  // namespace wsb
