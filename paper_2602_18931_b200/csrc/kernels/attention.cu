// K2 — grouped GQA attention of the verify / draft forward over the KV slot pool.
//
// One CTA per (group, kv head). A group is the set of rows of one request that share a
// context: a linear committed prefix (prefix_len consecutive slots from prefix_slot, visible to
// every row) followed by explicit "extra" slots (new rows, tree ancestors) whose visibility is
// causal (verify rows, catch-up prefill: row j sees extra[0 .. E-n+j]) or given by a per-row
// 64-bit mask (the worker's tree leaves: each leaf sees its own ancestor chain). Every K/V tile
// is read from HBM once per (group, kv head) and reused by all n_rows x (n_q / n_kv) query
// vectors: a request's k+1 verify rows and all its draft leaves share one pass.
//
// Math on the tensor cores with warp-level mma.sync m16n8k16 (bf16 in, fp32 accumulate): each
// warp owns 16 query vectors; S = Q·Kᵀ per 32-position tile (ldmatrix from a 128-byte-XOR-
// swizzled smem tile), online softmax on the accumulator fragments (exp2 domain), then P·V with
// the S fragments re-packed as the A operand and V loaded by ldmatrix.trans. K/V tiles are
// double-buffered with cp.async so the next tile's HBM reads overlap this tile's math. The
// kernel is HBM-bound on KV bytes; tensor-core throughput is not the limiter at these shapes.
#include <cuda_bf16.h>

#include <mutex>
#include <stdexcept>

#include "cuda_check.hpp"
#include "pdl.cuh"
#include "llama_ops.cuh"

namespace wsb {

namespace {

constexpr int kTile = 32;  // positions per K/V tile

__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ void ldsm_x4(std::uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(std::uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const std::uint32_t (&a)[4], std::uint32_t b0,
                                         std::uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ std::uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<std::uint32_t*>(&v);
}

// Tile of HD-wide bf16 rows, 16-byte chunks XOR-swizzled by (row & 7) (conflict-free ldmatrix).
template <int HD>
__device__ __forceinline__ int swz(int row, int chunk) {
  constexpr int C = HD / 8;
  return row * C + (chunk ^ (row & 7));
}

// VW x KS warps per CTA: VW vector warps (16 query vectors each) times KS key slices. Slice
// ks streams the K/V tiles t = ks, ks + KS, ... through its own STAGES-deep cp.async ring, so a
// CTA keeps KS * (STAGES - 1) tiles in flight; at the end of a pass the slices' softmax states
// merge in slice order. KS is fixed per head dim (never chosen from the group), so a row's
// result is the same in any group of any batch (batch invariance: speculative stream == greedy
// stream); STAGES only changes how far ahead the loads run.
template <int HD, int VW, int KS, int STAGES>
__global__ void __launch_bounds__(32 * VW * KS) attn_mma_kernel(const __nv_bfloat16* __restrict__ q,
                                                                 const __nv_bfloat16* __restrict__ kp,
                                                                 const __nv_bfloat16* __restrict__ vp,
                                                                 const AttnGroup* __restrict__ groups,
                                                                 const std::int32_t* __restrict__ extra,
                                                                 const unsigned long long* __restrict__ row_mask,
                                                                 int nq, int nkv, float scale_log2,
                                                                 __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();  // inputs come from the previous kernel of the chain
  constexpr int C = HD / 8;   // 16-byte chunks per row
  constexpr int KST = HD / 16; // k16 steps for S = Q·Kᵀ
  constexpr int NT = HD / 8;  // n8 tiles of the output
  constexpr int kSliceThreads = 32 * VW;
  constexpr int kVecPerPass = 16 * VW;
  constexpr int kMergeFloats = 4 + 4 * NT;  // m_lo, m_hi, l_lo, l_hi, o[NT][4] per lane
  static_assert((KS - 1) * VW * 32 * kMergeFloats * 4 <= KS * STAGES * 2 * kTile * C * 16, "merge scratch");
  static_assert(STAGES >= 2, "ring depth");
  // dynamic smem: Q tile, then [slice][stage][K | V] tiles (launch_attn's kSmem)
  extern __shared__ __align__(128) uint4 smem_dyn[];
  uint4* sQ = smem_dyn;
  uint4* sKV0 = smem_dyn + kVecPerPass * C;
  auto kv_tile = [&](int slice, int buf, int which) {
    return sKV0 + ((slice * STAGES + buf) * 2 + which) * (kTile * C);
  };

  const AttnGroup g = groups[blockIdx.x];
  const int kvh = blockIdx.y;
  const int G = nq / nkv;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int vw = warp % VW, ks = warp / VW;
  const int st = threadIdx.x % kSliceThreads;  // thread index within the slice
  const int nvec = g.n_rows * G;
  const int ctx = g.prefix_len + g.extra_len;
  const std::size_t slot_stride = static_cast<std::size_t>(nkv) * HD;
  // Causal groups: this entry's rows see keys up to the last row's own position, so the tiles past
  // it are masked for every row of the entry and are skipped (a fully masked tile leaves the
  // online-softmax state unchanged). Prompt-prefill groups of 127 rows come as many entries, the
  // early ones seeing only a fraction of the keys.
  int ctx_eff = ctx;
#ifndef WS_ATTN_SKIP
#define WS_ATTN_SKIP 1
#endif
  if (WS_ATTN_SKIP && !g.masked) {
    const int v_last = min(nvec, g.pad + 16 * VW) - 1;
    if (v_last >= 0) ctx_eff = min(ctx, g.prefix_len + g.extra_len - g.n_rows + v_last / G + 1);
  }
  const int n_tiles = (ctx_eff + kTile - 1) / kTile;
  const int n_iter = (n_tiles + KS - 1) / KS;

  auto slot_of = [&](int p) -> int {
    return p < g.prefix_len ? g.prefix_slot + p : (p < ctx ? extra[g.extra_off + p - g.prefix_len] : -1);
  };
  auto load_tile = [&](int t, int buf) {  // by the threads of this slice
    if (t >= n_tiles) return;
    for (int i = st; i < kTile * C; i += kSliceThreads) {
      const int r = i / C, c = i % C;
      const int s = slot_of(t * kTile + r);
      const std::size_t base = static_cast<std::size_t>(s < 0 ? 0 : s) * slot_stride + static_cast<std::size_t>(kvh) * HD;
      cp_async16(kv_tile(ks, buf, 0) + swz<HD>(r, c), kp + base + c * 8, s >= 0);
      cp_async16(kv_tile(ks, buf, 1) + swz<HD>(r, c), vp + base + c * 8, s >= 0);
    }
  };

  // one pass: the entry's query vectors [g.pad, g.pad + 16 VW) (large groups come as several
  // entries — attention_vectors_per_cta())
  for (int pass0 = g.pad; pass0 < nvec && pass0 < g.pad + kVecPerPass; pass0 += kVecPerPass) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < STAGES - 1; ++i) {  // ring prologue: this slice's first STAGES-1 tiles
      if (i < n_iter) load_tile(i * KS + ks, i);
      if (i == 0) {
        // Q for this pass, in the first group so its latency overlaps the first K/V tiles:
        // vector v -> (row j = v / G, head kvh*G + v % G), zero-filled past nvec
        for (int e = threadIdx.x; e < kVecPerPass * C; e += 32 * VW * KS) {
          const int vv = e / C, c = e % C, v = pass0 + vv;
          const bool ok = v < nvec;
          const int j = ok ? v / G : 0, h = ok ? kvh * G + v % G : 0;
          cp_async16(&sQ[swz<HD>(vv, c)], q + (static_cast<std::size_t>(g.row0 + j) * nq + h) * HD + c * 8, ok);
        }
      }
      cp_async_commit();
    }
    __syncthreads();

    // this warp's 16 query vectors; the thread's two accumulator rows
    const int wv0 = pass0 + vw * 16;
    const bool warp_live = wv0 < nvec;
    const int r_lo = lane / 4, r_hi = r_lo + 8;
    int last_lo = -1, last_hi = -1;
    unsigned long long m_lo = 0ull, m_hi = 0ull;
    bool live_lo = false, live_hi = false;
    {
      const int v_lo = wv0 + r_lo, v_hi = wv0 + r_hi;
      live_lo = v_lo < nvec;
      live_hi = v_hi < nvec;
      if (live_lo) {
        const int j = v_lo / G;
        if (g.masked) m_lo = row_mask[g.row0 + j]; else last_lo = g.extra_len - g.n_rows + j;
      }
      if (live_hi) {
        const int j = v_hi / G;
        if (g.masked) m_hi = row_mask[g.row0 + j]; else last_hi = g.extra_len - g.n_rows + j;
      }
    }
    // Q fragments (A operand) for all k16 steps: held in registers for hd 64; for hd 128 they
    // are re-read from smem per tile (32 fewer registers → one more CTA per SM)
    constexpr bool kQReg = HD <= 64;
    std::uint32_t qa[kQReg ? KST : 1][4];
    auto q_frag = [&](int kk, std::uint32_t (&f)[4]) {
      // lanes 0-15 rows 0-15 chunk 2kk, lanes 16-31 rows 0-15 chunk 2kk+1
      const int row = vw * 16 + (lane % 16);
      const int chunk = 2 * kk + lane / 16;
      ldsm_x4(f, &sQ[swz<HD>(row, chunk)]);
    };
    // (hd 64: the fragments are read once Q has landed, at the first tile)
    float o[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
    float mx_lo = -INFINITY, mx_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

    for (int it = 0; it < n_iter; ++it) {
      const int t = it * KS + ks;  // this slice's tile
      const int buf = it % STAGES;
      {  // refill the stage consumed last iteration; one (possibly empty) group per iteration
        const int ahead = it + STAGES - 1;
        if (ahead < n_iter) load_tile(ahead * KS + ks, ahead % STAGES);
        cp_async_commit();
        asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
      }
      __syncthreads();
      if constexpr (kQReg) {
        if (it == 0 && warp_live) {  // Q landed with the first group
#pragma unroll
          for (int kk = 0; kk < KST; ++kk) q_frag(kk, qa[kk]);
        }
      }
      if (warp_live && t < n_tiles) {
        // S = Q·Kᵀ over 32 positions: 4 n8 tiles
        float s[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KST; ++kk) {
          std::uint32_t qf[4];
          if constexpr (kQReg) {
#pragma unroll
            for (int e = 0; e < 4; ++e) qf[e] = qa[kk][e];
          } else {
            q_frag(kk, qf);
          }
#pragma unroll
          for (int np = 0; np < 2; ++np) {  // pairs of n8 tiles (16 positions) per ldmatrix.x4
            std::uint32_t kb[4];
            // matrices: (pos 0-7, k lo), (pos 0-7, k hi), (pos 8-15, k lo), (pos 8-15, k hi)
            const int pos = np * 16 + (lane % 8) + ((lane / 16) * 8);
            const int chunk = 2 * kk + ((lane / 8) & 1);
            ldsm_x4(kb, kv_tile(ks, buf, 0) + swz<HD>(pos, chunk));
            mma16816(s[2 * np], qf, kb[0], kb[1]);
            mma16816(s[2 * np + 1], qf, kb[2], kb[3]);
          }
        }
        // visibility + scale (exp2 domain)
        const int p0 = t * kTile;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int p = p0 + nt * 8 + (lane % 4) * 2 + (e & 1);
            const bool hi = e >= 2;
            bool vis = p < ctx && (hi ? live_hi : live_lo);
            if (vis && p >= g.prefix_len) {
              const int x = p - g.prefix_len;
              vis = g.masked ? (((hi ? m_hi : m_lo) >> (x & 63)) & 1ull) != 0ull : x <= (hi ? last_hi : last_lo);
            }
            s[nt][e] = vis ? s[nt][e] * scale_log2 : -INFINITY;
          }
        // online softmax per row (quad reductions)
        float tmax_lo = -INFINITY, tmax_hi = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          tmax_lo = fmaxf(tmax_lo, fmaxf(s[nt][0], s[nt][1]));
          tmax_hi = fmaxf(tmax_hi, fmaxf(s[nt][2], s[nt][3]));
        }
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
          tmax_lo = fmaxf(tmax_lo, __shfl_xor_sync(0xffffffffu, tmax_lo, off));
          tmax_hi = fmaxf(tmax_hi, __shfl_xor_sync(0xffffffffu, tmax_hi, off));
        }
        const float nmax_lo = fmaxf(mx_lo, tmax_lo), nmax_hi = fmaxf(mx_hi, tmax_hi);
        const float base_lo = nmax_lo == -INFINITY ? 0.f : nmax_lo;
        const float base_hi = nmax_hi == -INFINITY ? 0.f : nmax_hi;
        const float corr_lo = exp2f(mx_lo - base_lo), corr_hi = exp2f(mx_hi - base_hi);
        mx_lo = nmax_lo;
        mx_hi = nmax_hi;
        float rs_lo = 0.f, rs_hi = 0.f;
        std::uint32_t pa[2][4];  // P as the A operand: 2 k16 steps of 16 positions
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const float p0v = exp2f(s[nt][0] - base_lo), p1v = exp2f(s[nt][1] - base_lo);
          const float p2v = exp2f(s[nt][2] - base_hi), p3v = exp2f(s[nt][3] - base_hi);
          rs_lo += p0v + p1v;
          rs_hi += p2v + p3v;
          const int kk = nt / 2, half = nt % 2;
          pa[kk][half * 2 + 0] = pack_bf16(p0v, p1v);
          pa[kk][half * 2 + 1] = pack_bf16(p2v, p3v);
        }
        rs_lo += __shfl_xor_sync(0xffffffffu, rs_lo, 1);
        rs_lo += __shfl_xor_sync(0xffffffffu, rs_lo, 2);
        rs_hi += __shfl_xor_sync(0xffffffffu, rs_hi, 1);
        rs_hi += __shfl_xor_sync(0xffffffffu, rs_hi, 2);
        l_lo = l_lo * corr_lo + rs_lo;
        l_hi = l_hi * corr_hi + rs_hi;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          o[nt][0] *= corr_lo;
          o[nt][1] *= corr_lo;
          o[nt][2] *= corr_hi;
          o[nt][3] *= corr_hi;
        }
        // O += P·V: A = P (16 x 32 positions), B = V (32 positions x HD) via ldmatrix.trans
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
          for (int np = 0; np < NT / 2; ++np) {  // pairs of n8 output tiles (16 dims)
            std::uint32_t vb[4];
            // matrices: (pos lo 0-7, dims np*16+0-7), (pos 8-15, same), (pos 0-7, dims +8), (pos 8-15, +8)
            const int pos = kk * 16 + (lane % 8) + ((lane / 8) & 1) * 8;
            const int chunk = 2 * np + (lane / 16);
            ldsm_x4_t(vb, kv_tile(ks, buf, 1) + swz<HD>(pos, chunk));
            mma16816(o[2 * np], pa[kk], vb[0], vb[1]);
            mma16816(o[2 * np + 1], pa[kk], vb[2], vb[3]);
          }
        }
      }
      __syncthreads();  // stage `buf` of every slice is refilled next iteration
    }
    // merge the KS slices' states (slice order, in the K/V scratch), then normalise + store
    if constexpr (KS > 1) {
      float* scratch = reinterpret_cast<float*>(sKV0);
      if (ks > 0 && warp_live) {
        float* my = scratch + ((static_cast<std::size_t>(ks - 1) * VW + vw) * 32 + lane) * kMergeFloats;
        my[0] = mx_lo;
        my[1] = mx_hi;
        my[2] = l_lo;
        my[3] = l_hi;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) my[4 + nt * 4 + e] = o[nt][e];
      }
      __syncthreads();
      if (ks == 0 && warp_live) {
#pragma unroll 1
        for (int sl = 1; sl < KS; ++sl) {
          const float* ot = scratch + ((static_cast<std::size_t>(sl - 1) * VW + vw) * 32 + lane) * kMergeFloats;
          const float om_lo = ot[0], om_hi = ot[1];
          const float nm_lo = fmaxf(mx_lo, om_lo), nm_hi = fmaxf(mx_hi, om_hi);
          const float b_lo = nm_lo == -INFINITY ? 0.f : nm_lo, b_hi = nm_hi == -INFINITY ? 0.f : nm_hi;
          const float ca_lo = exp2f(mx_lo - b_lo), cb_lo = exp2f(om_lo - b_lo);
          const float ca_hi = exp2f(mx_hi - b_hi), cb_hi = exp2f(om_hi - b_hi);
          l_lo = l_lo * ca_lo + ot[2] * cb_lo;
          l_hi = l_hi * ca_hi + ot[3] * cb_hi;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            o[nt][0] = o[nt][0] * ca_lo + ot[4 + nt * 4 + 0] * cb_lo;
            o[nt][1] = o[nt][1] * ca_lo + ot[4 + nt * 4 + 1] * cb_lo;
            o[nt][2] = o[nt][2] * ca_hi + ot[4 + nt * 4 + 2] * cb_hi;
            o[nt][3] = o[nt][3] * ca_hi + ot[4 + nt * 4 + 3] * cb_hi;
          }
          mx_lo = nm_lo;
          mx_hi = nm_hi;
        }
      }
    }
    // epilogue: normalise and store this warp's rows (slice 0 holds the merged state)
    if (warp_live && ks == 0) {
      const float inv_lo = l_lo > 0.f ? 1.f / l_lo : 0.f, inv_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int v = wv0 + (half ? r_hi : r_lo);
        if (v >= nvec) continue;
        const int j = v / G, h = kvh * G + v % G;
        __nv_bfloat16* os = out + (static_cast<std::size_t>(g.row0 + j) * nq + h) * HD;
        const float inv = half ? inv_hi : inv_lo;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int d = nt * 8 + (lane % 4) * 2;
          *reinterpret_cast<__nv_bfloat162*>(os + d) =
              __floats2bfloat162_rn(o[nt][half * 2] * inv, o[nt][half * 2 + 1] * inv);
        }
      }
    }
  }
}

}  // namespace

template <int HD, int VW, int KS, int STAGES>
void launch_attn(const void* q, const void* k_pool, const void* v_pool, const AttnGroup* groups, int n_groups,
                 const std::int32_t* extra, const unsigned long long* row_mask, const AttnShape& s, float sl2,
                 void* out, cudaStream_t st) {
  if (n_groups <= 0) return;
  constexpr int C = HD / 8;
  constexpr int kSmem = (16 * VW * C + KS * STAGES * 2 * kTile * C) * 16;
  static std::atomic<std::uint32_t> attr_done{0};
  once_per_device(attr_done, [] {
    WS_CUDA(cudaFuncSetAttribute(attn_mma_kernel<HD, VW, KS, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmem));
  });
  launch_pdl(attn_mma_kernel<HD, VW, KS, STAGES>, dim3(n_groups, s.n_kv), dim3(32 * VW * KS), kSmem, st, 1,
             static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k_pool),
             static_cast<const __nv_bfloat16*>(v_pool), groups, extra, row_mask, s.n_q, s.n_kv, sl2,
             static_cast<__nv_bfloat16*>(out));
}

// One launch: every entry is one CTA's pass over <= attention_vectors_per_cta(hd) query vectors
// of its group (AttnGroup.pad = first vector). The vector-warp count and the key-slice count
// are fixed per head dim, so numerics never depend on the grouping.
int attention_vectors_per_cta(int hd) { return hd == 128 ? 32 : 16; }

void attention(const void* q, const void* k_pool, const void* v_pool, const AttnGroup* entries, int n_entries,
               const std::int32_t* extra, const unsigned long long* row_mask, const AttnShape& s, void* out,
               cudaStream_t st) {
  if (n_entries <= 0) return;
  const float sl2 = s.scale * 1.4426950408889634f;
  // A 2-deep K/V ring for both head dims. hd 64 (the 1B draft): one key slice (ncu launch lists
  // of scripts/forward_probe.py, profiles/r01_driver_policy.md): with Q riding in the first
  // cp.async group, 32.2 µs per layer against 37.2 with two slices and 47.7 with a 3-deep ring.
  // hd 128 (the 8B verify): two key slices — 32.6 µs per layer against 35.0 with one (105 x 5-row
  // groups over 176-position prefixes, WS_PROFILE_MODEL of scripts/forward_probe.py); 3-deep
  // rings and four slices were slower (profiles/r02_attention_hd128.md).
  if (s.hd == 128)
    launch_attn<128, 2, 2, 2>(q, k_pool, v_pool, entries, n_entries, extra, row_mask, s, sl2, out, st);
  else if (s.hd == 64)
    launch_attn<64, 1, 1, 2>(q, k_pool, v_pool, entries, n_entries, extra, row_mask, s, sl2, out, st);
  else
    throw std::invalid_argument("attention: head dim must be 64 or 128");
}

}  // namespace wsb
