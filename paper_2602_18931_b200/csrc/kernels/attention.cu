// K2 — grouped GQA attention of the verify / draft forward over the KV slot pool.
//
// One CTA per (group, kv head). A group is the set of rows of one request that share a
// context: a linear committed prefix (prefix_len consecutive slots from prefix_slot, visible to
// every row) followed by up to 64 explicit "extra" slots (new rows, tree ancestors) whose
// visibility is either causal (verify rows, catch-up prefill: row j sees extra[0 .. E-n+j]) or
// given by a per-row 64-bit mask (the worker's tree leaves: each leaf sees its own ancestor
// chain). Every K/V tile is read from HBM once per (group, kv head) and reused by all
// n_rows x (n_q / n_kv) query vectors — a request's k+1 verify rows and all its draft leaves
// share one pass over the prefix.
//
// Per tile of 32 positions: lane = position; the lane's K row lives in registers, query
// vectors stream from shared memory, online softmax per query vector (exp2 domain), P·V with
// the probabilities broadcast by shuffles. CUDA cores; the workload is HBM-bound on KV.
#include <cuda_bf16.h>

#include <stdexcept>

#include "cuda_check.hpp"
#include "llama_ops.cuh"

namespace wsb {

namespace {

constexpr int kThreads = 128;
constexpr int kTile = 32;
constexpr int kVPW = 8;  // query vectors per warp per pass

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int HD>
__global__ void __launch_bounds__(kThreads) attn_kernel(const __nv_bfloat16* __restrict__ q,
                                                        const __nv_bfloat16* __restrict__ kp,
                                                        const __nv_bfloat16* __restrict__ vp,
                                                        const AttnGroup* __restrict__ groups,
                                                        const std::int32_t* __restrict__ extra,
                                                        const unsigned long long* __restrict__ row_mask, int nq,
                                                        int nkv, float scale_log2, __nv_bfloat16* __restrict__ out) {
  constexpr int W = HD / 2;   // 32-bit words per head vector
  constexpr int RW = W + 1;   // padded smem row (bank-conflict-free row reads)
  constexpr int DPL = HD / 32;
  __shared__ std::uint32_t sK[kTile * RW];
  __shared__ std::uint32_t sV[kTile * RW];
  __shared__ __align__(16) float sQ[kThreads / 32][kVPW][HD];
  __shared__ std::int32_t sSlot[kTile];

  const AttnGroup g = groups[blockIdx.x];
  const int kvh = blockIdx.y;
  const int G = nq / nkv;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nvec = g.n_rows * G;
  const int ctx = g.prefix_len + g.extra_len;
  const std::size_t slot_stride = static_cast<std::size_t>(nkv) * HD;

  for (int pass0 = 0; pass0 < nvec; pass0 += (kThreads / 32) * kVPW) {
    float m[kVPW], l[kVPW], o[kVPW][DPL];
    unsigned long long vis[kVPW];  // masked groups: visibility bits over the extras (<= 64)
    int last[kVPW];                // causal groups: last visible extra index
    bool live[kVPW];
#pragma unroll
    for (int u = 0; u < kVPW; ++u) {
      m[u] = -INFINITY;
      l[u] = 0.f;
#pragma unroll
      for (int e = 0; e < DPL; ++e) o[u][e] = 0.f;
      const int v = pass0 + warp * kVPW + u;
      live[u] = v < nvec;
      vis[u] = 0ull;
      last[u] = -1;
      if (live[u]) {
        const int j = v / G, h = kvh * G + v % G;
        if (g.masked)
          vis[u] = row_mask[g.row0 + j];
        else
          last[u] = g.extra_len - g.n_rows + j;
        const __nv_bfloat16* qs = q + (static_cast<std::size_t>(g.row0 + j) * nq + h) * HD;
        for (int d = lane; d < HD; d += 32) sQ[warp][u][d] = __bfloat162float(qs[d]) * scale_log2;
      }
    }
    __syncwarp();
    for (int p0 = 0; p0 < ctx; p0 += kTile) {
      __syncthreads();
      if (threadIdx.x < kTile) {
        const int p = p0 + threadIdx.x;
        sSlot[threadIdx.x] = p < g.prefix_len ? g.prefix_slot + p : (p < ctx ? extra[g.extra_off + p - g.prefix_len] : -1);
      }
      __syncthreads();
      // K/V tile: 16-byte global loads, 4-byte smem stores into padded rows
      for (int t = threadIdx.x; t < kTile * (W / 4); t += kThreads) {
        const int r = t / (W / 4), c4 = t % (W / 4);
        const int s = sSlot[r];
        uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
        if (s >= 0) {
          const std::size_t base = static_cast<std::size_t>(s) * slot_stride + static_cast<std::size_t>(kvh) * HD;
          kv = reinterpret_cast<const uint4*>(kp + base)[c4];
          vv = reinterpret_cast<const uint4*>(vp + base)[c4];
        }
        std::uint32_t* dk = &sK[r * RW + 4 * c4];
        std::uint32_t* dv = &sV[r * RW + 4 * c4];
        dk[0] = kv.x;
        dk[1] = kv.y;
        dk[2] = kv.z;
        dk[3] = kv.w;
        dv[0] = vv.x;
        dv[1] = vv.y;
        dv[2] = vv.z;
        dv[3] = vv.w;
      }
      __syncthreads();
      const int p = p0 + lane;
      std::uint32_t krow[W];
#pragma unroll
      for (int w = 0; w < W; ++w) krow[w] = sK[lane * RW + w];
      const bool in_prefix = p < g.prefix_len;
      const int e = p - g.prefix_len;
#pragma unroll
      for (int u = 0; u < kVPW; ++u) {
        if (!live[u]) continue;  // warp-uniform
        const bool visible =
            p < ctx && (in_prefix || (g.masked ? ((vis[u] >> (e & 63)) & 1ull) != 0ull : e <= last[u]));
        float s = 0.f;
        const float2* qv = reinterpret_cast<const float2*>(sQ[warp][u]);
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&krow[w]));
          const float2 qf = qv[w];
          s = fmaf(qf.x, kf.x, s);
          s = fmaf(qf.y, kf.y, s);
        }
        s = visible ? s : -INFINITY;
        const float mt = warp_max(s);
        if (mt == -INFINITY) continue;  // nothing visible in this tile (warp-uniform)
        const float mn = fmaxf(m[u], mt);
        const float corr = exp2f(m[u] - mn);
        const float pr = exp2f(s - mn);
        l[u] = l[u] * corr + warp_sum(pr);
        m[u] = mn;
#pragma unroll
        for (int d = 0; d < DPL; ++d) o[u][d] *= corr;
#pragma unroll 4
        for (int jj = 0; jj < kTile; ++jj) {
          const float pj = __shfl_sync(0xffffffffu, pr, jj);
          const std::uint32_t* vr = &sV[jj * RW + lane * (DPL / 2)];
#pragma unroll
          for (int d = 0; d < DPL; d += 2) {
            const float2 vf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vr[d / 2]));
            o[u][d] = fmaf(pj, vf.x, o[u][d]);
            o[u][d + 1] = fmaf(pj, vf.y, o[u][d + 1]);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kVPW; ++u) {
      if (!live[u]) continue;
      const int v = pass0 + warp * kVPW + u;
      const int j = v / G, h = kvh * G + v % G;
      __nv_bfloat16* os = out + (static_cast<std::size_t>(g.row0 + j) * nq + h) * HD + lane * DPL;
      const float inv = l[u] > 0.f ? 1.f / l[u] : 0.f;
#pragma unroll
      for (int d = 0; d < DPL; d += 2)
        *reinterpret_cast<__nv_bfloat162*>(os + d) = __floats2bfloat162_rn(o[u][d] * inv, o[u][d + 1] * inv);
    }
  }
}

}  // namespace

void attention(const void* q, const void* k_pool, const void* v_pool, const AttnGroup* groups, int n_groups,
               const std::int32_t* extra, const unsigned long long* row_mask, const AttnShape& s, void* out,
               cudaStream_t st) {
  if (n_groups <= 0) return;
  dim3 grid(n_groups, s.n_kv);
  const float sl2 = s.scale * 1.4426950408889634f;
  if (s.hd == 128)
    attn_kernel<128><<<grid, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(q),
                                                static_cast<const __nv_bfloat16*>(k_pool),
                                                static_cast<const __nv_bfloat16*>(v_pool), groups, extra, row_mask,
                                                s.n_q, s.n_kv, sl2, static_cast<__nv_bfloat16*>(out));
  else if (s.hd == 64)
    attn_kernel<64><<<grid, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(q),
                                               static_cast<const __nv_bfloat16*>(k_pool),
                                               static_cast<const __nv_bfloat16*>(v_pool), groups, extra, row_mask,
                                               s.n_q, s.n_kv, sl2, static_cast<__nv_bfloat16*>(out));
  else
    throw std::invalid_argument("attention: head dim must be 64 or 128");
  WS_CUDA(cudaGetLastError());
}

}  // namespace wsb
