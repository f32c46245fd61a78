// Model-plumbing kernels: embedding gather, RMSNorm, RoPE + KV append, grouped GQA attention,
// planted bias, slot copies, Philox weight init. All HBM/latency bound; vectorised 16-byte
// accesses where the layout allows.
#include "llama_ops.cuh"

#include <algorithm>

#include <cuda_bf16.h>

#include <stdexcept>

#include "cuda_check.hpp"
#include "pdl.cuh"

namespace wsb {

namespace {

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

// One warp per 32-column chunk of a row: x = float(emb[tok]), xb = the bf16 copy (exact), and
// the chunk's sum of squares for the fused RMSNorm of the first projection (gemm_tc.cuh NormEpi).
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ emb, const std::int32_t* __restrict__ tok, int d,
                             float* __restrict__ x, __nv_bfloat16* __restrict__ xb, float* __restrict__ ss,
                             int ld_ss) {
  pdl_trigger();
  pdl_wait();  // inputs come from the previous kernel of the chain
  // One row per CTA; each thread moves 8 consecutive elements (one 16-byte load, two 16-byte fp32
  // stores, one 16-byte bf16 store). A 32-element norm-statistics chunk is 4 threads: each sums
  // its 8 squares in order, then the chunk combines ((t0 + t1) + (t2 + t3)) — a fixed order per
  // row, so the statistics are the same at any batch size.
  const int row = blockIdx.x;
  const __nv_bfloat16* e = emb + static_cast<std::size_t>(tok[row]) * d;
  for (int i8 = threadIdx.x; i8 < d / 8; i8 += blockDim.x) {
    const uint4 q = reinterpret_cast<const uint4*>(e)[i8];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
    float f[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 v = __bfloat1622float2(h[j]);
      f[2 * j] = v.x;
      f[2 * j + 1] = v.y;
    }
    float4* xo = reinterpret_cast<float4*>(x + static_cast<std::size_t>(row) * d) + 2 * i8;
    xo[0] = make_float4(f[0], f[1], f[2], f[3]);
    xo[1] = make_float4(f[4], f[5], f[6], f[7]);
    if (xb) reinterpret_cast<uint4*>(xb + static_cast<std::size_t>(row) * d)[i8] = q;
    if (ss) {
      float t = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) t = fmaf(f[j], f[j], t);
      const float t1 = __shfl_xor_sync(0xffffffffu, t, 1);
      const float a = (threadIdx.x & 1) ? t1 + t : t + t1;  // (t0 + t1) in the lower thread's order
      const float a2 = __shfl_xor_sync(0xffffffffu, a, 2);
      const float c = (threadIdx.x & 2) ? a2 + a : a + a2;
      if ((threadIdx.x & 3) == 0) ss[static_cast<std::size_t>(i8 / 4) * ld_ss + row] = c;  // chunk-major
    }
  }
}

__global__ void scale_cols_kernel(__nv_bfloat16* __restrict__ W, std::int64_t rows, int cols,
                                  const __nv_bfloat16* __restrict__ w) {
  const std::int64_t n = rows * cols;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    W[i] = __float2bfloat16_rn(__bfloat162float(W[i]) * __bfloat162float(w[i % cols]));
}

__global__ void rmsnorm_kernel(const float* __restrict__ x, int ld_x, const std::int32_t* __restrict__ idx,
                               const __nv_bfloat16* __restrict__ w, float eps, int d, __nv_bfloat16* __restrict__ y,
                               int ld_y) {
  pdl_trigger();
  pdl_wait();  // inputs come from the previous kernel of the chain
  const int row = blockIdx.x;
  const int src = idx ? idx[row] : row;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<std::size_t>(src) * ld_x);
  float ss = 0.f;
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = xr[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float r = rsqrtf(red[0] / static_cast<float>(d) + eps);
  __nv_bfloat162* yr = reinterpret_cast<__nv_bfloat162*>(y + static_cast<std::size_t>(row) * ld_y);
  const __nv_bfloat162* wr = reinterpret_cast<const __nv_bfloat162*>(w);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = xr[i];
    const float2 w0 = __bfloat1622float2(wr[2 * i]);
    const float2 w1 = __bfloat1622float2(wr[2 * i + 1]);
    yr[2 * i] = __floats2bfloat162_rn(v.x * r * w0.x, v.y * r * w0.y);
    yr[2 * i + 1] = __floats2bfloat162_rn(v.z * r * w1.x, v.w * r * w1.y);
  }
}

// One thread per (row, head, rotation pair i < hd/2): dims i and i + hd/2 (rotate-half).
__global__ void rope_append_kernel(const __nv_bfloat16* __restrict__ qkv, int nq, int nkv, int hd,
                                   const std::int32_t* __restrict__ pos, const std::int32_t* __restrict__ slot,
                                   const float* __restrict__ inv_freq, __nv_bfloat16* __restrict__ q_out,
                                   __nv_bfloat16* __restrict__ k_pool, __nv_bfloat16* __restrict__ v_pool) {
  const int row = blockIdx.x;
  const int half = hd / 2;
  const int heads = nq + 2 * nkv;
  const __nv_bfloat16* src = qkv + static_cast<std::size_t>(row) * heads * hd;
  const float p = static_cast<float>(pos[row]);
  const std::size_t sbase = static_cast<std::size_t>(slot[row]) * nkv * hd;
  for (int t = threadIdx.x; t < heads * half; t += blockDim.x) {
    const int h = t / half, i = t % half;
    const float a = __bfloat162float(src[h * hd + i]);
    const float b = __bfloat162float(src[h * hd + i + half]);
    if (h >= nq + nkv) {  // V: plain copy
      const std::size_t o = sbase + static_cast<std::size_t>(h - nq - nkv) * hd;
      v_pool[o + i] = src[h * hd + i];
      v_pool[o + i + half] = src[h * hd + i + half];
      continue;
    }
    float sn, cs;
    sincosf(p * inv_freq[i], &sn, &cs);
    const float r0 = a * cs - b * sn;
    const float r1 = b * cs + a * sn;
    if (h < nq) {
      __nv_bfloat16* o = q_out + (static_cast<std::size_t>(row) * nq + h) * hd;
      o[i] = __float2bfloat16(r0);
      o[i + half] = __float2bfloat16(r1);
    } else {
      __nv_bfloat16* o = k_pool + sbase + static_cast<std::size_t>(h - nq) * hd;
      o[i] = __float2bfloat16(r0);
      o[i + half] = __float2bfloat16(r1);
    }
  }
}

__global__ void plant_kernel(__nv_bfloat16* logits, int ld, const std::int32_t* plant, float bias, int rows) {
  pdl_trigger();
  pdl_wait();  // inputs come from the previous kernel of the chain
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int t = plant[r];
  if (t < 0) return;
  __nv_bfloat16* p = logits + static_cast<std::size_t>(r) * ld + t;
  *p = __float2bfloat16(__bfloat162float(*p) + bias);
}

__global__ void copy_slots_kernel(__nv_bfloat16* kp, __nv_bfloat16* vp, const std::int32_t* src, const std::int32_t* dst,
                                  std::int64_t layer_stride, int slot_stride) {
  const int pair = blockIdx.x, layer = blockIdx.y;
  const std::size_t s = static_cast<std::size_t>(layer) * layer_stride + static_cast<std::size_t>(src[pair]) * slot_stride;
  const std::size_t d = static_cast<std::size_t>(layer) * layer_stride + static_cast<std::size_t>(dst[pair]) * slot_stride;
  for (int i = threadIdx.x; i < slot_stride / 8; i += blockDim.x) {
    reinterpret_cast<uint4*>(kp + d)[i] = reinterpret_cast<const uint4*>(kp + s)[i];
    reinterpret_cast<uint4*>(vp + d)[i] = reinterpret_cast<const uint4*>(vp + s)[i];
  }
}

__device__ __forceinline__ void philox(std::uint32_t c[4], std::uint32_t k0, std::uint32_t k1) {
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

// Box-Muller on Philox words: 4 normals per counter.
__global__ void fill_normal_kernel(__nv_bfloat16* out, std::int64_t n, std::uint32_t k0, std::uint32_t k1,
                                   std::uint32_t sid, float std_, float mean) {
  for (std::int64_t i = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x * 4) {
    std::uint32_t c[4] = {static_cast<std::uint32_t>(i >> 2), static_cast<std::uint32_t>(i >> 34), sid, 0x5EEDu};
    philox(c, k0, k1);
    float z[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float u1 = (static_cast<float>(c[2 * h] >> 8) + 0.5f) * (1.0f / 16777216.0f);
      const float u2 = static_cast<float>(c[2 * h + 1] >> 8) * (1.0f / 16777216.0f);
      const float r = sqrtf(-2.0f * logf(u1));
      float sn, cs;
      sincospif(2.0f * u2, &sn, &cs);
      z[2 * h] = r * cs;
      z[2 * h + 1] = r * sn;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (i + e < n) out[i + e] = __float2bfloat16(std_ == 0.f ? mean : mean + std_ * z[e]);
  }
}

}  // namespace

void embed_rows(const void* emb, const std::int32_t* tok, int rows, int d, float* x, void* xb, float* ss, int ld_ss,
                cudaStream_t st) {
  if (rows <= 0) return;
  if (d % 32) throw std::invalid_argument("embed: d % 32");
  if (d % 256) throw std::invalid_argument("embed: d % 256");  // whole warps of 8-element threads
  launch_pdl(embed_kernel, dim3(rows), dim3(std::min(256, d / 8)), 0, st, 1, static_cast<const __nv_bfloat16*>(emb),
             tok, d, x, static_cast<__nv_bfloat16*>(xb), ss, ld_ss);
}

void fold_norm_weight(void* W, std::int64_t rows, int cols, const void* w, cudaStream_t st) {
  scale_cols_kernel<<<1184, 256, 0, st>>>(static_cast<__nv_bfloat16*>(W), rows, cols,
                                          static_cast<const __nv_bfloat16*>(w));
  WS_CUDA(cudaGetLastError());
}

void rmsnorm_rows(const float* x, int ld_x, const std::int32_t* idx, const void* w, float eps, int rows, int d,
                  void* y, int ld_y, cudaStream_t st) {
  if (rows <= 0) return;
  if (d % 4) throw std::invalid_argument("rmsnorm: d % 4");
  launch_pdl(rmsnorm_kernel, dim3(rows), dim3(256), 0, st, 1, x, ld_x, idx, static_cast<const __nv_bfloat16*>(w), eps,
             d, static_cast<__nv_bfloat16*>(y), ld_y);
}

void rope_kv_append(const void* qkv, int rows, int nq, int nkv, int hd, const std::int32_t* pos,
                    const std::int32_t* slot, const float* inv_freq, void* q_out, void* k_pool, void* v_pool,
                    cudaStream_t st) {
  if (rows <= 0) return;
  rope_append_kernel<<<rows, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(qkv), nq, nkv, hd, pos, slot, inv_freq,
                                           static_cast<__nv_bfloat16*>(q_out), static_cast<__nv_bfloat16*>(k_pool),
                                           static_cast<__nv_bfloat16*>(v_pool));
  WS_CUDA(cudaGetLastError());
}

void plant_bias(void* logits, int ld, const std::int32_t* plant, float bias, int rows, cudaStream_t st) {
  if (rows <= 0) return;
  launch_pdl(plant_kernel, dim3((rows + 127) / 128), dim3(128), 0, st, 1, static_cast<__nv_bfloat16*>(logits), ld,
             plant, bias, rows);
}

void copy_slots(void* k_pool, void* v_pool, const std::int32_t* src, const std::int32_t* dst, int n, int layers,
                std::int64_t layer_stride, int slot_stride, cudaStream_t st) {
  if (n <= 0) return;
  copy_slots_kernel<<<dim3(n, layers), 128, 0, st>>>(static_cast<__nv_bfloat16*>(k_pool),
                                                     static_cast<__nv_bfloat16*>(v_pool), src, dst, layer_stride,
                                                     slot_stride);
  WS_CUDA(cudaGetLastError());
}

void fill_normal_bf16(void* out, std::int64_t n, std::uint64_t seed, std::uint32_t sid, float std_, float mean,
                      cudaStream_t st) {
  if (n <= 0) return;
  fill_normal_kernel<<<148 * 8, 256, 0, st>>>(static_cast<__nv_bfloat16*>(out), n, static_cast<std::uint32_t>(seed),
                                              static_cast<std::uint32_t>(seed >> 32), sid, std_, mean);
  WS_CUDA(cudaGetLastError());
}

}  // namespace wsb
