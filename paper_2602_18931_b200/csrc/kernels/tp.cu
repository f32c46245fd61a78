// Tensor-parallel plumbing (see tp.cuh).
#include "tp.cuh"

#include <cuda_bf16.h>

#include <stdexcept>

#include "cuda_check.hpp"
#include "pdl.cuh"

namespace wsb {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) tp_allreduce_kernel(TPPeers p, int rank, int rows, int d, int ld_ss,
                                                                  unsigned long long epoch, int write_x_all) {
  // the row-parallel GEMM before this kernel is complete and its writes flushed: announce it
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x < p.tp) {
    __threadfence_system();
    st_release_sys(&p.flag_a[threadIdx.x][rank], epoch);
  }
  if (threadIdx.x < p.tp)
    while (ld_acquire_sys(&p.flag_a[rank][threadIdx.x]) < epoch) {
    }
  __syncthreads();
  const int r0 = static_cast<int>(static_cast<long long>(rows) * rank / p.tp);
  const int r1 = static_cast<int>(static_cast<long long>(rows) * (rank + 1) / p.tp);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int quads = d / 128;  // a warp covers 128 columns: lane = one float4, 8 lanes = one 32-column chunk
  float* xo = p.x[rank];
  const int gbase = lane & ~7;
  for (long long u = static_cast<long long>(blockIdx.x) * (kThreads / 32) + warp;
       u < static_cast<long long>(r1 - r0) * quads; u += static_cast<long long>(gridDim.x) * (kThreads / 32)) {
    const int row = r0 + static_cast<int>(u / quads);
    const int cq = static_cast<int>(u % quads);
    const std::size_t off = static_cast<std::size_t>(row) * d + cq * 128 + lane * 4;
    // every rank's partial in flight at once (NVLink reads for the peers), then the rank-ordered sum
    float4 a[kMaxTP];
#pragma unroll
    for (int t = 0; t < kMaxTP; ++t)
      if (t < p.tp) a[t] = *reinterpret_cast<const float4*>(p.part[t] + off);
    const float4 xv = *reinterpret_cast<const float4*>(xo + off);
    float4 s = a[0];
#pragma unroll
    for (int t = 1; t < kMaxTP; ++t)
      if (t < p.tp) {
        s.x += a[t].x;
        s.y += a[t].y;
        s.z += a[t].z;
        s.w += a[t].w;
      }
    const float4 v = make_float4(xv.x + s.x, xv.y + s.y, xv.z + s.z, xv.w + s.w);
    *reinterpret_cast<float4*>(xo + off) = v;
    // the 32-column chunk statistic: a sequential fmaf chain in column order (as the GEMM's
    // producer epilogue) over the 8 lanes of the chunk
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float wx = __shfl_sync(0xffffffffu, v.x, gbase + j), wy = __shfl_sync(0xffffffffu, v.y, gbase + j);
      const float wz = __shfl_sync(0xffffffffu, v.z, gbase + j), ww = __shfl_sync(0xffffffffu, v.w, gbase + j);
      q = fmaf(wx, wx, q);
      q = fmaf(wy, wy, q);
      q = fmaf(wz, wz, q);
      q = fmaf(ww, ww, q);
    }
    const __nv_bfloat162 b01 = __floats2bfloat162_rn(v.x, v.y), b23 = __floats2bfloat162_rn(v.z, v.w);
    uint2 pk;
    pk.x = *reinterpret_cast<const unsigned int*>(&b01);
    pk.y = *reinterpret_cast<const unsigned int*>(&b23);
    const int chunk = cq * 4 + (lane >> 3);
    for (int t = 0; t < p.tp; ++t) {
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.xb[t]) + off) = pk;
      if (write_x_all && t != rank) *reinterpret_cast<float4*>(p.x[t] + off) = v;
      if ((lane & 7) == 0) p.ss[t][static_cast<std::size_t>(chunk) * ld_ss + row] = q;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(p.counter, 1u);
    if (prev == gridDim.x - 1) {
      *p.counter = 0u;  // self-reset for the next all-reduce
      __threadfence_system();
      for (int t = 0; t < p.tp; ++t) st_release_sys(&p.flag_b[t][rank], epoch);
    }
  }
  // the kernel (and so the next GEMM on this stream) completes once every rank's broadcast
  // into this rank's replicas has landed
  if (blockIdx.x == 0 && threadIdx.x < p.tp)
    while (ld_acquire_sys(&p.flag_b[rank][threadIdx.x]) < epoch) {
    }
}

__device__ __forceinline__ void philox(std::uint32_t c[4], std::uint32_t k0, std::uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const std::uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const std::uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    c[0] = hi1 ^ c[1] ^ k0;
    c[1] = lo1;
    c[2] = hi0 ^ c[3] ^ k1;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__global__ void fill_2d_kernel(__nv_bfloat16* out, std::int64_t rows, std::int64_t cols, std::int64_t ld_full,
                               std::int64_t row0, std::int64_t col0, std::uint32_t k0, std::uint32_t k1,
                               std::uint32_t sid, float std_, float mean) {
  const std::int64_t n = rows * cols;
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t r = e / cols, c = e % cols;
    const std::int64_t i = (row0 + r) * ld_full + col0 + c;  // index in the full tensor
    const std::int64_t g = i & ~static_cast<std::int64_t>(3);  // its group of four (fill_normal_kernel)
    std::uint32_t w[4] = {static_cast<std::uint32_t>(g >> 2), static_cast<std::uint32_t>(g >> 34), sid, 0x5EEDu};
    philox(w, k0, k1);
    const int h = static_cast<int>((i & 3) >> 1);
    const float u1 = (static_cast<float>(w[2 * h] >> 8) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = static_cast<float>(w[2 * h + 1] >> 8) * (1.0f / 16777216.0f);
    const float rr = sqrtf(-2.0f * logf(u1));
    float sn, cs;
    sincospif(2.0f * u2, &sn, &cs);
    const float z = (i & 1) ? rr * sn : rr * cs;
    out[e] = __float2bfloat16(std_ == 0.f ? mean : mean + std_ * z);
  }
}

}  // namespace

void tp_allreduce_residual(const TPPeers& p, int rank, int rows, int d, int ld_ss, unsigned long long epoch,
                           bool write_x_all, cudaStream_t st) {
  if (p.tp < 2 || p.tp > kMaxTP || rank < 0 || rank >= p.tp) throw std::invalid_argument("tp_allreduce: bad rank");
  if (d % 128) throw std::invalid_argument("tp_allreduce: d % 128");
  // every CTA must become resident while others spin: at most one wave (148 SMs)
  const int owned = (rows + p.tp - 1) / p.tp;
  const long long units = static_cast<long long>(owned) * (d / 128);
  int grid = static_cast<int>(std::min<long long>(148, (units + kThreads / 32 - 1) / (kThreads / 32)));
  if (grid < 1) grid = 1;
  launch_pdl(tp_allreduce_kernel, dim3(grid), dim3(kThreads), 0, st, 1, p, rank, rows, d, ld_ss, epoch,
             write_x_all ? 1 : 0);
}

void fill_normal_bf16_2d(void* out, std::int64_t rows, std::int64_t cols, std::int64_t ld_full, std::int64_t row0,
                         std::int64_t col0, std::uint64_t seed, std::uint32_t sid, float std_, float mean,
                         cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  fill_2d_kernel<<<148 * 8, 256, 0, st>>>(static_cast<__nv_bfloat16*>(out), rows, cols, ld_full, row0, col0,
                                          static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32), sid,
                                          std_, mean);
  WS_CUDA(cudaGetLastError());
}

}  // namespace wsb
