// K1 — dense projections of the verify / draft forward on the 5th-gen tensor cores.
//
//   C[M, N] = A[M, K] · W[N, K]^T      (bf16 in, fp32 accumulate in TMEM)
//
// A = activations (rows = verify/draft rows), W = a weight matrix in its natural [out, in]
// (K-major) layout, so both operands are K-major and stream straight from HBM by TMA with the
// 128-byte swizzle the UMMA descriptors expect. Persistent and warp-specialised:
//   warp 0      TMA producer (one elected lane) over a STAGES-deep smem ring (mbarriers)
//   warp 1      TMEM allocator + MMA issuer (one lane issues tcgen05.mma 128xBNx16)
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> fused op -> global
// Each CTA walks work units u = blockIdx.x, +gridDim.x, ...; the accumulator is double-buffered
// in TMEM (2 x BN columns) so the epilogue of unit i overlaps the main loop of unit i+1.
// Epilogues: bf16 store (LM head), fp32 residual accumulate (O / down projections add into the
// fp32 residual stream), SwiGLU (gate/up rows interleaved in 16-row blocks), and QKV with RoPE
// + KV-pool scatter. Units are ordered M-fastest so all M-blocks of one weight tile run
// concurrently and each weight byte crosses HBM once per GEMM.
//
// Split-K for narrow outputs (N < 6144: the O / down projections, the 1B QKV): the K range of
// a tile is split into S parts chosen from (N, K) only; every split writes its fp32 partial and
// the last split to finish (ticket) sums the S partials in split order and runs the epilogue.
// Because S never depends on M, a row's result is bit-identical at any batch size, BN or
// schedule (batch invariance — the property behind "speculative stream == greedy stream").
#include "gemm_tc.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "cuda_check.hpp"
#include "pdl.cuh"
#include "sm100.cuh"

namespace wsb {

namespace {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle atom row
constexpr int kThreads = 192;
constexpr int kNumSMs = 148;

// Runtime tile width BN (multiple of 16, 64..256): the ring depth is whatever fits in
// shared memory, the two TMEM accumulators sit at columns 0 and 256 of a 512-column
// allocation (one CTA per SM).
constexpr int kSmemBudget = 232448;  // 227 KB opt-in
constexpr int kTmemCols = 512;
constexpr int kAccStride = 256;
// Per-CTA smem of one ring stage: the CTA's 128 A rows + its share of the BN weight rows (all
// of them for a single CTA, half for a CTA pair).
__host__ __device__ constexpr int a_bytes() { return BM * BK * 2; }
__host__ __device__ constexpr int b_bytes(int bn, int cg) { return bn / cg * BK * 2; }
__host__ __device__ constexpr int stage_bytes(int bn, int cg) { return a_bytes() + b_bytes(bn, cg); }
// cluster split-K (CS = 2): the receiving CTA's two 128 x 33 fp32 chunk buffers, after the ring
constexpr int kCsStride = 36;  // floats per row of a chunk buffer (16-byte rows, spread banks)
constexpr int kCsBufBytes = 2 * 128 * kCsStride * 4;
// fp32-residual epilogue staging (launches whose CTAs run several units): per epilogue warp a
// [32][33] fp32 tile + a [32][17] bf16-pair tile
constexpr int kEpiStageFloats = 32 * 33 + 32 * 17;
constexpr int kEpiStageBytes = 4 * kEpiStageFloats * 4;
inline int ring_stages(int bn, int cg, int cs = 1, bool epi_stage = false) {
  return std::min(8, (kSmemBudget - 2048 - (cs == 2 ? kCsBufBytes : 0) - (epi_stage ? kEpiStageBytes : 0)) /
                         stage_bytes(bn, cg));
}
inline int smem_bytes(int bn, int cg, int cs = 1, bool epi_stage = false) {
  return 1024 + ring_stages(bn, cg, cs, epi_stage) * stage_bytes(bn, cg) + 256 + (cs == 2 ? kCsBufBytes : 0) +
         (epi_stage ? kEpiStageBytes : 0);
}

__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ std::uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const std::uint32_t*>(&h);
}
// 32 bf16 (16 packed pairs) → dst[0, 32) with four 16-byte stores; every index is a constant
// after unrolling, so nothing here touches local memory.
__device__ __forceinline__ void store32_bf16(void* dst, const std::uint32_t (&pk)[16]) {
  uint4* o = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) o[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
}
__device__ __forceinline__ void store_bf16_tail(__nv_bfloat16* dst, const std::uint32_t (&pk)[16], int n) {
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j < n) {
      const std::uint32_t w = pk[j >> 1];
      dst[j] = __ushort_as_bfloat16(static_cast<unsigned short>((j & 1) ? (w >> 16) : (w & 0xFFFFu)));
    }
}

// Epilogue of one 128 x BN tile for this thread's row. fetch(col, r) yields the 32 fp32 values
// of tile columns [col, col+32) (from TMEM, or the summed split-K partials) and must be called
// by every lane (TMEM loads are warp-collective). wait() blocks until the accumulator is ready:
// inputs that do not depend on it (the residual row) are loaded before the call, so their L2
// latency overlaps the main loop instead of following it.
template <int EPI, bool STG, class Fetch, class Wait>
__device__ __forceinline__ void epilogue_tile(Fetch&& fetch, Wait&& wait, int BN, int row, int M, int N, int n_blk,
                                              void* out, int ldo, const RopeEpi& rp, const NormEpi& nm,
                                              float* estage = nullptr) {
  const bool live = row < M;
  if constexpr (EPI != kEpiAddF32 && EPI != kEpiQKVRope) wait();
  if constexpr (EPI == kEpiSwiGLU) {
    // W rows interleaved in 16-row blocks [gate 0..15 | up 0..15 | gate 16..31 | ...]: the
    // 32-column chunk c holds gate and up of output features f0 + c/2 .. +15.
    const int f0 = n_blk * (BN / 2);
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      std::uint32_t r[32];
      fetch(c, r);
      if (live && f0 + c / 2 < N / 2) {
        std::uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float a0 = silu(__uint_as_float(r[2 * j])) * __uint_as_float(r[16 + 2 * j]);
          const float a1 = silu(__uint_as_float(r[2 * j + 1])) * __uint_as_float(r[16 + 2 * j + 1]);
          pk[j] = pack_bf16(a0, a1);
        }
        uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + static_cast<std::size_t>(row) * ldo +
                                            f0 + c / 2);
        o[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        o[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  } else if constexpr (EPI == kEpiQKVRope) {
    // Per head of the tile: rotate-half RoPE on q/k (pairs i, i+hd/2; cos/sin from the
    // fp64-built table), then q → q_out[row], k and v → the KV pool at slot[row].
    const int hd = rp.hd, half = hd / 2;
    const int n0 = n_blk * BN;
    const int pos = live ? rp.pos[row] : 0;
    const int slot = live ? rp.slot[row] : 0;
    // (cos, sin) of the row's first 32 pairs, shared by every head of the tile: loaded before
    // the accumulator wait
    float4 cs0[16];
    if (live) {
      const float4* cs = reinterpret_cast<const float4*>(rp.cs + static_cast<std::size_t>(pos) * half);
#pragma unroll
      for (int j = 0; j < 16; ++j) cs0[j] = cs[j];
    }
    wait();
#pragma unroll 1
    for (int h0 = 0; h0 < BN; h0 += hd) {
      const int hh = (n0 + h0) / hd;  // warp-uniform
      if (hh >= rp.nq + 2 * rp.nkv) break;
      const bool rot = hh < rp.nq + rp.nkv;
      __nv_bfloat16* dst;
      if (hh < rp.nq)
        dst = static_cast<__nv_bfloat16*>(rp.q) + (static_cast<std::size_t>(row) * rp.nq + hh) * hd;
      else if (hh < rp.nq + rp.nkv)
        dst = static_cast<__nv_bfloat16*>(rp.k_pool) + (static_cast<std::size_t>(slot) * rp.nkv + (hh - rp.nq)) * hd;
      else
        dst = static_cast<__nv_bfloat16*>(rp.v_pool) +
              (static_cast<std::size_t>(slot) * rp.nkv + (hh - rp.nq - rp.nkv)) * hd;
#pragma unroll 1
      for (int c = 0; c < half; c += 32) {
        std::uint32_t a[32], b[32];
        fetch(h0 + c, a);
        fetch(h0 + c + half, b);
        if (!live) continue;
        std::uint32_t lo[16], hi[16];
        const float4* cs = reinterpret_cast<const float4*>(rp.cs + static_cast<std::size_t>(pos) * half + c);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float x0 = __uint_as_float(a[2 * j]), x1 = __uint_as_float(a[2 * j + 1]);
          float y0 = __uint_as_float(b[2 * j]), y1 = __uint_as_float(b[2 * j + 1]);
          if (rot) {
            const float4 cc = c == 0 ? cs0[j] : cs[j];  // (cos, sin) of pairs 2j and 2j + 1
            const float rx0 = x0 * cc.x - y0 * cc.y, ry0 = y0 * cc.x + x0 * cc.y;
            const float rx1 = x1 * cc.z - y1 * cc.w, ry1 = y1 * cc.z + x1 * cc.w;
            x0 = rx0;
            y0 = ry0;
            x1 = rx1;
            y1 = ry1;
          }
          lo[j] = pack_bf16(x0, x1);
          hi[j] = pack_bf16(y0, y1);
        }
        store32_bf16(dst + c, lo);
        store32_bf16(dst + c + half, hi);
      }
    }
  } else if constexpr (EPI == kEpiAddF32) {
    if constexpr (STG) {
    // Staged variant (launches whose CTAs run several units, where the epilogue overlaps the next
    // unit's main loop and its load/store traffic competes with it): the residual / output / bf16
    // tiles move through this warp's shared-memory staging (32 rows x 32 columns, padded rows),
    // so every global access is a coalesced row segment — lane l moves float4 column l % 8 of
    // rows l / 8 + 4 i (profiles/r02_prefill_probe.md). Same arithmetic as the direct path.
    const int n0 = n_blk * BN;
    const int ncols = min(BN, N - n0);
    const int lane = static_cast<int>(threadIdx.x & 31);
    const int row0 = row - lane;  // the warp's first row
    const int cq = lane & 7, rq = lane >> 3;
    float* ft = estage;                                                    // [32][33] fp32
    std::uint32_t* bt = reinterpret_cast<std::uint32_t*>(estage + 32 * 33);  // [32][17] bf16 pairs
    float* orow = static_cast<float*>(out) + static_cast<std::size_t>(row) * ldo + n0;
    const bool res = !nm.store_only;
    float4 cur[8], nxt[8];
    auto load = [&](int c, float4 (&v)[8]) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = row0 + rq + 4 * i;
        v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (res && rr < M && c + 32 <= ncols)
          v[i] = reinterpret_cast<const float4*>(static_cast<const float*>(out) + static_cast<std::size_t>(rr) * ldo +
                                                 n0 + c)[cq];
      }
    };
    load(0, cur);
    wait();
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      std::uint32_t r[32];
      fetch(c, r);
      if (c + 32 < BN) load(c + 32, nxt);
      if (c + 32 <= ncols) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float* d = ft + (rq + 4 * i) * 33 + 4 * cq;
          d[0] = cur[i].x;
          d[1] = cur[i].y;
          d[2] = cur[i].z;
          d[3] = cur[i].w;
        }
        __syncwarp();
        float x[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = ft[lane * 33 + j] + __uint_as_float(r[j]);
        if (nm.ss != nullptr && live) {
          float t = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) t = fmaf(x[j], x[j], t);
          nm.ss[static_cast<std::size_t>((n0 + c) / 32) * nm.ld_ss + row] = t;  // chunk-major: coalesced
#pragma unroll
          for (int j = 0; j < 16; ++j) bt[lane * 17 + j] = pack_bf16(x[2 * j], x[2 * j + 1]);
        }
        __syncwarp();  // every lane has read its residual row
#pragma unroll
        for (int j = 0; j < 32; ++j) ft[lane * 33 + j] = x[j];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = row0 + rq + 4 * i;
          if (rr < M) {
            const float* sp = ft + (rq + 4 * i) * 33 + 4 * cq;
            reinterpret_cast<float4*>(static_cast<float*>(out) + static_cast<std::size_t>(rr) * ldo + n0 + c)[cq] =
                make_float4(sp[0], sp[1], sp[2], sp[3]);
          }
        }
        if (nm.ss != nullptr) {
          const int bq = lane & 3, br = lane >> 2;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = row0 + br + 8 * i;
            if (rr < M) {
              const std::uint32_t* sp = bt + (br + 8 * i) * 17 + 4 * bq;
              *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(nm.xb) + static_cast<std::size_t>(rr) * nm.ld_xb +
                                        n0 + c + 8 * bq) = make_uint4(sp[0], sp[1], sp[2], sp[3]);
            }
          }
        }
        __syncwarp();  // the staging is reused by the next chunk
      } else if (live && c < ncols) {  // the ragged last chunk, element-wise
        float* o = orow + c;
        float x[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          x[j] = 0.f;
          if (c + j < ncols) {
            o[j] = (nm.store_only ? 0.f : o[j]) + __uint_as_float(r[j]);
            x[j] = o[j];
          }
        }
        if (nm.ss != nullptr) {
          float t = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) t = fmaf(x[j], x[j], t);
          nm.ss[static_cast<std::size_t>((n0 + c) / 32) * nm.ld_ss + row] = t;
          std::uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(x[2 * j], x[2 * j + 1]);
          store_bf16_tail(static_cast<__nv_bfloat16*>(nm.xb) + static_cast<std::size_t>(row) * nm.ld_xb + n0 + c, pk,
                          ncols - c);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
    }
    return;
    }

    // out[row, n] += acc (+ the fused-RMSNorm outputs of the new row). The residual chunk c + 32
    // is loaded while chunk c is processed, chunk 0 before the accumulator wait.
    const int n0 = n_blk * BN;
    const int ncols = min(BN, N - n0);  // valid columns of this tile (BN % 32 == 16: last chunk is half)
    float* orow = static_cast<float*>(out) + static_cast<std::size_t>(row) * ldo + n0;
    float4 cur[8], nxt[8];
    auto load = [&](int c, float4 (&v)[8]) {
      if (nm.store_only) {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
      }
      if (live && c + 32 <= ncols) {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = reinterpret_cast<const float4*>(orow + c)[q];
      }
    };
    load(0, cur);
    wait();
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      std::uint32_t r[32];
      fetch(c, r);
      if (c + 32 < BN) load(c + 32, nxt);
      if (live && c < ncols) {
        float* o = orow + c;
        float x[32];
        if (c + 32 <= ncols) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4 v = cur[q];
            v.x += __uint_as_float(r[4 * q + 0]);
            v.y += __uint_as_float(r[4 * q + 1]);
            v.z += __uint_as_float(r[4 * q + 2]);
            v.w += __uint_as_float(r[4 * q + 3]);
            reinterpret_cast<float4*>(o)[q] = v;
            x[4 * q] = v.x;
            x[4 * q + 1] = v.y;
            x[4 * q + 2] = v.z;
            x[4 * q + 3] = v.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            x[j] = 0.f;
            if (c + j < ncols) {
              o[j] = (nm.store_only ? 0.f : o[j]) + __uint_as_float(r[j]);
              x[j] = o[j];
            }
          }
        }
        if (nm.ss != nullptr) {
          float t = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) t = fmaf(x[j], x[j], t);
          nm.ss[static_cast<std::size_t>((n0 + c) / 32) * nm.ld_ss + row] = t;  // chunk-major: coalesced
          std::uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(x[2 * j], x[2 * j + 1]);
          __nv_bfloat16* xb = static_cast<__nv_bfloat16*>(nm.xb) + static_cast<std::size_t>(row) * nm.ld_xb + n0 + c;
          if (c + 32 <= ncols)
            store32_bf16(xb, pk);
          else
            store_bf16_tail(xb, pk, ncols - c);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
    }
  } else {
    const int n0 = n_blk * BN;
    const int ncols = min(BN, N - n0);  // valid columns of this tile (BN % 32 == 16: last chunk is half)
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      std::uint32_t r[32];
      fetch(c, r);
      if (!live || c >= ncols) continue;
      if constexpr (EPI == kEpiBF16) {
        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out) + static_cast<std::size_t>(row) * ldo + n0 + c;
        std::uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        if (c + 32 <= ncols)
          store32_bf16(o, pk);
        else
          store_bf16_tail(o, pk, ncols - c);
      }
    }
  }
}

// WS_GEMM_ABLATE bit 8: CTA 0 records a %globaltimer timeline of its first unit (diagnostics,
// read back with ws_debug_gemm_trace): entry, prologue done, dependency wait done, first ring
// slot full, last MMA of the unit issued, accumulator ready in the epilogue, epilogue done, exit.
__device__ unsigned long long g_gemm_trace[8];
constexpr int kEarlyTrigger = 1 << 16;  // (flag bit in `ablate`) trigger dependents at entry
constexpr int kLateTrigger = 1 << 17;   // (flag bit) trigger dependents once the last accumulator is ready
__device__ __forceinline__ void trace_point(int ablate, int i) {
  if ((ablate & 8) && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemm_trace[i] = t;
  }
}

struct SplitArgs {
  int splits = 1;
  // canonical K chunks of the whole K range (pick_chunks: from (N, K) only): every chunk
  // accumulates from zero in its own TMEM columns and the chunks are summed in order, so a
  // unit computing all of them in one CTA and `chunks` split units reducing their partials in
  // split order give identical bits — the split can then follow the batch size
  int chunks = 1;
  bool cluster = false;              // splits == 2 on CTA pairs: reduce through DSMEM (CS = 2)
  float* ws = nullptr;               // fp32 partials [splits][m_blocks*BM][N]
  unsigned int* tickets = nullptr;   // [m_blocks * n_tiles], zero-initialised, self-resetting
};

// CG = 1: one CTA per 128 x BN tile. CG = 2: a CTA pair (cluster of 2, cta_group::2) per
// 256 x BN tile — each CTA holds its 128 A rows and half of the BN weight rows, the leader's
// single thread issues the pair MMA over both CTAs' smem, and each CTA's TMEM receives its
// 128 rows; shared-memory traffic per MAC drops by a third (the main loop is smem-bound).
// CS = 2 (CTA pairs only): cluster split-K. A cluster of four CTAs is two pairs computing the
// same 256 x BN tile over the two halves of K; the second pair streams its fp32 accumulator
// through distributed shared memory into the first pair's CTAs, which add it to their own
// (split 0 + split 1, the order of the ordered global split-K sum) and run the epilogue. Half
// the K loop per SM, twice the tiles in flight, no partial traffic through L2.
template <int EPI, int CG, int CS = 1, bool STG = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, int m_blocks, int n_tiles, void* __restrict__ out, int ldo, const RopeEpi rope,
                   const SplitArgs sk, const NormEpi norm, int BN, int STAGES, int ablate) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~static_cast<std::uintptr_t>(1023));
  const int A_BYTES = a_bytes(), B_BYTES = b_bytes(BN, CG), STAGE_BYTES = stage_bytes(BN, CG);
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * A_BYTES;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + STAGES * STAGE_BYTES);
  std::uint64_t* empty = full + STAGES;
  std::uint64_t* tfull = empty + STAGES;  // [2]
  std::uint64_t* tempty = tfull + 2;      // [2]
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  std::uint32_t* last_flag = tmem_slot + 1;
  std::uint64_t* rfull = reinterpret_cast<std::uint64_t*>(tmem_slot + 2);  // [2] CS == 2: peer chunk landed
  std::uint64_t* sfree = rfull + 2;                                         // [2] CS == 2: chunk buffer consumed
  float* rbuf = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);  // CS == 2: [2][128][36]
  // the staged epilogue's per-warp blocks, after the CS buffers (kStagedEpi launches only)
  float* estage_base = STG ? reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256 + (CS == 2 ? kCsBufBytes : 0))
                            : nullptr;

  const int num_k = K / BK;
  const int S = sk.splits;  // 1 for pairs
  const int m_units = CG == 2 ? (m_blocks + 1) / 2 : m_blocks;
  const int total = m_units * n_tiles * S;
  const int crank = CG == 2 ? static_cast<int>(cluster_ctarank()) : 0;  // rank in the cluster
  const int rank = crank & 1;                      // role in the CTA pair (0 = leader)
  const int pair_base = crank & ~1;                // the pair's leader rank in the cluster
  const int ksplit = CS == 2 ? crank >> 1 : 0;     // cluster split-K: which half of K
  const std::uint16_t pair_mask = static_cast<std::uint16_t>(3u << pair_base);
  const int first = CG == 2 ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int step = CG == 2 ? static_cast<int>(cluster_count_x()) : static_cast<int>(gridDim.x);
  const bool leader = rank == 0;
  const std::uint32_t warp = warp_id(), lane = lane_id();
  // unit u → (M unit, n_blk, split), M fastest; this CTA's 128-row block is unit * CG + rank;
  // split s covers k-blocks [s*nk/S, (s+1)*nk/S)
  const int KSPLITS = CS == 2 ? 2 : S;  // K ranges per tile
  auto decode = [&](int u, int& m_blk, int& n_blk, int& split) {
    m_blk = (u % m_units) * CG + rank;
    const int r = u / m_units;
    split = CS == 2 ? ksplit : r % S;
    n_blk = r / S;
  };

  if (threadIdx.x == 0) {
    if (ablate & kEarlyTrigger) pdl_trigger_now();  // small grid: dependents may use the idle SMs
    trace_point(ablate, 0);
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * CG);  // one arrival per epilogue warp (of both CTAs for a pair)
      if constexpr (CS == 2) {
        mbar_init(&rfull[a], 4);  // one per sending epilogue warp, after the warp's stores
        mbar_init(&sfree[a], 4);  // one per receiving epilogue warp, after the warp's reads
      }
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2)
      tmem_alloc_pair<kTmemCols>(tmem_slot);
    else
      tmem_alloc<kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // the peer's barriers exist before any remote signal
  tc_fence_after();
  const std::uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) trace_point(ablate, 1);

  if (warp == 0) {
    // TMA producer: the whole warp runs the ring (operands stay warp-uniform), one elected lane
    // issues. The weight boxes of the first ring fill depend on nothing: they go out before the
    // wait for the previous kernel (PDL), the activation boxes after it.
    const std::uint32_t fill_bytes = CG == 2 ? 2 * STAGE_BYTES : STAGE_BYTES;
    int pre = 0;
    if (first < total) {
      int m_blk, n_blk, split;
      decode(first, m_blk, n_blk, split);
      const int kb0 = split * num_k / KSPLITS, kb1 = (split + 1) * num_k / KSPLITS;
      pre = min(STAGES, kb1 - kb0);
      if (elect_one()) {
        for (int i = 0; i < pre; ++i) {
          const int kb = kb0 + i;
          if constexpr (CG == 2) {
            if (leader) mbar_arrive_expect_tx(&full[i], fill_bytes);
            tma_load_2d_pair(sB + i * B_BYTES, &tmB, &full[i], kb * BK, n_blk * BN + rank * (BN / 2));
          } else {
            mbar_arrive_expect_tx(&full[i], fill_bytes);
            tma_load_2d(sB + i * B_BYTES, &tmB, &full[i], kb * BK, n_blk * BN);
          }
        }
      }
      __syncwarp();
    }
    pdl_wait();
    if (lane == 0) trace_point(ablate, 2);
    int stage = 0, it = 0;
    std::uint32_t phase = 0;
    for (int u = first; u < total; u += step) {
      int m_blk, n_blk, split;
      decode(u, m_blk, n_blk, split);
      const int kb0 = split * num_k / KSPLITS, kb1 = (split + 1) * num_k / KSPLITS;
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const bool prefilled = it < pre;  // weight box already in flight
        if (!prefilled) mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          if constexpr (CG == 2) {
            // both CTAs' boxes complete on the leader's barrier, which expects the pair's bytes
            if (!prefilled && leader) mbar_arrive_expect_tx(&full[stage], fill_bytes);
            tma_load_2d_pair(sA + stage * A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
            if (!prefilled)
              tma_load_2d_pair(sB + stage * B_BYTES, &tmB, &full[stage], kb * BK, n_blk * BN + rank * (BN / 2));
          } else {
            if (!prefilled) mbar_arrive_expect_tx(&full[stage], fill_bytes);
            tma_load_2d(sA + stage * A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
            if (!prefilled) tma_load_2d(sB + stage * B_BYTES, &tmB, &full[stage], kb * BK, n_blk * BN);
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // MMA issuer: the whole warp runs the loop, one elected lane issues
      const std::uint32_t idesc = idesc_bf16_f32(BM * CG, static_cast<std::uint32_t>(BN));
      const std::uint64_t da0 = smem_desc_sw128(sA), db0 = smem_desc_sw128(sB);
      int stage = 0;
      std::uint32_t phase = 0;
      int local = 0;
      for (int u = first; u < total; u += step, ++local) {
        int m_blk, n_blk, split;
        decode(u, m_blk, n_blk, split);
        const int kb0 = split * num_k / KSPLITS, kb1 = (split + 1) * num_k / KSPLITS;
        const int acc = local & 1;
        mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);  // epilogue drained this buffer
        tc_fence_after();
        const std::uint32_t d = tmem_base + acc * kAccStride;
        const int chunk_len = num_k / sk.chunks;
        for (int kb = kb0; kb < kb1; ++kb) {
          const int lk = kb - kb0;
          const std::uint32_t dc = d + static_cast<std::uint32_t>((lk / chunk_len) * BN);  // this chunk's columns
          const int in_chunk = lk % chunk_len;
          mbar_wait(&full[stage], phase);  // TMA → MMA: both async proxy, ordered by the mbarrier
          if (local == 0 && kb == kb0 && lane == 0) trace_point(ablate, 3);
          // descriptor start-address field is addr >> 4 (stage offsets are 16-byte multiples)
          const std::uint64_t da = da0 + static_cast<std::uint64_t>((stage * A_BYTES) >> 4);
          const std::uint64_t db = db0 + static_cast<std::uint64_t>((stage * B_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {  // advance 16 elements = 32 B = 2 descriptor units
              if (ablate & 1) continue;
              if constexpr (CG == 2)
                mma_bf16_pair(dc, da + 2 * k, db + 2 * k, idesc, (in_chunk | k) != 0);
              else
                mma_bf16(dc, da + 2 * k, db + 2 * k, idesc, (in_chunk | k) != 0);
            }
            // frees the smem slot (in both CTAs of a pair) when these MMAs retire
            if constexpr (CG == 2)
              mma_commit_pair(&empty[stage], pair_mask);
            else
              mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) {
          if constexpr (CG == 2)
            mma_commit_pair(&tfull[acc], pair_mask);
          else
            mma_commit(&tfull[acc]);
        }
        if (local == 0 && lane == 0) trace_point(ablate, 4);
        __syncwarp();
      }
    }
  } else {  // epilogue warps 2..5 → TMEM lane groups (warp % 4)
    pdl_wait();  // the epilogues read the residual / norm statistics / rope tables
    const int grp = static_cast<int>(warp & 3);
    float* estage = estage_base ? estage_base + grp * kEpiStageFloats : nullptr;
    const int m_slots = m_units * CG;  // 128-row blocks incl. a pair's padding block
    const int rows_pad = m_slots * BM;
    int local = 0;
    int cs_q = 0;  // CS == 2: chunks exchanged so far (buffer = cs_q & 1)
    for (int u = first; u < total; u += step, ++local) {
      int m_blk, n_blk, split;
      decode(u, m_blk, n_blk, split);
      const int acc = local & 1;
      const int row = m_blk * BM + grp * 32 + static_cast<int>(lane);
      // fused RMSNorm consumer: this row's scale from the producer's chunk statistics (read
      // coalesced, chunk-major, while the accumulator is still being computed; four partial
      // sums combined in a fixed order — deterministic)
      float rs = 1.f;
      if (norm.ss_in != nullptr && row < M) {
        const float* p = norm.ss_in + row;
        float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
        const int nc = K / 32;
        int c = 0;
        for (; c + 4 <= nc; c += 4) {
          t0 += p[static_cast<std::size_t>(c) * norm.ld_ss];
          t1 += p[static_cast<std::size_t>(c + 1) * norm.ld_ss];
          t2 += p[static_cast<std::size_t>(c + 2) * norm.ld_ss];
          t3 += p[static_cast<std::size_t>(c + 3) * norm.ld_ss];
        }
        for (; c < nc; ++c) t0 += p[static_cast<std::size_t>(c) * norm.ld_ss];
        rs = rsqrtf(((t0 + t1) + (t2 + t3)) / static_cast<float>(K) + norm.eps);
      }
      auto acc_wait = [&] {
        mbar_wait(&tfull[acc], (local >> 1) & 1);
        if (local == 0 && warp == 2 && lane == 0) trace_point(ablate, 5);
        // the CTA's last accumulator is complete: only its epilogue remains, so the next kernel
        // of the chain may start its prologue and weight prefetch on the SMs that free up
        if ((ablate & kLateTrigger) && u + step >= total && warp == 2 && lane == 0) pdl_trigger_now();
        tc_fence_after();
      };
      const std::uint32_t t_row = tmem_base + acc * kAccStride + (static_cast<std::uint32_t>(grp * 32) << 16);
      const int local_chunks = sk.chunks / KSPLITS;  // S == 1: all chunks; a split unit: one
      auto tmem_fetch = [&](int col, std::uint32_t (&r)[32]) {
        tmem_ld32(t_row + col, r);
        tmem_ld_wait();
        if (local_chunks > 1) {  // 0 + c0 + c1 + ...: the split path's ordered sum of partials
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f + __uint_as_float(r[j]);
          for (int c = 1; c < local_chunks; ++c) {
            tmem_ld32(t_row + static_cast<std::uint32_t>(c * BN + col), r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += __uint_as_float(r[j]);
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(v[j]);
        }
        if (norm.ss_in != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * rs);
        }
      };
      if constexpr (CS == 2) {
        const int rl = grp * 32 + static_cast<int>(lane);  // row within this CTA's 128
        if (ksplit == 1) {
          // sender: this CTA's accumulator, 32 columns at a time, into the split-0 CTA with the
          // same role (cluster rank - 2), double-buffered
          acc_wait();
          const std::uint32_t dst = static_cast<std::uint32_t>(crank - 2);
          const std::uint32_t rb = mapa_u32(rbuf, dst);
#pragma unroll 1
          for (int c = 0; c < BN; c += 32, ++cs_q) {
            const int b = cs_q & 1;
            mbar_wait_cluster(&sfree[b], ((cs_q >> 1) & 1) ^ 1);
            std::uint32_t r[32];
            tmem_ld32(t_row + c, r);
            tmem_ld_wait();
            const std::uint32_t a = rb + static_cast<std::uint32_t>((b * 128 * kCsStride + rl * kCsStride) * 4);
#pragma unroll
            for (int j = 0; j < 32; j += 4) st_cluster_v4(a + 4 * j, r[j], r[j + 1], r[j + 2], r[j + 3]);
            __syncwarp();  // orders the lanes' stores before lane 0's cluster-scope release
            if (lane == 0) mbar_arrive_cluster(&rfull[b], dst);
          }
        } else {
          // receiver: own (split 0) + peer (split 1), the ordered global split-K sum
          auto cs_fetch = [&](int col, std::uint32_t (&r)[32]) {
            tmem_ld32(t_row + col, r);
            tmem_ld_wait();
            const int b = cs_q & 1;
            mbar_wait_cluster(&rfull[b], (cs_q >> 1) & 1);
            const float4* pb = reinterpret_cast<const float4*>(rbuf + b * 128 * kCsStride + rl * kCsStride);
            float pv[32];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 t = pb[j];
              pv[4 * j] = t.x;
              pv[4 * j + 1] = t.y;
              pv[4 * j + 2] = t.z;
              pv[4 * j + 3] = t.w;
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              float v = __uint_as_float(r[j]) + pv[j];
              if (norm.ss_in != nullptr) v *= rs;
              r[j] = __float_as_uint(v);
            }
            // relaxed: the values are already consumed, and a release would first drain this
            // thread's residual stores of the previous chunk
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(&sfree[b], static_cast<std::uint32_t>(crank + 2));
            ++cs_q;
          };
          epilogue_tile<EPI, STG>(cs_fetch, acc_wait, BN, row, (ablate & 4) ? 0 : M, N, n_blk, out, ldo, rope, norm,
                            estage);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&tempty[acc], pair_base);
        continue;
      }
      if (S == 1) {
        epilogue_tile<EPI, STG>(tmem_fetch, acc_wait, BN, row, (ablate & 4) ? 0 : M, N, n_blk, out, ldo, rope, norm,
                          estage);
        if (local == 0 && warp == 2 && lane == 0) trace_point(ablate, 6);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {  // the accumulator is reused by the (leader's) MMA issuer
          if constexpr (CG == 2)
            mbar_arrive_cluster(&tempty[acc], pair_base);
          else
            mbar_arrive(&tempty[acc]);
        }
        continue;
      }
      // split-K: publish this split's fp32 partial, release TMEM, take a ticket
      acc_wait();
      const int ncols = min(BN, N - n_blk * BN);
      float* my = sk.ws + (static_cast<std::size_t>(split) * rows_pad + row) * N + static_cast<std::size_t>(n_blk) * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        std::uint32_t r[32];
        tmem_ld32(t_row + c, r);  // raw partial: the norm scale applies once, after the ordered sum
        tmem_ld_wait();
        if (c < ncols) {
          if (c + 32 <= ncols) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              __stcg(reinterpret_cast<float4*>(my + c) + q,
                     make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                 __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c + j < ncols) __stcg(my + c + j, __uint_as_float(r[j]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // the accumulator is reused by the (leader's) MMA issuer
        if constexpr (CG == 2)
          mbar_arrive_cluster(&tempty[acc], pair_base);
        else
          mbar_arrive(&tempty[acc]);
      }
      __threadfence();
      epi_bar();
      const int tile = n_blk * m_slots + m_blk;
      if (threadIdx.x == 64) {
        const unsigned int t = atomicAdd(&sk.tickets[tile], 1u);
        *last_flag = t == static_cast<unsigned int>(S - 1) ? 1u : 0u;
        if (t == static_cast<unsigned int>(S - 1)) sk.tickets[tile] = 0u;  // self-reset
      }
      epi_bar();
      if (*last_flag) {
        __threadfence();
        const float* base = sk.ws + static_cast<std::size_t>(row) * N + static_cast<std::size_t>(n_blk) * BN;
        const std::size_t sstride = static_cast<std::size_t>(rows_pad) * N;
        auto ws_fetch = [&](int col, std::uint32_t (&r)[32]) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
          if (col < ncols) {
            for (int s = 0; s < S; ++s) {  // fixed split order → deterministic
              const float* p = base + s * sstride + col;
              if (col + 32 <= ncols) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                  const float4 x = __ldcg(reinterpret_cast<const float4*>(p) + q);
                  v[4 * q] += x.x;
                  v[4 * q + 1] += x.y;
                  v[4 * q + 2] += x.z;
                  v[4 * q + 3] += x.w;
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (col + j < ncols) v[j] += __ldcg(p + j);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(norm.ss_in != nullptr ? v[j] * rs : v[j]);
        };
        epilogue_tile<EPI, STG>(ws_fetch, [] {}, BN, row, M, N, n_blk, out, ldo, rope, norm, estage);
      }
      epi_bar();  // last_flag is reused by the next unit
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_point(ablate, 7);
  if constexpr (CG == 2) {
    cluster_sync();  // neither CTA leaves while its peer's MMAs / signals may still target it
    if (warp == 1) tmem_dealloc_pair<kTmemCols>(tmem_base);
  } else {
    if (warp == 1) tmem_dealloc<kTmemCols>(tmem_base);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D K-major bf16 tensor [rows, cols] (row stride ld elements), box = box_rows x 64, SW128.
// Encoded maps are cached per host thread (direct-mapped on the parameters): a forward's weight
// maps and its activation buffers' maps repeat every forward, and a map holds only the address,
// shape and box, so a hit is exact.
CUtensorMap make_map(const void* ptr, std::uint64_t rows, std::uint64_t cols, std::uint64_t ld, std::uint32_t box_rows) {
  struct Entry {
    const void* p = nullptr;
    std::uint64_t rows = 0, cols = 0, ld = 0;
    std::uint32_t box = 0;
    CUtensorMap m;
  };
  thread_local Entry cache[512];
  std::uint64_t h = reinterpret_cast<std::uintptr_t>(ptr) * 0x9E3779B97F4A7C15ull;
  h ^= (rows * 0xBF58476D1CE4E5B9ull) ^ (cols << 20) ^ (ld << 7) ^ box_rows;
  h ^= h >> 29;
  Entry& e = cache[h % 512];
  if (e.p == ptr && e.rows == rows && e.cols == cols && e.ld == ld && e.box == box_rows) return e.m;
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  e.p = ptr;
  e.rows = rows;
  e.cols = cols;
  e.ld = ld;
  e.box = box_rows;
  e.m = m;
  return m;
}

template <int CSZ>
int max_clusters() {  // co-resident clusters of CSZ CTAs at one CTA per SM (same on every B200)
  static int n = [] {
    WS_CUDA(cudaFuncSetAttribute(gemm_tn_kernel<kEpiBF16, 2, CSZ / 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemBudget));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CSZ * (kNumSMs / CSZ), 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemBudget;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CSZ;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int c = 0;
    WS_CUDA(cudaOccupancyMaxActiveClusters(&c, gemm_tn_kernel<kEpiBF16, 2, CSZ / 2>, &cfg));
    return std::max(1, c);
  }();
  return n;
}
int pair_clusters() { return max_clusters<2>(); }

// the staged-epilogue instantiation exists for the fp32-residual epilogue only
template <int EPI, int CG, int CS>
auto pick_kernel(bool staged) {
  if constexpr (EPI == kEpiAddF32) {
    if (staged) return gemm_tn_kernel<EPI, CG, CS, true>;
  }
  return gemm_tn_kernel<EPI, CG, CS, false>;
}

template <int EPI, int CG, int CS = 1>
void launch(const GemmArgs& g, const SplitArgs& sk, int bn, cudaStream_t st) {
  static std::atomic<std::uint32_t> attr_done{0};
  once_per_device(attr_done, [] {
    WS_CUDA(cudaFuncSetAttribute(gemm_tn_kernel<EPI, CG, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemBudget));
    if constexpr (EPI == kEpiAddF32)
      WS_CUDA(cudaFuncSetAttribute(gemm_tn_kernel<EPI, CG, CS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kSmemBudget));
  });
  static const int ablate = [] {  // WS_GEMM_ABLATE (measurement only): 1 no MMA,
    const char* e = std::getenv("WS_GEMM_ABLATE");  // 4 no epilogue stores
    return e ? std::atoi(e) : 0;
  }();
  // grids at or below WS_PDL_EARLY_GRID CTAs trigger their dependents at entry (default 0 = off:
  // measured 1.28 -> 1.33 s per step at 64 requests with 96, no gain at 256)
  static const int early_grid = [] {
    const char* e = std::getenv("WS_PDL_EARLY_GRID");
    return e ? std::atoi(e) : 0;
  }();
  const int late = g.pdl_late > 0 ? kLateTrigger : 0;
  const CUtensorMap ta = make_map(g.A, g.M, g.K, g.lda, BM);
  const CUtensorMap tb = make_map(g.W, g.N, g.K, g.ldw, static_cast<std::uint32_t>(bn / CG));
  const int m_blocks = (g.M + BM - 1) / BM;
  const int n_tiles = (g.N + bn - 1) / bn;  // SwiGLU: N counts gate+up rows
  // The fp32-residual epilogue goes through shared-memory staging when CTAs run several units
  // (its traffic then overlaps the next unit's main loop); a single unit keeps the direct path,
  // which is shorter on the critical path (profiles/r02_prefill_probe.md). WS_EPI_STAGE=0: never.
  static const bool stage_ok = [] {
    const char* e = std::getenv("WS_EPI_STAGE");
    return !(e && e[0] == '0');
  }();
  bool staged = false;
  auto plan = [&](int units, int ctas_or_clusters, int& smem, int& stages, int& flags) {
    staged = EPI == kEpiAddF32 && stage_ok && units > ctas_or_clusters;
    smem = smem_bytes(bn, CG, CS, staged);
    stages = ring_stages(bn, CG, CS, staged);
    flags = ablate | late;
  };
  int smem = 0, stages = 0, flags = 0;
  if constexpr (CG == 1) {
    const int total = m_blocks * n_tiles * sk.splits;
    // max_ctas < 0: one CTA per unit (not persistent: SMs free up between units, so a
    // concurrent higher-priority stream's kernels get scheduled sooner)
    const int grid = g.max_ctas < 0 ? total : std::min(total, g.max_ctas > 0 ? g.max_ctas : kNumSMs);
    plan(total, grid, smem, stages, flags);
    flags |= (grid <= early_grid ? kEarlyTrigger : 0);
    launch_pdl(pick_kernel<EPI, 1, 1>(staged), dim3(grid), dim3(kThreads), smem, st,
               1, ta, tb, g.M, g.N, g.K, m_blocks, n_tiles, g.out, g.ldo, g.rope, sk, g.norm, bn, stages, flags);
  } else if constexpr (CS == 2) {
    const int total = (m_blocks + 1) / 2 * n_tiles;  // tiles; each cluster of 4 holds both K halves
    int clusters = g.max_ctas < 0 ? total : std::min(total, max_clusters<4>());
    if (g.max_ctas > 0) clusters = std::max(1, std::min(clusters, g.max_ctas / 4));
    plan(total, clusters, smem, stages, flags);
    static const bool dbg = std::getenv("WS_GEMM_DEBUG") != nullptr;
    if (dbg) std::fprintf(stderr, "[gemm] cluster split: %d tiles, %d co-resident clusters of 4, bn %d, %d stages\n",
                          total, max_clusters<4>(), bn, stages);
    flags |= (4 * clusters <= early_grid ? kEarlyTrigger : 0);
    launch_pdl(pick_kernel<EPI, 2, 2>(staged), dim3(4 * clusters),
               dim3(kThreads), smem, st, 4, ta, tb, g.M, g.N, g.K, m_blocks, n_tiles, g.out, g.ldo, g.rope, sk,
               g.norm, bn, stages, flags);
  } else {
    const int total = (m_blocks + 1) / 2 * n_tiles * sk.splits;
    int clusters = g.max_ctas < 0 ? total : std::min(total, pair_clusters());
    if (g.max_ctas > 0) clusters = std::max(1, std::min(clusters, g.max_ctas / 2));
    plan(total, clusters, smem, stages, flags);
    flags |= (2 * clusters <= early_grid ? kEarlyTrigger : 0);
    launch_pdl(pick_kernel<EPI, 2, 1>(staged), dim3(2 * clusters),
               dim3(kThreads), smem, st, 2, ta, tb, g.M, g.N, g.K, m_blocks, n_tiles, g.out, g.ldo, g.rope, sk,
               g.norm, bn, stages, flags);
  }
}

template <int EPI>
void launch_cg(const GemmArgs& g, const SplitArgs& sk, int bn, int cg, cudaStream_t st) {
  if (cg == 2) {
    if constexpr (EPI != kEpiQKVRope) {  // (the QKV epilogue reads chunks out of order)
      if (sk.splits == 2 && sk.cluster) {
        SplitArgs one = sk;
        one.splits = 1;  // the K halves live in the cluster, not in the unit index
        return launch<EPI, 2, 2>(g, one, bn, st);
      }
    }
    return launch<EPI, 2>(g, sk, bn, st);
  }
  return launch<EPI, 1>(g, sk, bn, st);
}

}  // namespace

// Tile choice from the measured shared-memory bound (profiles/r01_gemm_feed.md): per k-block an
// SM moves its A rows and its share of the weight rows through smem twice (TMA fill + MMA
// read) at ~128 B/cycle, against an MMA floor of 2 BN cycles:
//   single CTA, 128 x BN:  256 + 2 BN cycles   (always smem-bound)
//   CTA pair,   256 x BN:  max(2 BN, 256 + BN) (balanced at BN = 256)
// and a GEMM costs ceil(units / slots) of those (148 SMs, 74 pairs). Pick the (mode, BN) — BN a
// multiple of 32 and of the epilogue's granule — minimising that; wider on ties. Numerics do
// not depend on either (each output is the same K-ordered MMA chain): batch/tile invariance.
struct TileChoice {
  int cg, bn;
};
TileChoice pick_tile(int M, int N, int granule, bool allow_pair, int bn_max = 256) {
  const int step = std::max(32, granule);
  const int mb = (M + BM - 1) / BM;
  TileChoice best{1, step};
  long best_cost = -1;
  // WS_GEMM_PAIR1=1: CTA pairs also for a single 128-row block (the second CTA's A rows are all
  // padding; a pair tile moves half the weight rows per SM). Isolated small-batch forwards gain
  // 2-4 %, but a pair takes two SMs per tile and the 4-GPU bench, where both lanes share the
  // SMs, lost 1 % (profiles/r02_gemm_chunks.md): off by default.
  static const bool pair1 = [] {
    const char* e = std::getenv("WS_GEMM_PAIR1");
    return e && e[0] == '1';
  }();
  for (int cg = 1; cg <= (allow_pair && (mb > 1 || pair1) ? 2 : 1); ++cg) {
    for (int bn = bn_max / step * step; bn >= std::max(std::min(64, bn_max), step); bn -= step) {
      const long units = static_cast<long>((mb + cg - 1) / cg) * ((N + bn - 1) / bn);
      const long slots = cg == 2 ? kNumSMs / 2 : kNumSMs;
      const long per = cg == 2 ? std::max(2L * bn, 256L + bn) : 256L + 2L * bn;
      const long cost = ((units + slots - 1) / slots) * per;
      if (best_cost < 0 || cost < best_cost) {
        best_cost = cost;
        best = TileChoice{cg, bn};
      }
    }
  }
  return best;
}

int pick_bn(int M, int N, int granule) { return pick_tile(M, N, granule, false).bn; }

int pick_bn(int M, int N) { return pick_bn(M, N, 32); }

void gemm_debug_trace(unsigned long long* out8) {
  WS_CUDA(cudaMemcpyFromSymbol(out8, g_gemm_trace, sizeof(unsigned long long) * 8));
}

int pick_splits(int N, int K) {
  // From (N, K) only — never from M — so results stay batch-invariant. Measured on B200
  // (profiles/r01_splitk.md): at the verify/draft batch sizes the extra partial traffic and the
  // serialised last-split epilogue cost more than the extra parallelism buys (8B O-proj 187 →
  // 380 ms/run, 1B down 318 → 766 ms/run), so the model path does not split; the machinery
  // stays available (explicit splits) and tested.
  // WS_GEMM_SPLITS="N:K:S[,N:K:S...]" (experiments): a fixed split count for those shapes
  struct Rule {
    int n, k, s;
  };
  static const std::vector<Rule> rules = [] {
    std::vector<Rule> r;
    if (const char* e = std::getenv("WS_GEMM_SPLITS")) {
      std::string v(e);
      std::size_t at = 0;
      while (at < v.size()) {
        const std::size_t end = std::min(v.find(',', at), v.size());
        int n = 0, k = 0, sp = 0;
        if (std::sscanf(v.substr(at, end - at).c_str(), "%d:%d:%d", &n, &k, &sp) == 3 && sp >= 1) r.push_back({n, k, sp});
        at = end + 1;
      }
    }
    return r;
  }();
  for (const Rule& r : rules)
    if (r.n == N && r.k == K) return r.s;
  return 1;
}

int pick_chunks(int N, int K) {
  // Canonical K chunks, from (N, K) only (batch invariance). WS_GEMM_CHUNKS="N:K:C[,...]"
  // overrides / extends the defaults (experiments).
  struct Rule {
    int n, k, c;
  };
  static const std::vector<Rule> rules = [] {
    std::vector<Rule> r;
    if (const char* e = std::getenv("WS_GEMM_CHUNKS")) {
      std::string v(e);
      std::size_t at = 0;
      while (at < v.size()) {
        const std::size_t end = std::min(v.find(',', at), v.size());
        int n = 0, k = 0, c = 0;
        if (std::sscanf(v.substr(at, end - at).c_str(), "%d:%d:%d", &n, &k, &c) == 3 && c >= 1) r.push_back({n, k, c});
        at = end + 1;
      }
    }
    return r;
  }();
  for (const Rule& r : rules)
    if (r.n == N && r.k == K) return (K / BK) % r.c == 0 && r.c <= 4 ? r.c : 1;
  // Default: the 1B down projection (N 2048, K 8192: 128 k-blocks on 16-32 CTAs at draft
  // batches) in two chunks — split over two CTA sets below ~256 rows, -8 to -11 % per 1B
  // forward at 48-192 rows, neutral at 496 (profiles/r02_gemm_chunks.md). The 8B shapes lose
  // their BN = 256 pair tiles to the chunk accumulators (+11 % at 535 rows) and stay at one.
  if (N == 2048 && K == 8192) return 2;
  if (N == 4096 && K == 14336) return 2;  // the 8B down projection (224 k-blocks)
  return 1;
}

// Workspace layout (fixed, whatever the GEMM shape): [tickets: kMaxTiles u32 | fp32 partials].
// The self-resetting tickets must never move between launches of different shapes.
constexpr std::size_t kMaxTiles = 65536;
constexpr std::size_t kTicketBytes = kMaxTiles * sizeof(unsigned int);

std::size_t gemm_workspace_bytes(int max_rows) {
  const std::size_t rows = ((static_cast<std::size_t>(max_rows) + BM - 1) / BM) * BM;
  // max over split configurations of splits x N (pick_splits: 4 x <3072, 2 x <6144)
  return kTicketBytes + rows * 12288 * sizeof(float);
}

void gemm_tn(const GemmArgs& g, cudaStream_t st) {
  if (g.K % BK != 0) throw std::invalid_argument("gemm: K must be a multiple of 64");
  if (g.lda % 8 || g.ldw % 8) throw std::invalid_argument("gemm: leading dims must be multiples of 8");
  // epilogue granularity: SwiGLU tiles hold whole 64-row gate/up blocks, QKV tiles whole heads
  int granule = 16;
  if (g.epi == kEpiSwiGLU) granule = 32;
  if (g.epi == kEpiQKVRope) {
    if (g.rope.hd != 64 && g.rope.hd != 128) throw std::invalid_argument("gemm: qkv epilogue needs hd 64/128");
    if (g.N != (g.rope.nq + 2 * g.rope.nkv) * g.rope.hd) throw std::invalid_argument("gemm: qkv width");
    granule = g.rope.hd;
  }
  if (g.norm.ss_in && g.K % 32) throw std::invalid_argument("gemm: fused norm needs K % 32 == 0");
  if (g.norm.ss && (g.epi != kEpiAddF32 || !g.norm.xb)) throw std::invalid_argument("gemm: norm producer epilogue");
  if (g.norm.ss) granule = 32;  // statistics are per 32-column chunk
  // WS_GEMM_PAIR: "0" keeps every GEMM on single CTAs, "2" forces CTA pairs (tests, A/B)
  const char* pe = std::getenv("WS_GEMM_PAIR");
  const int pair_env = pe ? std::atoi(pe) : -1;
  const bool pair_ok = pair_env != 0 && g.cta_group != 1;
  // canonical K chunks (only on the automatic path): all chunks in one CTA's TMEM (BN <= 256 /
  // chunks), or — when even the split units fit in one wave of slots — one split unit per chunk
  // (without a split workspace only the distributed-shared-memory split — two chunks on CTA
  // pairs — can be taken; the unsplit in-CTA chunks need none)
  const int chunks = g.chunks_ > 0 ? g.chunks_
                     : (g.splits == 0 && !g.bn && g.epi != kEpiQKVRope) ? pick_chunks(g.N, g.K)
                                                                       : 1;
  // The C chunk accumulators of an unsplit unit take C x BN TMEM columns: within one of the two
  // 256-column buffers, or — when every CTA (pair) holds a single unit, so the second buffer is
  // never used — within all 512.
  auto units_of = [&](const TileChoice& t) {
    const long m_units = t.cg == 2 ? ((g.M + BM - 1) / BM + 1) / 2 : (g.M + BM - 1) / BM;
    return m_units * ((g.N + t.bn - 1) / t.bn);
  };
  auto slots_of = [&](const TileChoice& t) { return t.cg == 2 ? static_cast<long>(pair_clusters()) : kNumSMs; };
  // whether some CTA (pair) may run more than one unit (the launch's grid, see launch())
  auto multi_unit = [&](const TileChoice& t) {
    if (g.max_ctas < 0) return false;
    const long cap = g.max_ctas > 0 ? (t.cg == 2 ? std::max(1, g.max_ctas / 2) : g.max_ctas) : slots_of(t);
    return units_of(t) > std::min(cap, slots_of(t));
  };
  TileChoice tc = pick_tile(g.M, g.N, granule, pair_ok);
  if (g.cta_group == 2 || (pair_env == 2 && pair_ok)) tc.cg = 2;
  if (g.bn) tc.bn = g.bn;
  bool chunk_split = false;
  if (chunks > 1) {
    // Tile and split chosen together from the shared-memory cost model of pick_tile: unsplit
    // (all chunks in one CTA) or one unit per chunk (two chunks on CTA pairs reduce through
    // distributed shared memory, otherwise through global partials — the latter charged extra).
    const int step = std::max(32, granule);
    const int num_k = g.K / BK;
    const int mb = (g.M + BM - 1) / BM;
    long best = -1;
    static const bool pair1 = [] {
      const char* e = std::getenv("WS_GEMM_PAIR1");
      return e && e[0] == '1';
    }();
    for (int cg = 1; cg <= (pair_ok && (mb > 1 || pair1) ? 2 : 1); ++cg) {
      if (g.cta_group && cg != g.cta_group) continue;
      for (int bn = 256 / step * step; bn >= std::max(64, step); bn -= step) {
        const TileChoice t{cg, bn};
        const long per = cg == 2 ? std::max(2L * bn, 256L + bn) : 256L + 2L * bn;
        for (int sp : {1, chunks}) {
          if (sp == 1 && chunks * bn > kAccStride && (multi_unit(t) || chunks * bn > kTmemCols)) continue;
          if (sp > 1 && !g.ws && !(cg == 2 && chunks == 2)) continue;  // global partials need a workspace
          const long units = units_of(t) * sp;
          const long rounds = (units + slots_of(t) - 1) / slots_of(t);
          const long overhead = sp == 1 ? 0 : (cg == 2 && chunks == 2 ? 2048 : 8192);
          const long cost = rounds * per * (num_k / sp) + overhead;
          if (best < 0 || cost < best) {
            best = cost;
            tc = t;
            chunk_split = sp > 1;
          }
        }
      }
    }
    if (g.bn) tc.bn = g.bn;
  }
  bool csplit_now = false;
  // WS_GEMM_CSPLIT=1 (experiment): residual-epilogue projections (O, down) run as cluster
  // split-K on CTA pairs — a fixed split count whatever M, so results stay batch-invariant —
  // with BN from the pair cost model over 33 co-resident clusters of four.
  static const bool csplit = [] {
    const char* e = std::getenv("WS_GEMM_CSPLIT");
    return e && e[0] == '1';
  }();
  if (csplit && g.splits == 0 && g.epi == kEpiAddF32 && g.cta_group != 1 && !g.bn && g.K / BK >= 16) {
    csplit_now = true;
    tc.cg = 2;
    const int mu = ((g.M + BM - 1) / BM + 1) / 2;
    long best = -1;
    for (int b = 256; b >= 128; b -= 32) {
      const long tiles = static_cast<long>(mu) * ((g.N + b - 1) / b);
      const long cost = (tiles + 32) / 33 * std::max(2L * b, 256L + b);
      if (best < 0 || cost < best) {
        best = cost;
        tc.bn = b;
      }
    }
  }
  const int bn = tc.bn;
  if (bn < 16 || bn > 256 || bn % granule) throw std::invalid_argument("gemm: tile width must be a multiple of " +
                                                                       std::to_string(granule) + " in [16, 256]");
  if (bn % 32 && g.cta_group != 2) tc.cg = 1;  // an explicit odd-16 width runs on single CTAs
  if (tc.cg == 2 && bn % 32) throw std::invalid_argument("gemm: CTA pairs need BN % 32");
  SplitArgs sk;
  sk.splits = csplit_now ? 2 : g.splits > 0 ? g.splits : chunk_split ? chunks : (g.ws ? pick_splits(g.N, g.K) : 1);
  sk.chunks = csplit_now ? 1 : chunks;
  if (sk.chunks > 1 && sk.splits != 1 && sk.splits != sk.chunks)
    throw std::logic_error("gemm: canonical chunks need splits of 1 or chunks");
  if (sk.chunks > 1 && (g.K / BK) % sk.chunks) throw std::invalid_argument("gemm: K not a multiple of the chunks");
  if (sk.chunks / sk.splits * bn > kAccStride) {
    // only with one unit per CTA (pair): the unit's chunks may span both accumulator buffers
    TileChoice t = tc;
    t.bn = bn;
    if (sk.chunks / sk.splits * bn > kTmemCols || multi_unit(t))
      throw std::invalid_argument("gemm: chunk accumulators exceed TMEM (M " + std::to_string(g.M) + " N " +
                                  std::to_string(g.N) + " K " + std::to_string(g.K) + " bn " + std::to_string(bn) +
                                  " cg " + std::to_string(tc.cg) + " chunks " + std::to_string(sk.chunks) +
                                  " splits " + std::to_string(sk.splits) + " units " + std::to_string(units_of(t)) +
                                  " slots " + std::to_string(slots_of(t)) + ")");
  }

  // two K halves on CTA pairs reduce through distributed shared memory (no workspace);
  // WS_GEMM_DSMEM=0 keeps them on the global-partials path (tests compare the two bit for bit)
  const char* de = std::getenv("WS_GEMM_DSMEM");
  sk.cluster = sk.splits == 2 && tc.cg == 2 && g.epi != kEpiQKVRope && !(de && de[0] == '0');
  if (sk.splits > 1 && !sk.cluster) {
    if (!g.ws) throw std::invalid_argument("gemm: split-K needs a workspace");
    const int m_blocks = (g.M + BM - 1) / BM;
    const int m_slots = tc.cg == 2 ? (m_blocks + 1) / 2 * 2 : m_blocks;  // as in the kernel
    const int n_tiles = (g.N + bn - 1) / bn;
    const std::size_t need = kTicketBytes + static_cast<std::size_t>(sk.splits) * m_slots * BM * g.N * sizeof(float);
    if (need > g.ws_bytes || static_cast<std::size_t>(m_slots) * n_tiles > kMaxTiles) {
      // Rows are independent: run the GEMM in row slices that fit the workspace.
      if (g.ws_bytes <= kTicketBytes) throw std::invalid_argument("gemm: split-K workspace too small");
      const std::size_t per_row = static_cast<std::size_t>(sk.splits) * g.N * sizeof(float);
      const int unit = tc.cg == 2 ? 2 * BM : BM;  // pair slices keep whole CTA pairs
      const int per = std::max<int>(unit, static_cast<int>((g.ws_bytes - kTicketBytes) / per_row / unit * unit));
      if (per >= g.M) throw std::invalid_argument("gemm: split-K workspace too small");
      for (int r0 = 0; r0 < g.M; r0 += per) {
        GemmArgs s = g;
        s.M = std::min(per, g.M - r0);
        // the fused-norm statistics and the bf16 row copy are indexed by the launch-local row
        if (g.norm.ss_in) s.norm.ss_in = g.norm.ss_in + r0;
        if (g.norm.ss) s.norm.ss = g.norm.ss + r0;
        if (g.norm.xb) s.norm.xb = static_cast<__nv_bfloat16*>(g.norm.xb) + static_cast<std::size_t>(r0) * g.norm.ld_xb;
        s.A = static_cast<const __nv_bfloat16*>(g.A) + static_cast<std::size_t>(r0) * g.lda;
        if (g.epi == kEpiAddF32)
          s.out = static_cast<float*>(g.out) + static_cast<std::size_t>(r0) * g.ldo;
        else if (g.epi == kEpiQKVRope) {
          s.rope.pos = g.rope.pos + r0;
          s.rope.slot = g.rope.slot + r0;
          s.rope.q = static_cast<__nv_bfloat16*>(g.rope.q) + static_cast<std::size_t>(r0) * g.rope.nq * g.rope.hd;
        } else
          s.out = static_cast<__nv_bfloat16*>(g.out) + static_cast<std::size_t>(r0) * g.ldo;
        s.bn = bn;
        s.splits = sk.splits;
        s.cta_group = tc.cg;
        s.chunks_ = sk.chunks;
        gemm_tn(s, st);
      }
      return;
    }
    sk.tickets = static_cast<unsigned int*>(g.ws);
    sk.ws = reinterpret_cast<float*>(static_cast<unsigned char*>(g.ws) + kTicketBytes);
  }
  switch (g.epi) {
    case kEpiBF16: return launch_cg<kEpiBF16>(g, sk, bn, tc.cg, st);
    case kEpiAddF32: return launch_cg<kEpiAddF32>(g, sk, bn, tc.cg, st);
    case kEpiSwiGLU: return launch_cg<kEpiSwiGLU>(g, sk, bn, tc.cg, st);
    case kEpiQKVRope: return launch_cg<kEpiQKVRope>(g, sk, bn, tc.cg, st);
  }
  throw std::invalid_argument("gemm: unknown epilogue");
}

}  // namespace wsb
