// Microbenchmark: issue rate of tcgen05.mma kind::f16 (SS mode, M=128, K=16) for several N,
// one CTA per SM, operands resident in shared memory, no barriers inside the timed loop.
// Prints cycles per instruction and the implied fraction of the 128*N/256 floor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_18931_b200/csrc \
//        scripts/mma_probe.cu -o /tmp/mma_probe -lcuda
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/sm100.cuh"

using namespace wsb::sm100;

// variant bit 0: tcgen05.commit to a side barrier after every 4 MMAs (one k-block);
// variant bit 1: mbarrier wait on an already-completed barrier before every k-block.
template <int N>
__global__ void probe(int iters, long long* out, int variant) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~1023ull);
  __shared__ std::uint32_t tmem_slot;
  __shared__ __align__(8) std::uint64_t bar, side, done;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<std::uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&side, 1);
    mbar_init(&done, 1);
    mbar_arrive(&done);  // phase 0 complete
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t d = tmem_slot;
  if (threadIdx.x == 0) {
    const std::uint64_t da = smem_desc_sw128(smem);
    const std::uint64_t db = smem_desc_sw128(smem + 128 * 128);
    const std::uint32_t idesc = idesc_bf16_f32(128, N);
    // warm-up
    for (int i = 0; i < 64; ++i) mma_bf16(d, da + 2 * (i & 3), db + 2 * (i & 3), idesc, i != 0);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if ((variant & 2) && (i & 3) == 0) mbar_wait(&done, 0);
      mma_bf16(d, da + 2 * (i & 3), db + 2 * (i & 3), idesc, 1);
      if ((variant & 1) && (i & 3) == 3) mma_commit(&side);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 1);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *out = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(d);
}

template <int N>
void run(int ctas, int variant) {
  long long* d_out;
  cudaMalloc(&d_out, 8);
  const int smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  probe<N><<<ctas, 128, smem>>>(iters, d_out, variant);
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  const double per = static_cast<double>(cyc) / iters;
  std::printf("v%d N=%3d ctas=%3d  %.1f cycles/mma  floor %.1f  (%.0f%%)  %s\n", variant, N, ctas, per, 128.0 * N / 256.0,
              100.0 * (128.0 * N / 256.0) / per, cudaGetErrorString(e));
  cudaFree(d_out);
}

int main() {
  for (int v = 0; v < 4; ++v) {
    run<96>(148, v);
    run<160>(148, v);
    run<256>(148, v);
  }
  return 0;
}
