// tcgen05.mma throughput microbenchmark (development aid).  One CTA per SM;
// one warp runs the issue loop (descriptors warp-uniform), an elected lane
// issues ITER groups of 8 MMAs (K = 8 x 16), then commits and waits.
// Reports cycles per MMA instruction for the operand configurations the
// attention kernel can use.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench mma_bench.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2509_16518_b200/csrc/ptx.cuh"

using namespace fga;

constexpr int ITER = 512;

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) mbench(long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 192 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 192 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(slot, 512);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 1) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    constexpr int N = MODE == 1 ? 256 : (MODE == 4 || MODE == 5) ? 64 : 128;
    constexpr uint32_t idesc = idesc_bf16(128, N, false, MODE == 3 || MODE == 5);
    long long t0 = clock64();
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        uint64_t bd;
        if constexpr (MODE == 3 || MODE == 5) bd = sdesc(b + kk * 2048, 16384, 1024, 2);
        else bd = sdesc(b + off, 16, 1024, 2);
        const uint64_t ad = sdesc(a + off, 16, 1024, 2);
        if (elect_one()) {
          if constexpr (MODE == 2 || MODE == 3 || MODE == 5)
            umma_ts(tmem + 256, tmem + 384 + kk * 8, bd, idesc, kk > 0);
          else
            umma_ss(tmem, ad, bd, idesc, kk > 0);
        }
        __syncwarp();
      }
    }
    long long t1 = clock64();
    if (elect_one()) umma_commit(bar);
    __syncwarp();
    mbar_wait(bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 32) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int MODE>
void run(const char* name, int n, long long* d) {
  cudaFuncSetAttribute(mbench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  mbench<MODE><<<148, 128, 200 * 1024>>>(d);
  mbench<MODE><<<148, 128, 200 * 1024>>>(d);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double per = double(h[1]) / (ITER * 8);
  const double ideal = 128.0 * n / 256.0;
  printf("%-30s issue %6.1f  complete %6.1f cyc/MMA  ideal %4.0f -> %3.0f%% of peak (%s)\n", name,
         double(h[0]) / (ITER * 8), per, ideal, 100.0 * ideal / per, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<0>("SS M128 N128", 128, d);
  run<1>("SS M128 N256", 256, d);
  run<2>("TS M128 N128 B K-major", 128, d);
  run<3>("TS M128 N128 B MN-major", 128, d);
  run<4>("SS M128 N64", 64, d);
  run<5>("TS M128 N64 B MN-major", 64, d);
  return 0;
}
