// MUFU ex2 throughput on one SM: f32 vs packed bf16x2 and f16x2 ex2.approx (all 16 exps/clk/SM on B200).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ex2_rate ex2_rate.cu && ./ex2_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  uint32_t r[8];
  for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(-0.001f * (threadIdx.x + i));
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[i]));
      else if (MODE == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[i]));
      else asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[i]));
    }
  }
  const long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __uint_as_float(r[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 12);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int threads : {128, 256, 512, 1024}) {
      if (mode == 0) k<0><<<1, threads>>>(out, cyc, iters); else if (mode == 1) k<1><<<1, threads>>>(out, cyc, iters); else k<2><<<1, threads>>>(out, cyc, iters);
      if (mode == 0) k<0><<<1, threads>>>(out, cyc, iters); else if (mode == 1) k<1><<<1, threads>>>(out, cyc, iters); else k<2><<<1, threads>>>(out, cyc, iters);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double instr = double(threads / 32) * iters * 8;  // warp instructions
      const double elems = instr * 32 * (mode ? 2 : 1);
      printf("%s threads %4d: %.2f cycles per warp-instr per SM, %.1f exps/clk/SM\n", mode == 2 ? "f16x2 " : mode ? "bf16x2" : "f32   ",
             threads, c / instr, elems / c);
    }
  return 0;
}
