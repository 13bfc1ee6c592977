// MUFU.EX2 rate per SM sub-partition with 1 or 2 warps issuing the softmax's exp loop
// (FFMA2 argument, 2x MUFU.EX2, FADD2 row sum, F2FP pack), development aid:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu scripts/mufu_bench.cu && /tmp/mufu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

template <int MODE>
__global__ void bench(float* out, long long* cyc, int iters, float m) {
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = (threadIdx.x * 0.001f + i) * 0.01f;
  float acc = 0.f;
  uint32_t pk_acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float2 sc = make_float2(0.125f, 0.125f), nm = make_float2(-m, -m);
    float2 sum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      float2 x;
      if (MODE == 0 || MODE == 3) x = __ffma2_rn(make_float2(s[2 * k], s[2 * k + 1]), sc, nm);
      else x = make_float2(s[2 * k] - m, s[2 * k + 1] - m);
      float2 p;
      p.x = ex2f(x.x);
      p.y = ex2f(x.y);
      if (MODE == 0) {
        sum[k & 1] = __fadd2_rn(sum[k & 1], p);
        pk_acc ^= pack(p.x, p.y);
      } else if (MODE == 1 || MODE == 3) {
        sum[k & 1].x += p.x;
        sum[k & 1].y += p.y;
      } else if (MODE == 2) {
        pk_acc ^= pack(p.x, p.y);
      } else if (MODE == 4) {
        sum[k & 1] = __fadd2_rn(sum[k & 1], p);
      } else if (MODE == 5) {  // pack via integer ops (round-to-nearest-even by hand)
        uint32_t a = __float_as_uint(p.x), b = __float_as_uint(p.y);
        a = (a + 0x7fffu + ((a >> 16) & 1u)) >> 16;
        b = (b + 0x7fffu + ((b >> 16) & 1u)) & 0xffff0000u;
        pk_acc ^= a | b;
        sum[k & 1].x += p.x;
        sum[k & 1].y += p.y;
      }
    }
    acc += sum[0].x + sum[0].y + sum[1].x + sum[1].y;
    m += 1e-7f * acc;  // loop-carried, so iterations cannot be merged
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + pk_acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  const char* names[] = {"ffma2+ex2+fadd2+pack", "fadd+ex2+fadd", "fadd+ex2+pack", "ffma2+ex2+fadd", "fadd+ex2+fadd2", "fadd+ex2+fadd+intpack"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int wps = 1; wps <= 4; wps *= 2) {  // warps per sub-partition
      const int threads = 128 * wps;
      for (int rep = 0; rep < 2; ++rep) {
        switch (mode) {
          case 0: bench<0><<<148, threads>>>(out, cyc, iters, 1.f); break;
          case 1: bench<1><<<148, threads>>>(out, cyc, iters, 1.f); break;
          case 2: bench<2><<<148, threads>>>(out, cyc, iters, 1.f); break;
          case 3: bench<3><<<148, threads>>>(out, cyc, iters, 1.f); break;
          case 4: bench<4><<<148, threads>>>(out, cyc, iters, 1.f); break;
          default: bench<5><<<148, threads>>>(out, cyc, iters, 1.f); break;
        }
      }
      cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double exps = 128.0 * iters * 32 * wps;  // per sub-partition
      printf("mode %d (%s) warps/SMSP %d: %.1f cycles per 128-exp row per warp, %.2f ex2/clk/SMSP\n", mode,
             names[mode], wps, double(c) / iters / wps, exps / double(c));
    }
  }
  return 0;
}
