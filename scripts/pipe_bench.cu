// Pipe microbenchmark (development aid): cycles per warp instruction for MUFU.EX2,
// F2FP.BF16 pack, FFMA2, integer bf16 packing, and mixes, with 1 or 2 warps per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void kern(float* out, long long* cyc, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i * 0.01f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int n = 0; n < iters; ++n) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) {  // 2 MUFU
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
      } else if (MODE == 1) {  // 1 F2FP
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
        acc += r;
      } else if (MODE == 2) {  // 2 MUFU + 1 F2FP
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
        acc += r;
      } else if (MODE == 3) {  // 1 FFMA2
        float2 x = make_float2(a[i], a[i + 1]);
        x = __ffma2_rn(x, make_float2(1.0001f, 1.0001f), make_float2(0.5f, 0.5f));
        a[i] = x.x; a[i + 1] = x.y;
      } else if (MODE == 4) {  // integer RNE bf16 pack (3 ALU + PRMT)
        uint32_t u0 = __float_as_uint(a[i]), u1 = __float_as_uint(a[i + 1]);
        u0 += 0x7FFFu + ((u0 >> 16) & 1u);
        u1 += 0x7FFFu + ((u1 >> 16) & 1u);
        acc += __byte_perm(u0, u1, 0x7632);
        a[i] = __uint_as_float(u0 ^ 0x10);
        a[i + 1] = __uint_as_float(u1 ^ 0x10);
      } else if (MODE == 5) {  // truncating pack: PRMT only
        acc += __byte_perm(__float_as_uint(a[i]), __float_as_uint(a[i + 1]), 0x7632);
        a[i] = __uint_as_float(__float_as_uint(a[i]) + 1);
      } else if (MODE == 7) {  // 2 MUFU + 1 FFMA2 (independent)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        float2 x = make_float2(a[(i + 4) & 15], a[(i + 5) & 15]);
        x = __ffma2_rn(x, make_float2(1.0001f, 1.0001f), make_float2(0.5f, 0.5f));
        a[(i + 4) & 15] = x.x; a[(i + 5) & 15] = x.y;
      } else if (MODE == 8) {  // 2 MUFU + 2 FFMA (scalar, independent)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        a[(i + 4) & 15] = fmaf(a[(i + 4) & 15], 1.0001f, 0.5f);
        a[(i + 5) & 15] = fmaf(a[(i + 5) & 15], 1.0001f, 0.5f);
      } else if (MODE == 9) {  // 2 MUFU + 2 FFMA2 + 1 F2FP (the softmax pair mix)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        float2 x = make_float2(a[(i + 4) & 15], a[(i + 5) & 15]);
        x = __ffma2_rn(x, make_float2(1.0001f, 1.0001f), make_float2(0.5f, 0.5f));
        float2 y = make_float2(a[(i + 8) & 15], a[(i + 9) & 15]);
        y = __fadd2_rn(y, make_float2(0.5f, 0.5f));
        a[(i + 4) & 15] = x.x; a[(i + 5) & 15] = x.y; a[(i + 8) & 15] = y.x; a[(i + 9) & 15] = y.y;
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
        acc += r;
      } else if (MODE == 6) {  // 1 FMNMX3
        float m;
        asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(a[i]), "f"(a[i + 1]), "f"(a[(i + 2) & 15]));
        a[i] = m;
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps, int per_iter_instr) {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  kern<MODE><<<148, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  // per SMSP: warps/4 warps, each iters*8*per_iter_instr instructions
  const double instr_per_smsp = (warps / 4.0) * iters * 8 * per_iter_instr;
  printf("%-34s warps=%2d  %6.2f cycles per warp-instr per SMSP\n", name, warps, h / instr_per_smsp);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("MUFU.EX2", w, 2);
    run<1>("F2FP.BF16 pack", w, 1);
    run<2>("2 MUFU + 1 F2FP (per 3 instr)", w, 3);
    run<3>("FFMA2", w, 1);
    run<4>("int RNE pack (~8 instr)", w, 8);
    run<5>("PRMT pack + IADD", w, 2);
    run<6>("FMNMX3", w, 1);
    run<7>("2 MUFU + 1 FFMA2 (per 3)", w, 3);
    run<8>("2 MUFU + 2 FFMA (per 4)", w, 4);
    run<9>("2 MUFU+FFMA2+FADD2+F2FP (per 5)", w, 5);
  }
  return 0;
}
