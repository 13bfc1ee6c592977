// Gather-load microbenchmark (development aid): how fast can one SM pack
// 128 random 256-byte K rows into a 128B-swizzled smem slot?
//   mode 0: TMA tile::gather4, all 32 lanes of one warp issue (64 instr / 32 KB)
//   mode 1: TMA tile::gather4, one lane issues all 64
//   mode 2: cp.async 16B (LDGSTS) by W producer warps + cp.async.mbarrier.arrive.noinc
//   mode 3: TMA 2D box (128 contiguous rows) -- dense reference
// A consumer warp waits for each slot and frees it immediately.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gather_bench gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2509_16518_b200/csrc/ptx.cuh"

using namespace fga;

constexpr int HALF = 128 * 128;
constexpr int SLOT = 2 * HALF;  // 128 rows x 256 B

struct Args {
  const int* idx;  // [chunks_total * 128]
  const uint8_t* src;
  int chunks_per_cta;
  int mode;
  int nslot;
  int pwarps;
};

__global__ void __launch_bounds__(32 * 17, 1) gbench(const __grid_constant__ CUtensorMap tmg,
                                                    const __grid_constant__ CUtensorMap tmb, Args a) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.nslot * SLOT);
  uint64_t* empty = full + 16;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nprod = a.mode >= 2 && a.mode != 3 ? a.pwarps : 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.nslot; ++i) {
      mbar_init(&full[i], a.mode == 2 || a.mode == 4 || a.mode == 5 ? 32 * nprod : a.mode == 6 ? 32 * (nprod - 1) + 1 : 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * a.chunks_per_cta;
  if (warp < nprod) {
    const uint64_t pol = policy_evict_last();
    for (int c = 0; c < a.chunks_per_cta; ++c) {
      const int slot = c % a.nslot, use = c / a.nslot;
      mbar_wait(&empty[slot], (use & 1) ^ 1);
      uint8_t* dst = smem + slot * SLOT;
      const int* ix = a.idx + (c0 + c) * 128;
      if (a.mode == 0 || a.mode == 1) {
        int r[4];
        for (int e = 0; e < 4; ++e) r[e] = ix[lane * 4 + e];
        if (lane == 0) mbar_expect_tx(&full[slot], SLOT);
        __syncwarp();
        if (a.mode == 0) {
          tma_gather4(dst + lane * 512, &tmg, &full[slot], 0, r[0], r[1], r[2], r[3], pol);
          tma_gather4(dst + HALF + lane * 512, &tmg, &full[slot], 64, r[0], r[1], r[2], r[3], pol);
        } else {
          for (int l = 0; l < 32; ++l) {
            int rr[4];
            for (int e = 0; e < 4; ++e) rr[e] = __shfl_sync(0xffffffffu, r[e], l);
            if (lane == 0) {
              tma_gather4(dst + l * 512, &tmg, &full[slot], 0, rr[0], rr[1], rr[2], rr[3], pol);
              tma_gather4(dst + HALF + l * 512, &tmg, &full[slot], 64, rr[0], rr[1], rr[2], rr[3], pol);
            }
          }
        }
      } else if (a.mode == 2) {
        // each producer thread copies 16-byte chunks; row r, chunk ch (0..15)
        const int t = warp * 32 + lane, nt = nprod * 32;
        for (int e = t; e < 128 * 16; e += nt) {
          const int row = e >> 4, ch = e & 15;
          const int key = __ldg(ix + row);
          const uint8_t* g = a.src + static_cast<int64_t>(key) * 256 + ch * 16;
          const int h = ch >> 3, c = ch & 7;
          uint8_t* s = dst + h * HALF + row * 128 + ((c ^ (row & 7)) << 4);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[slot])) : "memory");
      } else if (a.mode == 4) {
        // indices preloaded per warp (one LDG per lane per 32 rows), broadcast by shuffle,
        // 16 lanes per 256-byte row -> each warp instruction moves 2 rows (512 B)
        const int rw = 128 / nprod;
        int my[4];
        for (int i = 0; i < 4; ++i) my[i] = (lane + 32 * i < rw) ? __ldg(ix + warp * rw + lane + 32 * i) : 0;
        const int ch = lane & 15, hh = ch >> 3, cc = ch & 7;
#pragma unroll 4
        for (int k = 0; k < rw / 2; ++k) {
          const int rl = 2 * k + (lane >> 4);
          int key = __shfl_sync(0xffffffffu, my[0], rl & 31);
          if (rw > 32) {
            const int k1 = __shfl_sync(0xffffffffu, my[1], rl & 31);
            const int k2 = __shfl_sync(0xffffffffu, my[2], rl & 31);
            const int k3 = __shfl_sync(0xffffffffu, my[3], rl & 31);
            key = (rl >> 5) == 0 ? key : (rl >> 5) == 1 ? k1 : (rl >> 5) == 2 ? k2 : k3;
          }
          const int row = warp * rw + rl;
          const uint8_t* g = a.src + static_cast<int64_t>(key) * 256 + ch * 16;
          uint8_t* s = dst + hh * HALF + row * 128 + ((cc ^ (row & 7)) << 4);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[slot])) : "memory");
      } else if (a.mode == 5) {
        // LDG.128 -> registers -> STS.128 (swizzled), 8 loads in flight per thread
        const int t = warp * 32 + lane, nt = nprod * 32;
        for (int e0 = t; e0 < 128 * 16; e0 += 8 * nt) {
          uint4 v[8];
          int rows_[8], chs[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * nt;
            rows_[u] = e >> 4; chs[u] = e & 15;
            if (e < 128 * 16) v[u] = __ldg(reinterpret_cast<const uint4*>(a.src + static_cast<int64_t>(__ldg(ix + rows_[u])) * 256 + chs[u] * 16));
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (e0 + u * nt < 128 * 16) {
              const int row = rows_[u], h = chs[u] >> 3, c = chs[u] & 7;
              *reinterpret_cast<uint4*>(dst + h * HALF + row * 128 + ((c ^ (row & 7)) << 4)) = v[u];
            }
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(&full[slot]);
      } else if (a.mode == 6) {
        // hybrid: warp 0 gathers rows [0, RT) with gather4, warps 1.. copy the rest with cp.async
        const int RT = a.pwarps >= 5 ? 32 : 48;  // rows via TMA (multiple of 4)
        if (warp == 0) {
          int r[4];
          const int rr = lane * 4;
          for (int e = 0; e < 4; ++e) r[e] = rr + e < RT ? ix[rr + e] : 0;
          if (lane == 0) mbar_expect_tx(&full[slot], RT * 256);
          __syncwarp();
          if (rr < RT) {
            tma_gather4(dst + lane * 512, &tmg, &full[slot], 0, r[0], r[1], r[2], r[3], pol);
            tma_gather4(dst + HALF + lane * 512, &tmg, &full[slot], 64, r[0], r[1], r[2], r[3], pol);
          }
        } else {
          const int t = (warp - 1) * 32 + lane, nt = (nprod - 1) * 32;
          for (int e = RT * 16 + t; e < 128 * 16; e += nt) {
            const int row = e >> 4, ch = e & 15;
            const int key = __ldg(ix + row);
            const uint8_t* g = a.src + static_cast<int64_t>(key) * 256 + ch * 16;
            const int h = ch >> 3, c = ch & 7;
            uint8_t* sp = dst + h * HALF + row * 128 + ((c ^ (row & 7)) << 4);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sp)), "l"(g) : "memory");
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[slot])) : "memory");
        }
      } else {
        if (lane == 0) {
          mbar_expect_tx(&full[slot], SLOT);
          const int row = ix[0] & ~127;
          tma_load_2d(dst, &tmb, &full[slot], 0, row, pol);
          tma_load_2d(dst + HALF, &tmb, &full[slot], 64, row, pol);
        }
      }
    }
  } else if (warp == nprod && lane == 0) {
    for (int c = 0; c < a.chunks_per_cta; ++c) {
      const int slot = c % a.nslot, use = c / a.nslot;
      mbar_wait(&full[slot], use & 1);
      mbar_arrive(&empty[slot]);
    }
  }
  __syncthreads();
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 32760;  // rows in the gathered region (one head)
  const int chunks_per_cta = 256;
  const int grid = 148;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(p);
  uint8_t* src;
  cudaMalloc(&src, rows * 256);
  cudaMemset(src, 1, rows * 256);
  const int64_t total = static_cast<int64_t>(grid) * chunks_per_cta * 128;
  std::vector<int> h(total);
  srand(1);
  for (auto& x : h) x = rand() % rows;
  int* idx;
  cudaMalloc(&idx, total * 4);
  cudaMemcpy(idx, h.data(), total * 4, cudaMemcpyHostToDevice);
  CUtensorMap tg, tb;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t str[1] = {256};
  cuuint32_t boxg[2] = {64, 1}, boxb[2] = {64, 128}, es[2] = {1, 1};
  enc(&tg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, boxg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(gbench, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * SLOT + 1024 + 512);
  printf("rows=%lld\n", (long long)rows);
  struct Cfg { int mode, nslot, pw; const char* name; };
  Cfg cfgs[] = {{0, 4, 1, "gather4 32-lane ring4"},     {3, 4, 1, "tma box ring4 (dense)"},
                {2, 6, 8, "cp.async 8 warps ring6"},      {2, 6, 12, "cp.async 12 warps ring6"},
                {2, 6, 16, "cp.async 16 warps ring6"},    {5, 6, 8, "ldg+sts 8 warps ring6"},
                {5, 6, 16, "ldg+sts 16 warps ring6"},     {6, 6, 5, "hybrid g4(48)+4w cp.async"},
                {6, 6, 9, "hybrid g4(32)+8w cp.async"},   {6, 6, 13, "hybrid g4(32)+12w cp.async"}};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& c : cfgs) {
    Args ar{idx, src, chunks_per_cta, c.mode, c.nslot, c.pw};
    const int threads = 32 * (c.pw + 1);
    const int sm = c.nslot * SLOT + 1024 + 512;
    gbench<<<grid, threads, sm>>>(tg, tb, ar);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) gbench<<<grid, threads, sm>>>(tg, tb, ar);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 5.0 * total * 256;
    cudaError_t e = cudaGetLastError();
    printf("%-28s %8.3f ms  %7.1f GB/s  %5.1f B/clk/SM@1.9GHz  %s\n", c.name, ms / 5, bytes / (ms * 1e-3) / 1e9,
           bytes / (ms * 1e-3) / 148 / 1.9e9, cudaGetErrorString(e));
  }
  return 0;
}
