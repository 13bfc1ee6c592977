// Gather-load microbenchmark v2 (development aid): L2 -> SMEM throughput of
// packing 128 listed 256-byte K/V rows into 32 KB SW128 slots, with the
// realistic access pattern of the attention kernel (all 148 CTAs reading one
// head's K and V, each chunk = 128 consecutive entries of a sorted random
// 45%-dense key list).
//   mode 0 CP   : cp.async 16 B, all NW warps cooperate on every item
//   mode 1 CPW  : cp.async 16 B, one warp per item (items round-robin over warps)
//   mode 2 G4W  : TMA tile::gather4, one warp per item (32 lanes x 2 gather4)
//   mode 3 ROW  : TMA 2D box {64 cols x 1 row} per row half, one warp per item
//   mode 4 BULK : cp.async.bulk 1D 256 B per row (linear dst: bandwidth only)
//   mode 5 BOX  : TMA 2D box 128 contiguous rows (dense reference)
//   mode 6 G4S  : gather4, one warp per item, only lane 0..7 issue (8 rows/lane)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gather_bench2 gather_bench2.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#include "../paper_2509_16518_b200/csrc/ptx.cuh"

using namespace fga;

constexpr int HALF = 128 * 128;
constexpr int SLOT = 2 * HALF;  // 128 rows x 256 B

struct Args {
  const int* idx;       // [groups, per_group] sorted lists
  int per_group;        // keys per list (multiple of 128)
  int groups;
  const uint8_t* k;     // [rows, 256 B]
  const uint8_t* v;
  int chunks_per_cta;
  int mode, nslot, nw;
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(32 * 25, 1) gbench(const __grid_constant__ CUtensorMap tk,
                                                    const __grid_constant__ CUtensorMap tv,
                                                    const __grid_constant__ CUtensorMap tkb,
                                                    const __grid_constant__ CUtensorMap tvb, Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.nslot * SLOT);
  uint64_t* empty = full + 16;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool coop = a.mode == 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.nslot; ++i) {
      mbar_init(&full[i], coop ? 32 * a.nw : (a.mode == 1 ? 32 : 1));
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int n_items = 2 * a.chunks_per_cta;
  const int g = blockIdx.x % a.groups;
  const int* list = a.idx + static_cast<int64_t>(g) * a.per_group;
  const int chunks_in_list = a.per_group / 128;
  const uint64_t pol = policy_evict_last();
  if (warp < a.nw) {
    for (int item = coop ? 0 : warp; item < n_items; item += coop ? 1 : a.nw) {
      const int slot = item % a.nslot, use = item / a.nslot;
      mbar_wait(&empty[slot], (use & 1) ^ 1);
      const int kv = item & 1;
      const int* ix = list + ((item >> 1) % chunks_in_list) * 128;
      const uint8_t* src = kv ? a.v : a.k;
      const CUtensorMap* tm = kv ? &tv : &tk;
      uint8_t* dst = smem + slot * SLOT;
      if (a.mode == 0) {
        const int t = warp * 32 + lane, nt = a.nw * 32;
        for (int e = t; e < 128 * 16; e += nt) {
          const int row = e >> 4, ch = e & 15;
          const int key = __ldg(ix + row);
          const int h = ch >> 3, c = ch & 7;
          cp_async16(smem_u32(dst + h * HALF + row * 128 + ((c ^ (row & 7)) << 4)),
                     src + static_cast<int64_t>(key) * 256 + ch * 16, 16);
        }
        cp_async_arrive_noinc(&full[slot]);
      } else if (a.mode == 1) {
        const int ch = lane & 15, h = ch >> 3, c = ch & 7;
        int keys[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) keys[i] = __ldg(ix + i * 32 + lane);
#pragma unroll 8
        for (int r2 = 0; r2 < 64; ++r2) {
          const int row = 2 * r2 + (lane >> 4);
          const int key = __shfl_sync(0xffffffffu, keys[row >> 5], row & 31);
          cp_async16(smem_u32(dst + h * HALF + row * 128 + ((c ^ (row & 7)) << 4)),
                     src + static_cast<int64_t>(key) * 256 + ch * 16, 16);
        }
        cp_async_arrive_noinc(&full[slot]);
      } else if (a.mode == 2 || a.mode == 6) {
        const int lanes = a.mode == 2 ? 32 : 8;
        const int per = 32 / lanes;  // gather4 groups per lane
        if (lane == 0) mbar_expect_tx(&full[slot], SLOT);
        __syncwarp();
        if (lane < lanes) {
          for (int q = 0; q < per; ++q) {
            const int r = (lane * per + q) * 4;
            const int4 kk = *reinterpret_cast<const int4*>(ix + r);
            tma_gather4(dst + r * 128, tm, &full[slot], 0, kk.x, kk.y, kk.z, kk.w, pol);
            tma_gather4(dst + HALF + r * 128, tm, &full[slot], 64, kk.x, kk.y, kk.z, kk.w, pol);
          }
        }
      } else if (a.mode == 3) {
        if (lane == 0) mbar_expect_tx(&full[slot], SLOT);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = i * 32 + lane;
          const int key = __ldg(ix + row);
          tma_load_2d(dst + row * 128, tm, &full[slot], 0, key, pol);
          tma_load_2d(dst + HALF + row * 128, tm, &full[slot], 64, key, pol);
        }
      } else if (a.mode == 4) {
        if (lane == 0) mbar_expect_tx(&full[slot], SLOT);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = i * 32 + lane;
          const int key = __ldg(ix + row);
          bulk_g2s(smem_u32(dst + row * 256), src + static_cast<int64_t>(key) * 256, 256, &full[slot]);
        }
      } else if (a.mode == 5) {
        if (lane == 0) {
          mbar_expect_tx(&full[slot], SLOT);
          const int row = ix[0] & ~127;
          tma_load_2d(dst, kv ? &tvb : &tkb, &full[slot], 0, row, pol);
          tma_load_2d(dst + HALF, kv ? &tvb : &tkb, &full[slot], 64, row, pol);
        }
      }
    }
  } else if (warp == a.nw && lane == 0) {
    for (int item = 0; item < n_items; ++item) {
      const int slot = item % a.nslot, use = item / a.nslot;
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
  const int rows = 32760;
  const double dens = argc > 1 ? atof(argv[1]) : 0.45;
  const int per_group = (static_cast<int>(dens * rows) / 128) * 128;
  const int groups = 256;
  const int chunks_per_cta = 400;
  const int grid = 148;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(p);
  uint8_t *k, *v;
  cudaMalloc(&k, static_cast<size_t>(rows) * 256);
  cudaMalloc(&v, static_cast<size_t>(rows) * 256);
  cudaMemset(k, 1, static_cast<size_t>(rows) * 256);
  cudaMemset(v, 2, static_cast<size_t>(rows) * 256);
  std::vector<int> h(static_cast<size_t>(groups) * per_group);
  std::mt19937 rng(1);
  std::vector<int> perm(rows);
  for (int gi = 0; gi < groups; ++gi) {
    std::iota(perm.begin(), perm.end(), 0);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::sort(perm.begin(), perm.begin() + per_group);
    std::copy(perm.begin(), perm.begin() + per_group, h.begin() + static_cast<size_t>(gi) * per_group);
  }
  int* idx;
  cudaMalloc(&idx, h.size() * 4);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tk, tv, tkb, tvb;
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  cuuint64_t str[1] = {256};
  cuuint32_t box1[2] = {64, 1}, boxb[2] = {64, 128}, es[2] = {1, 1};
  const auto prom = argc > 2 && atoi(argv[2]) == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  enc(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, dims, str, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, v, dims, str, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tkb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, dims, str, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tvb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, v, dims, str, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(gbench, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * SLOT + 512);
  printf("rows=%d density=%.2f keys/list=%d promotion=%s\n", rows, dens, per_group,
         prom == CU_TENSOR_MAP_L2_PROMOTION_NONE ? "none" : "256B");
  struct Cfg { int mode, nslot, nw; const char* name; };
  const Cfg cfgs[] = {
      {5, 4, 1, "BOX  dense 128-row box"}, {5, 6, 2, "BOX  dense, 2 warps"},
      {0, 4, 8, "CP   coop"},  {0, 5, 11, "CP   coop"}, {0, 5, 15, "CP   coop"}, {0, 6, 16, "CP   coop"},
      {0, 6, 20, "CP   coop"}, {0, 6, 24, "CP   coop"},
      {1, 4, 4, "CPW  warp/item"}, {1, 6, 6, "CPW  warp/item"}, {1, 3, 3, "CPW  warp/item"},
      {2, 4, 1, "G4W  gather4 warp/item"}, {2, 4, 2, "G4W  gather4 warp/item"}, {2, 6, 3, "G4W  gather4 warp/item"},
      {2, 6, 6, "G4W  gather4 warp/item"}, {2, 3, 3, "G4W  gather4 warp/item"},
      {6, 6, 6, "G4S  gather4 8 lanes"},
      {3, 4, 2, "ROW  tma box 1 row"}, {3, 6, 6, "ROW  tma box 1 row"},
      {4, 4, 2, "BULK 1D 256B/row"}, {4, 6, 6, "BULK 1D 256B/row"},
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const auto& c : cfgs) {
    Args ar{idx, per_group, groups, k, v, chunks_per_cta, c.mode, c.nslot, c.nw};
    const int threads = 32 * (c.nw + 1);
    const int sm = c.nslot * SLOT + 512;
    gbench<<<grid, threads, sm>>>(tk, tv, tkb, tvb, ar);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) gbench<<<grid, threads, sm>>>(tk, tv, tkb, tvb, ar);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = static_cast<double>(reps) * grid * chunks_per_cta * 2 * SLOT;
    const cudaError_t err = cudaGetLastError();
    printf("%-26s nslot=%d nw=%2d  %7.3f ms  %7.1f GB/s  %5.1f B/clk/SM@1.965GHz  %s\n", c.name, c.nslot, c.nw,
           ms / reps, bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / grid / 1.965e9, cudaGetErrorString(err));
    if (err != cudaSuccess) return 1;
  }
  return 0;
}
