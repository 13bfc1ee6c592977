// gather_rows (/root/reference/pkg/src/sliceattn/sparse.py:95-108) on the TMA
// tile::gather4 engine: the packed tile is written back to global memory so its
// bytes can be compared bitwise with the reference.  This is the public gather
// primitive, NOT the attention kernel's producer: the hot path gathers with
// 16-byte cp.async from four producer warps (attn_ws.cu producer_half; tested by
// itself through fga_gather_ring_probe), which measured faster than gather4 issued
// from the producer warps (profiles/r02/gather4_vs_ldgsts.md).
//
// One CTA (one warp) per 128 indices.  Lane l gathers rows 4l..4l+3 of the
// chunk with one gather4 per 64-column half into a 128B-swizzled stage (the
// same SW128 image as the attention ring slots), then the warp un-swizzles it.
#include "internal.h"
#include "ptx.cuh"

namespace fga {
namespace {

constexpr int CH = 128;         // rows per CTA
constexpr int HALF = CH * 128;  // 128 rows x 64 bf16

template <int D>
__global__ void __launch_bounds__(32, 1)
    fga_gather_kernel(const __grid_constant__ CUtensorMap tm, const int32_t* __restrict__ indices, int64_t n_idx,
                      uint16_t* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (D / 64) * HALF);
  const int lane = threadIdx.x;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * CH;
  const int nvalid = static_cast<int>(n_idx - base < CH ? n_idx - base : CH);
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const int first = __ldg(indices + base);
  int r[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int i = lane * 4 + e;
    r[e] = i < nvalid ? __ldg(indices + base + i) : first;
  }
  if (lane == 0) mbar_expect_tx(bar, CH * D * 2);
  __syncwarp();
  const uint64_t pol = policy_evict_first();
#pragma unroll
  for (int h = 0; h < D / 64; ++h) tma_gather4(smem + h * HALF + lane * 512, &tm, bar, h * 64, r[0], r[1], r[2], r[3], pol);
  mbar_wait(bar, 0);
  // un-swizzle: row r, 16-byte chunk c of half h lives at h*HALF + r*128 + ((c ^ (r&7)) << 4)
  for (int row = lane; row < nvalid; row += 32) {
    uint4* dst = reinterpret_cast<uint4*>(out + (base + row) * D);
#pragma unroll
    for (int h = 0; h < D / 64; ++h)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        dst[h * 8 + c] = *reinterpret_cast<const uint4*>(smem + h * HALF + row * 128 + ((c ^ (row & 7)) << 4));
  }
}

template <int D>
int launch_d(const CUtensorMap& tm, const int32_t* idx, int64_t n_idx, void* out, cudaStream_t st) {
  const int smem = (D / 64) * HALF + 64 + 1024;
  auto kern = fga_gather_kernel<D>;
  if (const int rc = smem_opt_in(reinterpret_cast<const void*>(kern), smem, "gather"); rc != FGA_OK)
    return rc;
  const int64_t grid = (n_idx + CH - 1) / CH;
  kern<<<static_cast<unsigned>(grid), 32, smem, st>>>(tm, idx, n_idx, static_cast<uint16_t*>(out));
  return check_launch("fga_gather_kernel");
}

}  // namespace

int launch_gather(const void* matrix, int64_t rows, int64_t d, const int32_t* indices, int64_t n_idx, void* out,
                  cudaStream_t stream) {
  if (d <= 0 || d % 64 != 0 || d > 256) return fail(FGA_EUNSUPPORTED, "gather_rows: d must be 64, 128, 192 or 256");
  if (rows <= 0 || rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "gather_rows: rows out of range");
  if (n_idx == 0) return FGA_OK;
  if ((n_idx + CH - 1) / CH >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "gather_rows: too many indices");
  CUtensorMap tm;
  int rc = make_tmap_bf16_2d(&tm, matrix, rows, d, 64, 1);
  if (rc != FGA_OK) return rc;
  switch (d) {
    case 64: return launch_d<64>(tm, indices, n_idx, out, stream);
    case 128: return launch_d<128>(tm, indices, n_idx, out, stream);
    case 192: return launch_d<192>(tm, indices, n_idx, out, stream);
    default: return launch_d<256>(tm, indices, n_idx, out, stream);
  }
}

}  // namespace fga
