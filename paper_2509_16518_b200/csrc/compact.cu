// K1b: slice-mask compaction.  keep[row, :] (uint8) -> ascending kept key
// positions + count, bit-exact with
//   /root/reference/pkg/src/sliceattn/masks.py:75-91   (_lists_from_keep: np.nonzero,
//                                                        empty -> [argmax(scores)])
//   /root/reference/pkg/src/sliceattn/sparse.py:165-175 (export_padded: -1 tail)
//
// One CTA per (b,h,g) row.  Each thread reads one aligned 16-byte block of
// keep bytes per round, turns it into a 16-bit occupancy mask, and a
// warp-shuffle + shared-memory block scan of the popcounts gives every
// thread its output offset, so positions are written in ascending order
// without any sort.  HBM-bound: read n bytes, write 4*count (+4*(n-count)).
#include "internal.h"

namespace fga {
namespace {

constexpr int T = 256;
constexpr int W = T / 32;

__device__ __forceinline__ uint32_t nonzero_bytes(uint32_t x) {
  uint32_t m = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) m |= ((x >> (8 * e)) & 0xFFu) ? (1u << e) : 0u;
  return m;
}

__global__ void __launch_bounds__(T) fga_compact_kernel(const uint8_t* __restrict__ keep,
                                                        const float* __restrict__ scores, int64_t n,
                                                        int32_t* __restrict__ idx, int64_t stride,
                                                        int32_t* __restrict__ counts, int fill) {
  __shared__ int s_warp[W];
  __shared__ int s_total;
  __shared__ float s_bv[W];
  __shared__ int s_bi[W];
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint8_t* kr = keep + row * n;
  int32_t* out = idx + row * stride;
  const int head = static_cast<int>(reinterpret_cast<uintptr_t>(kr) & 15u);
  const uint8_t* abase = kr - head;  // 16-byte aligned
  const int64_t span = head + n;
  const int64_t nblk = (span + 15) >> 4;

  int running = 0;
  for (int64_t b0 = 0; b0 < nblk; b0 += T) {
    const int64_t blk = b0 + tid;
    uint32_t bits = 0;
    if (blk < nblk) {
      const int64_t lo = blk * 16;
      if (lo >= head && lo + 16 <= span) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(abase + lo));
        bits = nonzero_bytes(w.x) | (nonzero_bytes(w.y) << 4) | (nonzero_bytes(w.z) << 8) | (nonzero_bytes(w.w) << 12);
      } else {
#pragma unroll 4
        for (int e = 0; e < 16; ++e) {
          const int64_t pos = lo + e;
          if (pos >= head && pos < span && abase[pos] != 0) bits |= 1u << e;
        }
      }
    }
    const int cnt = __popc(bits);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int v = lane < W ? s_warp[lane] : 0;
      int sc = v;
#pragma unroll
      for (int o = 1; o < W; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, sc, o);
        if (lane >= o) sc += t;
      }
      if (lane < W) s_warp[lane] = sc - v;  // exclusive warp prefix
      if (lane == W - 1) s_total = sc;
    }
    __syncthreads();
    int off = running + s_warp[warp] + incl - cnt;
    const int key0 = static_cast<int>(blk * 16 - head);
    while (bits) {
      const int b = __ffs(bits) - 1;
      out[off++] = key0 + b;
      bits &= bits - 1;
    }
    running += s_total;
    __syncthreads();
  }

  if (running == 0 && scores != nullptr) {
    // argmax fallback, first maximum (np.argmax semantics)
    const float* sr = scores + row * n;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int64_t i = tid; i < n; i += T) {
      const float x = sr[i];
      if (x > bv || (x == bv && i < bi)) { bv = x; bi = static_cast<int>(i); }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { s_bv[warp] = bv; s_bi[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < W; ++w)
        if (s_bv[w] > bv || (s_bv[w] == bv && s_bi[w] < bi)) { bv = s_bv[w]; bi = s_bi[w]; }
      out[0] = bi == 0x7fffffff ? 0 : bi;  // all -inf / NaN rows: index 0 like np.argmax
    }
    running = 1;
  }
  if (tid == 0) counts[row] = running;
  if (fill)
    for (int64_t i = running + tid; i < n; i += T) out[i] = -1;
}

}  // namespace

int launch_compact(const uint8_t* keep, const float* scores, int64_t rows, int64_t n, int32_t* idx,
                   int64_t idx_stride, int32_t* counts, int fill, cudaStream_t stream) {
  if (rows < 0 || n <= 0 || idx_stride < n) return fail(FGA_EINVAL, "compact: need rows >= 0, n > 0, idx_stride >= n");
  if (n >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact: n must be < 2^31");
  if (rows == 0) return FGA_OK;
  if (rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact: too many rows");
  fga_compact_kernel<<<static_cast<unsigned>(rows), T, 0, stream>>>(keep, scores, n, idx, idx_stride, counts, fill);
  return check_launch("fga_compact_kernel");
}

}  // namespace fga
