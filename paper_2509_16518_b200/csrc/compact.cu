// K1b: slice-mask compaction.  keep[row, :] (uint8) -> ascending kept key
// positions + count, bit-exact with
//   /root/reference/pkg/src/sliceattn/masks.py:75-91   (_lists_from_keep: np.nonzero,
//                                                        empty -> [argmax(scores)])
//   /root/reference/pkg/src/sliceattn/sparse.py:165-175 (export_padded: -1 tail)
//
// Two input formats: uint8 keep bytes (fga_compact) and bit-packed keep words
// (fga_compact_bits, 8x fewer bytes to read or to ship from the host).
//
// One CTA per (b,h,g) row.  Each thread reads one aligned 16-byte block of
// keep bytes per round, turns it into a 16-bit occupancy mask, and a
// warp-shuffle + shared-memory block scan of the popcounts gives every
// thread its offset in a shared-memory stage, so positions come out in
// ascending order without any sort and leave the CTA as coalesced stores.
// HBM-bound: read n bytes (n/8 for bits), write 4*count (+4*(n-count)).
#include "internal.h"

namespace fga {
namespace {

constexpr int T = 256;
#ifndef FGA_COMPACT_T
#define FGA_COMPACT_T 256
#endif
constexpr int TC = FGA_COMPACT_T;  // keep-byte kernel: threads per row (one 16-byte block each per round)
constexpr int WC = TC / 32;
constexpr int W = T / 32;

__device__ __forceinline__ uint32_t nonzero_bytes(uint32_t x) {
  uint32_t m = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) m |= ((x >> (8 * e)) & 0xFFu) ? (1u << e) : 0u;
  return m;
}

__global__ void __launch_bounds__(TC) fga_compact_kernel(const uint8_t* __restrict__ keep,
                                                        const float* __restrict__ scores, int64_t n,
                                                        int32_t* __restrict__ idx, int64_t stride,
                                                        int32_t* __restrict__ counts, int fill) {
  __shared__ int s_warp[WC];
  __shared__ int s_total;
  __shared__ float s_bv[WC];
  __shared__ int s_bi[WC];
  __shared__ int s_stage[TC * 16];  // one round's positions, written out coalesced
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint8_t* kr = keep + row * n;
  int32_t* out = idx + row * stride;
  const int head = static_cast<int>(reinterpret_cast<uintptr_t>(kr) & 15u);
  const uint8_t* abase = kr - head;  // 16-byte aligned
  const int64_t span = head + n;
  const int64_t nblk = (span + 15) >> 4;

  // the next round's 16-byte block is loaded before this round's scan (two loads in flight)
  auto load = [&](int64_t blk) -> uint4 {
    const int64_t lo = blk * 16;
    return (blk < nblk && lo >= head && lo + 16 <= span) ? __ldg(reinterpret_cast<const uint4*>(abase + lo))
                                                         : make_uint4(0u, 0u, 0u, 0u);
  };
  uint4 wn = load(tid);
  int running = 0;
  for (int64_t b0 = 0; b0 < nblk; b0 += TC) {
    const int64_t blk = b0 + tid;
    const uint4 w = wn;
    wn = load(blk + TC);
    uint32_t bits = 0;
    if (blk < nblk) {
      const int64_t lo = blk * 16;
      if (lo >= head && lo + 16 <= span) {
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
      const int v = lane < WC ? s_warp[lane] : 0;
      int sc = v;
#pragma unroll
      for (int o = 1; o < WC; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, sc, o);
        if (lane >= o) sc += t;
      }
      if (lane < WC) s_warp[lane] = sc - v;  // exclusive warp prefix
      if (lane == WC - 1) s_total = sc;
    }
    __syncthreads();
    int off = s_warp[warp] + incl - cnt;
    const int key0 = static_cast<int>(blk * 16 - head);
    while (bits) {
      s_stage[off++] = key0 + __ffs(bits) - 1;
      bits &= bits - 1;
    }
    __syncthreads();
    const int total = s_total;
    for (int i = tid; i < total; i += TC) out[running + i] = s_stage[i];
    running += total;
    __syncthreads();
  }

  if (running == 0 && scores != nullptr) {
    // argmax fallback, first maximum (np.argmax semantics)
    const float* sr = scores + row * n;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int64_t i = tid; i < n; i += TC) {
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
      for (int w = 1; w < WC; ++w)
        if (s_bv[w] > bv || (s_bv[w] == bv && s_bi[w] < bi)) { bv = s_bv[w]; bi = s_bi[w]; }
      out[0] = bi == 0x7fffffff ? 0 : bi;  // all -inf / NaN rows: index 0 like np.argmax
    }
    running = 1;
  }
  if (tid == 0) counts[row] = running;
  if (fill)
    for (int64_t i = running + tid; i < n; i += TC) out[i] = -1;
}

// ---------------------------------------------------------------- bit-packed masks
// keep bits: uint32 words, bit b of word w = key 32w + b.  Packing (one warp
// ballot per 32 keys) and compaction from bits: each thread scans WPT words
// per round, so a CTA covers 256 * WPT * 32 keys per round with one block scan.
__global__ void __launch_bounds__(256) fga_pack_bits_kernel(const uint8_t* __restrict__ keep, int64_t rows, int64_t n,
                                                             int64_t words, uint32_t* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t wi = warp; wi < rows * words; wi += nwarps) {
    const int64_t row = wi / words, w = wi % words;
    const int64_t key = w * 32 + lane;
    const bool on = key < n && keep[row * n + key] != 0;
    const uint32_t b = __ballot_sync(0xffffffffu, on);
    if (lane == 0) bits[wi] = b;
  }
}

constexpr int WPT = 1;

__global__ void __launch_bounds__(T) fga_compact_bits_kernel(const uint32_t* __restrict__ bits, int64_t words,
                                                             int64_t n, int32_t* __restrict__ idx, int64_t stride,
                                                             int32_t* __restrict__ counts, int fill) {
  __shared__ int s_warp[W];
  __shared__ int s_total;
  __shared__ int s_stage[T * WPT * 32];
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t* br = bits + row * words;
  int32_t* out = idx + row * stride;
  int running = 0;
  for (int64_t w0 = 0; w0 < words; w0 += int64_t(T) * WPT) {
    uint32_t m[WPT];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < WPT; ++u) {
      const int64_t w = w0 + int64_t(tid) * WPT + u;
      uint32_t v = w < words ? __ldg(br + w) : 0u;
      const int64_t k0 = w * 32;
      if (k0 + 32 > n) v &= (k0 >= n) ? 0u : ((1u << (n - k0)) - 1u);  // keys past n are not keys
      m[u] = v;
      cnt += __popc(v);
    }
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
      if (lane < W) s_warp[lane] = sc - v;
      if (lane == W - 1) s_total = sc;
    }
    __syncthreads();
    int off = s_warp[warp] + incl - cnt;
#pragma unroll
    for (int u = 0; u < WPT; ++u) {
      uint32_t v = m[u];
      const int key0 = static_cast<int>((w0 + int64_t(tid) * WPT + u) * 32);
      while (v) {
        s_stage[off++] = key0 + __ffs(v) - 1;
        v &= v - 1;
      }
    }
    __syncthreads();
    const int total = s_total;
    for (int i = tid; i < total; i += T) out[running + i] = s_stage[i];
    running += total;
    __syncthreads();
  }
  if (tid == 0) counts[row] = running;
  if (fill)
    for (int64_t i = running + tid; i < n; i += T) out[i] = -1;
}

}  // namespace

int launch_pack_bits(const uint8_t* keep, int64_t rows, int64_t n, uint32_t* bits, cudaStream_t stream) {
  if (rows < 0 || n <= 0) return fail(FGA_EINVAL, "pack_bits: need rows >= 0, n > 0");
  if (rows == 0) return FGA_OK;
  const int64_t words = (n + 31) / 32;
  const int64_t warps = rows * words;
  const int64_t blocks = (warps + 7) / 8 < 148 * 16 ? (warps + 7) / 8 : 148 * 16;
  fga_pack_bits_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(keep, rows, n, words, bits);
  return check_launch("fga_pack_bits_kernel");
}

int launch_compact_bits(const uint32_t* bits, int64_t rows, int64_t n, int32_t* idx, int64_t idx_stride,
                        int32_t* counts, int fill, cudaStream_t stream) {
  if (rows < 0 || n <= 0 || idx_stride < n) return fail(FGA_EINVAL, "compact_bits: need rows >= 0, n > 0, idx_stride >= n");
  if (n >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact_bits: n must be < 2^31");
  if (rows == 0) return FGA_OK;
  if (rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact_bits: too many rows");
  fga_compact_bits_kernel<<<static_cast<unsigned>(rows), T, 0, stream>>>(bits, (n + 31) / 32, n, idx, idx_stride,
                                                                           counts, fill);
  return check_launch("fga_compact_bits_kernel");
}

int launch_compact(const uint8_t* keep, const float* scores, int64_t rows, int64_t n, int32_t* idx,
                   int64_t idx_stride, int32_t* counts, int fill, cudaStream_t stream) {
  if (rows < 0 || n <= 0 || idx_stride < n) return fail(FGA_EINVAL, "compact: need rows >= 0, n > 0, idx_stride >= n");
  if (n >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact: n must be < 2^31");
  if (rows == 0) return FGA_OK;
  if (rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact: too many rows");
  fga_compact_kernel<<<static_cast<unsigned>(rows), TC, 0, stream>>>(keep, scores, n, idx, idx_stride, counts, fill);
  return check_launch("fga_compact_kernel");
}

// FGM1 mask payload (io.py) -> device index layout.  Row r's list
// is words[starts[r] .. starts[r] + words[starts[r] - 1]); one CTA per row copies it
// into idx[r, :len] (coalesced u32 loads / stores), writes counts[r] and optionally
// the -1 tail.  HBM-bound: 4 B read + 4 B written per index.
__global__ void fga_fgm1_unpack_kernel(const int32_t* __restrict__ words, const int64_t* __restrict__ starts, int64_t n,
                                       int32_t* __restrict__ idx, int64_t idx_stride, int32_t* __restrict__ counts,
                                       int fill) {
  const int64_t r = blockIdx.x;
  const int64_t s = starts[r];
  const int len = words[s - 1];
  int32_t* dst = idx + r * idx_stride;
  for (int i = threadIdx.x; i < len; i += blockDim.x) dst[i] = words[s + i];
  if (fill)
    for (int64_t i = len + threadIdx.x; i < n; i += blockDim.x) dst[i] = -1;
  if (threadIdx.x == 0) counts[r] = len;
}

int launch_fgm1_unpack(const int32_t* words, const int64_t* starts, int64_t rows, int64_t n, int32_t* idx,
                       int64_t idx_stride, int32_t* counts, int fill, cudaStream_t stream) {
  if (rows < 0 || n <= 0 || idx_stride < n) return fail(FGA_EINVAL, "fgm1_unpack: need rows >= 0, n > 0, idx_stride >= n");
  if (rows == 0) return FGA_OK;
  if (rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "fgm1_unpack: too many rows");
  fga_fgm1_unpack_kernel<<<static_cast<unsigned>(rows), 256, 0, stream>>>(words, starts, n, idx, idx_stride, counts,
                                                                           fill);
  return check_launch("fga_fgm1_unpack_kernel");
}

}  // namespace fga
