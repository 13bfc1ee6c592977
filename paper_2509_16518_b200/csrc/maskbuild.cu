// K1a: slice-mask construction on the GPU (the step before compaction).
//
//   fga_pooled_scores    masks.py:108-118  exp((k_j . mean_g q) * scale) / D  [bf16-rounded]
//   fga_threshold_keep   masks.py:104 / :132  keep = s >= tau
//   fga_topk_keep        masks.py:133-147  top_k largest, ties -> smaller index
//   fga_cached_group_max oracle.py:45-52 + masks.py:66-72  max over a group's rows of
//                        the normalised attention map, without materialising it
//   fga_random_keep      sparse.py:216-232 count rule (device RNG, benchmark masks)
// (paths relative to /root/reference/pkg/src/sliceattn/)
//
// Scores are fp32 CUDA-core dot products with a sequential-in-d FMA chain so
// results sit within a few ulp of NumPy; keep bits are compared exactly in
// tests (report any flip with |s - tau| within ulps).
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace fga {
namespace {

__device__ __forceinline__ float bf16_rne(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float ld_bf16(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// ------------------------------------------------------------ pooled scores
// qbar[bhg, d] = (sum_{i in g} q[bh, i, d]) / rows   (sequential fp32 sum, as np.mean over axis 2)
__global__ void pooled_mean_kernel(const __nv_bfloat16* __restrict__ q, float* __restrict__ qbar, int N, int D,
                                   int M, int G) {
  const int64_t bhg = blockIdx.x;
  const int g = static_cast<int>(bhg % G);
  const int64_t bh = bhg / G;
  const int lo = g * M, hi = min(lo + M, N);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.f;
    for (int i = lo; i < hi; ++i) acc = __fadd_rn(acc, ld_bf16(q + (bh * N + i) * D + d));
    qbar[bhg * D + d] = __fdiv_rn(acc, static_cast<float>(hi - lo));
  }
}

// Same sums (each column added row by row, in order) with the group's rows -- one contiguous
// M x D bf16 block -- brought into shared memory by TMA bulk copies first: one CTA of D threads
// per group, thread = column.  Used when the block is 16-byte aligned and fits in 64 KB.  With
// parts != null it also writes the three bf16 parts of q̄ the tensor-core score pass reads
// (split3_kernel's split, parts_n = B*H*G*D elements per part).  zero_word (nullable) is set to 0
// by block 0 (the fused threshold's empty-row counter, instead of a separate memset).
constexpr int PM_MAX_BYTES = 64 * 1024;
__global__ void pooled_mean_bulk_kernel(const __nv_bfloat16* __restrict__ q, float* __restrict__ qbar, int N, int D,
                                        int M, int G, __nv_bfloat16* __restrict__ parts, int64_t parts_n,
                                        int32_t* __restrict__ zero_word) {
  if (zero_word != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *zero_word = 0;
  extern __shared__ __align__(16) __nv_bfloat16 s_rows[];
  __shared__ __align__(8) uint64_t bar;
  const int64_t bhg = blockIdx.x;
  const int g = static_cast<int>(bhg % G);
  const int64_t bh = bhg / G;
  const int lo = g * M, hi = min(lo + M, N);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bytes = static_cast<uint32_t>(hi - lo) * D * 2;
    mbar_expect_tx(&bar, bytes);
    const char* src = reinterpret_cast<const char*>(q + (bh * N + lo) * D);
    for (uint32_t off = 0; off < bytes; off += 32768u)
      bulk_g2s(reinterpret_cast<char*>(s_rows) + off, src + off, min(32768u, bytes - off), &bar);
  }
  mbar_wait(&bar, 0);
  const int d = threadIdx.x;
  float acc = 0.f;
#pragma unroll 8
  for (int i = 0; i < hi - lo; ++i) acc = __fadd_rn(acc, __bfloat162float(s_rows[i * D + d]));
  const float v = __fdiv_rn(acc, static_cast<float>(hi - lo));
  qbar[bhg * D + d] = v;
  if (parts != nullptr) split3(v, parts, parts_n, bhg * D + d);
}

// 64x64 fp32 tile of A[rows, D] . B[cols, D]^T, 256 threads, 4x4 per thread.
// A and B rows are fetched through loader functors (bf16 or fp32 sources).
constexpr int TILE = 64, DK = 32;

template <typename LA, typename LB>
__device__ __forceinline__ void dot_tile(LA la, LB lb, int D, float (&acc)[4][4]) {
  __shared__ float As[TILE][DK + 1];
  __shared__ float Bs[TILE][DK + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;
  for (int d0 = 0; d0 < D; d0 += DK) {
    for (int e = tid; e < TILE * DK; e += 256) {
      const int rr = e / DK, dd = e % DK;
      As[rr][dd] = la(rr, d0 + dd);
      Bs[rr][dd] = lb(rr, d0 + dd);
    }
    __syncthreads();
#pragma unroll 8
    for (int dd = 0; dd < DK; ++dd) {
      float a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = As[ty + 16 * r][dd];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[tx + 16 * c][dd];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = __fmaf_rn(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
}

// scores[bh, g, j] for a 128(g) x 128(j) tile, 256 threads x (8 x 8): each thread reads
// 4 float4 of the transposed SMEM tiles per d and issues 64 FMAs (FMA-bound, not LDS-bound);
// the per-score FMA chain still runs over d in ascending order.  grid: (key tiles, group tiles, B*H)
constexpr int PT = 128, PDK = 32, PPAD = 4;
__global__ void __launch_bounds__(256) pooled_scores128_kernel(const float* __restrict__ qbar,
                                                               const __nv_bfloat16* __restrict__ k,
                                                               float* __restrict__ scores,
                                                               uint16_t* __restrict__ scores16, int N, int D, int G,
                                                               float scale, int round) {
  __shared__ __align__(16) float As[PDK][PT + PPAD];  // [d][g]
  __shared__ __align__(16) float Bs[PDK][PT + PPAD];  // [d][j]
  const int64_t bh = blockIdx.z;
  const int g0 = blockIdx.y * PT, j0 = blockIdx.x * PT;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
  for (int d0 = 0; d0 < D; d0 += PDK) {
    // stage: thread t loads row (t / 2) ... 16 consecutive d of 128 rows -> transposed stores
    for (int e = tid; e < PT * PDK; e += 256) {
      const int rr = e / PDK, dd = e % PDK;
      const int g = g0 + rr, j = j0 + rr;
      As[dd][rr] = g < G ? qbar[(bh * G + g) * D + d0 + dd] : 0.f;
      Bs[dd][rr] = j < N ? ld_bf16(k + (bh * N + j) * D + d0 + dd) : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int dd = 0; dd < PDK; ++dd) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[dd][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[dd][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[dd][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[dd][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = __fmaf_rn(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
  const float dd = static_cast<float>(D);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int g = g0 + (r < 4 ? ty * 4 + r : 64 + ty * 4 + r - 4);
    if (g >= G) continue;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = j0 + (c < 4 ? tx * 4 + c : 64 + tx * 4 + c - 4);
      if (j >= N) continue;
      float s = __fdiv_rn(expf(__fmul_rn(acc[r][c], scale)), dd);
      if (scores16 != nullptr) {
        scores16[(bh * G + g) * N + j] = __bfloat16_as_ushort(__float2bfloat16_rn(s));
        continue;
      }
      if (round) s = bf16_rne(s);
      scores[(bh * G + g) * N + j] = s;
    }
  }
}


// ------------------------------------------------------------ group max of an explicit map
__global__ void group_max_map_kernel(const float* __restrict__ map, int64_t n, int64_t m, int64_t g_count,
                                     int round, float* __restrict__ gmax) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t g = blockIdx.y, bh = blockIdx.z;
  if (j >= n) return;
  const int64_t lo = g * m, hi = lo + m < n ? lo + m : n;
  const float* col = map + bh * n * n + j;
  float best = -INFINITY;
  for (int64_t i = lo; i < hi; ++i) best = fmaxf(best, col[i * n]);
  if (round) best = bf16_rne(best);
  gmax[(bh * g_count + g) * n + j] = best;
}

// ------------------------------------------------------------ threshold
__global__ void threshold_kernel(const float* __restrict__ s, int64_t n, float tau, uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    keep[i] = s[i] >= tau ? 1 : 0;
}

// ------------------------------------------------------------ top-k / random
__device__ __forceinline__ uint32_t float_key(float x) {  // order-preserving float -> uint32
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint32_t mix32(uint64_t x) {  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return static_cast<uint32_t>(x >> 32);
}

struct FloatKeys {
  const float* s;
  __device__ uint32_t operator()(int64_t row, int64_t n, int64_t i) const { return float_key(s[row * n + i]); }
};
struct HashKeys {
  uint64_t seed;
  __device__ uint32_t operator()(int64_t row, int64_t n, int64_t i) const {
    return mix32(seed * 0xD1B54A32D192ED03ull ^ (static_cast<uint64_t>(row) * n + i));
  }
};

constexpr int TK = 512;

// Keep the k largest keys of each row; among keys equal to the k-th largest,
// keep the ones with the smallest indices.  Radix select on the 32-bit ordered keys with
// digits of 12 + 12 + 8 bits (12 + 4 for rows of bf16-valued scores, detected in the first
// pass: two keys with equal top 16 bits are then equal), then one ordered pass.  The wide
// first digit spreads rows whose values share a few exponents (the builders' scores) over
// many histogram bins instead of serialising their atomics on two or three.
constexpr int TK_BINS = 4096;
#ifndef FGA_TOPK_EQ_MAX
#define FGA_TOPK_EQ_MAX 256
#endif
constexpr int TK_EQ_MAX = FGA_TOPK_EQ_MAX > 0 ? FGA_TOPK_EQ_MAX : 1;  // ties at the threshold resolved by rank counting up to this many
#ifndef FGA_TOPK_ORD_N
#define FGA_TOPK_ORD_N 81920
#endif
constexpr int TK_ORD_N = FGA_TOPK_ORD_N;  // rows up to this long resolve many ties with one block scan
template <typename Keys>
__global__ void __launch_bounds__(TK) topk_kernel(Keys keys, int64_t n, int64_t k, uint8_t* __restrict__ keep) {
  __shared__ uint32_t hist[TK_BINS];
  __shared__ uint32_t s_prefix;
  __shared__ int64_t s_rem;
  __shared__ int64_t s_wsum[TK / 32];
  __shared__ int s_warp[TK / 32];
  __shared__ int s_tot;
  __shared__ int64_t s_eqcnt;
  __shared__ int s_eqidx[TK_EQ_MAX];
  __shared__ uint32_t s_ordmask[TK_ORD_N / 32];  // per (512-key iteration, warp): ballot of tied keys
  __shared__ int s_ordcnt[TK_ORD_N / 32];        // its popcount, then its exclusive rank base
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t prefix = 0, mask = 0;
  int64_t rem = k;
  int shift = 32;
  bool bf16_row = false;
  for (int pass = 0; shift > (bf16_row ? 16 : 0); ++pass) {
    const int width = pass == 0 ? 12 : bf16_row ? 4 : (shift > 8 ? 12 : 8);
    shift -= width;
    const int nb = 1 << width;
    for (int b = tid; b < nb; b += TK) hist[b] = 0;
    __syncthreads();
    uint32_t low = 0;
    for (int64_t i = tid; i < n; i += TK) {
      const uint32_t key = keys(row, n, i);
      if (pass == 0) low |= ((key & 0x80000000u) ? key : ~key) & 0xFFFFu;
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & (nb - 1)], 1u);
    }
    if (pass == 0) bf16_row = !__syncthreads_or(low != 0);
    __syncthreads();
    // the digit b with  sum_{d > b} hist[d] < rem <= sum_{d >= b} hist[d]: thread t owns the 8 bins
    // nb-1-8t .. nb-8-8t (descending); a block scan of the segment sums finds the owner
    const int nseg = nb / 8;
    int64_t own = 0;
    if (tid < nseg) {
#pragma unroll
      for (int e = 0; e < 8; ++e) own += hist[nb - 1 - 8 * tid - e];
    }
    int64_t incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    int64_t before = 0;
    for (int w = 0; w < warp; ++w) before += s_wsum[w];
    const int64_t excl = before + incl - own;
    if (tid < nseg && excl < rem && rem <= excl + own) {
      int64_t cum = excl;
      int b = nb - 1 - 8 * tid;
      for (int e = 0; e < 7; ++e, --b) {
        const uint32_t hb = hist[b];
        if (cum + hb >= rem) break;
        cum += hb;
      }
      s_prefix = prefix | (static_cast<uint32_t>(b) << shift);
      s_rem = rem - cum;
      s_eqcnt = hist[b];  // after the last digit: the keys equal to the k-th largest
    }
    __syncthreads();
    prefix = s_prefix;
    rem = s_rem;
    mask |= static_cast<uint32_t>(nb - 1) << shift;
    __syncthreads();
  }
  if (bf16_row) prefix |= (prefix & 0x80000000u) ? 0u : 0xFFFFu;  // the low half every such key has
  // prefix is the k-th largest key; keep all larger keys and the first `rem` equal ones.
  const int64_t n_eq = s_eqcnt;  // keys equal to prefix
  if (rem == n_eq) {  // every equal key is kept: no order needed
    for (int64_t i = tid; i < n; i += TK) keep[row * n + i] = keys(row, n, i) >= prefix ? 1 : 0;
    return;
  }
  if (FGA_TOPK_EQ_MAX > 0 && n_eq <= TK_EQ_MAX) {
    // few ties: decide the rest in parallel, list the tied indices, keep the rem smallest of them
    if (tid == 0) s_tot = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += TK) {
      const uint32_t key = keys(row, n, i);
      keep[row * n + i] = key > prefix ? 1 : 0;
      if (key == prefix) s_eqidx[atomicAdd(&s_tot, 1)] = static_cast<int>(i);
    }
    __syncthreads();
    for (int e = tid; e < n_eq; e += TK) {
      const int me = s_eqidx[e];
      int rank = 0;
      for (int f = 0; f < n_eq; ++f) rank += s_eqidx[f] < me;
      if (rank < rem) keep[row * n + me] = 1;
    }
    return;
  }
  if (n <= TK_ORD_N) {
    // many ties: one coalesced pass keeps the larger keys and records, per (iteration, warp),
    // the ballot of keys equal to the threshold; one block scan over those counts in index
    // order gives every tied key its rank; the first `rem` of them are kept.
    const int nit = static_cast<int>((n + TK - 1) / TK);
    for (int it = 0; it < nit; ++it) {
      const int64_t i = static_cast<int64_t>(it) * TK + tid;
      uint32_t key = 0;
      if (i < n) key = keys(row, n, i);
      const bool eq = i < n && key == prefix;
      const unsigned bal = __ballot_sync(0xffffffffu, eq);
      if (i < n) keep[row * n + i] = key > prefix ? 1 : 0;
      if (lane == 0) {
        s_ordmask[it * (TK / 32) + warp] = bal;
        s_ordcnt[it * (TK / 32) + warp] = __popc(bal);
      }
    }
    __syncthreads();
    // exclusive scan of the nit * (TK/32) counts (iteration-major = index order)
    const int ne = nit * (TK / 32);
    const int per = (ne + TK - 1) / TK;
    int own = 0;
    for (int e = tid * per; e < min(ne, tid * per + per); ++e) own += s_ordcnt[e];
    int incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int run = incl - own;
    for (int w = 0; w < warp; ++w) run += s_warp[w];
    for (int e = tid * per; e < min(ne, tid * per + per); ++e) {
      const int c = s_ordcnt[e];
      s_ordcnt[e] = run;
      run += c;
    }
    __syncthreads();
    for (int it = 0; it < nit; ++it) {
      const uint32_t m = s_ordmask[it * (TK / 32) + warp];
      if ((m >> lane) & 1u) {
        const int rank = s_ordcnt[it * (TK / 32) + warp] + __popc(m & ((1u << lane) - 1u));
        if (rank < rem) keep[row * n + static_cast<int64_t>(it) * TK + tid] = 1;
      }
    }
    return;
  }
  int64_t taken = 0;
  for (int64_t base = 0; base < n; base += TK) {
    const int64_t i = base + tid;
    uint32_t key = 0;
    if (i < n) key = keys(row, n, i);
    const bool gt = i < n && key > prefix;
    const bool eq = i < n && key == prefix;
    const unsigned bal = __ballot_sync(0xffffffffu, eq);
    const int in_warp = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int w = 0; w < TK / 32; ++w) { const int t = s_warp[w]; s_warp[w] = run; run += t; }
      s_tot = run;
    }
    __syncthreads();
    const int64_t rank = taken + s_warp[warp] + in_warp;
    if (i < n) keep[row * n + i] = (gt || (eq && rank < rem)) ? 1 : 0;
    taken += s_tot;
    __syncthreads();
  }
}

// ------------------------------------------------------------ cached builder
// Pass 1: per query row, max_j s_ij (mode 0) or sum_j exp(s_ij - max) in fp64 (mode 1).
// grid: (query tiles, B*H); each block walks every key tile.
template <int MODE>
__global__ void __launch_bounds__(256) row_stats_kernel(const __nv_bfloat16* __restrict__ q,
                                                        const __nv_bfloat16* __restrict__ k, int N, int D,
                                                        float scale, float* __restrict__ row_max,
                                                        double* __restrict__ row_den) {
  const int64_t bh = blockIdx.y;
  const int i0 = blockIdx.x * TILE;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  __shared__ float red_f[TILE][17];
  __shared__ double red_d[TILE][17];
  float mx[4];
  double den[4];
  float mrow[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    mx[r] = -INFINITY;
    den[r] = 0.0;
    const int i = i0 + ty + 16 * r;
    mrow[r] = (MODE == 1 && i < N) ? row_max[bh * N + i] : 0.f;
  }
  for (int j0 = 0; j0 < N; j0 += TILE) {
    float acc[4][4];
    dot_tile([&](int r, int d) { const int i = i0 + r; return i < N ? ld_bf16(q + (bh * N + i) * D + d) : 0.f; },
             [&](int r, int d) { const int j = j0 + r; return j < N ? ld_bf16(k + (bh * N + j) * D + d) : 0.f; }, D,
             acc);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = j0 + tx + 16 * c;
        if (j >= N) continue;
        const float s = __fmul_rn(acc[r][c], scale);
        if (MODE == 0) mx[r] = fmaxf(mx[r], s);
        else den[r] += static_cast<double>(expf(__fsub_rn(s, mrow[r])));
      }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (MODE == 0) red_f[ty + 16 * r][tx] = mx[r];
    else red_d[ty + 16 * r][tx] = den[r];
  }
  __syncthreads();
  if (threadIdx.x < TILE) {
    const int rr = threadIdx.x, i = i0 + rr;
    if (i < N) {
      if (MODE == 0) {
        float m = -INFINITY;
        for (int t = 0; t < 16; ++t) m = fmaxf(m, red_f[rr][t]);
        row_max[bh * N + i] = m;
      } else {
        double s = 0.0;
        for (int t = 0; t < 16; ++t) s += red_d[rr][t];
        row_den[bh * N + i] = s;
      }
    }
  }
}

// Pass 2: gmax[bh, g, j] = max_{i in g} float(exp(s_ij - max_i) / den_i).  grid: (key tiles, G, B*H)
__global__ void __launch_bounds__(256) group_max_kernel(const __nv_bfloat16* __restrict__ q,
                                                        const __nv_bfloat16* __restrict__ k, int N, int D, int M,
                                                        int G, float scale, const float* __restrict__ row_max,
                                                        const double* __restrict__ row_den, int round,
                                                        float* __restrict__ gmax) {
  const int64_t bh = blockIdx.z;
  const int g = blockIdx.y, j0 = blockIdx.x * TILE;
  const int lo = g * M, hi = min(lo + M, N);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  __shared__ float red[16][TILE];
  float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int i0 = lo; i0 < hi; i0 += TILE) {
    float acc[4][4];
    dot_tile([&](int r, int d) { const int i = i0 + r; return i < hi ? ld_bf16(q + (bh * N + i) * D + d) : 0.f; },
             [&](int r, int d) { const int j = j0 + r; return j < N ? ld_bf16(k + (bh * N + j) * D + d) : 0.f; }, D,
             acc);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + ty + 16 * r;
      if (i >= hi) continue;
      const float m = row_max[bh * N + i];
      const double den = row_den[bh * N + i];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float s = __fmul_rn(acc[r][c], scale);
        const float a = static_cast<float>(static_cast<double>(expf(__fsub_rn(s, m))) / den);
        best[c] = fmaxf(best[c], a);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) red[ty][tx + 16 * c] = best[c];
  __syncthreads();
  if (threadIdx.x < TILE) {
    const int j = j0 + threadIdx.x;
    if (j < N) {
      float m = -INFINITY;
      for (int t = 0; t < 16; ++t) m = fmaxf(m, red[t][threadIdx.x]);
      if (round) m = bf16_rne(m);
      gmax[(bh * G + g) * N + j] = m;
    }
  }
}

int grid1d(int64_t n) { const int64_t b = (n + 255) / 256; return static_cast<int>(b < 148 * 32 ? b : 148 * 32); }

}  // namespace

size_t ws_pooled_bytes(const fga_shape& s) {
  const int64_t G = (s.seq_len + s.group_size - 1) / s.group_size;
  const int64_t qrows = s.batch * s.heads * G;
  return Workspace::align(sizeof(float) * qrows * s.head_dim) + Workspace::align(sizeof(__nv_bfloat16) * 3 * qrows * s.head_dim);
}

size_t ws_cached_bytes(const fga_shape& s) {
  const int64_t rows = s.batch * s.heads * s.seq_len;
  return Workspace::align(sizeof(float) * rows) + Workspace::align(sizeof(double) * rows);
}

int launch_pooled_scores(const void* q, const void* k, const fga_shape& s, int round, const PooledOut& out,
                         Workspace& ws, cudaStream_t st) {
  const int64_t B = s.batch, H = s.heads, N = s.seq_len, D = s.head_dim, M = s.group_size;
  const int64_t G = (N + M - 1) / M;
  if (D % DK != 0) return fail(FGA_EUNSUPPORTED, "pooled_scores: head_dim must be a multiple of 32");
  float* qbar = ws.take<float>(B * H * G * D);
  __nv_bfloat16* parts = ws.take<__nv_bfloat16>(3 * B * H * G * D);
  if (qbar == nullptr || parts == nullptr) return fail(FGA_EINVAL, "pooled_scores: workspace too small (fga_workspace_bytes)");
  const int64_t blk = M * D * 2;
  bool parts_ready = false;
  if (D % 8 == 0 && D <= 1024 && blk <= PM_MAX_BYTES && (reinterpret_cast<uintptr_t>(q) & 15u) == 0) {
    if (const int rc = smem_opt_in(reinterpret_cast<const void*>(pooled_mean_bulk_kernel), static_cast<int>(blk),
                                   "pooled_mean_bulk");
        rc != FGA_OK)
      return rc;
    pooled_mean_bulk_kernel<<<static_cast<unsigned>(B * H * G), static_cast<unsigned>(D), static_cast<size_t>(blk),
                              st>>>(static_cast<const __nv_bfloat16*>(q), qbar, static_cast<int>(N),
                                    static_cast<int>(D), static_cast<int>(M), static_cast<int>(G), parts, B * H * G * D,
                                    out.fix_count);
    parts_ready = true;
  } else {
    if (out.fix_count != nullptr && cudaMemsetAsync(out.fix_count, 0, sizeof(int32_t), st) != cudaSuccess)
      return check_launch("memset");
    pooled_mean_kernel<<<static_cast<unsigned>(B * H * G), 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(q), qbar, static_cast<int>(N), static_cast<int>(D), static_cast<int>(M),
        static_cast<int>(G));
  }
  const char* cc = std::getenv("FGA_POOLED_CC");  // 1: the CUDA-core tile kernel below
  if (out.keep_bits != nullptr || cc == nullptr || cc[0] != '1') {
    const int rc = launch_pooled_scores_tc(qbar, parts, parts_ready, k, s, round, out, st);
    if (rc != FGA_EUNSUPPORTED || out.keep_bits != nullptr) return rc;  // fused bits: tensor-core pass only
  }
  const float scale = s.scale > 0.f ? s.scale : 1.0f / std::sqrt(static_cast<float>(D));
  dim3 grid(static_cast<unsigned>((N + PT - 1) / PT), static_cast<unsigned>((G + PT - 1) / PT),
            static_cast<unsigned>(B * H));
  pooled_scores128_kernel<<<grid, 256, 0, st>>>(qbar, static_cast<const __nv_bfloat16*>(k), out.scores, out.scores16,
                                                static_cast<int>(N), static_cast<int>(D), static_cast<int>(G), scale,
                                                round);
  return check_launch("pooled_scores128_kernel");
}

int launch_group_max_map(const float* map, int64_t bh, int64_t n, int64_t m, int round, float* gmax,
                         cudaStream_t st) {
  if (bh < 1 || n < 1 || m < 1 || m > n) return fail(FGA_EINVAL, "group_max_map: bad shape");
  const int64_t g = (n + m - 1) / m;
  if (g > 65535 || bh > 65535) return fail(FGA_EINVAL, "group_max_map: too many groups or heads");
  dim3 grid(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(g), static_cast<unsigned>(bh));
  group_max_map_kernel<<<grid, 256, 0, st>>>(map, n, m, g, round, gmax);
  return check_launch("group_max_map_kernel");
}

int launch_threshold(const float* s, int64_t n, float tau, uint8_t* keep, cudaStream_t st) {
  if (n == 0) return FGA_OK;
  threshold_kernel<<<grid1d(n), 256, 0, st>>>(s, n, tau, keep);
  return check_launch("threshold_kernel");
}

int launch_topk(const float* s, int64_t rows, int64_t n, int64_t k, uint8_t* keep, cudaStream_t st) {
  if (k < 1 || k > n) return fail(FGA_EINVAL, "top_k must be in [1, n]");
  if (rows == 0) return FGA_OK;
  topk_kernel<<<static_cast<unsigned>(rows), TK, 0, st>>>(FloatKeys{s}, n, k, keep);
  return check_launch("topk_kernel");
}

int launch_random_keep(int64_t rows, int64_t n, int64_t count, uint64_t seed, uint8_t* keep, cudaStream_t st) {
  if (count < 1 || count > n) return fail(FGA_EINVAL, "random_keep: count must be in [1, n]");
  if (rows == 0) return FGA_OK;
  topk_kernel<<<static_cast<unsigned>(rows), TK, 0, st>>>(HashKeys{seed}, n, count, keep);
  return check_launch("topk_kernel(random)");
}

int launch_cached_group_max(const void* q, const void* k, const fga_shape& s, int round, float* gmax, Workspace& ws,
                            cudaStream_t st) {
  const int64_t B = s.batch, H = s.heads, N = s.seq_len, D = s.head_dim, M = s.group_size;
  const int64_t G = (N + M - 1) / M;
  float* row_max = ws.take<float>(B * H * N);
  double* row_den = ws.take<double>(B * H * N);  // the tensor-core passes use its first B*H*N floats (1/den)
  if (row_max == nullptr || row_den == nullptr) return fail(FGA_EINVAL, "cached_group_max: workspace too small (fga_workspace_bytes)");
  // tensor-core passes for M = 128, D in {64, 128} (maskbuild_tc.cu); FGA_CACHED_CC=1 forces this file's
  // CUDA-core passes (kept for other shapes and as a cross-check)
  const char* cc = std::getenv("FGA_CACHED_CC");
  if (cc == nullptr || cc[0] != '1') {
    const int rc = launch_cached_group_max_tc(q, k, s, round, gmax, row_max, reinterpret_cast<float*>(row_den), st);
    if (rc != FGA_EUNSUPPORTED) return rc;
  }
  if (D % DK != 0) return fail(FGA_EUNSUPPORTED, "cached_group_max: head_dim must be a multiple of 32");
  const float scale = s.scale > 0.f ? s.scale : 1.0f / std::sqrt(static_cast<float>(D));
  const auto* qb = static_cast<const __nv_bfloat16*>(q);
  const auto* kb = static_cast<const __nv_bfloat16*>(k);
  dim3 g1(static_cast<unsigned>((N + TILE - 1) / TILE), static_cast<unsigned>(B * H));
  row_stats_kernel<0><<<g1, 256, 0, st>>>(qb, kb, static_cast<int>(N), static_cast<int>(D), scale, row_max, row_den);
  row_stats_kernel<1><<<g1, 256, 0, st>>>(qb, kb, static_cast<int>(N), static_cast<int>(D), scale, row_max, row_den);
  dim3 g2(static_cast<unsigned>((N + TILE - 1) / TILE), static_cast<unsigned>(G), static_cast<unsigned>(B * H));
  group_max_kernel<<<g2, 256, 0, st>>>(qb, kb, static_cast<int>(N), static_cast<int>(D), static_cast<int>(M),
                                       static_cast<int>(G), scale, row_max, row_den, round, gmax);
  return check_launch("cached_group_max");
}

}  // namespace fga
