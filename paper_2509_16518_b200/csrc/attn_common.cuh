// Shared definitions of the FG-Attn attention kernels (tile decode, params,
// epilogue stores).
#pragma once

#include <cuda_bf16.h>

#include <cstdint>

#include "../../include/fgattn.h"
#include "ptx.cuh"

namespace fga {

constexpr int BM = 128;         // query rows per tile (UMMA M)
constexpr int BN = 128;         // keys per chunk
constexpr int HALF = BM * 128;  // one SW128 block: 128 rows x 64 bf16 = 16 KB

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct AttnParams {
  const void* k;  // raw bf16 [B*H*N, D] (cp.async gather source)
  const void* v;
  const int32_t* idx;
  int64_t idx_group_stride;
  const int32_t* counts;
  void* out;
  float* lse;
  int64_t tile_begin;  // first tile of this launch (multi-GPU shards run tile ranges)
  int64_t n_tiles;     // one past the last tile
  int heads, seq_len, group_size, groups, tiles_per_group;
  float scale_log2;
  int dense;
  long long* trace;  // debug timeline (FGA_TRACE=<file>): CTA 0, tile iteration trace_it, clock64 per phase
  int trace_it;      // FGA_TRACE_IT (default 0)
  int32_t* status;       // nullable device word: FGA_STATUS_* bits of mask violations seen (atomicOr)
  unsigned int* sched;   // dynamic tile counter (self-resetting, attn_ws.cu); null = static stride
  const int32_t* order;  // nullable: work index -> tile offset from tile_begin (LPT order)
  long long* cta_ns;     // nullable: %globaltimer at start / end of CTA b in [2b], [2b + 1] (b < cta_ns_len / 2)
  int64_t cta_ns_len;
};
__device__ __forceinline__ void record_cta_ns(const AttnParams& p, int end) {
  if (p.cta_ns != nullptr && threadIdx.x == 0 && 2 * static_cast<int64_t>(blockIdx.x) + 1 < p.cta_ns_len)
    p.cta_ns[2 * blockIdx.x + end] = global_ns();
}

// Mask violations the kernels detect while running are ORed into p.status as the FGA_STATUS_*
// bits of fgattn.h (sparse.py:47-52 raises for these).  The kernels stay memory-safe: counts are
// clamped to [0, stride] and out-of-range keys read row 0.

// Debug timeline hooks (FGA_TRACE=<file>).  Chunk level: slot s of chunk j
// (j < 64) of CTA 0's tile iteration p.trace_it.  Tile level: slot s of CTA 0's
// tile iteration it (< 32).  CTA level: %globaltimer at start / end of every CTA.
#define FGA_TRACE_SLOTS 16
#define FGA_TRACE_TILE_OFF (64 * FGA_TRACE_SLOTS)
#define FGA_TRACE_CTA_OFF (FGA_TRACE_TILE_OFF + 32 * 8)
#define FGA_TRACE_WARP_OFF (FGA_TRACE_CTA_OFF + 2 * 1024)  // per softmax warp: p_full arrive of chunk j < 64
#define FGA_TRACE_LEN (FGA_TRACE_WARP_OFF + 64 * 16)
#ifndef FGA_TRACE_ON
#define FGA_TRACE_ON 0  // timeline hooks are compiled in only for the trace build (scripts/trace_run.py)
#endif
#if FGA_TRACE_ON
#define FGA_TS(p, it, j, slot)                                                                         \
  do {                                                                                                  \
    if ((p).trace != nullptr && blockIdx.x == 0 && (it) == (p).trace_it && (j) < 64)                    \
      (p).trace[(j) * FGA_TRACE_SLOTS + (slot)] = clock64();                                            \
  } while (0)
#define FGA_TT(p, it, slot)                                                                            \
  do {                                                                                                  \
    if ((p).trace != nullptr && blockIdx.x == 0 && (it) < 32)                                           \
      (p).trace[FGA_TRACE_TILE_OFF + (it) * 8 + (slot)] = clock64();                                    \
  } while (0)
#define FGA_TW(p, it, j, w)                                                                            \
  do {                                                                                                  \
    if ((p).trace != nullptr && blockIdx.x == 0 && (it) == (p).trace_it && (j) < 64)                    \
      (p).trace[FGA_TRACE_WARP_OFF + (j) * 16 + (w)] = clock64();                                       \
  } while (0)
#else
#define FGA_TW(p, it, j, w) \
  do {                      \
  } while (0)
#define FGA_TS(p, it, j, slot) \
  do {                         \
  } while (0)
#define FGA_TT(p, it, slot) \
  do {                      \
  } while (0)
#endif

// One work tile: <=128 query rows of group (b,h,g) and that group's key list.
struct Tile {
  int64_t bhg;
  int q0;       // first query row within the head
  int rows;     // valid query rows in this tile
  int row0;     // first row of head (b,h) in the [B*H*N, D] view
  int count;    // keys in the list (clamped to [0, stride])
  int nchunks;  // ceil(count / BN)
  int32_t bad;  // FGA_STATUS_* bits of this tile's count
  const int32_t* list;
};

__device__ __forceinline__ Tile decode_tile(const AttnParams& p, int64_t tile) {
  Tile t;
  const int sub = static_cast<int>(tile % p.tiles_per_group);
  t.bhg = tile / p.tiles_per_group;
  const int g = static_cast<int>(t.bhg % p.groups);
  const int64_t bh = t.bhg / p.groups;
  t.q0 = g * p.group_size + sub * BM;
  const int q_end = min(g * p.group_size + p.group_size, p.seq_len);
  t.rows = min(BM, q_end - t.q0);
  t.row0 = static_cast<int>(bh * p.seq_len);
  t.bad = 0;
  if (p.dense) {
    t.count = p.seq_len;
  } else {
    const int c = __ldg(p.counts + t.bhg);
    t.bad = (c < 1 ? FGA_STATUS_EMPTY : 0) | (c > p.idx_group_stride ? FGA_STATUS_STRIDE : 0);
    t.count = static_cast<int>(min(static_cast<int64_t>(max(c, 0)), p.idx_group_stride));
  }
  t.nchunks = (t.count + BN - 1) / BN;
  t.list = p.dense ? nullptr : p.idx + t.bhg * p.idx_group_stride;
  return t;
}

// Store N (multiple of 8) fp32 accumulator columns (scaled) of one output row.
template <bool OUT_F32, int N>
__device__ __forceinline__ void store_row(void* out, int64_t off, const uint32_t (&o)[N], float scale) {
  if constexpr (OUT_F32) {
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(out) + off);
#pragma unroll
    for (int i = 0; i < N / 4; ++i)
      dst[i] = make_float4(__uint_as_float(o[4 * i]) * scale, __uint_as_float(o[4 * i + 1]) * scale,
                           __uint_as_float(o[4 * i + 2]) * scale, __uint_as_float(o[4 * i + 3]) * scale);
  } else {
    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + off);
#pragma unroll
    for (int i = 0; i < N / 8; ++i)
      dst[i] = make_uint4(pack_bf16(__uint_as_float(o[8 * i]) * scale, __uint_as_float(o[8 * i + 1]) * scale),
                          pack_bf16(__uint_as_float(o[8 * i + 2]) * scale, __uint_as_float(o[8 * i + 3]) * scale),
                          pack_bf16(__uint_as_float(o[8 * i + 4]) * scale, __uint_as_float(o[8 * i + 5]) * scale),
                          pack_bf16(__uint_as_float(o[8 * i + 6]) * scale, __uint_as_float(o[8 * i + 7]) * scale));
  }
}
template <bool OUT_F32>
__device__ __forceinline__ void store_row32(void* out, int64_t off, const uint32_t (&o)[32], float scale) {
  store_row<OUT_F32, 32>(out, off, o, scale);
}

int launch_attn_ws(const CUtensorMap* maps, const void* q, const AttnParams& p, int d, bool out_f32,
                   cudaStream_t stream);
int launch_attn_dual(const CUtensorMap* maps, const AttnParams& p, int d, bool out_f32, cudaStream_t stream);
int launch_ring_probe(const AttnParams& p, int d, void* out_k, void* out_v, cudaStream_t stream);

// Producer-side memory safety.  The producers load their keys before waiting for a free ring
// slot (the load latency hides behind the wait); clamp_key() then maps a listed key to
// min(key, N-1) as unsigned (a negative or too large key reads a valid row, never out of bounds)
// and returns -1 (the zero-fill sentinel) past the list end: one IMNMX per key.  Range and order
// violations are reported by the validation kernel (fga_validate_mask, or FGA_ATTN_CHECK), not
// here: an in-kernel vote per chunk measured 2% on the producers, which bound the kernel.
// report_tile() ORs a tile's count violations into p.status (once per tile).
__device__ __forceinline__ int clamp_key(const AttnParams& p, int key, bool listed) {
  return listed ? static_cast<int>(min(static_cast<unsigned>(key), static_cast<unsigned>(p.seq_len - 1))) : -1;
}
__device__ __forceinline__ void report_tile(const AttnParams& p, const Tile& t) {
  if (t.bad && p.status != nullptr) atomicOr(p.status, t.bad);
}

}  // namespace fga
