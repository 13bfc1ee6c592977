// FG-Attn forward on sm_100a: K2 (TMA tile::gather4 producer) + K3 (tcgen05
// consumer with S/O accumulators in TMEM and an online softmax).
//
// Semantics follow the reference sparse kernel
//   /root/reference/pkg/src/sliceattn/sparse.py:111-156  (per (b,h,g) chunk loop)
//   /root/reference/pkg/src/sliceattn/tiled.py:48-77     (online softmax + finalize)
// One work tile = up to 128 query rows of one group (b, h, g); its key list is
// consumed in chunks of 128 gathered keys.  A short last chunk is gathered
// full-width with a repeated valid key and its extra score columns are set to
// -inf, so they contribute exactly zero (sparse.py:145-146 processes it short).
//
// This file holds the host launcher (tensor maps, parameters, dispatch) and
// version 1 ("sync"), kept as a debugging reference selectable with
// FGA_ATTN_KERNEL=sync: 4 warps, thread t owns query row t (TMEM lane t), K/V
// stages double-buffered, QK^T / softmax / PV serialised inside the CTA.
// The default path is the warp-specialised kernel in attn_ws.cu.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "attn_common.cuh"

#include "internal.h"
#include "ptx.cuh"

namespace fga {

namespace {

constexpr int NST = 2;          // K/V pipeline stages
constexpr int TMEM_COLS = 256;  // S: 128 fp32 columns, O: D columns

template <int D>
struct Smem {
  static constexpr int KV = (D / 64) * HALF;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + KV;
  static constexpr int OFF_V = OFF_K + NST * KV;
  static constexpr int OFF_P = OFF_V + NST * KV;
  static constexpr int OFF_BAR = OFF_P + 2 * HALF;
  static constexpr int BYTES = OFF_BAR + 128;
  static constexpr int ALLOC = BYTES + 1024;  // 1024 B alignment slack (SW128 atoms)
};

// K2: one warp gathers chunk j (128 keys) of K and V into one stage.  Lane l
// owns keys 4l..4l+3 of the chunk and issues one gather4 per 64-column half
// per tensor; the mbarrier completes when all 2*128*D*2 bytes have landed.
template <int D>
__device__ __forceinline__ void produce_chunk(const AttnParams& p, const CUtensorMap* tmK,
                                              const CUtensorMap* tmV, const int32_t* list, int count,
                                              int row0, int j, uint8_t* ks, uint8_t* vs, uint64_t* bar,
                                              uint64_t pol, int lane) {
  const int base = j * BN;
  const int first = p.dense ? base : __ldg(list + base);
  int r[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int kk = base + lane * 4 + e;
    const int key = kk < count ? (p.dense ? kk : __ldg(list + kk)) : first;
    r[e] = row0 + key;
  }
  if (lane == 0) mbar_expect_tx(bar, 2 * BN * D * 2);
  __syncwarp();
#pragma unroll
  for (int h = 0; h < D / 64; ++h) {
    tma_gather4(ks + h * HALF + lane * 512, tmK, bar, h * 64, r[0], r[1], r[2], r[3], pol);
    tma_gather4(vs + h * HALF + lane * 512, tmV, bar, h * 64, r[0], r[1], r[2], r[3], pol);
  }
}

template <int D, bool OUT_F32>
__global__ void __launch_bounds__(128, 1)
    fga_attn_sync_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sP = smem + L::OFF_P;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);  // [NST]
  uint64_t* mma_bar = full + NST;
  uint64_t* q_bar = mma_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_bar + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  const Tile tl = decode_tile(p, p.tile_begin + blockIdx.x);
  const int q0 = tl.q0, rows = tl.rows, row0 = tl.row0, count = tl.count, nchunks = tl.nchunks;
  const int32_t* list = tl.list;

  if (tid == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1);
    mbar_init(mma_bar, 1);
    mbar_init(q_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;        // 128 columns fp32 scores
  const uint32_t tO = tmem + 128;  // D columns fp32 output accumulator
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;

  const uint64_t pol_kv = policy_evict_last();
  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_bar, BM * D * 2);
#pragma unroll
      for (int h = 0; h < D / 64; ++h) tma_load_2d(sQ + h * HALF, &tmQ, q_bar, h * 64, row0 + q0, policy_evict_first());
    }
    for (int j = 0; j < NST && j < nchunks; ++j)
      produce_chunk<D>(p, &tmK, &tmV, list, count, row0, j, sK + j * L::KV, sV + j * L::KV, &full[j], pol_kv, lane);
  }

  constexpr uint32_t IDESC_S = idesc_bf16(BM, BN, false, false);  // S = Q K^T, both K-major
  constexpr uint32_t IDESC_O = idesc_bf16(BM, D, false, true);    // O += P V, V is MN-major

  float m_run = -INFINITY, l_run = 0.f;
  uint32_t mma_phase = 0;
  mbar_wait(q_bar, 0);

  for (int j = 0; j < nchunks; ++j) {
    const int s = j % NST;
    uint8_t* ks = sK + s * L::KV;
    uint8_t* vs = sV + s * L::KV;
    mbar_wait(&full[s], (j / NST) & 1);

    // ---- S = Q K^T  (M=128, N=128, K=D; 16 deep per instruction)
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int h = kk >> 2, off = (kk & 3) * 32;
        const uint64_t a = sdesc_sw128(smem_u32(sQ + h * HALF + off), 16, 1024);
        const uint64_t b = sdesc_sw128(smem_u32(ks + h * HALF + off), 16, 1024);
        umma_ss(tS, a, b, IDESC_S, kk > 0);
      }
      umma_commit(mma_bar);
    }
    mbar_wait(mma_bar, mma_phase);
    mma_phase ^= 1;
    tc_fence_after();

    // ---- online softmax on this thread's row (tiled.py:48-70)
    uint32_t sr[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld32(tS + lane_off + c * 32, sr[c]);
    tmem_ld_wait();
    const int nvalid = min(BN, count - j * BN);
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < BN; ++c) {
      float x = __uint_as_float(sr[c >> 5][c & 31]) * p.scale_log2;
      x = c < nvalid ? x : -INFINITY;
      sr[c >> 5][c & 31] = __float_as_uint(x);
      mx = fmaxf(mx, x);
    }
    const float m_new = fmaxf(m_run, mx);
    const float alpha = ex2(m_run - m_new);  // 0 on the first chunk
    float rsum = 0.f;
    uint32_t pk[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      const float p0 = ex2(__uint_as_float(sr[(2 * c) >> 5][(2 * c) & 31]) - m_new);
      const float p1 = ex2(__uint_as_float(sr[(2 * c + 1) >> 5][(2 * c + 1) & 31]) - m_new);
      rsum += p0 + p1;
      pk[c] = pack_bf16(p0, p1);
    }
    l_run = l_run * alpha + rsum;
    m_run = m_new;

    // P (bf16) -> smem in the canonical K-major SW128 layout (A operand of PV)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const int pi = h * 32 + ch * 4;
        *reinterpret_cast<uint4*>(sP + h * HALF + tid * 128 + ((ch ^ (tid & 7)) << 4)) =
            make_uint4(pk[pi], pk[pi + 1], pk[pi + 2], pk[pi + 3]);
      }
    }
    // rescale the running O in TMEM (skipped when no row of the warp moved its max)
    if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + lane_off + c * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
        tmem_st32(tO + lane_off + c * 32, o);
      }
      tmem_st_wait();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();

    // ---- O += P V  (M=128, N=D, K=128 keys)
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk) {
        const int h = kk >> 2, off = (kk & 3) * 32;
        const uint64_t a = sdesc_sw128(smem_u32(sP + h * HALF + off), 16, 1024);
        const uint64_t b = sdesc_sw128(smem_u32(vs + kk * 16 * 128), HALF, 1024);
        umma_ss(tO, a, b, IDESC_O, (j > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit(mma_bar);
    }
    mbar_wait(mma_bar, mma_phase);
    mma_phase ^= 1;
    tc_fence_after();
    // stage s is free again: prefetch chunk j+NST into it
    if (warp == 0 && j + NST < nchunks)
      produce_chunk<D>(p, &tmK, &tmV, list, count, row0, j + NST, ks, vs, &full[s], pol_kv, lane);
  }

  // ---- epilogue: O / l  (tiled.py:73-77)
  const bool valid = tid < rows;
  const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
  const int64_t out_row = static_cast<int64_t>(row0) + q0 + tid;
#pragma unroll
  for (int c = 0; c < D / 32; ++c) {
    uint32_t o[32];
    if (nchunks > 0) {
      tmem_ld32(tO + lane_off + c * 32, o);
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = 0u;
    }
    if (valid) store_row32<OUT_F32>(p.out, out_row * D + c * 32, o, inv_l);
  }
  if (valid && p.lse != nullptr)
    p.lse[out_row] = l_run > 0.f ? m_run * 0.69314718055994531f + logf(l_run) : -INFINITY;

  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, TMEM_COLS);
}

template <int D, bool F32>
int launch_typed(const CUtensorMap* maps, const AttnParams& p, cudaStream_t stream) {
  auto kern = fga_attn_sync_kernel<D, F32>;
  const int smem = Smem<D>::ALLOC;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return check_launch("cudaFuncSetAttribute(attn)");
  kern<<<static_cast<unsigned>(p.n_tiles - p.tile_begin), 128, smem, stream>>>(maps[0], maps[1], maps[2], p);
  return check_launch("fga_attn_sync_kernel");
}

}  // namespace

int launch_attn_sync(const CUtensorMap* maps, const AttnParams& p, int d, bool out_f32, cudaStream_t stream) {
  if (d == 64) return out_f32 ? launch_typed<64, true>(maps, p, stream) : launch_typed<64, false>(maps, p, stream);
  return out_f32 ? launch_typed<128, true>(maps, p, stream) : launch_typed<128, false>(maps, p, stream);
}

int launch_attn(const void* q, const void* k, const void* v, const int32_t* idx, int64_t idx_group_stride,
                const int32_t* counts, void* o, int o_dtype, float* lse, const fga_shape& s, bool dense,
                cudaStream_t stream, int64_t tile_begin, int64_t tile_end) {
  const int64_t B = s.batch, H = s.heads, N = s.seq_len, D = s.head_dim, M = s.group_size;
  if (D != 64 && D != 128) return fail(FGA_EUNSUPPORTED, "head_dim must be 64 or 128");
  const int64_t rows = B * H * N;
  if (rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "B*H*N must be < 2^31");
  const int64_t G = (N + M - 1) / M;
  const int64_t tpg = (M + BM - 1) / BM;
  const int64_t n_tiles = B * H * G * tpg;
  if (n_tiles >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "too many tiles");
  if (tile_end < 0) tile_end = n_tiles;
  if (tile_begin < 0 || tile_begin > tile_end || tile_end > n_tiles)
    return fail(FGA_EINVAL, "tile range must satisfy 0 <= begin <= end <= B*H*G*ceil(M/128)");

  // maps: Q (128-row box), K and V (1-row box for gather4), K and V (128-row box, dense path)
  CUtensorMap maps[5];
  int rc;
  if ((rc = make_tmap_bf16_2d(&maps[0], q, rows, D, 64, BM)) != FGA_OK) return rc;
  if ((rc = make_tmap_bf16_2d(&maps[1], k, rows, D, 64, 1)) != FGA_OK) return rc;
  if ((rc = make_tmap_bf16_2d(&maps[2], v, rows, D, 64, 1)) != FGA_OK) return rc;
  if ((rc = make_tmap_bf16_2d(&maps[3], k, rows, D, 64, BN)) != FGA_OK) return rc;
  if ((rc = make_tmap_bf16_2d(&maps[4], v, rows, D, 64, BN)) != FGA_OK) return rc;

  AttnParams p{};
  p.k = k;
  p.v = v;
  p.idx = idx;
  p.idx_group_stride = idx_group_stride;
  p.counts = counts;
  p.out = o;
  p.lse = lse;
  p.tile_begin = tile_begin;
  p.n_tiles = tile_end;
  p.heads = static_cast<int>(H);
  p.seq_len = static_cast<int>(N);
  p.group_size = static_cast<int>(M);
  p.groups = static_cast<int>(G);
  p.tiles_per_group = static_cast<int>(tpg);
  const float scale = s.scale > 0.f ? s.scale : 1.0f / std::sqrt(static_cast<float>(D));
  p.scale_log2 = scale * 1.4426950408889634f;
  p.dense = dense ? 1 : 0;
  if (tile_end == tile_begin) return FGA_OK;

  const bool f32 = o_dtype == FGA_OUT_F32;
  const char* trace_file = std::getenv("FGA_TRACE");
  if (trace_file != nullptr && cudaMalloc(&p.trace, FGA_TRACE_LEN * sizeof(long long)) == cudaSuccess)
    cudaMemsetAsync(p.trace, 0, FGA_TRACE_LEN * sizeof(long long), stream);
  const char* which = std::getenv("FGA_ATTN_KERNEL");
  if (const char* ti = std::getenv("FGA_TRACE_IT")) p.trace_it = std::atoi(ti);
  if (p.trace != nullptr) {
    int rc2 = (which != nullptr && std::strcmp(which, "sync") == 0)
                  ? launch_attn_sync(maps, p, static_cast<int>(D), f32, stream)
              : (which != nullptr && std::strcmp(which, "pp") == 0)
                  ? launch_attn_pp(maps, p, static_cast<int>(D), f32, stream)
                  : launch_attn_ws(maps, q, p, static_cast<int>(D), f32, stream);
    static long long host[FGA_TRACE_LEN];
    cudaMemcpyAsync(host, p.trace, sizeof(host), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    cudaFree(p.trace);
    if (FILE* f = std::fopen(trace_file, "w")) {
      for (int j = 0; j < 64; ++j) {
        for (int k = 0; k < FGA_TRACE_SLOTS; ++k) std::fprintf(f, "%lld ", host[j * FGA_TRACE_SLOTS + k]);
        std::fprintf(f, "\n");
      }
      for (int it = 0; it < 32; ++it) {
        for (int k = 0; k < 8; ++k) std::fprintf(f, "%lld ", host[FGA_TRACE_TILE_OFF + it * 8 + k]);
        std::fprintf(f, "\n");
      }
      for (int b = 0; b < 1024; ++b)
        std::fprintf(f, "%lld %lld\n", host[FGA_TRACE_CTA_OFF + 2 * b], host[FGA_TRACE_CTA_OFF + 2 * b + 1]);
      for (int j = 0; j < 64; ++j) {
        for (int w = 0; w < 16; ++w) std::fprintf(f, "%lld ", host[FGA_TRACE_WARP_OFF + j * 16 + w]);
        std::fprintf(f, "\n");
      }
      std::fclose(f);
    }
    return rc2;
  }
  if (which != nullptr && std::strcmp(which, "sync") == 0) return launch_attn_sync(maps, p, static_cast<int>(D), f32, stream);
  if (which != nullptr && std::strcmp(which, "pp") == 0) return launch_attn_pp(maps, p, static_cast<int>(D), f32, stream);
  // groups of 129..256 rows: both tiles of a group share each gathered chunk (attn_dual.cu, 1-7%
  // faster than attn_ws.cu there); FGA_ATTN_KERNEL=ws forces attn_ws.cu
  if (which == nullptr || std::strcmp(which, "ws") != 0) {
    const int rc = launch_attn_dual(maps, p, static_cast<int>(D), f32, stream);
    if (rc != FGA_EUNSUPPORTED) return rc;
  }
  return launch_attn_ws(maps, q, p, static_cast<int>(D), f32, stream);
}

}  // namespace fga
