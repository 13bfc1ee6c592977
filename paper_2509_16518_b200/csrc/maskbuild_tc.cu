// K1a cached-threshold builder on the tensor cores (M = 128, D in {64, 128}).
//
// Reference: oracle.py:45-52 (attention_map: s = (q k^T) * scale, a = exp(s - max_row) /
// sum_row in fp64, as fp32) + masks.py:66-72 (_group_max over a group's rows, after the
// bf16 rounding of analysis_scores, core.py:196-200), used by build_mask_cached
// (masks.py:94-105); paths relative to /root/reference/pkg/src/sliceattn/.
//
// The CUDA-core version (maskbuild.cu) streams Q K^T three times through FP32 FMA chains
// (~0.4 s at Wan 480p).  Here every score tile is a tcgen05 SS-MMA (bf16 x bf16 products
// are exact in fp32; only the accumulation order differs from NumPy's BLAS) and the
// per-element work stays in fp32/fp64 on the CUDA cores:
//
//   pass 0 (rows):  S = Q_t K_c^T, thread = query row.  Running row max m and the
//                   denominator sum_j exp(s_ij - m) (per-chunk fp32 partial sums of MUFU
//                   ex2 terms, accumulated and rescaled in fp64); writes m_i and 1/den_i.
//   pass 1 (group): S^T = K_c Q_g^T, thread = key j, columns = the group's 128 queries.
//                   The transposed tile turns the column max over a group into a per-thread
//                   max: y_j = max_i s_ij - (m_i + ln den_i) (half an FFMA2 and half an FMNMX3
//                   per element, -(m_i + ln den_i) in registers), gmax_gj = expf(y_j), bf16-
//                   rounded.  exp(y) = exp(s - m) / den up to ~1e-6 relative (the rounding of
//                   m + ln den), far below a bf16 step: at N = 4000-4096 5.7-6.3e-5 of the values
//                   land one bf16 step away from NumPy's, against 4.2-5.5e-5 when the argmax
//                   query is selected and a_i*j = expf(s - m_i*) / den_i* is evaluated as the
//                   reference does (-DFGA_CB_EXACT_SELECT: 3 more instructions per element,
//                   pass 1 ~25% slower).
//
// Warps (18, one CTA per SM, persistent over (b, h, tile) units): 0-15 epilogue (four per TMEM
// lane quadrant, 32 columns each), 16 MMA issuer, 17 TMA producer (Q tile + 4-slot K ring).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "attn_common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace fga {
namespace {

#ifndef FGA_CB_POLY
#define FGA_CB_POLY 3
#endif
constexpr int CB_POLY = FGA_CB_POLY;  // pass 0: every CB_POLY-th pair of exps on the FMA pipe (0: none)
constexpr int CB_EW = 4;              // epilogue warps per TMEM lane quadrant
constexpr int CB_EPI = 4 * CB_EW;      // epilogue warps 0..15
constexpr int CB_WARPS = CB_EPI + 2;   // + MMA issuer + TMA producer
#ifdef FGA_CB_EXACT_SELECT
constexpr int CB_P1G = 1;  // pass 1: groups per unit (the exact-select variant keeps one)
#else
constexpr int CB_P1G = 2;  // pass 1: two groups per unit share every K chunk (half the L2 -> SMEM bytes)
#endif
#ifndef FGA_CB_P1N256
#define FGA_CB_P1N256 1  // pass 1: the unit's two group tiles as one N = 256 MMA per K step
#endif
#ifndef FGA_CB_P0G
#define FGA_CB_P0G 1  // 2 measured slower: 3.6 -> 4.2 ms (bitwise the same output)
#endif
constexpr int CB_P0G = FGA_CB_P0G;  // pass 0: query tiles per unit sharing every K chunk
// Q-side tiles per unit: pass 2 q̄ hi/mid/lo (accumulated into one score tile), pass 1 the unit's
// CB_P1G groups (one score tile each), pass 0 CB_P0G query tiles (one score tile each)
// (pass 3 = the argmax fix-up of a fused threshold pass: pass 2's tiles for the rows listed)
constexpr int cb_nq(int pass) { return pass >= 2 ? 3 : pass == 1 ? CB_P1G : CB_P0G; }
constexpr int cb_sbw(int pass) { return pass == 1 ? 128 * CB_P1G : pass == 0 ? 128 * CB_P0G : 128; }  // TMEM columns per S buffer
constexpr int cb_ns(int pass) { return pass >= 2 ? 3 : 4; }  // K ring slots
constexpr int CB_NS = 4;                                      // barrier slots (max ring)
constexpr int CB_SB = 4;  // S buffers in TMEM (4 x 128 columns): the MMA runs up to 3 tiles ahead
constexpr int CB_BARS = 2 + 2 * CB_NS + 2 * CB_SB;

template <int D, int PASS>
struct CbSmem {
  static constexpr int KV = (D / 64) * HALF;  // one 128-row tile
  static constexpr int NQ = cb_nq(PASS), NS = cb_ns(PASS);
  static constexpr int SBW = cb_sbw(PASS), NSB = 128 * CB_SB / SBW;  // S buffer width / count in TMEM
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = NQ * KV;
  static constexpr int OFF_BAR = OFF_K + NS * KV;
  static constexpr int OFF_TAB = OFF_BAR + 256;       // pass 1: (m_i, 1/den_i, m_i + ln den_i) per query
  static constexpr int OFF_NZ = OFF_TAB + CB_P1G * 128 * 16;  // pass 1: -(m_i + ln den_i) of the unit's groups
  static constexpr int OFF_XCH = OFF_NZ + CB_P1G * 128 * 4;     // pass 0: (m, den) per slice; pass 1: candidates x 2
  static constexpr int BYTES = OFF_XCH + 2 * 3 * CB_EW * 128 * 4;
  static_assert(CB_P0G * CB_EW * 128 * 12 <= 2 * 3 * CB_EW * 128 * 4, "exchange area");
  static_assert(BYTES <= 232448, "exceeds the 227 KB of shared memory per CTA");
  static_assert(CB_BARS * 8 + 8 <= 256, "barrier area");
};

struct CbBars {
  uint64_t *q_full, *q_empty, *k_full, *k_empty, *s_full, *s_empty;
  uint32_t* tmem_slot;
};

template <int D, int PASS>
__device__ __forceinline__ CbBars cb_bars(uint8_t* smem) {
  uint64_t* b = reinterpret_cast<uint64_t*>(smem + CbSmem<D, PASS>::OFF_BAR);
  CbBars r;
  r.q_full = b;
  r.q_empty = b + 1;
  r.k_full = b + 2;
  r.k_empty = r.k_full + CB_NS;
  r.s_full = r.k_empty + CB_NS;
  r.s_empty = r.s_full + CB_SB;
  r.tmem_slot = reinterpret_cast<uint32_t*>(r.s_empty + CB_SB);
  return r;
}

struct CbParams {
  int64_t bh;   // B * H
  int n;        // sequence length
  int tiles;    // units per (b, h): ceil(n / 128) query tiles (pass 0), ceil(G / CB_P1G) group pairs (pass 1), ceil(G / 128) group tiles (pass 2)
  int nch;      // key chunks per unit: ceil(n / 128)
  int groups;   // pass 2: G
  int64_t part_rows;  // pass 2: rows of one q̄ part (B*H*G)
  float* scores;      // pass 2: [B*H*G*N] fp32, or
  uint16_t* scores16; // pass 2: [B*H*G*N] bf16 bits (the builders' input; p.round must be 1), or
  uint32_t* keep_bits;            // pass 2: [B*H*G, words] threshold decisions (bf16 score >= tau)
  float tau;
  float a_mid, hb;                // pass 2 with keep_bits: accumulator threshold and band (threshold_band)
  const int32_t* fix_rows;        // pass 3: rows (b*h*G + g) whose threshold kept nothing
  const int32_t* fix_count;       //         their number (device)
  int32_t* fix_idx;               //         idx[row * fix_stride] = the row's argmax key
  int64_t fix_stride;
  int words;                      // ceil(N / 32)
  float scale;
  int round;
  float* row_max;  // [B*H*N]
  float* row_rinv; // [B*H*N]
  float* gmax;     // [B*H*G*N]
  long long* dbg;  // FGA_CB_TRACE builds: clock64 timeline of CTA 0's first 256 chunks (pass 0)
};

#ifdef FGA_CB_TRACE
#define CB_TS(kc, slot_) \
  do { if (PASS == 0 && p.dbg != nullptr && blockIdx.x == 0 && (kc) < 256) p.dbg[(kc) * 8 + (slot_)] = clock64(); } while (0)
#else
#define CB_TS(kc, slot_) do { } while (0)
#endif
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * CB_EPI) : "memory"); }

template <int D, int PASS>
__global__ void __launch_bounds__(32 * CB_WARPS, 1)
    cached_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const CbParams p) {
  using L = CbSmem<D, PASS>;
  extern __shared__ __align__(1024) uint8_t smem_cb[];
  uint8_t* smem = smem_cb;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  if (PASS == 3 && blockIdx.x >= *p.fix_count) return;  // (usually every CTA: no row kept nothing)
  const CbBars bar = cb_bars<D, PASS>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n_units = PASS == 3 ? static_cast<int64_t>(*p.fix_count) : p.bh * p.tiles;
  // unit u of passes 0 and 3 -> (b*h, tile t, key chunks [c_lo, c_hi))
  auto unit = [&](int64_t u, int64_t& bh, int& t, int& c_lo, int& c_hi) {
    if (PASS == 3) {  // one listed row: its group tile over every key chunk
      const int r = __ldg(p.fix_rows + u);
      bh = r / p.groups;
      t = (r % p.groups) / BM;
    } else {
      bh = u / p.tiles;
      t = static_cast<int>(u % p.tiles);
    }
    c_lo = 0;
    c_hi = p.nch;
  };
  // This CTA's units.  Passes 1 and 2 split the flattened (b*h, tile, key chunk) space into gridDim.x
  // contiguous ranges (balanced to one chunk), cut at tile boundaries: a unit is a (b*h, tile)
  // with a key chunk range.  Passes 0 (row statistics over every key) and 3 stride over whole units.
  constexpr bool FLAT = PASS == 1 || PASS == 2;
  const int64_t flat_n = p.bh * p.tiles * static_cast<int64_t>(p.nch);
  constexpr bool P1W = PASS == 1 && CB_P1G == 2 && FGA_CB_P1N256;  // pass 1 as N = 256 MMAs
  struct Seq {
    int64_t u, f, hi;
  };
  auto seq_init = [&]() {
    Seq q;
    q.u = blockIdx.x;
    q.f = flat_n * blockIdx.x / gridDim.x;
    q.hi = flat_n * (blockIdx.x + 1) / gridDim.x;
    return q;
  };
  auto seq_next = [&](Seq& q, int64_t& bh, int& t, int& c_lo, int& c_hi, int64_t& uid) -> bool {
    uid = q.u;
    if (FLAT) {
      if (q.f >= q.hi) return false;
      const int64_t r = q.f / p.nch;
      bh = r / p.tiles;
      t = static_cast<int>(r % p.tiles);
      c_lo = static_cast<int>(q.f % p.nch);
      c_hi = static_cast<int>(min(static_cast<int64_t>(p.nch), c_lo + (q.hi - q.f)));
      q.f += c_hi - c_lo;
      ++q.u;
      return true;
    }
    if (q.u >= n_units) return false;
    unit(q.u, bh, t, c_lo, c_hi);
    q.u += gridDim.x;
    return true;
  };
  if (tid == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    mbar_init(bar.q_full, 1);
    mbar_init(bar.q_empty, 1);
    for (int i = 0; i < L::NS; ++i) {
      mbar_init(&bar.k_full[i], 1);
      mbar_init(&bar.k_empty[i], 1);
    }
    for (int i = 0; i < CB_SB; ++i) {
      mbar_init(&bar.s_full[i], 1);
      mbar_init(&bar.s_empty[i], CB_EPI);
    }
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(bar.tmem_slot, 128 * CB_SB);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *bar.tmem_slot;

  if (warp == CB_EPI + 1) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first(), pol_k = policy_evict_last();
      uint32_t kc = 0;
      int it = 0;
      Seq sq = seq_init();
      int64_t bh, u;
      int t, c_lo, c_hi;
      for (; seq_next(sq, bh, t, c_lo, c_hi, u); ++it) {
        const int row0 = static_cast<int>(bh * p.n);
        mbar_wait(bar.q_empty, (it & 1) ^ 1);
        mbar_expect_tx(bar.q_full, L::NQ * BM * D * 2);
#pragma unroll
        for (int qp = 0; qp < L::NQ; ++qp) {
          const int qrow = PASS >= 2 ? static_cast<int>(qp * p.part_rows + bh * p.groups) + t * BM
                                     : row0 + (t * L::NQ + qp) * BM;  // pass 1: group CB_P1G*t + qp
#pragma unroll
          for (int h = 0; h < D / 64; ++h)
            // (pass 1 with N = 256: the groups' tiles interleaved per 64-column half, so each half
            // holds 256 consecutive rows for one B descriptor)
            tma_load_2d(smem + L::OFF_Q + (P1W ? h * L::NQ * HALF + qp * HALF : qp * L::KV + h * HALF), &tmQ,
                        bar.q_full, h * 64, qrow, pol_q);
        }
        for (int c = c_lo; c < c_hi; ++c, ++kc) {
          const uint32_t slot = kc % L::NS, use = kc / L::NS;
          CB_TS(kc, 0);
          mbar_wait(&bar.k_empty[slot], (use & 1) ^ 1);
          CB_TS(kc, 1);
          mbar_expect_tx(&bar.k_full[slot], BN * D * 2);
#pragma unroll
          for (int h = 0; h < D / 64; ++h)
            tma_load_2d(smem + L::OFF_K + slot * L::KV + h * HALF, &tmK, &bar.k_full[slot], h * 64, row0 + c * BN, pol_k);
        }
      }
    }
    __syncwarp();
  } else if (warp == CB_EPI) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t IDESC = idesc_bf16(BM, BN, false, false);  // both operands K-major in SMEM
    const uint64_t dq0 = sdesc_sw128(smem_u32(smem + L::OFF_Q), 16, 1024);
    const uint64_t dk0 = sdesc_sw128(smem_u32(smem + L::OFF_K), 16, 1024);
    uint32_t kc = 0, sc = 0;
    int it = 0;
    Seq sq = seq_init();
    int64_t bh, u;
    int t, c_lo, c_hi;
    for (; seq_next(sq, bh, t, c_lo, c_hi, u); ++it) {
      mbar_wait(bar.q_full, it & 1);
      for (int c = c_lo; c < c_hi; ++c, ++kc, ++sc) {
        const uint32_t slot = kc % L::NS, use = kc / L::NS, b = sc % L::NSB;
        CB_TS(kc, 2);
        mbar_wait(&bar.k_full[slot], use & 1);
        CB_TS(kc, 3);
        mbar_wait(&bar.s_empty[b], ((sc / L::NSB) & 1) ^ 1);
        CB_TS(kc, 4);
        tc_fence_after();
        const uint64_t dk = dk0 + ((slot * L::KV) >> 4);
        if (P1W) {
          if (elect_one()) {
            constexpr uint32_t IDESC_W = idesc_bf16(BM, 2 * BN, false, false);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = ((kk >> 2) * HALF + (kk & 3) * 32) >> 4;
              const uint32_t offq = ((kk >> 2) * 2 * HALF + (kk & 3) * 32) >> 4;
              umma_ss(tmem + b * L::SBW, dk + off, dq0 + offq, IDESC_W, kk > 0 ? 1u : 0u);
            }
            umma_commit(&bar.s_full[b]);
            umma_commit(&bar.k_empty[slot]);
            if (c == c_hi - 1) umma_commit(bar.q_empty);
          }
        } else if (elect_one()) {
#pragma unroll
          for (int qp = 0; qp < L::NQ; ++qp) {  // pass 2: S^T = K (q̄_hi + q̄_mid + q̄_lo)^T, exact splits
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = ((kk >> 2) * HALF + (kk & 3) * 32) >> 4;
              const uint64_t dq = dq0 + ((qp * L::KV) >> 4) + off;
              if (PASS == 0)  // S = Q K^T, one 128-column tile per query tile of the unit
                umma_ss(tmem + b * L::SBW + qp * 128, dq, dk + off, IDESC, kk > 0 ? 1u : 0u);
              else if (PASS == 1)  // S^T = K Q_g^T, one 128-column tile per group of the unit
                umma_ss(tmem + b * L::SBW + qp * 128, dk + off, dq, IDESC, kk > 0 ? 1u : 0u);
              else umma_ss(tmem + b * L::SBW, dk + off, dq, IDESC, (qp > 0 || kk > 0) ? 1u : 0u);
            }
          }
          umma_commit(&bar.s_full[b]);
          umma_commit(&bar.k_empty[slot]);
          if (c == c_hi - 1) umma_commit(bar.q_empty);
        }
        __syncwarp();
      }
    }
  } else if (warp < CB_EPI) {
    // ---------------------------------------------------------------- epilogue
    // warp (w, q): TMEM lane quadrant q, columns [32w, 32w + 32) of the 128-column tile
    const int q = warp & 3, w = warp >> 2;
    const int row = q * 32 + lane;  // TMEM lane: query row (pass 0) or key row (pass 1)
    const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16) + w * 32;
    const float4* tab = reinterpret_cast<const float4*>(smem + L::OFF_TAB);
    const float scale = p.scale;  // parameters hoisted into registers for the per-score loops
    const int rnd = p.round;
    const int n_keys = p.n;
    uint16_t* const s16 = p.scores16;
    float* const s32 = p.scores;
    uint32_t* const bits_out = p.keep_bits;
    const uint32_t tau_b16 = __bfloat16_as_ushort(__float2bfloat16_ru(p.tau));  // p.tau > 0
    const float a_mid = p.a_mid, hb = p.hb;
    const float sl0 = scale * 1.4426950408889634f;  // pass 0: scale * log2e
    (void)rnd; (void)s16; (void)s32; (void)bits_out; (void)tau_b16; (void)a_mid; (void)hb;
    // s = fl(fl(expf(fl(acc * scale))) / D), bf16 bits (masks.py:108-118, rounded as core.py:196-200)
    auto score_b16 = [&](float acc) {
      constexpr float inv_d = 1.0f / D;  // D is a power of two: x / D == x * (1/D) exactly
      return static_cast<uint32_t>(
          __bfloat16_as_ushort(__float2bfloat16_rn(__fmul_rn(expf(__fmul_rn(acc, scale)), inv_d))));
    };
    uint32_t sc = 0;
    Seq sq = seq_init();
    int64_t bh, u;
    int t, c_lo, c_hi;
    for (; seq_next(sq, bh, t, c_lo, c_hi, u);) {
      const int64_t row0 = bh * p.n;
      const int q0 = t * L::NQ * BM;  // pass 1: the first query of the unit's first group
      if (PASS == 1) {
        // the groups' (m_i, 1/den_i, m_i + ln den_i); rows past the sequence end are never selected
        if (tid < L::NQ * 128) {
          const int i = q0 + tid;
          float4 e = make_float4(0.f, 0.f, INFINITY, 0.f);
          if (i < p.n) {
            const float mi = p.row_max[row0 + i], ri = p.row_rinv[row0 + i];
            e = make_float4(mi, ri, mi - logf(ri), 0.f);
          }
          reinterpret_cast<float4*>(smem + L::OFF_TAB)[tid] = e;
          reinterpret_cast<float*>(smem + L::OFF_NZ)[tid] = -e.z;
        }
        epi_bar();
      }
      float nz[1][32];  // pass 1: -(m_i + ln den_i) of this warp's 32 queries of the unit's first group
      if (PASS == 1) {  // (the second group's are read from shared memory per chunk: registers)
#pragma unroll
        for (int k = 0; k < 32; ++k) nz[0][k] = -tab[w * 32 + k].z;
      }
      float m = -INFINITY;
      float ml0 = -INFINITY;  // pass 0: m * log2e
      double den = 0.0;
      float m_1 = -INFINITY, ml0_1 = -INFINITY;  // pass 0: the second query tile's row (CB_P0G == 2)
      double den_1 = 0.0;
      // pass 3: the listed row's group column and this thread's best (bf16 score + 1, key) so far
      const int fix_r = PASS == 3 ? __ldg(p.fix_rows + u) : 0;
      const int fix_col = (fix_r % (p.groups > 0 ? p.groups : 1)) % BM;
      uint32_t best_rank = 0, best_j = 0xFFFFFFFFu;
      for (int c = c_lo; c < c_hi; ++c, ++sc) {
        const uint32_t b = sc % L::NSB;
        if (tid == 0) CB_TS(sc, 5);
        mbar_wait(&bar.s_full[b], (sc / L::NSB) & 1);
        if (tid == 0) CB_TS(sc, 6);
        tc_fence_after();
        if constexpr (PASS == 3) {
          // exact score of key j for the row's group (the fused pass's arithmetic), running argmax:
          // highest bf16 bits (NaN above inf, as np.argmax), the smallest key among equals
          if (w == fix_col / 32) {
            const uint32_t x = tmem_ld1(tmem + (static_cast<uint32_t>(q * 32) << 16) + b * L::SBW + fix_col);
            tmem_ld_wait();
            const int j = c * BN + row;
            const uint32_t rank = score_b16(__uint_as_float(x)) + 1u;
            if (j < n_keys && rank > best_rank) {
              best_rank = rank;
              best_j = static_cast<uint32_t>(j);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar.s_empty[b]);
          continue;
        }
        uint32_t v[32];
        tmem_ld32(tl + b * L::SBW, v);
        tmem_ld_wait();
        if ((PASS != 1 || CB_P1G == 1) && (PASS != 0 || CB_P0G == 1)) {  // (passes 0 / 1 read their second tile first)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar.s_empty[b]);
        }
        if (PASS == 2) {
          // row: key j = c*128 + row; columns: groups g = 128t + 32w + k (masks.py:108-118):
          // s = exp(k_j . q̄_g * scale) / D, bf16-rounded
          const int j = c * BN + row;
          constexpr float inv_d = 1.0f / D;  // D is a power of two: x / D == x * (1/D) exactly
          if (bits_out != nullptr || j < n_keys) {
            if (j >= n_keys) {  // keys past N: never kept, never the argmax
#pragma unroll
              for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(-INFINITY);
            }
            const int64_t off = (bh * p.groups + t * BM + w * 32) * static_cast<int64_t>(n_keys) + j;
            const int kmax = min(32, p.groups - (t * BM + w * 32));
            // s = fl(fl(expf(fl(acc * scale))) / D); one pointer step of n per group column, no
            // per-element predicate for a full 32-group slice
            if (bits_out != nullptr) {
              // threshold fused into the epilogue (masks.py:131-132), per group column one ballot of
              // this warp's 32 consecutive keys -> keep word.  The bf16 score is a non-decreasing
              // function of the accumulator, and outside a narrow band around a_mid (threshold_band)
              // "score >= tau" is exactly "acc >= a_mid": one compare per score.  A 32 x 32 block
              // with an accumulator in the band (or a NaN) is evaluated exactly.  Rows that keep
              // nothing get their argmax from the pass-3 fix-up (masks.py:86-87).
              bool band = false;
#pragma unroll
              for (int k = 0; k < 32; ++k) band |= !(fabsf(__uint_as_float(v[k]) - a_mid) >= hb);
              uint32_t* xw = reinterpret_cast<uint32_t*>(smem + L::OFF_XCH) + warp * 32;
              if (__any_sync(0xffffffffu, band)) {
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                  const uint32_t b16 = score_b16(__uint_as_float(v[k]));
                  xw[k] = __ballot_sync(0xffffffffu, b16 >= tau_b16 && b16 <= 0x7F80u);
                }
              } else {
#pragma unroll
                for (int k = 0; k < 32; ++k) xw[k] = __ballot_sync(0xffffffffu, __uint_as_float(v[k]) >= a_mid);
              }
              __syncwarp();
              const uint32_t myword = xw[lane];
              __syncwarp();
              const int g = t * BM + w * 32 + lane;
              if (g < p.groups && c * BN + q * 32 < n_keys)  // a word past N belongs to no row
                bits_out[(bh * p.groups + g) * p.words + (c * BN + q * 32) / 32] = myword;
            } else if (s16 != nullptr) {
              uint16_t* dst = s16 + off;
              if (kmax == 32) {
#pragma unroll
                for (int k = 0; k < 32; ++k, dst += n_keys)
                  *dst = __bfloat16_as_ushort(__float2bfloat16_rn(__fmul_rn(expf(__fmul_rn(__uint_as_float(v[k]), scale)), inv_d)));
              } else {
#pragma unroll
                for (int k = 0; k < 32; ++k, dst += n_keys)
                  if (k < kmax)
                    *dst = __bfloat16_as_ushort(__float2bfloat16_rn(__fmul_rn(expf(__fmul_rn(__uint_as_float(v[k]), scale)), inv_d)));
              }
            } else {
              float* dst = s32 + off;
#pragma unroll
              for (int k = 0; k < 32; ++k, dst += n_keys) {
                if (k < kmax) {
                  float sc = __fmul_rn(expf(__fmul_rn(__uint_as_float(v[k]), scale)), inv_d);
                  if (rnd) sc = __bfloat162float(__float2bfloat16_rn(sc));
                  *dst = sc;
                }
              }
            }
          }
        } else if (PASS == 0) {
          auto row_chunk = [&](uint32_t (&v)[32], float& m, float& ml0, double& den) {
            // columns: keys j = c*128 + 32w + k.  Each term exp(s - m) is one FFMA2 + MUFU ex2 on
            // acc * scale * log2e - m * log2e; their rounding errors average out over the row's N
            // terms, each chunk's 32 summed in fp32, the row in fp64.  m is a lazy running max (in
            // the units of s = fl(acc * scale), attention_map's s): the exps use it until a score
            // beats it by more than 8 log2 units, which shows up as a chunk sum above 2^8 (all terms
            // are positive) and sends the warp to the exact path -- the chunk's max on the raw dot
            // products (scale > 0 and rounding is monotonic, so fl(max(acc) * scale) = max(s)), den
            // rescaled in fp64, the chunk re-summed.  Pass 1 needs only m + ln den, which any such m
            // gives exactly; the per-chunk max and the fp64 exp are off the common path.
            const int jbase = c * BN + w * 32;
            if (jbase + 32 > n_keys) {
#pragma unroll
              for (int k = 0; k < 32; ++k)
                if (jbase + k >= n_keys) v[k] = __float_as_uint(-INFINITY);
            }
            auto chunk_sum = [&](float ml) {
              float2 acc = make_float2(0.f, 0.f);
#pragma unroll
              for (int k = 0; k < 32; k += 2) {
                const float2 x = __ffma2_rn(make_float2(__uint_as_float(v[k]), __uint_as_float(v[k + 1])),
                                            make_float2(sl0, sl0), make_float2(-ml, -ml));
                if (CB_POLY > 0 && (k / 2) % (CB_POLY > 0 ? CB_POLY : 1) == CB_POLY - 1)
                  acc = __fadd2_rn(acc, ex2_poly2<5>(x));  // this pair on the FMA pipe
                else
                  acc = __fadd2_rn(acc, make_float2(ex2(x.x), ex2(x.y)));
              }
              return acc;
            };
            float2 acc = make_float2(0.f, 0.f);
            bool exact = m == -INFINITY;
            if (!exact) {
              acc = chunk_sum(ml0);
              exact = !(acc.x + acc.y <= 256.f);
            }
            if (__any_sync(0xffffffffu, exact) && exact) {
              float amax = -INFINITY;
#pragma unroll
              for (int k = 0; k < 32; k += 2) amax = fmax3f(amax, __uint_as_float(v[k]), __uint_as_float(v[k + 1]));
              const float cmax = __fmul_rn(amax, scale);
              if (cmax > m) {
                den = m == -INFINITY ? 0.0 : den * exp(static_cast<double>(m) - static_cast<double>(cmax));
                m = cmax;
                ml0 = m * 1.4426950408889634f;
              }
              acc = m == -INFINITY ? make_float2(0.f, 0.f) : chunk_sum(ml0);
            }
            if (m != -INFINITY) den += static_cast<double>(acc.x) + static_cast<double>(acc.y);
          };
          row_chunk(v, m, ml0, den);
          if (tid == 0) CB_TS(sc, 7);
          if (CB_P0G == 2) {  // the second query tile's slice, then the buffer goes back to the MMA
            tmem_ld32(tl + b * L::SBW + 128, v);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar.s_empty[b]);
            row_chunk(v, m_1, ml0_1, den_1);
          }
        } else {
          // columns: the group's queries i = 32w + k; row: key j = c*128 + row.
          float* xy = reinterpret_cast<float*>(smem + L::OFF_XCH) + (sc & 1) * (3 * CB_EW * 128);
#ifndef FGA_CB_EXACT_SELECT
          // y_j = max_i s_ij - (m_i + ln den_i); gmax_gj = exp(y_j), for each group of the unit
          auto col_max = [&](const float (&nzg)[32]) {
            float y = -INFINITY;
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
              const float2 y2 = __ffma2_rn(make_float2(__uint_as_float(v[k]), __uint_as_float(v[k + 1])),
                                           make_float2(scale, scale), make_float2(nzg[k], nzg[k + 1]));
              y = fmax3f(y, y2.x, y2.y);
            }
            return y;
          };
          float by[CB_P1G];
          by[0] = col_max(nz[0]);
          if (CB_P1G == 2) {  // the second group's tile, then the buffer goes back to the MMA
            tmem_ld32(tl + b * L::SBW + 128, v);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar.s_empty[b]);
            float nz1[32];
            const float4* nzs = reinterpret_cast<const float4*>(smem + L::OFF_NZ + (128 + w * 32) * 4);
#pragma unroll
            for (int k4 = 0; k4 < 8; ++k4) {
              const float4 z = nzs[k4];
              nz1[4 * k4] = z.x; nz1[4 * k4 + 1] = z.y; nz1[4 * k4 + 2] = z.z; nz1[4 * k4 + 3] = z.w;
            }
            by[CB_P1G - 1] = col_max(nz1);
          }
          if (w > 0) {
#pragma unroll
            for (int gi = 0; gi < CB_P1G; ++gi) xy[(gi * CB_EW + w) * 128 + row] = by[gi];
          }
          epi_bar();  // double-buffered by chunk parity: one barrier per chunk
          if (w == 0) {
            const int j = c * BN + row;
#pragma unroll
            for (int gi = 0; gi < CB_P1G; ++gi) {
              float y = by[gi];
#pragma unroll
              for (int o = 1; o < CB_EW; ++o) y = fmaxf(y, xy[(gi * CB_EW + o) * 128 + row]);
              float g = expf(y);
              if (p.round) g = __bfloat162float(__float2bfloat16_rn(g));
              const int grp = t * CB_P1G + gi;
              if (j < p.n && grp < p.groups) p.gmax[(bh * p.groups + grp) * static_cast<int64_t>(p.n) + j] = g;
            }
          }
#else
          // select the query maximising s_ij - (m_i + ln den_i), then evaluate
          // a_ij = expf(s_ij - m_i) / den_i as the reference does for that one query
          float by = -INFINITY, bacc = 0.f;
          int bi = 0;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float y = fmaf(__uint_as_float(v[k]), p.scale, nz[0][k]);
            if (y > by) {
              by = y;
              bacc = __uint_as_float(v[k]);
              bi = w * 32 + k;
            }
          }
          if (w > 0) {
            xy[(w * 3 + 0) * 128 + row] = by;
            xy[(w * 3 + 1) * 128 + row] = bacc;
            xy[(w * 3 + 2) * 128 + row] = __int_as_float(bi);
          }
          epi_bar();  // double-buffered by chunk parity: one barrier per chunk
          if (w == 0) {
#pragma unroll
            for (int o = 1; o < CB_EW; ++o) {
              const float yo = xy[(o * 3 + 0) * 128 + row];
              if (yo > by) {
                by = yo;
                bacc = xy[(o * 3 + 1) * 128 + row];
                bi = __float_as_int(xy[(o * 3 + 2) * 128 + row]);
              }
            }
            const float4 e = tab[bi];
            float g = __fmul_rn(expf(__fsub_rn(__fmul_rn(bacc, p.scale), e.x)), e.y);
            if (p.round) g = __bfloat162float(__float2bfloat16_rn(g));
            const int j = c * BN + row;
            if (j < p.n) p.gmax[(bh * p.groups + t) * static_cast<int64_t>(p.n) + j] = g;
          }
#endif
        }
      }
      if (PASS == 0) {
        // merge the column slices of each row: den relative to the common max (per query tile of
        // the unit, its own exchange area)
#pragma unroll
        for (int g = 0; g < CB_P0G; ++g) {
          float* xf = reinterpret_cast<float*>(smem + L::OFF_XCH + g * CB_EW * 128 * 12);
          double* xd = reinterpret_cast<double*>(smem + L::OFF_XCH + g * CB_EW * 128 * 12 + CB_EW * 128 * 4);
          if (w > 0) {
            xf[w * 128 + row] = g == 0 ? m : m_1;
            xd[w * 128 + row] = g == 0 ? den : den_1;
          }
        }
        epi_bar();
        if (w == 0) {
#pragma unroll
          for (int g = 0; g < CB_P0G; ++g) {
            const float* xf = reinterpret_cast<const float*>(smem + L::OFF_XCH + g * CB_EW * 128 * 12);
            const double* xd =
                reinterpret_cast<const double*>(smem + L::OFF_XCH + g * CB_EW * 128 * 12 + CB_EW * 128 * 4);
            const float mg = g == 0 ? m : m_1;
            const double dg = g == 0 ? den : den_1;
            float mx = mg;
#pragma unroll
            for (int o = 1; o < CB_EW; ++o) mx = fmaxf(mx, xf[o * 128 + row]);
            double tot = mg == -INFINITY ? 0.0 : dg * exp(static_cast<double>(mg) - static_cast<double>(mx));
#pragma unroll
            for (int o = 1; o < CB_EW; ++o) {
              const float mo = xf[o * 128 + row];
              if (mo != -INFINITY) tot += xd[o * 128 + row] * exp(static_cast<double>(mo) - static_cast<double>(mx));
            }
            const int i = q0 + g * BM + row;
            if (i < p.n) {
              p.row_max[row0 + i] = mx;
              p.row_rinv[row0 + i] = static_cast<float>(1.0 / tot);
            }
          }
        }
      }
      if (PASS == 3) {
        uint32_t* xu = reinterpret_cast<uint32_t*>(smem + L::OFF_XCH);
        if (w == fix_col / 32) {
          const uint32_t mr = __reduce_max_sync(0xffffffffu, best_rank);
          const uint32_t mj = __reduce_min_sync(0xffffffffu, best_rank == mr ? best_j : 0xFFFFFFFFu);
          if (lane == 0) {
            xu[2 * q] = mr;
            xu[2 * q + 1] = mj;
          }
        }
        epi_bar();
        if (tid == 0) {
          uint32_t mr = xu[0], mj = xu[1];
          for (int o = 1; o < 4; ++o)
            if (xu[2 * o] > mr || (xu[2 * o] == mr && xu[2 * o + 1] < mj)) {
              mr = xu[2 * o];
              mj = xu[2 * o + 1];
            }
          p.fix_idx[fix_r * p.fix_stride] = static_cast<int32_t>(mj);
        }
      }
      epi_bar();  // exchange / table space free for the next unit
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128 * CB_SB);
  }
}

template <int D, int PASS>
int launch_pass(const CUtensorMap* maps, const CbParams& p, cudaStream_t st) {
  auto kern = cached_tc_kernel<D, PASS>;
  const int smem = CbSmem<D, PASS>::BYTES;
  if (const int rc = smem_opt_in(reinterpret_cast<const void*>(kern), smem, "cached_tc"); rc != FGA_OK)
    return rc;
  const int sms = sm_count();
  // pass 3: the listed rows are counted on the device; at most one CTA per row
  // passes 1 and 2: one contiguous range of (b*h, tile, key chunk) per CTA; pass 3: listed rows
  // (counted on the device), at most one CTA per row
  const int64_t units = PASS == 3 ? p.bh * p.groups : PASS == 0 ? p.bh * p.tiles : p.bh * p.tiles * p.nch;
  kern<<<static_cast<unsigned>(units < sms ? units : sms), 32 * CB_WARPS, smem, st>>>(maps[0], maps[1], p);
  return check_launch("cached_tc_kernel");
}

}  // namespace

// Tensor-core cached builder; returns FGA_EUNSUPPORTED (caller uses the CUDA-core kernel)
// unless M == 128 and D is 64 or 128.
int launch_cached_group_max_tc(const void* q, const void* k, const fga_shape& s, int round, float* gmax,
                               float* row_max, float* rinv, cudaStream_t st) {
  const int64_t B = s.batch, H = s.heads, N = s.seq_len, D = s.head_dim, M = s.group_size;
  if (M != 128 || (D != 64 && D != 128)) return FGA_EUNSUPPORTED;
  const int64_t rows = B * H * N;
  if (rows >= (int64_t(1) << 31)) return FGA_EUNSUPPORTED;
  CUtensorMap maps[2];
  int rc;
  if ((rc = make_tmap_bf16_2d(&maps[0], q, rows, D, 64, BM)) != FGA_OK) return rc;
  if ((rc = make_tmap_bf16_2d(&maps[1], k, rows, D, 64, BN)) != FGA_OK) return rc;
  CbParams p{};
#ifdef FGA_CB_TRACE
  static long long* dbg = nullptr;
  if (dbg == nullptr) cudaMalloc(&dbg, 256 * 8 * sizeof(long long));
  cudaMemsetAsync(dbg, 0, 256 * 8 * sizeof(long long), st);
  p.dbg = dbg;
#endif
  p.bh = B * H;
  p.n = static_cast<int>(N);
  p.tiles = static_cast<int>((N + BM - 1) / BM);
  p.nch = p.tiles;
  p.scale = s.scale > 0.f ? s.scale : 1.0f / std::sqrt(static_cast<float>(D));
  p.round = round;
  p.row_max = row_max;
  p.row_rinv = rinv;
  p.gmax = gmax;
  p.groups = p.tiles;  // M = 128: one query tile per group
  CbParams p0 = p;
  p0.tiles = (p.tiles + CB_P0G - 1) / CB_P0G;  // units per (b, h): CB_P0G query tiles each
  rc = D == 64 ? launch_pass<64, 0>(maps, p0, st) : launch_pass<128, 0>(maps, p0, st);
#ifdef FGA_CB_TRACE
  if (const char* f = std::getenv("FGA_CB_TRACE_FILE")) {
    long long host[256 * 8];
    cudaMemcpyAsync(host, p.dbg, sizeof(host), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE* fp = std::fopen(f, "w")) {
      for (int i = 0; i < 256; ++i) {
        for (int j = 0; j < 8; ++j) std::fprintf(fp, "%lld ", host[i * 8 + j]);
        std::fprintf(fp, "\n");
      }
      std::fclose(fp);
    }
  }
#endif
  if (rc == FGA_OK) {
    CbParams p1 = p;
    p1.tiles = (p.groups + CB_P1G - 1) / CB_P1G;  // units per (b, h): CB_P1G groups each
    rc = D == 64 ? launch_pass<64, 1>(maps, p1, st) : launch_pass<128, 1>(maps, p1, st);
  }
  return rc;
}

// Accumulator threshold of the fused threshold epilogue (pass 2 with keep_bits).  keep <=>
// bf16_rn(y) >= t with t = tau rounded up to bf16 and y = fl(E / D), E = expf(s), s = fl(acc * scale).
// Round-to-nearest-even gives bf16_rn(y) >= t for y > mid and < t for y < mid, mid = (t_prev + t) / 2
// (a float); y = E / D exactly while E / D is normal (D is a power of two); expf is within 2 ulp of
// e^s.  So with L = ln(mid * D): s > L + d  =>  E > mid * D  =>  kept, and s < L - d  =>  not kept,
// for any d well above 2 ulp.  a_mid = L / scale and hb = 2e-5 max(1, |L|) / scale leave d >= 1.9e-5
// after the roundings of acc * scale, a_mid and acc - a_mid; accumulators within hb of a_mid (about
// 1e-5 of them at unit-scale scores) are evaluated exactly.  Thresholds whose mid is subnormal or
// near overflow put every accumulator in the band (hb = inf): exact everywhere.
static void threshold_band(float tau, int d, float scale, float* a_mid, float* hb) {
  uint32_t bits;
  std::memcpy(&bits, &tau, 4);
  uint32_t t16 = (bits >> 16) + ((bits & 0xFFFFu) != 0u ? 1u : 0u);  // round up (tau > 0)
  auto bf = [](uint32_t h) {
    const uint32_t b = h << 16;
    float f;
    std::memcpy(&f, &b, 4);
    return static_cast<double>(f);
  };
  const double mid = t16 >= 0x7F80u ? 0.0 : 0.5 * (bf(t16) + bf(t16 - 1));
  const char* ex = std::getenv("FGA_THRESHOLD_EXACT");  // 1: every score evaluated (tests / A/B)
  if (!(mid >= std::ldexp(1.0, -120)) || mid * d > std::ldexp(1.0, 120) || (ex != nullptr && ex[0] == '1')) {
    *a_mid = 0.f;
    *hb = INFINITY;
    return;
  }
  const double L = std::log(mid * d);
  *a_mid = static_cast<float>(L / scale);
  *hb = static_cast<float>(2e-5 * std::max(1.0, std::fabs(L)) / scale);
}

// q̄ (fp32) -> three bf16 parts with hi + mid + lo == q̄ exactly (8 + 8 + 8 significand bits),
// so K q̄^T is three exact-product bf16 MMAs accumulated in fp32.
__global__ void split3_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ parts, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    split3(x[i], parts, n, i);
}

// Avg-query scores s[b,h,g,j] = exp(k_j . q̄_g * scale) / D on the tensor cores (pass 2);
// FGA_EUNSUPPORTED unless D is 64 or 128.  qbar: fp32 [B*H*G, D] (pooled_mean_kernel).
int launch_pooled_scores_tc(const float* qbar, __nv_bfloat16* parts, bool parts_ready, const void* k,
                            const fga_shape& s, int round, const PooledOut& out, cudaStream_t st) {
  const int64_t B = s.batch, H = s.heads, N = s.seq_len, D = s.head_dim, M = s.group_size;
  if (D != 64 && D != 128) return FGA_EUNSUPPORTED;
  const int64_t G = (N + M - 1) / M;
  const int64_t rows = B * H * N, qrows = B * H * G;
  if (rows >= (int64_t(1) << 31) || 3 * qrows >= (int64_t(1) << 31)) return FGA_EUNSUPPORTED;
  int rc = FGA_OK;
  if (!parts_ready) {
    split3_kernel<<<static_cast<unsigned>(std::min<int64_t>((qrows * D + 255) / 256, 148 * 16)), 256, 0, st>>>(
        qbar, parts, qrows * D);
    rc = check_launch("split3_kernel");
  }
  CUtensorMap maps[2];
  if (rc == FGA_OK) rc = make_tmap_bf16_2d(&maps[0], parts, 3 * qrows, D, 64, BM);
  if (rc == FGA_OK) rc = make_tmap_bf16_2d(&maps[1], k, rows, D, 64, BN);
  if (rc == FGA_OK) {
    CbParams p{};
    p.bh = B * H;
    p.n = static_cast<int>(N);
    p.tiles = static_cast<int>((G + BM - 1) / BM);
    p.nch = static_cast<int>((N + BN - 1) / BN);
    p.groups = static_cast<int>(G);
    p.part_rows = qrows;
    p.scores = out.scores;
    p.scores16 = out.scores16;
    p.keep_bits = out.keep_bits;
    p.tau = out.tau;
    if (out.keep_bits != nullptr) threshold_band(out.tau, static_cast<int>(D), s.scale > 0.f ? s.scale : 1.0f / std::sqrt(static_cast<float>(D)), &p.a_mid, &p.hb);
    p.words = static_cast<int>((N + 31) / 32);
    p.scale = s.scale > 0.f ? s.scale : 1.0f / std::sqrt(static_cast<float>(D));
    p.round = round;
    rc = D == 64 ? launch_pass<64, 2>(maps, p, st) : launch_pass<128, 2>(maps, p, st);
    if (rc == FGA_OK && out.keep_bits != nullptr && out.idx != nullptr) {
      rc = launch_compact_bits(out.keep_bits, qrows, N, out.idx, out.idx_stride, out.counts, out.fill, st,
                               out.fix_rows, out.fix_count);
      if (rc == FGA_OK) {  // argmax of the rows that kept nothing: their tiles again, exact scores
        CbParams p3 = p;
        p3.keep_bits = nullptr;
        p3.fix_rows = out.fix_rows;
        p3.fix_count = out.fix_count;
        p3.fix_idx = out.idx;
        p3.fix_stride = out.idx_stride;
        rc = D == 64 ? launch_pass<64, 3>(maps, p3, st) : launch_pass<128, 3>(maps, p3, st);
      }
    }
  }
  return rc;
}

}  // namespace fga
