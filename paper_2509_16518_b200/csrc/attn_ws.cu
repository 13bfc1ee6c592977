// FG-Attn forward on sm_100a, warp-specialised persistent kernel (v2).
//
// Reference semantics: /root/reference/pkg/src/sliceattn/sparse.py:111-156
// (per-(b,h,g) chunk loop over the key list) with the online softmax of
// tiled.py:48-77.  One work tile = <=128 query rows of one group; its key list
// is consumed in chunks of 128 gathered keys (a short last chunk is gathered
// full-width with a repeated valid key and its extra columns get -inf).
//
// Roles (one CTA per SM, persistent, tiles strided over the grid):
//   warps 0-3       softmax + epilogue: thread t owns query row t = TMEM lane t
//   warp  4         MMA issuer (one warp, elected lane): S_c = Q K_c^T (SS)
//                   into S[c%2], then O += P_{c-1} V_{c-1} (TS: P from TMEM)
//   warps 5..5+NP-1 producers: Q by 2D TMA; each K/V chunk (one ring item of
//                   128 rows) is packed into a 128B-swizzled slot -- the first
//                   G4 rows by TMA tile::gather4, the rest by 16-byte cp.async
//                   spread over all producer lanes.  Measured on B200
//                   (scripts/gather_bench.cu): gather4 alone tops out near
//                   2.1 TB/s chip-wide (~7.5 B/clk/SM, the per-SM TMA unit),
//                   cp.async scales with producer warps (~8.2 TB/s at 16), so
//                   the wide cp.async producer carries the gather and the TMA
//                   unit adds an independent share.
// Registers are rebalanced with setmaxnreg: softmax 232, everything else 48
// (.inc only draws from what the CTA released: see the static_assert).
// TMEM (512 cols): S0 | S1 | O0 | O1.  P_c (bf16) overwrites S[c%2] cols 0-63.
// Issue order S_0, S_1, PV_0, S_2, PV_1, ... gives softmax(c) the window
// PV_{c-1} + S_{c+1} to run while the tensor core stays busy.
// Lazy rescale: the running max used for exp only moves when the row max grows
// by more than 8 (log2 units); O in TMEM is rescaled only then (rarely).
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>

#include "attn_common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace fga {
namespace {

#ifndef FGA_PINGPONG
#define FGA_PINGPONG 1
#endif
// softmax warps: ping-pong = two warpgroups on alternate chunks, else one warpgroup
constexpr int NSOFT = FGA_PINGPONG ? 8 : 4;
constexpr int WARP_MMA = NSOFT;
constexpr int WARP_PROD0 = NSOFT + 1;
constexpr int REG_SOFTMAX = FGA_PINGPONG ? 176 : 232;
constexpr int REG_OTHER = FGA_PINGPONG ? 40 : 48;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units (factor 256)
#ifndef FGA_EMU_EVERY
#define FGA_EMU_EVERY (1 << 20)
#endif
constexpr int EMU_EVERY = FGA_EMU_EVERY;   // 1 in EMU_EVERY exp2 pairs on the FMA pipe

template <int D>
struct WsSmem {
  static constexpr int KV = (D / 64) * HALF;  // one K or V chunk (also one Q tile)
  static constexpr int NSLOT = D == 128 ? 5 : 8;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = OFF_Q + 2 * KV;
  static constexpr int OFF_BAR = OFF_KV + NSLOT * KV;
  static constexpr int NBAR = 2 + 2 + 2 * NSLOT + 2 + 2 + 2 + 2 + 2;
  static constexpr int OFF_XCH = OFF_BAR + ((NBAR * 8 + 16 + 15) / 16) * 16;  // ping-pong merge: 2 WG x (m, l) x 128
  static constexpr int BYTES = OFF_XCH + (FGA_PINGPONG ? 2 * 2 * 128 * 4 : 0);
  static constexpr int ALLOC = BYTES;  // extern smem is declared __align__(1024)
};

struct Bars {
  uint64_t* q_full;    // [2]
  uint64_t* q_empty;   // [2]
  uint64_t* kv_full;   // [NSLOT]
  uint64_t* kv_empty;  // [NSLOT]
  uint64_t* s_full;    // [2]
  uint64_t* p_full;    // [2]
  uint64_t* pv_done;   // [2] (ping-pong: one per O accumulator)
  uint64_t* o_full;    // [2]
  uint64_t* o_empty;   // [2]
  uint32_t* tmem_slot;
};

template <int D>
__device__ __forceinline__ Bars carve_bars(uint8_t* smem) {
  using L = WsSmem<D>;
  uint64_t* b = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  Bars r;
  r.q_full = b;
  r.q_empty = b + 2;
  r.kv_full = b + 4;
  r.kv_empty = b + 4 + L::NSLOT;
  r.s_full = b + 4 + 2 * L::NSLOT;
  r.p_full = r.s_full + 2;
  r.pv_done = r.p_full + 2;
  r.o_full = r.pv_done + 2;
  r.o_empty = r.o_full + 2;
  r.tmem_slot = reinterpret_cast<uint32_t*>(r.o_empty + 2);
  return r;
}

// ------------------------------------------------------------------ producers
// Producer warp pw (0..NP-1).  Rows [0, G4) of every K/V item are gathered by
// warp 0 with gather4 (lane l: rows 4l..4l+3); rows [G4, 128) are split into
// warp instructions of RPI rows (LPR lanes x 16 B per row), instruction i
// belonging to warp i % NP.  Each lane of a warp holds the key of one of the
// warp's rows for the current chunk (shuffled to the copying lanes); keys of
// chunk j+1 are loaded while chunk j is copied.  Rows past the list end are
// zero-filled (src-size 0), so no stale or NaN bytes reach the MMA.
template <int D, int NP, int G4>
struct ProdGeom {
  static constexpr int LPR = D / 8;                 // lanes per row
  static constexpr int RPI = 32 / LPR;              // rows per warp instruction
  static constexpr int NINST = (BN - G4) / RPI;     // cp.async instructions per item
  static constexpr int MAXI = (NINST + NP - 1) / NP;  // per warp
  static_assert(G4 % 4 == 0 && G4 <= BN && (BN - G4) % RPI == 0, "bad G4");
  static_assert(MAXI * RPI <= 32, "a warp must be able to hold its row keys in one register");
};

template <int D, int NP, int G4>
__device__ __forceinline__ void load_chunk_keys(const AttnParams& p, const Tile& t, int j, int pw, int lane,
                                                int& mykey, int4& g4key) {
  using G = ProdGeom<D, NP, G4>;
  const int base = j * BN;
  mykey = -1;
  if (lane < G::MAXI * G::RPI) {
    const int inst = pw + NP * (lane / G::RPI);
    const int row = G4 + inst * G::RPI + lane % G::RPI;
    if (inst < G::NINST && base + row < t.count) mykey = __ldg(t.list + base + row);
  }
  if constexpr (G4 > 0) {
    if (pw == 0 && lane * 4 < G4) {
      const int first = __ldg(t.list + base);
      int r[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kk = base + lane * 4 + e;
        r[e] = t.row0 + (kk < t.count ? __ldg(t.list + kk) : first);
      }
      g4key = make_int4(r[0], r[1], r[2], r[3]);
    }
  }
}

template <int D, int NP, int G4>
__device__ __forceinline__ void producer(const AttnParams& p, const CUtensorMap* tmQ, const CUtensorMap* tmK,
                         const CUtensorMap* tmV, const CUtensorMap* tmK2, const CUtensorMap* tmV2, uint8_t* smem,
                         const Bars& bar, int pw, int lane) {
  using L = WsSmem<D>;
  using G = ProdGeom<D, NP, G4>;
  const uint64_t pol_kv = policy_evict_last();
  const uint64_t pol_q = policy_evict_first();
  const int sub = lane / G::LPR, ch = lane % G::LPR;
  const uint32_t lane_off = static_cast<uint32_t>((ch >> 3) * HALF);  // 64-column half of this lane's 16 B
  const int cc = ch & 7;
  const char* gsrc[2] = {static_cast<const char*>(p.k) + ch * 16, static_cast<const char*>(p.v) + ch * 16};
  const uint32_t kv_base = smem_u32(smem + L::OFF_KV);
  uint32_t item = 0;
  int it = 0;
  for (int64_t tile = p.tile_begin + blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const Tile t = decode_tile(p, tile);
    const int qs = it & 1;
    if (pw == 0) {
      mbar_wait(&bar.q_empty[qs], ((it >> 1) & 1) ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&bar.q_full[qs], BM * D * 2);
#pragma unroll
        for (int h = 0; h < D / 64; ++h)
          tma_load_2d(smem + L::OFF_Q + qs * L::KV + h * HALF, tmQ, &bar.q_full[qs], h * 64, t.row0 + t.q0, pol_q);
      }
    }
    int key = -1;
    int4 g4 = make_int4(0, 0, 0, 0);
    if (!p.dense && t.nchunks > 0) load_chunk_keys<D, NP, G4>(p, t, 0, pw, lane, key, g4);
    for (int j = 0; j < t.nchunks; ++j) {
      int key_n = -1;
      int4 g4_n = g4;
      if (!p.dense && j + 1 < t.nchunks) load_chunk_keys<D, NP, G4>(p, t, j + 1, pw, lane, key_n, g4_n);
#pragma unroll
      for (int kv = 0; kv < 2; ++kv) {
        const uint32_t slot = item % L::NSLOT;
        const uint32_t use = item / L::NSLOT;
        ++item;
        mbar_wait(&bar.kv_empty[slot], (use & 1) ^ 1);
        const uint32_t dst = kv_base + slot * L::KV;
        uint64_t* full = &bar.kv_full[slot];
        if (p.dense) {
          // contiguous keys: whole 128-row boxes by TMA (one lane), everyone else just arrives
          if (pw == 0 && lane == 0) {
            mbar_expect_tx(full, BN * D * 2);
#pragma unroll
            for (int h = 0; h < D / 64; ++h)
              tma_load_2d(smem + L::OFF_KV + slot * L::KV + h * HALF, kv ? tmV2 : tmK2, full, h * 64,
                          t.row0 + j * BN, pol_kv);
          }
          mbar_arrive(full);
          continue;
        }
        if (pw == 0 && lane == 0) mbar_expect_tx(full, G4 * D * 2);  // the +1 arrival (0 bytes when G4 == 0)
        if constexpr (G4 > 0) {
          __syncwarp();
          if (pw == 0 && lane * 4 < G4) {
#pragma unroll
            for (int h = 0; h < D / 64; ++h)
              tma_gather4(smem + L::OFF_KV + slot * L::KV + h * HALF + lane * 512, kv ? tmV : tmK, full, h * 64,
                          g4.x, g4.y, g4.z, g4.w, pol_kv);
          }
        }
        const char* src = gsrc[kv];
#pragma unroll
        for (int m = 0; m < G::MAXI; ++m) {
          const int inst = pw + NP * m;
          if (inst < G::NINST) {
            const int rk = __shfl_sync(0xffffffffu, key, m * G::RPI + sub);
            const int row = G4 + inst * G::RPI + sub;
            const uint32_t d = dst + lane_off + row * 128 + ((cc ^ (row & 7)) << 4);
            const char* sp = rk >= 0 ? src + static_cast<int64_t>(t.row0 + rk) * (D * 2) : src;
            cp_async16(d, sp, rk >= 0 ? 16u : 0u);
          }
        }
        cp_async_arrive_noinc(full);
      }
      key = key_n;
      g4 = g4_n;
    }
  }
}

// ------------------------------------------------------------------ MMA issuer (one warp)
// The whole warp runs the loop (waits, descriptor arithmetic stay warp-uniform);
// one elected lane issues each batch of tcgen05.mma + commits.
template <int D>
__device__ __forceinline__ void mma_issuer(const AttnParams& p, uint8_t* smem, const Bars& bar, uint32_t tmem) {
  using L = WsSmem<D>;
  constexpr uint32_t IDESC_S = idesc_bf16(BM, BN, false, false);  // Q, K both K-major
  constexpr uint32_t IDESC_O = idesc_bf16(BM, D, false, true);    // P from TMEM, V MN-major
  // descriptor templates; the start-address field (addr >> 4) is advanced by adding offset >> 4
  const uint64_t dq0 = sdesc_sw128(smem_u32(smem + L::OFF_Q), 16, 1024);
  const uint64_t dk0 = sdesc_sw128(smem_u32(smem + L::OFF_KV), 16, 1024);
  const uint64_t dv0 = sdesc_sw128(smem_u32(smem + L::OFF_KV), HALF, 1024);
  uint32_t chunk = 0;
  int it = 0;
  for (int64_t tile = p.tile_begin + blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const Tile t = decode_tile(p, tile);
    const int qs = it & 1, ob = it & 1;
    mbar_wait(&bar.q_full[qs], (it >> 1) & 1);
    if (!FGA_PINGPONG) mbar_wait(&bar.o_empty[ob], ((it >> 1) & 1) ^ 1);
    tc_fence_after();
    const uint64_t dq = dq0 + ((qs * L::KV) >> 4);
    for (int j = 0; j <= t.nchunks; ++j) {
      if (j < t.nchunks) {
        const uint32_t c = chunk + j;
        const uint32_t item = 2 * c, slot = item % L::NSLOT, use = item / L::NSLOT;
        FGA_TS(p, it, j, 8);
        mbar_wait(&bar.kv_full[slot], use & 1);
        FGA_TS(p, it, j, 9);
        fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05.mma (async proxy) reads
        tc_fence_after();
        FGA_TS(p, it, j, 13);
        const uint64_t dk = dk0 + ((slot * L::KV) >> 4);
        const uint32_t tS = tmem + (c & 1) * 128;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * HALF + (kk & 3) * 32) >> 4;
            umma_ss(tS, dq + off, dk + off, IDESC_S, kk > 0);
          }
          umma_commit(&bar.s_full[c & 1]);
          umma_commit(&bar.kv_empty[slot]);
        }
        __syncwarp();
        FGA_TS(p, it, j, 14);
      }
      if (j >= 1) {
        const uint32_t c = chunk + j - 1;
        // ping-pong: O[c&1] per softmax warpgroup, one O set per tile (freed by the merged epilogue)
        const uint32_t tO = tmem + 256 + (FGA_PINGPONG ? (c & 1) : ob) * 128;
        const bool first_pv = FGA_PINGPONG ? (j - 1 < 2) : (j == 1);
        if (FGA_PINGPONG && j == 1) {
          mbar_wait(&bar.o_empty[0], (it & 1) ^ 1);
          tc_fence_after();
        }
        FGA_TS(p, it, j - 1, 10);
        mbar_wait(&bar.p_full[c & 1], (c >> 1) & 1);
        FGA_TS(p, it, j - 1, 11);
        const uint32_t item = 2 * c + 1, slot = item % L::NSLOT, use = item / L::NSLOT;
        mbar_wait(&bar.kv_full[slot], use & 1);
        fence_proxy_async_smem();
        tc_fence_after();
        const uint64_t dv = dv0 + ((slot * L::KV) >> 4);
        const uint32_t tP = tmem + (c & 1) * 128;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            umma_ts(tO, tP + kk * 8, dv + ((kk * 16 * 128) >> 4), IDESC_O, (!first_pv || kk > 0) ? 1u : 0u);
          umma_commit(&bar.kv_empty[slot]);
          umma_commit(&bar.pv_done[FGA_PINGPONG ? (c & 1) : 0]);
        }
        __syncwarp();
        FGA_TS(p, it, j - 1, 12);
      }
    }
    if (elect_one()) {
      umma_commit(&bar.o_full[FGA_PINGPONG ? 0 : ob]);
      umma_commit(&bar.q_empty[qs]);
    }
    __syncwarp();
    chunk += t.nchunks;
  }
}

// ------------------------------------------------------------------ softmax + epilogue (128 threads)
template <int D, bool OUT_F32>
__device__ __forceinline__ void softmax_wg(const AttnParams& p, const Bars& bar, uint32_t tmem, int tid) {
  const int warp = tid >> 5;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const float sl2 = p.scale_log2;
  uint32_t chunk = 0;
  int it = 0;
  for (int64_t tile = p.tile_begin + blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const Tile t = decode_tile(p, tile);
    const int ob = it & 1;
    const uint32_t tO = tmem + 256 + ob * 128 + lane_off;
    float m_use = -INFINITY;  // running max actually used as the exp shift (log2-scaled)
    float l_run = 0.f;
    for (int j = 0; j < t.nchunks; ++j) {
      const uint32_t c = chunk + j;
      const uint32_t tS = tmem + (c & 1) * 128 + lane_off;
      if (tid == 0) FGA_TS(p, it, j, 0);
      mbar_wait(&bar.s_full[c & 1], (c >> 1) & 1);
      if (tid == 0) FGA_TS(p, it, j, 1);
      tc_fence_after();
      uint32_t s[4][32];
#pragma unroll
      for (int q = 0; q < 4; ++q) tmem_ld32(tS + q * 32, s[q]);
      tmem_ld_wait();
      if (tid == 0) FGA_TS(p, it, j, 2);
      const int nvalid = min(BN, t.count - j * BN);
      if (nvalid < BN) {
#pragma unroll
        for (int i = 0; i < BN; ++i)
          if (i >= nvalid) s[i >> 5][i & 31] = __float_as_uint(-INFINITY);
      }
      // row max with 8 independent chains
      float mx[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) mx[a] = __uint_as_float(s[0][a]);
#pragma unroll
      for (int i = 8; i < BN; ++i) mx[i & 7] = fmaxf(mx[i & 7], __uint_as_float(s[i >> 5][i & 31]));
      const float rmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * sl2;
      if (tid == 0) FGA_TS(p, it, j, 3);
      float alpha = 1.f;
      bool rescale = false;
      if (j == 0) {
        m_use = rmax;
      } else if (rmax - m_use > RESCALE_THRESHOLD) {
        alpha = ex2(m_use - rmax);
        m_use = rmax;
        rescale = true;
      }
      const float neg_m = -m_use;
      float sum[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) sum[a] = 0.f;
      uint32_t pk[2][32];
#pragma unroll
      for (int i = 0; i < BN / 2; ++i) {
        const float x0 = fmaf(__uint_as_float(s[(2 * i) >> 5][(2 * i) & 31]), sl2, neg_m);
        const float x1 = fmaf(__uint_as_float(s[(2 * i + 1) >> 5][(2 * i + 1) & 31]), sl2, neg_m);
        const bool emu = (i % EMU_EVERY) == EMU_EVERY - 1;  // optional FMA-pipe exp2 share (off by default)
        const float p0 = emu ? ex2_poly(x0) : ex2(x0);
        const float p1 = emu ? ex2_poly(x1) : ex2(x1);
        sum[(2 * i) & 7] += p0;
        sum[(2 * i + 1) & 7] += p1;
        pk[i >> 5][i & 31] = pack_bf16(p0, p1);
      }
      const float rsum = ((sum[0] + sum[1]) + (sum[2] + sum[3])) + ((sum[4] + sum[5]) + (sum[6] + sum[7]));
      if (tid == 0) FGA_TS(p, it, j, 4);
      l_run = l_run * alpha + rsum;
      tmem_st32(tS, pk[0]);
      tmem_st32(tS + 32, pk[1]);
      if (__any_sync(0xffffffffu, rescale)) {
        // O holds PV_{c-1}: wait for it, then scale this warp's rows in place
        mbar_wait(&bar.pv_done[0], (c - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int q = 0; q < D / 32; ++q) {
          uint32_t o[32];
          tmem_ld32(tO + q * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tO + q * 32, o);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&bar.p_full[c & 1]);
      if (tid == 0) FGA_TS(p, it, j, 5);
    }
    // ---- epilogue: O / l -> global  (tiled.py:73-77)
    mbar_wait(&bar.o_full[ob], (it >> 1) & 1);
    tc_fence_after();
    const bool valid = tid < t.rows;
    const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
    const int64_t out_row = static_cast<int64_t>(t.row0) + t.q0 + tid;
#pragma unroll
    for (int q = 0; q < D / 32; ++q) {
      uint32_t o[32];
      tmem_ld32(tO + q * 32, o);
      tmem_ld_wait();
      if (t.nchunks == 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = 0u;  // empty list: TMEM holds stale data
      }
      if (valid) store_row32<OUT_F32>(p.out, out_row * D + q * 32, o, inv_l);
    }
    tc_fence_before();
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&bar.o_empty[ob]);
    if (valid && p.lse != nullptr)
      p.lse[out_row] = l_run > 0.f ? m_use * 0.69314718055994531f + logf(l_run) : -INFINITY;
    chunk += t.nchunks;
  }
}

// ------------------------------------------------------------------ ping-pong softmax (256 threads)
// Warpgroup wg (warps 4wg..4wg+3) owns the chunks with c % 2 == wg: S/P buffer
// S[wg], its own running max / sum and its own accumulator O[wg].  The two
// groups are never lock-stepped, so one group's MUFU-heavy exp phase overlaps
// the other's TMEM loads, max and stores (two softmax warps per SMSP).  The
// epilogue merges (m, l, O) of both groups:
//   O = (O0 2^(m0-M) + O1 2^(m1-M)) / (l0 2^(m0-M) + l1 2^(m1-M)),  M = max(m0, m1)
// each group writing half of the output columns.  (A two-pass TMEM read to save
// registers cost six load->wait round trips per chunk and ran 1.7x slower.)
__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <int D, bool OUT_F32>
__device__ __forceinline__ void softmax_pp(const AttnParams& p, const Bars& bar, uint32_t tmem, int tid, float* xch) {
  const int warp = tid >> 5, wg = warp >> 2, row = tid & 127;
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t tS = tmem + wg * 128 + lane_off;
  const uint32_t tOw = tmem + 256 + wg * 128 + lane_off;
  const float sl2 = p.scale_log2;
  uint32_t chunk = 0;
  int it = 0;
  for (int64_t tile = p.tile_begin + blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const Tile t = decode_tile(p, tile);
    float m_use = -INFINITY, l_run = 0.f;
    const int j0 = (wg - static_cast<int>(chunk & 1)) & 1;
    for (int j = j0; j < t.nchunks; j += 2) {
      const uint32_t c = chunk + j;
      if (row == 0 && wg == 0) FGA_TS(p, it, j, 0);
      mbar_wait(&bar.s_full[wg], (c >> 1) & 1);
      if (row == 0 && wg == 0) FGA_TS(p, it, j, 1);
      tc_fence_after();
      const int nvalid = min(BN, t.count - j * BN);
      uint32_t sv[4][32];
#pragma unroll
      for (int q = 0; q < 4; ++q) tmem_ld32(tS + q * 32, sv[q]);
      tmem_ld_wait();
      if (row == 0 && wg == 0) FGA_TS(p, it, j, 2);
      if (nvalid < BN) {
#pragma unroll
        for (int i = 0; i < BN; ++i)
          if (i >= nvalid) sv[i >> 5][i & 31] = __float_as_uint(-INFINITY);
      }
      float mx[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) mx[a] = __uint_as_float(sv[0][a]);
#pragma unroll
      for (int i = 8; i < BN; ++i) mx[i & 7] = fmaxf(mx[i & 7], __uint_as_float(sv[i >> 5][i & 31]));
      const float rmax =
          fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * sl2;
      if (row == 0 && wg == 0) FGA_TS(p, it, j, 3);
      float alpha = 1.f;
      bool rescale = false;
      if (j < 2) {  // this group's first chunk of the tile
        m_use = rmax;
      } else if (rmax - m_use > RESCALE_THRESHOLD) {
        alpha = ex2(m_use - rmax);
        m_use = rmax;
        rescale = true;
      }
      const float neg_m = -m_use;
      float sum[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) sum[a] = 0.f;
      uint32_t pk[2][32];
#pragma unroll
      for (int i = 0; i < BN / 2; ++i) {
        const float p0 = ex2(fmaf(__uint_as_float(sv[(2 * i) >> 5][(2 * i) & 31]), sl2, neg_m));
        const float p1 = ex2(fmaf(__uint_as_float(sv[(2 * i + 1) >> 5][(2 * i + 1) & 31]), sl2, neg_m));
        sum[(2 * i) & 7] += p0;
        sum[(2 * i + 1) & 7] += p1;
        pk[i >> 5][i & 31] = pack_bf16(p0, p1);
      }
      tmem_st32(tS, pk[0]);
      tmem_st32(tS + 32, pk[1]);
      const float rsum = ((sum[0] + sum[1]) + (sum[2] + sum[3])) + ((sum[4] + sum[5]) + (sum[6] + sum[7]));
      if (row == 0 && wg == 0) FGA_TS(p, it, j, 4);
      l_run = l_run * alpha + rsum;
      if (__any_sync(0xffffffffu, rescale)) {
        // O[wg] holds PV of this group's previous chunk (c - 2): wait for it, then scale in place
        mbar_wait(&bar.pv_done[wg], ((c - 2) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int q = 0; q < D / 32; ++q) {
          uint32_t o[32];
          tmem_ld32(tOw + q * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tOw + q * 32, o);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&bar.p_full[wg]);
      if (row == 0 && wg == 0) FGA_TS(p, it, j, 5);
    }
    // ---- epilogue: merge the two groups' partial softmax, O / l -> global (tiled.py:73-77)
    xch[(wg * 2) * 128 + row] = m_use;
    xch[(wg * 2 + 1) * 128 + row] = l_run;
    softmax_bar();
    const float m0 = xch[row], l0 = xch[128 + row], m1 = xch[256 + row], l1 = xch[384 + row];
    softmax_bar();  // both groups have read before the next tile rewrites xch
    const float M = fmaxf(l0 > 0.f ? m0 : -INFINITY, l1 > 0.f ? m1 : -INFINITY);
    const float s0 = l0 > 0.f ? ex2(m0 - M) : 0.f;
    const float s1 = l1 > 0.f ? ex2(m1 - M) : 0.f;
    const float L = l0 * s0 + l1 * s1;
    const float inv = L > 0.f ? 1.f / L : 0.f;
    mbar_wait(&bar.o_full[0], it & 1);
    tc_fence_after();
    const bool valid = row < t.rows;
    const int64_t out_row = static_cast<int64_t>(t.row0) + t.q0 + row;
#pragma unroll
    for (int q = 0; q < D / 64; ++q) {
      const int col = wg * (D / 2) + q * 32;
      uint32_t o0[32], o1[32];
      tmem_ld32(tmem + 256 + lane_off + col, o0);
      tmem_ld32(tmem + 384 + lane_off + col, o1);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float a = s0 > 0.f ? __uint_as_float(o0[i]) * s0 : 0.f;  // an unused accumulator holds stale bits
        const float b = s1 > 0.f ? __uint_as_float(o1[i]) * s1 : 0.f;
        o0[i] = __float_as_uint(a + b);
      }
      if (valid) store_row32<OUT_F32>(p.out, out_row * D + col, o0, inv);
    }
    tc_fence_before();
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&bar.o_empty[0]);
    if (wg == 0 && valid && p.lse != nullptr)
      p.lse[out_row] = L > 0.f ? M * 0.69314718055994531f + logf(L) : -INFINITY;
    chunk += t.nchunks;
  }
}

template <int D, bool OUT_F32, int NP, int G4>
__global__ void __launch_bounds__(32 * (NSOFT + 1 + NP), 1)
    fga_attn_ws_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmK2,
                       const __grid_constant__ CUtensorMap tmV2, const AttnParams p) {
  using L = WsSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_ws[];
  uint8_t* smem = smem_ws;
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 atoms need 1 KB alignment
  const Bars bar = carve_bars<D>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(p.dense ? &tmK2 : &tmK);
    prefetch_tmap(p.dense ? &tmV2 : &tmV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar.q_full[i], 1);
      mbar_init(&bar.q_empty[i], 1);
      mbar_init(&bar.s_full[i], 1);
      mbar_init(&bar.p_full[i], FGA_PINGPONG ? 4 : NSOFT);
      mbar_init(&bar.o_full[i], 1);
      mbar_init(&bar.o_empty[i], NSOFT);  // every softmax warp arrives once per tile
    }
    for (int i = 0; i < L::NSLOT; ++i) {
      mbar_init(&bar.kv_full[i], NP * 32 + 1);
      mbar_init(&bar.kv_empty[i], 1);
    }
    mbar_init(&bar.pv_done[0], 1);
    mbar_init(&bar.pv_done[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(bar.tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *bar.tmem_slot;

  static_assert((NSOFT + 1 + NP) % 4 == 0, "whole warpgroups are needed for setmaxnreg");
  // setmaxnreg.inc can only take registers this CTA released with .dec (its pool is threads x launch regs)
  constexpr int kThreads = 32 * (NSOFT + 1 + NP);
  constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8 > 255 ? 248 : (65536 / kThreads) / 8 * 8;
  static_assert(32 * NSOFT * (REG_SOFTMAX - kLaunchRegs) <= (kThreads - 32 * NSOFT) * (kLaunchRegs - REG_OTHER),
                "setmaxnreg budget would deadlock");
  if (warp < NSOFT) {
    setmaxnreg_inc<REG_SOFTMAX>();
    if constexpr (FGA_PINGPONG)
      softmax_pp<D, OUT_F32>(p, bar, tmem, tid, reinterpret_cast<float*>(smem + L::OFF_XCH));
    else
      softmax_wg<D, OUT_F32>(p, bar, tmem, tid);
  } else {
    setmaxnreg_dec<REG_OTHER>();
    if (warp == WARP_MMA) {
      mma_issuer<D>(p, smem, bar, tmem);
    } else {
      producer<D, NP, G4>(p, &tmQ, &tmK, &tmV, &tmK2, &tmV2, smem, bar, warp - WARP_PROD0, lane);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

#ifndef FGA_NPROD
#define FGA_NPROD (FGA_PINGPONG ? 11 : 15)
#endif
#ifndef FGA_G4ROWS
#define FGA_G4ROWS 0
#endif
constexpr int NPROD = FGA_NPROD;    // producer warps (NSOFT + 1 + NPROD must be a multiple of 4)
constexpr int G4ROWS = FGA_G4ROWS;  // rows per K/V item gathered by TMA gather4 (rest by cp.async)

template <int D, bool F32>
int launch_ws(const CUtensorMap* maps, const AttnParams& p, cudaStream_t stream) {
  auto kern = fga_attn_ws_kernel<D, F32, NPROD, G4ROWS>;
  const int smem = WsSmem<D>::ALLOC;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return check_launch("cudaFuncSetAttribute(attn_ws)");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t span = p.n_tiles - p.tile_begin;
  const int64_t grid = span < sms ? span : sms;
  kern<<<static_cast<unsigned>(grid), 32 * (NSOFT + 1 + NPROD), smem, stream>>>(maps[0], maps[1], maps[2], maps[3], maps[4], p);
  return check_launch("fga_attn_ws_kernel");
}

}  // namespace

int launch_attn_ws(const CUtensorMap* maps, const AttnParams& p, int d, bool out_f32, cudaStream_t stream) {
  if (d == 64) return out_f32 ? launch_ws<64, true>(maps, p, stream) : launch_ws<64, false>(maps, p, stream);
  return out_f32 ? launch_ws<128, true>(maps, p, stream) : launch_ws<128, false>(maps, p, stream);
}

}  // namespace fga
