// FG-Attn forward on sm_100a for query groups of 129..256 rows: both 128-row tiles of a
// group share every gathered K/V chunk (shared-gather dual-tile kernel).
//
// Reference semantics: /root/reference/pkg/src/sliceattn/sparse.py:111-156 -- all rows of a
// group attend to the SAME key list.  With M = 128 each tile has its own list and every chunk
// is gathered for one tile (attn_ws.cu); with 128 < M <= 256 the group's two tiles need the
// same rows, so gathering them once per group halves the L2->SMEM bytes per FLOP, which is
// what bounds the single-tile kernel.
//
// Work unit = one group.  Per chunk c of its list and 64-key half h of the chunk:
//   S_r,c,h = Q_r K_c,h^T   tcgen05 SS-MMA (N = 64), r = tile 0 / 1 (Q tiles in SMEM, TMA)
//   P_r,c,h = 2^(S * scale * log2e - m_r)   softmax warpgroup r (thread = query row)
//   O_r    += P_r,c,h V_c,h  TS-MMA (K = 64; P from TMEM, V from SMEM)
// TMEM (512 columns): O_0 | O_1 | S_0,0 S_0,1 | S_1,0 S_1,1 (64 columns each); each tile keeps its
// own running max and accumulator, so the epilogues need no exchange.  The two halves are two
// chains per tile (S_c+1,h reuses the buffer PV_c,h reads, issued right behind it), and the two
// warpgroups take turns on each sub-partition's MUFU (named-barrier turns, as in the ping-pong
// kernel of round 1, git history) so one
// exponentiates while the tensor core serves the other.  Default for 129..256-row groups
// (1-7% faster than attn_ws.cu there).
//
// Warps (16): 0-3 softmax tile 0, 4-7 softmax tile 1, 8/9 MMA issuer of tile 0/1, 10-13
// gather producers (64-row halves of every K / V chunk, one per sub-partition), 14 Q loader.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>

#include "attn_common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace fga {
namespace {

constexpr int NWARPS = 16;
constexpr int NSOFT = 8;
constexpr int WARP_MMA0 = 8;
constexpr int WARP_PROD0 = 10;
constexpr int WARP_QLOAD = 14;
constexpr int NSK = 3, NSV = 2;  // K / V ring slots (the two Q tiles take 2 x 32 KB)
constexpr int REG_SOFTMAX = 184;
constexpr int REG_OTHER = 72;
constexpr float RESCALE_THRESHOLD = 8.0f;
constexpr float RESCALE_SUM = 256.0f;
constexpr uint32_t TM_O = 0, TM_S = 256;  // O_r at r*128, S_r at 256 + r*128
#ifndef DU_TURNS
#define DU_TURNS 1  // the two tiles' softmax warps take turns on each sub-partition's MUFU
#endif

template <int D>
struct DuSmem {
  static constexpr int KV = (D / 64) * HALF;
  static constexpr int OFF_Q = 0;  // Q tiles 0, 1
  static constexpr int OFF_K = OFF_Q + 2 * KV;
  static constexpr int OFF_V = OFF_K + NSK * KV;
  static constexpr int OFF_BAR = OFF_V + NSV * KV;
  static constexpr int NBAR = 3 * (NSK + NSV) + 4 + 4 + 2 + 2 + 2 + 2;
  static constexpr int OFF_TURN = OFF_BAR + ((NBAR * 8 + 16 + 15) / 16) * 16;
  static constexpr int BYTES = OFF_TURN + 4 + 256 * 4;  // the 0.0f word + one scratch word per softmax thread
  static_assert(BYTES <= 232448, "exceeds the 227 KB of shared memory per CTA");
};

struct Bars {
  uint64_t* k_full;   // [NSK] count 64 (two producer halves)
  uint64_t* k_empty;  // [2][NSK] issuer r's S read the chunk (the producers wait for both)
  uint64_t* v_full;   // [NSV] count 64
  uint64_t* v_empty;  // [2][NSV] issuer r's PV read the chunk
  uint64_t* s_full;   // [2][2] issuer r, 64-key half h
  uint64_t* p_full;   // [2][2] count 4 (warpgroup r)
  uint64_t* pv_done;  // [2] issuer r: one completion per PV (two per chunk)
  uint64_t* o_full;   // [2] issuer r: tile r's last PV complete
  uint64_t* o_empty;  // [2] count 4: warpgroup r read and cleared O_r
  uint64_t* q_full;   // Q loader expect_tx (both tiles)
  uint64_t* q_empty;  // count 2: both issuers' last S of the group complete
  uint32_t* tmem_slot;
};

template <int D>
__device__ __forceinline__ Bars carve_bars(uint8_t* smem) {
  uint64_t* b = reinterpret_cast<uint64_t*>(smem + DuSmem<D>::OFF_BAR);
  Bars r;
  r.k_full = b;
  r.k_empty = r.k_full + NSK;
  r.v_full = r.k_empty + 2 * NSK;
  r.v_empty = r.v_full + NSV;
  r.s_full = r.v_empty + 2 * NSV;
  r.p_full = r.s_full + 4;
  r.pv_done = r.p_full + 4;
  r.o_full = r.pv_done + 2;
  r.o_empty = r.o_full + 2;
  r.q_full = r.o_empty + 2;
  r.q_empty = r.q_full + 1;
  r.tmem_slot = reinterpret_cast<uint32_t*>(r.q_empty + 1);
  return r;
}

// group u (tiles 2u, 2u + 1 in launch order) of this launch
__device__ __forceinline__ int64_t n_groups(const AttnParams& p) { return (p.n_tiles - p.tile_begin) / 2; }
__device__ __forceinline__ Tile group_tile(const AttnParams& p, int64_t u, int r) {
  return decode_tile(p, p.tile_begin + 2 * u + r);
}

// ------------------------------------------------------------------ producers (attn_ws.cu)
template <int D>
__device__ __forceinline__ void producer_half(const AttnParams& p, uint8_t* smem, const Bars& bar, int kv, int part,
                                              int lane) {
  using L = DuSmem<D>;
  // 8 lanes per 128-byte half row, each lane copying its 16 bytes of every half of its row with
  // one key shuffle (attn_ws.cu's producer_half mapping)
  constexpr int LPR = 8, NH = D / 64, RPI = 32 / LPR, ROWS = BN / 2, PER = 8 / RPI;
  const int nslot = kv ? NSV : NSK;
  const int sub = lane / LPR, ch = lane % LPR;
  const uint32_t lane_off = static_cast<uint32_t>((ch >> 3) * HALF);
  const int cc = ch & 7;
  const uint32_t ring_base = smem_u32(smem + (kv ? L::OFF_V : L::OFF_K)) + part * ROWS * 128;
  uint64_t* fullb = kv ? bar.v_full : bar.k_full;
  uint64_t* emptyb = kv ? bar.v_empty : bar.k_empty;
  uint32_t item = 0;
  for (int64_t u = blockIdx.x; u < n_groups(p); u += gridDim.x) {
    const Tile t = group_tile(p, u, 0);
    if (kv == 0 && part == 0 && lane == 0) report_tile(p, t);
    const char* gsrc = static_cast<const char*>(kv ? p.v : p.k) + static_cast<int64_t>(t.row0) * (D * 2) + ch * 16;
    for (int c = 0; c < t.nchunks; ++c, ++item) {
      const uint32_t slot = item % nslot, use = item / nslot;
      int keys[ROWS / 32];
#pragma unroll
      for (int i = 0; i < ROWS / 32; ++i) {
        const int row = c * BN + part * ROWS + i * 32 + lane;
        keys[i] = row < t.count ? __ldg(t.list + row) : -1;
      }
      mbar_wait(&emptyb[slot], (use & 1) ^ 1);          // tile 0's reads of the slot done
      mbar_wait(&emptyb[nslot + slot], (use & 1) ^ 1);  // and tile 1's
      // this thread's copies into the slot's previous use completed before the slot filled (the
      // empty waits imply it); the wait states it for tools that track cp.async per thread
      // (compute-sanitizer racecheck), and is a no-op here
      if (use > 0) asm volatile("cp.async.wait_group %0;" ::"n"(NSK > NSV ? NSV - 1 : NSK - 1) : "memory");
#pragma unroll
      for (int i = 0; i < ROWS / 32; ++i) keys[i] = clamp_key(p, keys[i], c * BN + part * ROWS + i * 32 + lane < t.count);
      const char* src = gsrc;
      asm volatile("mov.b64 %0, %0;" : "+l"(src));
      uint32_t dstb[PER];
#pragma unroll
      for (int w = 0; w < PER; ++w)
        dstb[w] = ring_base + slot * L::KV + lane_off + sub * 128 + ((cc ^ ((w * RPI + sub) & 7)) << 4);
      if (c * BN + part * ROWS + ROWS <= t.count) {
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i) {
#pragma unroll
          for (int mm = 0; mm < 32 / RPI; ++mm) {
            const uint32_t key = static_cast<uint32_t>(__shfl_sync(0xffffffffu, keys[i], mm * RPI + sub));
            const char* g = src + static_cast<size_t>(key) * (D * 2);
#pragma unroll
            for (int hh = 0; hh < NH; ++hh)
              cp_async16_full(dstb[mm % PER] + hh * HALF + (i * 32 + mm * RPI) * 128, g + hh * 128);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i) {
#pragma unroll
          for (int mm = 0; mm < 32 / RPI; ++mm) {
            const int key = __shfl_sync(0xffffffffu, keys[i], mm * RPI + sub);
            const char* g = src + static_cast<size_t>(static_cast<uint32_t>(max(key, 0))) * (D * 2);
#pragma unroll
            for (int hh = 0; hh < NH; ++hh)
              cp_async16(dstb[mm % PER] + hh * HALF + (i * 32 + mm * RPI) * 128, g + hh * 128, key >= 0 ? 16u : 0u);
          }
        }
      }
      cp_async_arrive_noinc(&fullb[slot]);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }
}

template <int D>
__device__ __forceinline__ void q_loader(const AttnParams& p, const CUtensorMap* tmQ, uint8_t* smem, const Bars& bar,
                                         int lane) {
  using L = DuSmem<D>;
  const uint64_t pol_q = policy_evict_first();
  int it = 0;
  for (int64_t u = blockIdx.x; u < n_groups(p); u += gridDim.x, ++it) {
    mbar_wait(bar.q_empty, (it & 1) ^ 1);
    if (lane == 0) {
      mbar_expect_tx(bar.q_full, 2 * BM * D * 2);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const Tile t = group_tile(p, u, r);
#pragma unroll
        for (int h = 0; h < D / 64; ++h)
          tma_load_2d(smem + L::OFF_Q + r * L::KV + h * HALF, tmQ, bar.q_full, h * 64, t.row0 + t.q0, pol_q);
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ MMA issuers
// Issuer r drives tile r through two chains, one per 64-key half h of each chunk: S_r,c,h =
// Q_r K_c,h^T (N = 64) into S_r,h, and O_r += P_r,c,h V_c,h (K = 64).  Issue order
//   S_0,0 S_0,1 | PV_0,0 S_1,0 PV_0,1 S_1,1 | PV_1,0 S_2,0 PV_1,1 S_2,1 | ...
// puts each S right behind the PV that frees its buffer (tcgen05 executes one thread's ops in
// order), so while the softmax works on half 1 the tensor core already computes the next half 0.
template <int D>
__device__ __forceinline__ void mma_chain(const AttnParams& p, uint8_t* smem, const Bars& bar, uint32_t tmem, int r) {
  using L = DuSmem<D>;
  constexpr uint32_t IDESC_S = idesc_bf16(BM, BN / 2, false, false);  // N = 64 keys
  constexpr uint32_t IDESC_O = idesc_bf16(BM, D, false, true);
  const uint64_t dq = sdesc_sw128(smem_u32(smem + L::OFF_Q + r * L::KV), 16, 1024);
  const uint64_t dk0 = sdesc_sw128(smem_u32(smem + L::OFF_K), 16, 1024);
  const uint64_t dv0 = sdesc_sw128(smem_u32(smem + L::OFF_V), HALF, 1024);
  const uint32_t tO = tmem + TM_O + r * 128, tS = tmem + TM_S + r * 128;
  uint32_t kc = 0;  // CTA-wide chunk counter
  int it = 0;
  auto issue_s = [&](uint32_t cc, int h, bool last) {  // S_r,cc,h
    const uint32_t slot = cc % NSK;
    if (h == 0) {
      mbar_wait(&bar.k_full[slot], (cc / NSK) & 1);
      fence_proxy_async_smem();
      tc_fence_after();
    }
    const uint64_t dk = dk0 + ((slot * L::KV + h * 64 * 128) >> 4);
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off = ((kk >> 2) * HALF + (kk & 3) * 32) >> 4;
        umma_ss(tS + h * 64, dq + off, dk + off, IDESC_S, kk > 0 ? 1u : 0u);
      }
      umma_commit(&bar.s_full[2 * r + h]);
      if (h == 1) umma_commit(&bar.k_empty[r * NSK + slot]);
      if (h == 1 && last) umma_commit(bar.q_empty);
    }
    __syncwarp();
  };
  auto issue_pv = [&](uint32_t cc, int h, bool last) {  // O_r += P_r,cc,h V_cc,h
    mbar_wait(&bar.p_full[2 * r + h], cc & 1);
    const uint32_t slot = cc % NSV;
    if (h == 0) {
      mbar_wait(&bar.v_full[slot], (cc / NSV) & 1);
      fence_proxy_async_smem();
    }
    tc_fence_after();
    const uint64_t dv = dv0 + ((slot * L::KV + h * 64 * 128) >> 4);
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < BN / 32; ++kk)
        umma_ts(tO, tS + h * 64 + kk * 8, dv + ((kk * 16 * 128) >> 4), IDESC_O, 1u);
      umma_commit(&bar.pv_done[r]);
      if (h == 1) umma_commit(&bar.v_empty[r * NSV + slot]);
      if (h == 1 && last) umma_commit(&bar.o_full[r]);
    }
    __syncwarp();
  };
  for (int64_t u = blockIdx.x; u < n_groups(p); u += gridDim.x, ++it) {
    const Tile t = group_tile(p, u, r);
    const int n = t.nchunks;
    mbar_wait(bar.q_full, it & 1);
    tc_fence_after();
    issue_s(kc, 0, n == 1);
    issue_s(kc, 1, n == 1);
    mbar_wait(&bar.o_empty[r], it & 1);  // O_r cleared by the previous group's epilogue
    tc_fence_after();
    for (int c = 0; c < n; ++c) {
      const uint32_t cc = kc + c;
      const bool more = c + 1 < n;
      issue_pv(cc, 0, !more);
      if (more) issue_s(cc + 1, 0, c + 2 == n);
      issue_pv(cc, 1, !more);
      if (more) issue_s(cc + 1, 1, c + 2 == n);
    }
    kc += n;
  }
}

// ------------------------------------------------------------------ softmax
// MUFU turns between the two warps of a sub-partition (attn_pp.cu): tile 0's warp, then
// tile 1's, for every chunk.  The barriers are tied to the exps through shared memory.
__device__ __forceinline__ void turn_wait(int q, int r, float& m, uint32_t zero_addr) {
  if (DU_TURNS) asm volatile("{\n.reg .f32 z;\nbar.sync %1, 64;\nld.shared.f32 z, [%2];\nadd.f32 %0, %0, z;\n}\n"
               : "+f"(m)
               : "r"(2 + 2 * q + r), "r"(zero_addr)
               : "memory");
}
__device__ __forceinline__ void turn_pass(int q, int r, float2 a, float2 b, uint32_t junk_addr) {
  if (DU_TURNS) asm volatile("{\n.reg .f32 z;\nadd.f32 z, %0, %1;\nadd.f32 z, z, %2;\nadd.f32 z, z, %3;\n"
               "st.shared.f32 [%5], z;\nbar.arrive %4, 64;\n}\n" ::"f"(a.x),
               "f"(a.y), "f"(b.x), "f"(b.y), "r"(2 + 2 * q + (r ^ 1)), "r"(junk_addr)
               : "memory");
}

// 64-key half of a row: 2 x 32 scores
__device__ __forceinline__ void load_s(uint32_t tS, uint32_t (&s)[2][32]) {
  tmem_ld32(tS, s[0]);
  tmem_ld32(tS + 32, s[1]);
  tmem_ld_wait();
}

__device__ __forceinline__ void mask_tail(uint32_t (&s)[2][32], int nvalid) {
  if (nvalid < 64) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (32 * i + k >= nvalid) s[i][k] = __float_as_uint(-INFINITY);
  }
}

__device__ __forceinline__ float row_max(const uint32_t (&s)[2][32]) {
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int k = 0; k < 32; k += 2) m = fmax3f(m, __uint_as_float(s[i][k]), __uint_as_float(s[i][k + 1]));
  }
  return m;
}

// P = 2^(s * scale * log2e - m) for the 64 scores: packed FFMA2 arguments, MUFU ex2, packed
// FADD2 partial sums, key pairs (2i, 2i+1) packed into bf16x2 column i of P.
__device__ __forceinline__ float exp_half(const uint32_t (&s)[2][32], float sl2, float m, uint32_t (&pk)[32], int q,
                                          int r, bool pass, uint32_t junk) {
  const float2 sc2 = make_float2(sl2, sl2), nm = make_float2(-m, -m);
  float2 sum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[i][2 * k]), __uint_as_float(s[i][2 * k + 1])), sc2, nm);
      const float2 pr = make_float2(ex2(x.x), ex2(x.y));
      sum[k & 1] = __fadd2_rn(sum[k & 1], pr);
      pk[16 * i + k] = pack_bf16(pr.x, pr.y);
    }
  }
  if (pass) turn_pass(q, r, sum[0], sum[1], junk);
  const float2 u = __fadd2_rn(sum[0], sum[1]);
  return u.x + u.y;
}

template <int D, bool OUT_F32>
__device__ __forceinline__ void softmax(const AttnParams& p, const Bars& bar, uint32_t tmem, int tid, uint32_t zaddr) {
  const uint32_t junk = zaddr + 4 + 4 * tid;  // per-thread scratch word: no write-write sharing
  const int warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, r = warp >> 2;  // lane quadrant, tile of the group
  const int row = q * 32 + lane;
  const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
  const uint32_t tSr = tmem + TM_S + r * 128 + lanes;
  const uint32_t tOr = tmem + TM_O + r * 128 + lanes;
  const float sl2 = p.scale_log2;
  uint32_t zero[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) zero[i] = 0u;
  if (static_cast<int64_t>(blockIdx.x) < n_groups(p)) {
#pragma unroll
    for (int i = 0; i < D / 32; ++i) tmem_st32(tOr + i * 32, zero);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bar.o_empty[r]);
    if (r == 1) turn_pass(q, r, make_float2(0.f, 0.f), make_float2(0.f, 0.f), junk);  // tile 0 goes first
  }
  uint32_t kc = 0;
  int it = 0;
  for (int64_t u = blockIdx.x; u < n_groups(p); u += gridDim.x, ++it) {
    const Tile t = group_tile(p, u, r);
    float m = -INFINITY, l = 0.f;
    for (int c = 0; c < t.nchunks; ++c, ++kc) {
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const uint32_t tS = tSr + h * 64;
        mbar_wait(&bar.s_full[2 * r + h], kc & 1);
        tc_fence_after();
        uint32_t s[2][32];
        load_s(tS, s);
        const int nvalid = min(64, t.count - c * BN - h * 64);  // may be <= 0 in a short last chunk
        mask_tail(s, nvalid);
        uint32_t pk[32];
        float alpha = 1.f, sum;
        bool rescale = false;
        if (c == 0 && h == 0) {
          m = row_max(s) * sl2;
          turn_wait(q, r, m, zaddr);
          sum = exp_half(s, sl2, m, pk, q, r, true, junk);
        } else {
          turn_wait(q, r, m, zaddr);
          sum = exp_half(s, sl2, m, pk, q, r, true, junk);
          if (__any_sync(0xffffffffu, !(sum <= RESCALE_SUM))) {
            load_s(tS, s);  // S is intact (P not yet stored)
            mask_tail(s, nvalid);
            const float rmax = row_max(s) * sl2;
            if (rmax - m > RESCALE_THRESHOLD) {
              alpha = ex2(m - rmax);
              m = rmax;
              rescale = true;
            }
            sum = exp_half(s, sl2, m, pk, q, r, false, junk);
          }
        }
        if (__any_sync(0xffffffffu, rescale)) {
          // every PV issued into O_r so far (2*kc + h of them) must have landed before O_r scales
          const uint32_t done = 2 * kc + h;
          mbar_wait(&bar.pv_done[r], (done - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int i = 0; i < D / 32; ++i) {
            uint32_t o[32];
            tmem_ld32(tOr + 32 * i, o);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
            tmem_st32(tOr + 32 * i, o);
          }
        }
        l = l * alpha + sum;
        tmem_st32(tS, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar.p_full[2 * r + h]);
      }
    }
    // ---- epilogue of tile r (tiled.py:73-77)
    mbar_wait(&bar.o_full[r], it & 1);
    tc_fence_after();
    const bool valid = row < t.rows;
    const int64_t out_row = static_cast<int64_t>(t.row0) + t.q0 + row;
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int i = 0; i < D / 32; ++i) {
      uint32_t o[32];
      tmem_ld32(tOr + 32 * i, o);
      tmem_ld_wait();
      tmem_st32(tOr + 32 * i, zero);
      if (valid) store_row32<OUT_F32>(p.out, out_row * D + 32 * i, o, inv);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bar.o_empty[r]);
    if (valid && p.lse != nullptr) p.lse[out_row] = l > 0.f ? m * 0.69314718055994531f + logf(l) : -INFINITY;
  }
  if (kc > 0 && r == 0) {  // the turn tile 1's warp passed after the last half-chunk
    float dummy = 0.f;
    turn_wait(q, r, dummy, zaddr);
  }
}

template <int D, bool OUT_F32>
__global__ void __launch_bounds__(32 * NWARPS, 1)
    fga_attn_dual_kernel(const __grid_constant__ CUtensorMap tmQ, const AttnParams p) {
  using L = DuSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_du[];
  uint8_t* smem = smem_du;
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  const Bars bar = carve_bars<D>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    prefetch_tmap(&tmQ);
    for (int i = 0; i < NSK; ++i) mbar_init(&bar.k_full[i], 64);
    for (int i = 0; i < 2 * NSK; ++i) mbar_init(&bar.k_empty[i], 1);
    for (int i = 0; i < NSV; ++i) mbar_init(&bar.v_full[i], 64);
    for (int i = 0; i < 2 * NSV; ++i) mbar_init(&bar.v_empty[i], 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&bar.s_full[i], 1);
      mbar_init(&bar.p_full[i], NSOFT / 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar.pv_done[i], 1);
      mbar_init(&bar.o_full[i], 1);
      mbar_init(&bar.o_empty[i], NSOFT / 2);
    }
    mbar_init(bar.q_full, 1);
    mbar_init(bar.q_empty, 2);
    *reinterpret_cast<float*>(smem + L::OFF_TURN) = 0.f;
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(bar.tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  record_cta_ns(p, 0);
  tc_fence_after();
  const uint32_t tmem = *bar.tmem_slot;
  constexpr int kThreads = 32 * NWARPS;
  constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8 > 255 ? 248 : (65536 / kThreads) / 8 * 8;
  static_assert(32 * NSOFT * (REG_SOFTMAX - kLaunchRegs) <= (kThreads - 32 * NSOFT) * (kLaunchRegs - REG_OTHER),
                "setmaxnreg budget would deadlock");
  if (warp < NSOFT) {
    setmaxnreg_inc<REG_SOFTMAX>();
    softmax<D, OUT_F32>(p, bar, tmem, tid, smem_u32(smem + L::OFF_TURN));
  } else {
    setmaxnreg_dec<REG_OTHER>();
    if (warp < WARP_PROD0) {
      mma_chain<D>(p, smem, bar, tmem, warp - WARP_MMA0);
    } else if (warp < WARP_PROD0 + 4) {
      producer_half<D>(p, smem, bar, (warp - WARP_PROD0) >> 1, (warp - WARP_PROD0) & 1, lane);
    } else if (warp == WARP_QLOAD) {
      q_loader<D>(p, &tmQ, smem, bar, lane);
    }
  }
  tc_fence_before();
  __syncthreads();
  record_cta_ns(p, 1);
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool F32>
int launch_dual(const CUtensorMap* maps, const AttnParams& p, cudaStream_t stream) {
  auto kern = fga_attn_dual_kernel<D, F32>;
  const int smem = DuSmem<D>::BYTES;
  if (const int rc = smem_opt_in(reinterpret_cast<const void*>(kern), smem, "attn_dual"); rc != FGA_OK)
    return rc;
  const int sms = sm_count();
  const int64_t groups = (p.n_tiles - p.tile_begin) / 2;
  const int64_t grid = groups < sms ? groups : sms;
  kern<<<static_cast<unsigned>(grid), 32 * NWARPS, smem, stream>>>(maps[0], p);
  return check_launch("fga_attn_dual_kernel");
}

}  // namespace

// Sparse attention for groups of 129..256 rows with both tiles of a group sharing every gathered
// chunk; FGA_EUNSUPPORTED (caller uses attn_ws.cu) unless tiles_per_group == 2, the launch covers
// whole groups and the keys are gathered (not dense).
int launch_attn_dual(const CUtensorMap* maps, const AttnParams& p, int d, bool out_f32, cudaStream_t stream) {
  if (p.dense || p.tiles_per_group != 2 || (p.tile_begin % 2) != 0 || ((p.n_tiles - p.tile_begin) % 2) != 0)
    return FGA_EUNSUPPORTED;
  if (d == 64) return out_f32 ? launch_dual<64, true>(maps, p, stream) : launch_dual<64, false>(maps, p, stream);
  return out_f32 ? launch_dual<128, true>(maps, p, stream) : launch_dual<128, false>(maps, p, stream);
}

}  // namespace fga
