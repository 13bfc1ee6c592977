// FG-Attn forward on sm_100a, ping-pong softmax (v11).
//
// Reference semantics: /root/reference/pkg/src/sliceattn/sparse.py:111-156 (per-(b,h,g)
// chunk loop over the key list) with the online softmax of tiled.py:48-77.  Same work
// tiles, chunks, gather producers and MMA issuers as attn_ws.cu (v9); what changes is how
// the softmax overlaps with itself:
//
//   v9:  all 8 softmax warps work on the same chunk (two warps per TMEM lane quadrant,
//        each row split over a quad of threads), so a chunk's TMEM load, barrier and
//        store latency is exposed once per chunk on every sub-partition.
//   v11: two softmax warpgroups on alternate chunks.  Warpgroup r (warps 4r..4r+3) owns
//        every chunk of CTA-wide parity r, its S/P buffer S_r, its own running max per row
//        and its own accumulator O_r; thread = query row (32x32b TMEM shapes, 128 scores
//        per thread).  While one warpgroup waits for S or stores P, the other one keeps
//        the sub-partition's MUFU busy.  The two partial results are merged in the
//        epilogue: O = (2^(m0-m) O_0 + 2^(m1-m) O_1) / (2^(m0-m) l_0 + 2^(m1-m) l_1).
//
// TMEM (512 columns): O_0 [0,128) | O_1 [128,256) | S_0 [256,384) | S_1 [384,512); P_c
// (bf16 pairs, 64 columns) overwrites S_r.  The second accumulator takes the columns v9
// used for Q, so Q lives in SMEM again (one 32 KB buffer loaded by TMA, S by SS-MMA) and
// a Q-loader warp refills it once both issuers' last S of the tile has completed.
//
// Because O_r only ever receives PVs from issuer r, and tcgen05 ops of one thread
// complete in order, "S_c is complete" (s_full) already implies that the previous PV into
// O_r is complete: a lazy rescale of O_r needs no extra barrier.
//
// Warps (16, one CTA per SM):
//   0-3 softmax warpgroup 0 (even chunks), 4-7 softmax warpgroup 1 (odd chunks)
//   8, 9  MMA issuers for buffer 0 / 1
//   10-13 gather producers (K rows 0-63, K rows 64-127, V rows 0-63, V rows 64-127:
//         one per SM sub-partition, so their LDGSTS load the MIO queues evenly)
//   14    Q loader (TMA), 15 idle
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
constexpr int NSK = 3, NSV = 3;  // K / V ring slots
constexpr int REG_SOFTMAX = 184;
constexpr int REG_OTHER = 72;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units (factor 256)
constexpr float RESCALE_SUM = 256.0f;      // 2^RESCALE_THRESHOLD
constexpr uint32_t TM_O = 0, TM_S = 256;   // O_r at r*128, S_r at 256 + r*128
#ifndef PP_TURNS
#define PP_TURNS 1  // the two softmax groups take turns on the MUFU (see turn_wait)
#endif
#ifndef PP_PASS_AT
#define PP_PASS_AT 4  // the MUFU turn passes after this many of the row's four 32-score blocks
#endif
#ifndef PP_NOGATHER
#define PP_NOGATHER 0  // timing experiment only: zeroed K/V, no copies
#endif
#ifndef PP_POLY
#define PP_POLY 0  // 1 in PP_POLY exp pairs by the FMA-pipe polynomial (0: none)
#endif
#ifndef PP_POLY_DEG
#define PP_POLY_DEG 3
#endif
#ifndef PP_NOEXP
#define PP_NOEXP 0  // timing experiment only: P = S bits, no exp
#endif

template <int D>
struct PpSmem {
  static constexpr int KV = (D / 64) * HALF;  // one K or V chunk, or the Q tile
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + KV;
  static constexpr int OFF_V = OFF_K + NSK * KV;
  static constexpr int OFF_BAR = OFF_V + NSV * KV;
  static constexpr int NBAR = 2 * (NSK + NSV) + 2 + 2 + 4;
  static constexpr int OFF_XCH = OFF_BAR + ((NBAR * 8 + 16 + 15) / 16) * 16;  // epilogue: m, l per row per group
  static constexpr int OFF_TURN = OFF_XCH + 4 * 128 * 4;  // a 0.0f word and a scratch word (turn_wait/pass)
  static constexpr int BYTES = OFF_TURN + 4 + 8 * 4;  // the 0.0f word + one scratch word per softmax warp (SMEM is full)
  static_assert(BYTES <= 232448, "exceeds the 227 KB of shared memory per CTA");
};

struct Bars {
  uint64_t* k_full;   // [NSK] count 64 (two producer warps x 32 cp.async arrivals)
  uint64_t* k_empty;  // [NSK] S-issuer commit
  uint64_t* v_full;   // [NSV] count 64
  uint64_t* v_empty;  // [NSV] PV-issuer commit
  uint64_t* s_full;   // [2] issuer r commit
  uint64_t* p_full;   // [2] count 4 (the warps of softmax group r)
  uint64_t* q_full;   // Q loader expect_tx
  uint64_t* q_empty;  // count 2: both issuers' last S of the tile complete
  uint64_t* o_full;   // count 2: both chains' last PV of the tile complete
  uint64_t* o_empty;  // count 8: both accumulators read and cleared
  uint32_t* tmem_slot;
};

template <int D>
__device__ __forceinline__ Bars carve_bars(uint8_t* smem) {
  using L = PpSmem<D>;
  uint64_t* b = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  Bars r;
  r.k_full = b;
  r.k_empty = r.k_full + NSK;
  r.v_full = r.k_empty + NSK;
  r.v_empty = r.v_full + NSV;
  r.s_full = r.v_empty + NSV;
  r.p_full = r.s_full + 2;
  r.q_full = r.p_full + 2;
  r.q_empty = r.q_full + 1;
  r.o_full = r.q_empty + 1;
  r.o_empty = r.o_full + 1;
  r.tmem_slot = reinterpret_cast<uint32_t*>(r.o_empty + 1);
  return r;
}

// ------------------------------------------------------------------ producers
// Warp (kv, part) packs rows 64*part .. 64*part+63 of every chunk of ring kv with 16-byte
// cp.async into the 128B-swizzled slot (rows past the list end zero-filled).  A slot
// completes with both halves' 64 arrivals, so every warp sees every use of every slot of
// its ring and the empty-barrier parity can never be two phases behind.
template <int D>
__device__ __forceinline__ void producer_half(const AttnParams& p, const CUtensorMap* tmK2, const CUtensorMap* tmV2,
                                              uint8_t* smem, const Bars& bar, int kv, int part, int lane) {
  using L = PpSmem<D>;
  constexpr int LPR = D / 8;     // lanes per 2*D-byte row
  constexpr int RPI = 32 / LPR;  // rows per warp instruction
  constexpr int ROWS = BN / 2;
  constexpr int nslot = NSK;
  static_assert(NSK == NSV, "one slot count for both rings");
  const uint64_t pol_kv = policy_evict_last();
  const int sub = lane / LPR, ch = lane % LPR;
  const uint32_t lane_off = static_cast<uint32_t>((ch >> 3) * HALF);
  const int cc = ch & 7;
  uint8_t* ring = smem + (kv ? L::OFF_V : L::OFF_K);
  const uint32_t ring_base = smem_u32(ring) + part * ROWS * 128;
  uint64_t* fullb = kv ? bar.v_full : bar.k_full;
  uint64_t* emptyb = kv ? bar.v_empty : bar.k_empty;
  const CUtensorMap* tm = kv ? tmV2 : tmK2;
  constexpr int PER = 8 / RPI;
  uint32_t item = 0;
  for (int64_t tile = p.tile_begin + blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    const Tile t = decode_tile(p, tile);
    const char* gsrc = static_cast<const char*>(kv ? p.v : p.k) + static_cast<int64_t>(t.row0) * (D * 2) + ch * 16;
    for (int c = 0; c < t.nchunks; ++c, ++item) {
      const uint32_t slot = item % nslot, use = item / nslot;
      uint64_t* full = &fullb[slot];
      if (p.dense) {
        mbar_wait(&emptyb[slot], (use & 1) ^ 1);
        if (part == 0 && lane == 0) {
          mbar_expect_tx(full, BN * D * 2);
#pragma unroll
          for (int h = 0; h < D / 64; ++h)
            tma_load_2d(ring + slot * L::KV + h * HALF, tm, full, h * 64, t.row0 + c * BN, pol_kv);
        } else {
          mbar_arrive(full);
        }
        continue;
      }
      int keys[ROWS / 32];
#pragma unroll
      for (int i = 0; i < ROWS / 32; ++i) {
        const int row = c * BN + part * ROWS + i * 32 + lane;
        keys[i] = row < t.count ? __ldg(t.list + row) : -1;
      }
      mbar_wait(&emptyb[slot], (use & 1) ^ 1);
      const char* src = gsrc;
      // opaque to the optimiser, so src + key * 2D stays one IMAD.WIDE.U32 per copy
      asm volatile("mov.b64 %0, %0;" : "+l"(src));
      // SW128: row r's 16-byte chunk cc lands at r*128 + ((cc ^ (r & 7)) << 4)
      uint32_t dstb[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u)
        dstb[u] = ring_base + slot * L::KV + lane_off + sub * 128 + ((cc ^ ((u * RPI + sub) & 7)) << 4);
      if (PP_NOGATHER) {
      } else if (c * BN + part * ROWS + ROWS <= t.count) {
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i) {
#pragma unroll
          for (int mm = 0; mm < 32 / RPI; ++mm) {
            const uint32_t key = static_cast<uint32_t>(__shfl_sync(0xffffffffu, keys[i], mm * RPI + sub));
            cp_async16_full(dstb[mm % PER] + (i * 32 + mm * RPI) * 128, src + static_cast<size_t>(key) * (D * 2));
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i) {
#pragma unroll
          for (int mm = 0; mm < 32 / RPI; ++mm) {
            const int key = __shfl_sync(0xffffffffu, keys[i], mm * RPI + sub);
            const char* g = src + static_cast<size_t>(static_cast<uint32_t>(max(key, 0))) * (D * 2);
            cp_async16(dstb[mm % PER] + (i * 32 + mm * RPI) * 128, g, key >= 0 ? 16u : 0u);
          }
        }
      }
      cp_async_arrive_noinc(full);
    }
  }
}

// Q loader: one TMA load of the tile's 128 query rows into the Q buffer once both issuers'
// last S of the previous tile has completed; the tile after next is prefetched into L2.
template <int D>
__device__ __forceinline__ void q_loader(const AttnParams& p, const CUtensorMap* tmQ, uint8_t* smem, const Bars& bar,
                                         int lane) {
  using L = PpSmem<D>;
  const uint64_t pol_q = policy_evict_first();  // each Q tile is read once
  int it = 0;
  for (int64_t tile = p.tile_begin + blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const Tile t = decode_tile(p, tile);
    mbar_wait(bar.q_empty, (it & 1) ^ 1);
    if (lane == 0) FGA_TT(p, it, 0);
    if (lane == 0) {
      mbar_expect_tx(bar.q_full, BM * D * 2);
#pragma unroll
      for (int h = 0; h < D / 64; ++h) tma_load_2d(smem + L::OFF_Q + h * HALF, tmQ, bar.q_full, h * 64, t.row0 + t.q0, pol_q);
      if (tile + gridDim.x < p.n_tiles) {
        const Tile n = decode_tile(p, tile + gridDim.x);
#pragma unroll
        for (int h = 0; h < D / 64; ++h) tma_prefetch_2d(tmQ, h * 64, n.row0 + n.q0);
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ MMA issuers
// Issuer r owns the chunks of CTA-wide parity r: S_c = Q K_c^T into S_r (SS-MMA), then,
// after softmax group r has written P_c, O_r += P_c V_c (TS-MMA).  S_{c+2} reuses the
// buffer PV_c reads and comes from the same thread, so tcgen05's in-order execution is
// the only ordering needed.
template <int D>
__device__ __forceinline__ void mma_chain(const AttnParams& p, uint8_t* smem, const Bars& bar, uint32_t tmem, int r) {
  using L = PpSmem<D>;
  constexpr uint32_t IDESC_S = idesc_bf16(BM, BN, false, false);  // Q, K both K-major in SMEM
  constexpr uint32_t IDESC_O = idesc_bf16(BM, D, false, true);    // P (TMEM), V MN-major
  const uint64_t dq0 = sdesc_sw128(smem_u32(smem + L::OFF_Q), 16, 1024);
  const uint64_t dk0 = sdesc_sw128(smem_u32(smem + L::OFF_K), 16, 1024);
  const uint64_t dv0 = sdesc_sw128(smem_u32(smem + L::OFF_V), HALF, 1024);
  const uint32_t tO = tmem + TM_O + r * 128, tS = tmem + TM_S + r * 128;
  uint32_t c0 = 0;  // CTA-wide index of the tile's first chunk
  int it = 0;
  for (int64_t tile = p.tile_begin + blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const Tile t = decode_tile(p, tile);
    mbar_wait(bar.q_full, it & 1);
    FGA_TT(p, it, 6 + r);
    tc_fence_after();
    bool o_free = false, q_done = false;
    for (int j = (r - static_cast<int>(c0 & 1)) & 1; j < t.nchunks; j += 2) {
      const uint32_t c = c0 + j;
      {  // ---- S_c = Q K_c^T
        const uint32_t slot = c % NSK, use = c / NSK;
        FGA_TS(p, it, j, 8);
        mbar_wait(&bar.k_full[slot], use & 1);
        FGA_TS(p, it, j, 9);
        fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05.mma (async proxy) reads
        tc_fence_after();
        const uint64_t dk = dk0 + ((slot * L::KV) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * HALF + (kk & 3) * 32) >> 4;
            umma_ss(tS, dq0 + off, dk + off, IDESC_S, kk > 0 ? 1u : 0u);
          }
          umma_commit(&bar.s_full[r]);
          umma_commit(&bar.k_empty[slot]);
          if (j + 2 >= t.nchunks) umma_commit(bar.q_empty);  // this chain's last read of Q in the tile
        }
        __syncwarp();
        if (j + 2 >= t.nchunks) q_done = true;
      }
      {  // ---- O_r += P_c V_c
        if (!o_free) {
          mbar_wait(bar.o_empty, it & 1);  // both accumulators cleared by the previous epilogue
          tc_fence_after();
          o_free = true;
        }
        FGA_TS(p, it, j, 10);
        mbar_wait(&bar.p_full[r], (c >> 1) & 1);
        FGA_TS(p, it, j, 11);
        const uint32_t slot = c % NSV, use = c / NSV;
        mbar_wait(&bar.v_full[slot], use & 1);
        FGA_TS(p, it, j, 12);
        fence_proxy_async_smem();
        tc_fence_after();
        const uint64_t dv = dv0 + ((slot * L::KV) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) umma_ts(tO, tS + kk * 8, dv + ((kk * 16 * 128) >> 4), IDESC_O, 1u);
          umma_commit(&bar.v_empty[slot]);
        }
        __syncwarp();
        FGA_TS(p, it, j, 13);
      }
    }
    if (elect_one()) {
      if (!q_done) umma_commit(bar.q_empty);  // no chunk of this tile on this chain
    }
    __syncwarp();
    if (!o_free) mbar_wait(bar.o_empty, it & 1);  // keep the phase in step on a tile without our chunks
    if (elect_one()) umma_commit(bar.o_full);
    __syncwarp();
    c0 += static_cast<uint32_t>(t.nchunks);
  }
}

// ------------------------------------------------------------------ softmax
__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
// MUFU turn-taking between the two softmax warps of one SM sub-partition (lane quadrant q):
// named barrier 2 + 2q + r is "warp (r, q) may exponentiate"; the other group's warp
// arrives on it when it has finished its own exps.  Strict alternation follows the chunk
// order (group r owns the chunks of parity r), so at most one arrival is ever pending.
// The exps are register-only instructions that ptxas may move across a barrier, so the
// barriers are tied to them through shared memory, which bar.sync / bar.arrive do order:
// after the wait, m += (a shared 0.0f) makes every exp argument depend on a load issued
// after the barrier; before the pass, the partial sums (which depend on every exp so far)
// are stored to a scratch word.
__device__ __forceinline__ void turn_wait(int q, int r, float& m, uint32_t zero_addr) {
  if (PP_TURNS)
    asm volatile("{\n.reg .f32 z;\nbar.sync %1, 64;\nld.shared.f32 z, [%2];\nadd.f32 %0, %0, z;\n}\n"
                 : "+f"(m)
                 : "r"(2 + 2 * q + r), "r"(zero_addr)
                 : "memory");
}
__device__ __forceinline__ void turn_pass(int q, int r, float2 a, float2 b, uint32_t junk_addr) {
  if (PP_TURNS)
    asm volatile("{\n.reg .f32 z;\nadd.f32 z, %0, %1;\nadd.f32 z, z, %2;\nadd.f32 z, z, %3;\n"
                 "st.shared.f32 [%5], z;\nbar.arrive %4, 64;\n}\n" ::"f"(a.x),
                 "f"(a.y), "f"(b.x), "f"(b.y), "r"(2 + 2 * q + (r ^ 1)), "r"(junk_addr)
                 : "memory");
}

__device__ __forceinline__ void load_s(uint32_t tS, uint32_t (&s)[4][32]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) tmem_ld32(tS + 32 * i, s[i]);
  tmem_ld_wait();
}

__device__ __forceinline__ void mask_tail(uint32_t (&s)[4][32], int nvalid) {
  if (nvalid < BN) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (32 * i + k >= nvalid) s[i][k] = __float_as_uint(-INFINITY);
  }
}

__device__ __forceinline__ float row_max(const uint32_t (&s)[4][32]) {
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int k = 0; k < 32; k += 2) m = fmax3f(m, __uint_as_float(s[i][k]), __uint_as_float(s[i][k + 1]));
  }
  return m;
}

// P = 2^(s * scale * log2e - m) for this thread's row: packed FFMA2 arguments, MUFU ex2,
// packed FADD2 partial sums, key pairs (2i, 2i+1) packed into bf16x2 column i of P.
__device__ __forceinline__ float exp_row(const uint32_t (&s)[4][32], float sl2, float m, uint32_t (&pk)[64], int q,
                                         int r, bool pass, uint32_t junk) {
  const float2 sc2 = make_float2(sl2, sl2), nm = make_float2(-m, -m);
  float2 sum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[i][2 * k]), __uint_as_float(s[i][2 * k + 1])), sc2, nm);
      float2 pr;
      if (PP_NOEXP) {
        pr = x;  // timing experiment only
      } else if (PP_POLY > 0 && (16 * i + k) % PP_POLY == PP_POLY - 1) {
        pr = ex2_poly2<PP_POLY_DEG>(x);  // FMA pipe: a single warp cannot saturate the MUFU
      } else {
        pr.x = ex2(x.x);
        pr.y = ex2(x.y);
      }
      sum[k & 1] = __fadd2_rn(sum[k & 1], pr);
      pk[16 * i + k] = pack_bf16(pr.x, pr.y);
    }
    if (i == PP_PASS_AT - 1 && pass) turn_pass(q, r, sum[0], sum[1], junk);
  }
  const float2 u = __fadd2_rn(sum[0], sum[1]);
  return PP_NOEXP ? 1.f : u.x + u.y;
}

template <int D, bool OUT_F32>
__device__ __forceinline__ void softmax(const AttnParams& p, const Bars& bar, uint32_t tmem, int tid, float* xch,
                                        uint32_t zaddr) {
  const uint32_t junk = zaddr + 4 + 4 * (tid >> 5);  // per-warp scratch word (its lanes write the same word: benign)
  const int warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, r = warp >> 2;  // lane quadrant, softmax group (= chunk parity)
  const int row = q * 32 + lane;
  const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
  const uint32_t tS = tmem + TM_S + r * 128 + lanes;
  const uint32_t tOr = tmem + TM_O + r * 128 + lanes;
  const float sl2 = p.scale_log2;
  const bool tr = (tid & 127) == 0;
  uint32_t zero[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) zero[i] = 0u;
  int64_t tile = p.tile_begin + blockIdx.x;
  if (tile < p.n_tiles) {
#pragma unroll
    for (int i = 0; i < D / 32; ++i) tmem_st32(tOr + i * 32, zero);  // every PV accumulates into O_r
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(bar.o_empty);
    if (r == 1) {  // chunk 0 belongs to group 0
      turn_pass(q, r, make_float2(0.f, 0.f), make_float2(0.f, 0.f), junk);
    }
  }
  uint32_t c0 = 0;
  for (int it = 0; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const Tile t = decode_tile(p, tile);
    float m = -INFINITY, l = 0.f;  // this group's running max (log2 units) and row sum
    bool first = true;
    for (int j = (r - static_cast<int>(c0 & 1)) & 1; j < t.nchunks; j += 2) {
      const uint32_t c = c0 + j;
      if (tr) FGA_TS(p, it, j, 0);
      mbar_wait(&bar.s_full[r], (c >> 1) & 1);
      tc_fence_after();
      uint32_t s[4][32];
      load_s(tS, s);
      if (tr) FGA_TS(p, it, j, 1);
      const int nvalid = min(BN, t.count - j * BN);
      mask_tail(s, nvalid);
      uint32_t pk[64];
      float alpha = 1.f, sum;
      bool rescale = false;
      if (first) {
        m = row_max(s) * sl2;
        turn_wait(q, r, m, zaddr);
        sum = exp_row(s, sl2, m, pk, q, r, true, junk);
        first = false;
      } else {
        // fast path: P with the running max.  A score above it by more than
        // RESCALE_THRESHOLD makes the row sum exceed 2^THRESHOLD (all terms are positive)
        turn_wait(q, r, m, zaddr);
        sum = exp_row(s, sl2, m, pk, q, r, true, junk);
        if (__any_sync(0xffffffffu, !(sum <= RESCALE_SUM))) {
          // slow path (rare): S is still intact in TMEM (P not yet stored), reload it,
          // move the running max, recompute P; O_r is rescaled below
          load_s(tS, s);
          mask_tail(s, nvalid);
          const float rmax = row_max(s) * sl2;
          if (rmax - m > RESCALE_THRESHOLD) {
            alpha = ex2(m - rmax);
            m = rmax;
            rescale = true;
          }
          sum = exp_row(s, sl2, m, pk, q, r, false, junk);
        }
      }
      if (__any_sync(0xffffffffu, rescale)) {
        // S_c complete => the previous PV into O_r (same issuer, issued before S_c) is complete
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
      if (tr) FGA_TS(p, it, j, 2);
      {
        uint32_t a[32], b[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          a[k] = pk[k];
          b[k] = pk[32 + k];
        }
        tmem_st32(tS, a);
        tmem_st32(tS + 32, b);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar.p_full[r]);
      if (tr) FGA_TS(p, it, j, 3);
    }
    c0 += static_cast<uint32_t>(t.nchunks);
    if (tr) FGA_TT(p, it, 2 + r);
    // ---- epilogue: merge the two groups' partial results (tiled.py:73-77 per group)
    xch[r * 256 + row] = m;
    xch[r * 256 + 128 + row] = l;
    softmax_bar();
    const float mo = xch[(r ^ 1) * 256 + row], lo = xch[(r ^ 1) * 256 + 128 + row];
    softmax_bar();  // all reads done before the next tile rewrites xch
    const float mx = fmaxf(m, mo);
    const float ss = m == -INFINITY ? 0.f : ex2(m - mx), so = mo == -INFINITY ? 0.f : ex2(mo - mx);
    const float lt = l * ss + lo * so;
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    const float c_0 = (r == 0 ? ss : so) * inv, c_1 = (r == 0 ? so : ss) * inv;
    mbar_wait(bar.o_full, it & 1);
    if (tr) FGA_TT(p, it, 4 + r);
    tc_fence_after();
    const bool valid = row < t.rows;
    const int64_t out_row = static_cast<int64_t>(t.row0) + t.q0 + row;
    // group r finalises columns [r*D/2, (r+1)*D/2) of both accumulators
#pragma unroll
    for (int i = 0; i < D / 64; ++i) {
      const int col = r * (D / 2) + 32 * i;
      uint32_t a[32], b[32];
      tmem_ld32(tmem + TM_O + lanes + col, a);
      tmem_ld32(tmem + TM_O + 128 + lanes + col, b);
      tmem_ld_wait();
      tmem_st32(tmem + TM_O + lanes + col, zero);  // cleared for the next tile
      tmem_st32(tmem + TM_O + 128 + lanes + col, zero);
#pragma unroll
      for (int k = 0; k < 32; ++k) a[k] = __float_as_uint(__uint_as_float(a[k]) * c_0 + __uint_as_float(b[k]) * c_1);
      if (valid) store_row32<OUT_F32>(p.out, out_row * D + col, a, 1.0f);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(bar.o_empty);
    if (r == 0 && valid && p.lse != nullptr) p.lse[out_row] = lt > 0.f ? mx * 0.69314718055994531f + logf(lt) : -INFINITY;
  }
  if (c0 > 0 && static_cast<int>(c0 & 1) == r) {  // the turn passed after the last chunk
    float dummy = 0.f;
    turn_wait(q, r, dummy, zaddr);
  }
}

template <int D, bool OUT_F32>
__global__ void __launch_bounds__(32 * NWARPS, 1)
    fga_attn_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK2,
                       const __grid_constant__ CUtensorMap tmV2, const AttnParams p) {
  using L = PpSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_pp[];
  uint8_t* smem = smem_pp;
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 atoms need 1 KB alignment
  const Bars bar = carve_bars<D>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    prefetch_tmap(&tmQ);
    if (p.dense) {
      prefetch_tmap(&tmK2);
      prefetch_tmap(&tmV2);
    }
    for (int i = 0; i < NSK; ++i) {
      mbar_init(&bar.k_full[i], 64);
      mbar_init(&bar.k_empty[i], 1);
    }
    for (int i = 0; i < NSV; ++i) {
      mbar_init(&bar.v_full[i], 64);
      mbar_init(&bar.v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar.s_full[i], 1);
      mbar_init(&bar.p_full[i], NSOFT / 2);
    }
    mbar_init(bar.q_full, 1);
    mbar_init(bar.q_empty, 2);
    mbar_init(bar.o_full, 2);
    mbar_init(bar.o_empty, NSOFT);
    *reinterpret_cast<float*>(smem + L::OFF_TURN) = 0.f;
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
  if (PP_NOGATHER) {
    for (int i = tid; i < (L::OFF_BAR - L::OFF_K) / 16; i += 32 * NWARPS)
      reinterpret_cast<uint4*>(smem + L::OFF_K)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
  }

  constexpr int kThreads = 32 * NWARPS;
  constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8 > 255 ? 248 : (65536 / kThreads) / 8 * 8;
  static_assert(32 * NSOFT * (REG_SOFTMAX - kLaunchRegs) <= (kThreads - 32 * NSOFT) * (kLaunchRegs - REG_OTHER),
                "setmaxnreg budget would deadlock");
  if (warp < NSOFT) {
    setmaxnreg_inc<REG_SOFTMAX>();
    softmax<D, OUT_F32>(p, bar, tmem, tid, reinterpret_cast<float*>(smem + L::OFF_XCH), smem_u32(smem + L::OFF_TURN));
  } else {
    setmaxnreg_dec<REG_OTHER>();
    if (warp < WARP_PROD0) {
      mma_chain<D>(p, smem, bar, tmem, warp - WARP_MMA0);
    } else if (warp < WARP_PROD0 + 4) {
      producer_half<D>(p, &tmK2, &tmV2, smem, bar, (warp - WARP_PROD0) >> 1, (warp - WARP_PROD0) & 1, lane);
    } else if (warp == WARP_QLOAD) {
      q_loader<D>(p, &tmQ, smem, bar, lane);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool F32>
int launch_pp(const CUtensorMap* maps, const AttnParams& p, cudaStream_t stream) {
  auto kern = fga_attn_pp_kernel<D, F32>;
  const int smem = PpSmem<D>::BYTES;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return check_launch("cudaFuncSetAttribute(attn_pp)");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t span = p.n_tiles - p.tile_begin;
  const int64_t grid = span < sms ? span : sms;
  kern<<<static_cast<unsigned>(grid), 32 * NWARPS, smem, stream>>>(maps[0], maps[3], maps[4], p);
  return check_launch("fga_attn_pp_kernel");
}

}  // namespace

int launch_attn_pp(const CUtensorMap* maps, const AttnParams& p, int d, bool out_f32, cudaStream_t stream) {
  if (d == 64) return out_f32 ? launch_pp<64, true>(maps, p, stream) : launch_pp<64, false>(maps, p, stream);
  return out_f32 ? launch_pp<128, true>(maps, p, stream) : launch_pp<128, false>(maps, p, stream);
}

}  // namespace fga
