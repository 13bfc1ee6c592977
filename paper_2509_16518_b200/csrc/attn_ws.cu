// FG-Attn forward on sm_100a: warp-specialised persistent kernel (v9).
//
// Reference semantics: /root/reference/pkg/src/sliceattn/sparse.py:111-156
// (per-(b,h,g) chunk loop over the key list) with the online softmax of
// tiled.py:48-77.  One work tile = <=128 query rows of one group; its key list
// is consumed in chunks of 128 gathered keys (a short last chunk is zero-filled
// past the list end and its extra score columns are set to -inf).
//
// Per chunk j:
//   S_j  = Q K_j^T   tcgen05 TS-MMA: Q (bf16) resident in TMEM, K_j from SMEM
//   P_j  = 2^(S_j * scale * log2e - m)   softmax warps, written over S_j in TMEM
//   O   += P_j V_j   tcgen05 TS-MMA: P_j from TMEM, V_j from SMEM
// With Q in TMEM the tensor core reads only the gathered K and V from SMEM
// (64 KB per chunk instead of 96 KB), which leaves SMEM bandwidth for the
// gather's 64 KB of writes, and all 224 KB of SMEM for the K/V rings.
//
// Softmax: 8 warps, two per TMEM lane quadrant.  Warp w owns the 16 query rows
// 32(w%4) + 16(w/4) .. +15 (tcgen05 16x256b / 16x128b shapes: each thread holds
// two rows x 32 of the 128 scores, row max reduced over the 4-thread quad), so
// every row has exactly one owner and one running max: a single O accumulator,
// both warpgroups working on the same chunk at once.
//
// Warps (16, one CTA per SM, persistent over tiles strided by the grid):
//   0-7   softmax + epilogue (+ writing the next tile's Q into TMEM)
//   8, 9  MMA issuers, one per S/P buffer (chunks of CTA-wide parity 0 / 1)
//   10-13 gather producers: K rows 0-63, K rows 64-127, V rows 0-63, V rows 64-127 of
//         every chunk, one warp per SM sub-partition, 16-byte cp.async into the
//         128B-swizzled ring slots (3 K + 3 V)
//   14    tile scheduler: claims tiles from a global counter (atomicAdd, in the order of
//         p.order when given: the host's per-head longest-first order) and hands them to every
//         role through a 2-entry shared ring (one tile claimed ahead), so CTAs that draw short
//         lists take more tiles
//   15    idle
// TMEM (512 cols): O [0, D) | Q [128, 128 + D/2) | S0 [256, 384) | S1 [384, 512).
// P_j (bf16 pairs) overwrites S[j%2] cols 0..63.
// Lazy rescale: the running max used for exp only moves when the row max grows
// by more than 8 (log2 units); O rows in TMEM are rescaled only then (rarely).
//
// Variants measured against this kernel and not kept (TMA gather4 producers, dedicated
// epilogue warps, S prefetch, FMA-pipe exp2, ...) are listed in DESIGN.md section 4; their
// code is in the git history (e.g. commit 3cb3ba1).
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>

#include "attn_common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace fga {
namespace {

constexpr int NSOFT = 8;      // softmax warps
constexpr int WARP_MMA0 = 8;  // MMA issuers 8 (buffer 0) and 9 (buffer 1)
constexpr int WARP_PROD0 = 10;
constexpr int NPROD = 4;      // gather producers 10-13
constexpr int WARP_SCHED = 14;
#ifndef FGA_NSCHED
#define FGA_NSCHED 2  // 16 (round-2 first cut) claimed 16 tiles per CTA up front: tail 1.10 vs 1.02
#endif
constexpr int NSCHED = FGA_NSCHED;  // tile ring entries = how far the scheduler claims ahead
constexpr int NCONSUMERS = NSOFT + 2 + NPROD;  // warps that read every tile ring entry
constexpr int NWARPS = 16;
constexpr int REG_SOFTMAX = 184;
constexpr int REG_OTHER = 72;  // producers and issuers: measured 13% slower at 64
#ifndef FGA_NSK
#define FGA_NSK 3
#endif
#ifndef FGA_NSV
#define FGA_NSV 3
#endif
constexpr int NSK = FGA_NSK, NSV = FGA_NSV;  // K / V ring slots
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units (factor 256)
constexpr float RESCALE_SUM = 256.0f;      // 2^RESCALE_THRESHOLD
constexpr uint32_t TM_O = 0, TM_Q = 128, TM_S = 256;
// Timing-experiment builds (DESIGN.md section 4 "structural floors"); all 0 in production.
#ifndef FGA_NOGATHER
#define FGA_NOGATHER 0  // producers copy nothing
#endif
#ifndef FGA_NOMMA
#define FGA_NOMMA 0  // issuers commit without MMAs
#endif
#ifndef FGA_NOEXP
#define FGA_NOEXP 0  // P = S bits, no exp
#endif
#ifndef FGA_PROD_HALF
#define FGA_PROD_HALF 1  // producers: lanes per 128-byte half row, one key shuffle per row for all its copies
#endif
#ifndef FGA_KFREE_LATE
#define FGA_KFREE_LATE 0  // A/B knob: free chunk c's K slot with PV_c's commit instead of S_c's
#endif
#ifndef FGA_QPF
#define FGA_QPF 1  // the first producer prefetches each tile's Q rows into L2 when it starts the tile
#endif
#ifndef FGA_PROD_SWAP
#define FGA_PROD_SWAP 0  // A/B knob: 1 puts the K producers on sub-partitions 0/1 and the V producers on 2/3
#endif
#ifndef FGA_PROD_LPR
#define FGA_PROD_LPR 8  // FGA_PROD_HALF: lanes per half row (8: 16 bytes each; 4 / 2: 32 / 64 bytes each)
#endif
#ifndef FGA_POLY
#define FGA_POLY 0  // A/B knob: every FGA_POLY-th exp pair on the FMA pipe (0: all on MUFU)
#endif
#ifndef FGA_POLY_DEG
#define FGA_POLY_DEG 3
#endif

constexpr int FULL_COUNT = 64;  // cp.async arrivals per K / V ring slot (two producer warps)

template <int D>
struct WsSmem {
  static constexpr int KV = (D / 64) * HALF;  // one K or V chunk
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + NSK * KV;
  static constexpr int OFF_BAR = OFF_V + NSV * KV;
  static constexpr int NBAR = 2 * (NSK + NSV) + 2 + 2 + 2 + 3 + 1 + 2 * NSCHED;
  static constexpr int OFF_XCH = OFF_BAR + ((NBAR * 8 + 16 + 15) / 16) * 16;  // epilogue: m, l per row
  static constexpr int OFF_SCHED = OFF_XCH + 2 * 128 * 4;                      // tile ring: int64 ids
  static constexpr int BYTES = OFF_SCHED + NSCHED * 8;
  static_assert(BYTES <= 232448, "exceeds the 227 KB of shared memory per CTA");
  static_assert(WARP_PROD0 + NPROD <= NWARPS, "too many producer warps");
};

struct Bars {
  uint64_t* k_full;     // [NSK] count FULL_COUNT (cp.async arrivals of the lanes that copy K)
  uint64_t* k_empty;    // [NSK] S-issuer commit
  uint64_t* v_full;     // [NSV] count FULL_COUNT
  uint64_t* v_empty;    // [NSV] PV-issuer commit
  uint64_t* s_full;     // [2]
  uint64_t* p_full;     // [2] count 8 (every softmax warp)
  uint64_t* pv_done;    // [2] completion of PV into S buffer b's P
  uint64_t* pv_issued;  // count 1: PV_c has been issued (PVs enter the tensor pipe in chunk order)
  uint64_t* q_full;     // count 8 (every softmax warp writes a part of Q)
  uint64_t* o_full;
  uint64_t* o_empty;    // count 8
  uint64_t* sched_full;   // [NSCHED] count 1 (the scheduler's arrival after writing the entry)
  uint64_t* sched_empty;  // [NSCHED] count NCONSUMERS
  int64_t* sched_tile;    // [NSCHED] tile id, -1 = no more work
  uint32_t* tmem_slot;
};

template <int D>
__device__ __forceinline__ Bars carve_bars(uint8_t* smem) {
  using L = WsSmem<D>;
  uint64_t* b = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  Bars r;
  r.k_full = b;
  r.k_empty = r.k_full + NSK;
  r.v_full = r.k_empty + NSK;
  r.v_empty = r.v_full + NSV;
  r.s_full = r.v_empty + NSV;
  r.p_full = r.s_full + 2;
  r.pv_done = r.p_full + 2;
  r.q_full = r.pv_done + 2;
  r.o_full = r.q_full + 1;
  r.o_empty = r.o_full + 1;
  r.pv_issued = r.o_empty + 1;
  r.sched_full = r.pv_issued + 1;
  r.sched_empty = r.sched_full + NSCHED;
  r.tmem_slot = reinterpret_cast<uint32_t*>(r.sched_empty + NSCHED);
  r.sched_tile = reinterpret_cast<int64_t*>(smem + L::OFF_SCHED);
  return r;
}

// ------------------------------------------------------------------ tile sequence
// Every role walks the same tile sequence.  Static (p.sched == null): tile_begin + blockIdx.x,
// strided by the grid.  Dynamic: the scheduler warp's ring; each consumer warp reads every entry
// once, in order, and releases it.
struct TileSeq {
  uint32_t i = 0;
  int64_t next_static;
  __device__ explicit TileSeq(const AttnParams& p) : next_static(p.tile_begin + blockIdx.x) {}
  __device__ __forceinline__ int64_t next(const AttnParams& p, const Bars& bar) {
    if (p.sched == nullptr) {
      const int64_t t = next_static;
      next_static += gridDim.x;
      return t < p.n_tiles ? t : -1;
    }
    const uint32_t slot = i % NSCHED;
    mbar_wait(&bar.sched_full[slot], (i / NSCHED) & 1);
    // lane 0 reads the entry and releases it (its read is ordered before its own arrival), the
    // warp gets the id by shuffle
    long long t = 0;
    if ((threadIdx.x & 31) == 0) {
      t = *reinterpret_cast<volatile int64_t*>(&bar.sched_tile[slot]);
      mbar_arrive(&bar.sched_empty[slot]);
    }
    ++i;
    return __shfl_sync(0xffffffffu, t, 0);
  }
};

// Claims work items from p.sched until they run out; the CTA that draws the last of the
// n_work + gridDim.x claims (every CTA makes exactly one failing claim) resets the counter to
// zero for the next launch that uses this slot.
__device__ __forceinline__ void tile_scheduler(const AttnParams& p, const Bars& bar) {
  const uint32_t n_work = static_cast<uint32_t>(p.n_tiles - p.tile_begin);
  for (uint32_t i = 0;; ++i) {
    const uint32_t slot = i % NSCHED;
    mbar_wait(&bar.sched_empty[slot], ((i / NSCHED) & 1) ^ 1);
    const uint32_t w = atomicAdd(p.sched, 1u);
    int64_t tile = -1;
    if (w < n_work) {
      tile = p.tile_begin + (p.order != nullptr ? __ldg(p.order + w) : static_cast<int64_t>(w));
    } else if (w == n_work + gridDim.x - 1) {
      atomicExch(p.sched, 0u);
    }
    *reinterpret_cast<volatile int64_t*>(&bar.sched_tile[slot]) = tile;
    mbar_arrive(&bar.sched_full[slot]);
    if (tile < 0) return;
  }
}

// ------------------------------------------------------------------ producers
// Four warps, one per SM sub-partition, each packing one 64-row half of every chunk of one
// ring (warp 10: K rows 0-63, 11: K rows 64-127, 12: V rows 0-63, 13: V rows 64-127 ->
// sub-partitions 2, 3, 0, 1): the LDGSTS traffic, which competes with the softmax's
// MUFU.EX2 for each sub-partition's issue/MIO resources, is the same in every TMEM lane
// quadrant.  The rings are filled and drained in chunk order; the two issuers free
// neighbouring chunks out of order, but a slot completes only with both halves' 64
// arrivals, so each producer sees every use of every slot of its ring and the empty-barrier
// parity can never be two phases behind.  Per 16 bytes: SHFL of the key, IMAD.WIDE address,
// LDGSTS into the 128B-swizzled slot; rows past the list end are zero-filled (src-size 0),
// so no stale or NaN bytes reach the MMA.
template <int D>
__device__ __forceinline__ void producer_half(const AttnParams& p, const CUtensorMap* tmK2, const CUtensorMap* tmV2,
                                              uint8_t* smem, const Bars& bar, int kv, int part, int lane,
                                              const void* qptr = nullptr) {
  using L = WsSmem<D>;
  // Lane mapping.  FGA_PROD_HALF: LPR lanes per 128-byte half row (64 columns), 32 / LPR rows per
  // instruction; each lane copies 16-byte chunks ch, ch + LPR, ... of every half of its row with
  // the same key (one SHFL per (8 / LPR) * (D / 64) copies; every instruction still covers whole
  // 32-byte sectors).  Otherwise D/8 lanes cover a whole row (one SHFL per copy).  c2 A/B (min of
  // 30 flushed launches): whole rows 2.472 ms, 8 lanes per half row 2.400 ms.
  constexpr int LPR = FGA_PROD_HALF ? FGA_PROD_LPR : D / 8;  // lanes per row (per copy instruction)
  constexpr int CPL = FGA_PROD_HALF ? 8 / FGA_PROD_LPR : 1;  // chunks per lane per half row
  constexpr int NH = FGA_PROD_HALF ? D / 64 : 1;             // halves copied per row with one key
  constexpr int RPI = 32 / LPR;  // rows per warp instruction
  constexpr int ROWS = BN / 2;
  const int nslot = kv ? NSV : NSK;
  const uint64_t pol_kv = policy_evict_last();
  const int sub = lane / LPR, ch = lane % LPR;
  const uint32_t lane_off = static_cast<uint32_t>((ch >> 3) * HALF);
  const int cc = ch & 7;
  uint8_t* ring = smem + (kv ? L::OFF_V : L::OFF_K);
  const uint32_t ring_base = smem_u32(ring) + part * ROWS * 128;
  uint64_t* fullb = kv ? bar.v_full : bar.k_full;
  uint64_t* emptyb = kv ? bar.v_empty : bar.k_empty;
  const CUtensorMap* tm = kv ? tmV2 : tmK2;
  // SW128 destination: row r's 16-byte chunk cc lands at r*128 + ((cc ^ (r & 7)) << 4).  This
  // lane's rows are mm*RPI + sub (+32i), so (r & 7) cycles with period PER = 8 / RPI in mm and
  // the address is dstb[mm % PER] + compile-time immediate.
  constexpr int PER = RPI >= 8 ? 1 : 8 / RPI;
  uint32_t item = 0;
  TileSeq seq(p);
  for (int64_t tile = seq.next(p, bar); tile >= 0; tile = seq.next(p, bar)) {
    const Tile t = decode_tile(p, tile);
    if (kv == 0 && part == 0 && lane == 0) {
      report_tile(p, t);
      // the producers start a tile ~3 chunks before the softmax warps load its Q rows
      // (write_q at the end of the previous tile): have them in L2 by then
      if (FGA_QPF && qptr != nullptr)
        bulk_prefetch_l2(static_cast<const __nv_bfloat16*>(qptr) + (static_cast<int64_t>(t.row0) + t.q0) * D,
                         static_cast<uint32_t>(t.rows) * D * 2);
    }
    const char* gsrc = static_cast<const char*>(kv ? p.v : p.k) + static_cast<int64_t>(t.row0) * (D * 2) + ch * 16;
    for (int c = 0; c < t.nchunks; ++c, ++item) {
      const uint32_t slot = item % nslot, use = item / nslot;
      uint64_t* full = &fullb[slot];
      if (p.dense) {  // contiguous keys: one TMA box per 64 columns (lane 0 of part 0), 63 arrivals
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
#pragma unroll
      for (int i = 0; i < ROWS / 32; ++i) keys[i] = clamp_key(p, keys[i], c * BN + part * ROWS + i * 32 + lane < t.count);
      const char* src = gsrc;
      // opaque to the optimiser, so src + key * 2D stays one IMAD.WIDE.U32 per copy
      asm volatile("mov.b64 %0, %0;" : "+l"(src));
      uint32_t dstb[PER][CPL];
#pragma unroll
      for (int u = 0; u < PER; ++u)
#pragma unroll
        for (int x = 0; x < CPL; ++x)
          dstb[u][x] = ring_base + slot * L::KV + lane_off + sub * 128 + (((cc + LPR * x) ^ ((u * RPI + sub) & 7)) << 4);
      if (FGA_NOGATHER) {
        // timing experiment only: no data movement
      } else if (c * BN + part * ROWS + ROWS <= t.count) {
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i) {
#pragma unroll
          for (int mm = 0; mm < 32 / RPI; ++mm) {
            const uint32_t key = static_cast<uint32_t>(__shfl_sync(0xffffffffu, keys[i], mm * RPI + sub));
            const char* g = src + static_cast<size_t>(key) * (D * 2);
#pragma unroll
            for (int hh = 0; hh < NH; ++hh)
#pragma unroll
              for (int x = 0; x < CPL; ++x)
                cp_async16_full(dstb[mm % PER][x] + hh * HALF + (i * 32 + mm * RPI) * 128, g + hh * 128 + x * LPR * 16);
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
#pragma unroll
              for (int x = 0; x < CPL; ++x)
                cp_async16(dstb[mm % PER][x] + hh * HALF + (i * 32 + mm * RPI) * 128, g + hh * 128 + x * LPR * 16,
                           key >= 0 ? 16u : 0u);
          }
        }
      }
      cp_async_arrive_noinc(full);
    }
  }
}

// ------------------------------------------------------------------ MMA issuers
// Two issuer warps, one per S/P buffer: issuer r owns the chunks of CTA-wide parity r
// and issues, for each of them in order, S_c = Q K_c^T into S[r] and then (after the
// softmax) O += P_c V_c.  S_{c+2} reuses the buffer PV_c reads, and both come from the
// same thread, so tcgen05's in-order execution is all the ordering needed: no
// completion wait sits between PV_c and S_{c+2}.  Two issuers matter because a
// tcgen05.mma issue stalls until the MMA unit takes it: while one chain waits for its
// softmax, the other keeps the tensor core fed.  O starts each tile at zero (the
// epilogue clears it), so every PV accumulates and the two chains' PVs commute.
template <int D>
__device__ __forceinline__ void mma_chain(const AttnParams& p, uint8_t* smem, const Bars& bar, uint32_t tmem, int r) {
  using L = WsSmem<D>;
  constexpr uint32_t IDESC_S = idesc_bf16(BM, BN, false, false);  // Q (TMEM), K K-major
  constexpr uint32_t IDESC_O = idesc_bf16(BM, D, false, true);    // P (TMEM), V MN-major
  const uint64_t dk0 = sdesc_sw128(smem_u32(smem + L::OFF_K), 16, 1024);
  const uint64_t dv0 = sdesc_sw128(smem_u32(smem + L::OFF_V), HALF, 1024);
  const uint32_t tQ = tmem + TM_Q, tO = tmem + TM_O, tS = tmem + TM_S + r * 128;
  uint32_t c0 = 0;  // CTA-wide index of the tile's first chunk
  int it = 0;
  TileSeq seq(p);
  for (int64_t tile = seq.next(p, bar); tile >= 0; tile = seq.next(p, bar), ++it) {
    const Tile t = decode_tile(p, tile);
    mbar_wait(bar.q_full, it & 1);  // waited every tile, so the phase never runs two ahead
    if (r == 0) FGA_TT(p, it, 1);
    tc_fence_after();
    bool o_free = false;
    for (int j = (r - static_cast<int>(c0 & 1)) & 1; j < t.nchunks; j += 2) {
      const uint32_t c = c0 + j;
      // ---- S_c = Q K_c^T
      {
        const uint32_t slot = c % NSK, use = c / NSK;
        if (r == 0) FGA_TS(p, it, j, 8);
        mbar_wait(&bar.k_full[slot], use & 1);
        if (r == 0) FGA_TS(p, it, j, 9);
        fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05.mma (async proxy) reads
        tc_fence_after();
        const uint64_t dk = dk0 + ((slot * L::KV) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * HALF + (kk & 3) * 32) >> 4;
            if (!FGA_NOMMA) umma_ts(tS, tQ + kk * 8, dk + off, IDESC_S, kk > 0 ? 1u : 0u);
          }
          umma_commit(&bar.s_full[r]);
          if (!FGA_KFREE_LATE) umma_commit(&bar.k_empty[slot]);
        }
        __syncwarp();
        if (r == 0) FGA_TS(p, it, j, 14);
      }
      // ---- O += P_c V_c
      {
        if (!o_free) {
          mbar_wait(bar.o_empty, it & 1);  // O cleared by the previous tile's epilogue
          tc_fence_after();
          o_free = true;
        }
        if (r == 0) FGA_TS(p, it, j, 10);
        mbar_wait(&bar.p_full[r], (c >> 1) & 1);
        if (r == 0) FGA_TS(p, it, j, 11);
        const uint32_t slot = c % NSV, use = c / NSV;
        mbar_wait(&bar.v_full[slot], use & 1);
        if (r == 0) FGA_TS(p, it, j, 6);
        fence_proxy_async_smem();
        tc_fence_after();
        const uint64_t dv = dv0 + ((slot * L::KV) >> 4);
        // Deterministic accumulation: PV_c enters the tensor pipe only after PV_{c-1} (the other
        // issuer's) has been issued, so O sums the chunks in list order on every run.
        if (c > 0) mbar_wait(bar.pv_issued, (c - 1) & 1);
        if (r == 0) FGA_TS(p, it, j, 7);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            if (!FGA_NOMMA) umma_ts(tO, tS + kk * 8, dv + ((kk * 16 * 128) >> 4), IDESC_O, 1u);
          umma_commit(&bar.v_empty[slot]);
          if (FGA_KFREE_LATE) umma_commit(&bar.k_empty[c % NSK]);  // S_c is done when PV_c is
          umma_commit(&bar.pv_done[r]);
          mbar_arrive(bar.pv_issued);
        }
        __syncwarp();
        if (r == 0) FGA_TS(p, it, j, 12);
      }
    }
    if (!o_free) mbar_wait(bar.o_empty, it & 1);  // keep the phase in step on a tile without our chunks
    if (elect_one()) umma_commit(bar.o_full);      // count 2: both chains' PVs of this tile complete
    __syncwarp();
    if (r == 0) FGA_TT(p, it, 3);
    c0 += t.nchunks;
  }
}

// ------------------------------------------------------------------ softmax warps
__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Q rows of tile t -> TMEM (A operand of S = Q K^T): warp (q, h) writes lanes
// 32q..32q+31 (thread = row), packed bf16 columns [h*D/4, (h+1)*D/4).
template <int D>
__device__ __forceinline__ void write_q(const AttnParams& p, const void* qptr, const Tile& t, uint32_t tmem, int q,
                                        int h, int lane) {
  constexpr int NC = D / 4;  // 32-bit TMEM columns per warp
  const int row = q * 32 + lane;
  uint32_t v[32];
  const bool ok = row < t.rows;
  const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(qptr) +
                                                    (static_cast<int64_t>(t.row0) + t.q0 + row) * D + h * (D / 2));
#pragma unroll
  for (int i = 0; i < NC / 4; ++i) {
    const uint4 x = ok ? __ldg(src + i) : make_uint4(0u, 0u, 0u, 0u);
    v[4 * i] = x.x; v[4 * i + 1] = x.y; v[4 * i + 2] = x.z; v[4 * i + 3] = x.w;
  }
  const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + TM_Q + h * NC;
  if constexpr (NC == 32) {
    tmem_st32(taddr, v);
  } else {
    uint32_t v16[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v16[i] = v[i];
    tmem_st16(taddr, v16);
  }
}

// P = 2^(s*scale*log2e - m) for this thread's 2 rows x 32 scores: packed FFMA2 for the
// argument, MUFU ex2, packed FADD2 row sums, bf16 pairs in the 16x128b register order.
__device__ __forceinline__ void exp_chunk(const uint32_t (&sv)[2][32], float sl2, const float (&m_use)[2],
                                          uint32_t (&pk)[32], float2 (&sum2)[2][2]) {
  const float2 sc2 = make_float2(sl2, sl2);
  const float2 nm[2] = {make_float2(-m_use[0], -m_use[0]), make_float2(-m_use[1], -m_use[1])};
#pragma unroll
  for (int r = 0; r < 2; ++r) sum2[r][0] = sum2[r][1] = make_float2(0.f, 0.f);
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float2 sx = make_float2(__uint_as_float(sv[hh][4 * k + 2 * r]), __uint_as_float(sv[hh][4 * k + 2 * r + 1]));
        const float2 x = __ffma2_rn(sx, sc2, nm[r]);
        // A/B knob FGA_POLY = p > 0: every p-th pair on the FMA pipe (ex2_poly2), the rest on MUFU
        constexpr int PP = FGA_POLY > 0 ? FGA_POLY : 1;
        const float2 pr = (FGA_POLY > 0 && (16 * hh + 2 * k + r) % PP == PP - 1)
                              ? ex2_poly2<FGA_POLY_DEG>(x)
                              : make_float2(ex2(x.x), ex2(x.y));
        sum2[r][k & 1] = __fadd2_rn(sum2[r][k & 1], pr);
        pk[2 * (8 * hh + k) + r] = pack_bf16(pr.x, pr.y);
      }
    }
  }
}

template <int D, bool OUT_F32>
__device__ __forceinline__ void softmax(const AttnParams& p, const void* qptr, const Bars& bar, uint32_t tmem, int tid,
                                        float* xch) {
  const int warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, h = warp >> 2, a = lane & 3, b = lane >> 2;
  const uint32_t lanes16 = static_cast<uint32_t>(q * 32 + h * 16) << 16;  // this warp's 16 rows
  const int r0 = q * 32 + h * 16 + b;                                       // rows r0 and r0 + 8
  const float sl2 = p.scale_log2;
  const bool tr = tid == 0;
  uint32_t chunk = 0;
  int it = 0;
  constexpr int NQ32 = D / 64;  // 32-column blocks of O per warp (rows 32q.., columns h*D/2..)
  const uint32_t tOw = tmem + TM_O + (static_cast<uint32_t>(q * 32) << 16) + h * (D / 2);
  uint32_t zero[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) zero[i] = 0u;
  TileSeq seq(p);
  int64_t tile = seq.next(p, bar);
  if (tile >= 0) {
    write_q<D>(p, qptr, decode_tile(p, tile), tmem, q, h, lane);
#pragma unroll
    for (int i = 0; i < NQ32; ++i) tmem_st32(tOw + i * 32, zero);  // every PV accumulates into O
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(bar.q_full);
      mbar_arrive(bar.o_empty);
    }
  }
  for (int64_t next_tile; tile >= 0; tile = next_tile, ++it) {
    const Tile t = decode_tile(p, tile);
    float m_use[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};  // l_run: this thread's partial sums
    uint32_t sv[2][32];  // [column half][4k + 2*row + e]: rows r0/r0+8, col 64*half + 8k + 2a + e
    for (int j = 0; j < t.nchunks; ++j) {
      const uint32_t c = chunk + j;
      const uint32_t tS = tmem + TM_S + (c & 1) * 128 + lanes16;
      if (tr) FGA_TS(p, it, j, 0);
      mbar_wait(&bar.s_full[c & 1], (c >> 1) & 1);
      if (tr) FGA_TS(p, it, j, 1);
      tc_fence_after();
      tmem_ld16x256_x8(tS, sv[0]);
      tmem_ld16x256_x8(tS + 64, sv[1]);
      tmem_ld_wait();
      if (tr) FGA_TS(p, it, j, 2);
      const int nvalid = min(BN, t.count - j * BN);
      if (nvalid < BN) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (64 * hh + 8 * k + 2 * a + e >= nvalid) {
                sv[hh][4 * k + e] = __float_as_uint(-INFINITY);
                sv[hh][4 * k + 2 + e] = __float_as_uint(-INFINITY);
              }
      }
      // Fast path (every chunk after the first): P with the current running max -- no row max,
      // no quad shuffles.  A score above the running max by more than RESCALE_THRESHOLD shows
      // up as a partial row sum above 2^THRESHOLD (all terms are positive), which sends the
      // warp to the slow path: quad-reduced row max, new running max (O rescaled), P recomputed.
      float alpha[2] = {1.f, 1.f};
      bool rescale = false;
      uint32_t pk[32];  // 16x128b: pk[2K + r] = (row r0 + 8r, P col 4K + a), K = 8*half + k
      float2 sum2[2][2];
      bool slow = j == 0 && !FGA_NOEXP;
      if (FGA_NOEXP) {  // timing experiment only: P = S bits, no exp
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = sv[i >> 4][i & 15];
        sum2[0][0] = sum2[0][1] = sum2[1][0] = sum2[1][1] = make_float2(1.f, 1.f);
        if (j == 0) m_use[0] = m_use[1] = 0.f;
      } else if (!slow) {
        exp_chunk(sv, sl2, m_use, pk, sum2);
        const float2 u0 = __fadd2_rn(sum2[0][0], sum2[0][1]), u1 = __fadd2_rn(sum2[1][0], sum2[1][1]);
        const bool over = !(u0.x + u0.y <= RESCALE_SUM) || !(u1.x + u1.y <= RESCALE_SUM);
        slow = __any_sync(0xffffffffu, over);
      }
      if (slow) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          float mh[2];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            // the 16 values of row r in this half: sv[hh][4*(i/2) + 2r + i%2], i = 0..15
#define FGA_SV(i) __uint_as_float(sv[hh][4 * ((i) >> 1) + 2 * r + ((i) & 1)])
            float m = fmax3f(FGA_SV(0), FGA_SV(1), FGA_SV(2));
#pragma unroll
            for (int i = 3; i < 15; i += 2) m = fmax3f(m, FGA_SV(i), FGA_SV(i + 1));
            mh[hh] = fmaxf(m, FGA_SV(15));
#undef FGA_SV
          }
          float m = fmaxf(mh[0], mh[1]);
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
          const float rmax = m * sl2;
          if (j == 0) {
            m_use[r] = rmax;
          } else if (rmax - m_use[r] > RESCALE_THRESHOLD) {
            alpha[r] = ex2(m_use[r] - rmax);
            m_use[r] = rmax;
            rescale = true;
          }
        }
        exp_chunk(sv, sl2, m_use, pk, sum2);
      }
      if (tr) FGA_TS(p, it, j, 3);
      tmem_st16x128_x16(tS, pk);
      if (tr) FGA_TS(p, it, j, 4);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float2 s = __fadd2_rn(sum2[r][0], sum2[r][1]);
        l_run[r] = l_run[r] * alpha[r] + (s.x + s.y);
      }
      if (__any_sync(0xffffffffu, rescale)) {
        // O holds PV_{c-1}: wait for it (PV_{c-3} is done, so the parity is unambiguous), then
        // scale this warp's rows in place (the PV of this chunk waits for our p_full arrival)
        if (j > 0) {
          mbar_wait(&bar.pv_done[(c - 1) & 1], ((c - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int hh = 0; hh < D / 64; ++hh) {
            uint32_t o[32];
            tmem_ld16x256_x8(tmem + TM_O + lanes16 + hh * 64, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha[(i >> 1) & 1]);
            tmem_st16x256_x8(tmem + TM_O + lanes16 + hh * 64, o);
          }
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar.p_full[c & 1]);
      if (tr) FGA_TS(p, it, j, 5);
      if (lane == 0) FGA_TW(p, it, j, warp);
    }
    chunk += t.nchunks;
    // every S of this tile has been consumed, so Q may be replaced by the next tile's
    next_tile = seq.next(p, bar);
    if (next_tile >= 0) {
      write_q<D>(p, qptr, decode_tile(p, next_tile), tmem, q, h, lane);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar.q_full);
    }
    // ---- epilogue: O / l -> global (tiled.py:73-77).  Row sums over the quad; the
    //      row owners publish (m, l), then warp (q, h) stores rows 32q.. of columns h*D/2..
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
      l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (a == 0) {
        xch[r0 + 8 * r] = m_use[r];
        xch[128 + r0 + 8 * r] = l_run[r];
      }
    softmax_bar();
    const int row = q * 32 + lane;
    const float mrow = xch[row], lrow = xch[128 + row];
    softmax_bar();  // all rows read before the next tile rewrites xch
    const float inv = lrow > 0.f ? 1.f / lrow : 0.f;
    mbar_wait(bar.o_full, it & 1);
    if (tid == 0) FGA_TT(p, it, 4);
    tc_fence_after();
    const bool valid = row < t.rows;
    const int64_t out_row = static_cast<int64_t>(t.row0) + t.q0 + row;
    uint32_t o[NQ32][32];
#pragma unroll
    for (int i = 0; i < NQ32; ++i) tmem_ld32(tOw + i * 32, o[i]);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < NQ32; ++i) tmem_st32(tOw + i * 32, zero);  // cleared for the next tile
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(bar.o_empty);  // O is in registers and zero again: the next tile's PVs may start
#pragma unroll
    for (int i = 0; i < NQ32; ++i)
      if (valid) store_row32<OUT_F32>(p.out, out_row * D + h * (D / 2) + i * 32, o[i], inv);
    if (h == 0 && valid && p.lse != nullptr)
      p.lse[out_row] = lrow > 0.f ? mrow * 0.69314718055994531f + logf(lrow) : -INFINITY;
    if (tid == 0) FGA_TT(p, it, 5);
  }
}

template <int D, bool OUT_F32>
__global__ void __launch_bounds__(32 * NWARPS, 1)
    fga_attn_ws_kernel(const __grid_constant__ CUtensorMap tmK2, const __grid_constant__ CUtensorMap tmV2,
                       const void* __restrict__ qptr, const AttnParams p) {
  using L = WsSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_ws[];
  uint8_t* smem = smem_ws;
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 atoms need 1 KB alignment
  const Bars bar = carve_bars<D>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    if (p.dense) {
      prefetch_tmap(&tmK2);
      prefetch_tmap(&tmV2);
    }
    for (int i = 0; i < NSK; ++i) {
      mbar_init(&bar.k_full[i], FULL_COUNT);  // every copying lane's arrival (dense: lane 0's expect_tx + the rest)
      mbar_init(&bar.k_empty[i], 1);
    }
    for (int i = 0; i < NSV; ++i) {
      mbar_init(&bar.v_full[i], FULL_COUNT);
      mbar_init(&bar.v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar.s_full[i], 1);
      mbar_init(&bar.p_full[i], NSOFT);
      mbar_init(&bar.pv_done[i], 1);
    }
    mbar_init(bar.q_full, NSOFT);
    mbar_init(bar.o_full, 2);
    mbar_init(bar.o_empty, NSOFT);
    mbar_init(bar.pv_issued, 1);
    for (int i = 0; i < NSCHED; ++i) {
      mbar_init(&bar.sched_full[i], 1);
      mbar_init(&bar.sched_empty[i], NCONSUMERS);
    }
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
  if (p.trace != nullptr && tid == 0 && blockIdx.x < 1024) p.trace[FGA_TRACE_CTA_OFF + 2 * blockIdx.x] = global_ns();
  record_cta_ns(p, 0);

  static_assert(NWARPS % 4 == 0, "whole warpgroups are needed for setmaxnreg");
  // setmaxnreg.inc can only take registers this CTA released with .dec (its pool is threads x launch regs)
  constexpr int kThreads = 32 * NWARPS;
  constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8 > 255 ? 248 : (65536 / kThreads) / 8 * 8;
  static_assert(32 * NSOFT * (REG_SOFTMAX - kLaunchRegs) <= (kThreads - 32 * NSOFT) * (kLaunchRegs - REG_OTHER),
                "setmaxnreg budget would deadlock");
  if (warp < NSOFT) {
    setmaxnreg_inc<REG_SOFTMAX>();
    softmax<D, OUT_F32>(p, qptr, bar, tmem, tid, reinterpret_cast<float*>(smem + L::OFF_XCH));
  } else {
    setmaxnreg_dec<REG_OTHER>();
    if (warp < WARP_PROD0) {
      mma_chain<D>(p, smem, bar, tmem, warp - WARP_MMA0);
    } else if (warp < WARP_PROD0 + NPROD) {
      producer_half<D>(p, &tmK2, &tmV2, smem, bar, ((warp - WARP_PROD0) >> 1) ^ FGA_PROD_SWAP, (warp - WARP_PROD0) & 1,
                       lane, qptr);
    } else if (warp == WARP_SCHED && p.sched != nullptr && lane == 0) {
      tile_scheduler(p, bar);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.trace != nullptr && tid == 0 && blockIdx.x < 1024) p.trace[FGA_TRACE_CTA_OFF + 2 * blockIdx.x + 1] = global_ns();
  record_cta_ns(p, 1);
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool F32>
int launch_ws(const CUtensorMap* maps, const void* q, const AttnParams& p, cudaStream_t stream) {
  auto kern = fga_attn_ws_kernel<D, F32>;
  const int smem = WsSmem<D>::BYTES;
  if (const int rc = smem_opt_in(reinterpret_cast<const void*>(kern), smem, "attn_ws"); rc != FGA_OK)
    return rc;
  const int sms = sm_count();
  const int64_t span = p.n_tiles - p.tile_begin;
  const int64_t grid = span < sms ? span : sms;
  kern<<<static_cast<unsigned>(grid), 32 * NWARPS, smem, stream>>>(maps[3], maps[4], q, p);
  return check_launch("fga_attn_ws_kernel");
}

// ------------------------------------------------------------------ K2 in isolation
// The hot path's own producer warps (producer_half, warps 10-13) filling the K and V rings for
// one tile, with warp 0 standing in for the MMA issuers: it waits for each chunk's slots, copies
// them out of the 128B swizzle into rows [128c, 128c + 128) of out_k / out_v and frees them.
// Bitwise the packed tiles the tensor core reads (rows past the list end zero-filled), so the
// gather is tested by itself (sparse.py:95-108), not only through the attention tolerance.
template <int D>
__global__ void __launch_bounds__(32 * NWARPS, 1)
    fga_ring_probe_kernel(const AttnParams p, __nv_bfloat16* __restrict__ out_k, __nv_bfloat16* __restrict__ out_v) {
  using L = WsSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_ws[];
  uint8_t* smem = smem_ws;
  const Bars bar = carve_bars<D>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NSK; ++i) { mbar_init(&bar.k_full[i], FULL_COUNT); mbar_init(&bar.k_empty[i], 1); }
    for (int i = 0; i < NSV; ++i) { mbar_init(&bar.v_full[i], FULL_COUNT); mbar_init(&bar.v_empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp >= WARP_PROD0 && warp < WARP_PROD0 + NPROD) {
    producer_half<D>(p, nullptr, nullptr, smem, bar, (warp - WARP_PROD0) >> 1, (warp - WARP_PROD0) & 1, lane);
  } else if (warp == 0) {
    const Tile t = decode_tile(p, p.tile_begin);
    for (int c = 0; c < t.nchunks; ++c) {
      for (int kv = 0; kv < 2; ++kv) {
        const int nslot = kv ? NSV : NSK;
        const uint32_t slot = c % nslot, use = c / nslot;
        mbar_wait(&(kv ? bar.v_full : bar.k_full)[slot], use & 1);
        const uint8_t* ring = smem + (kv ? L::OFF_V : L::OFF_K) + slot * L::KV;
        __nv_bfloat16* out = kv ? out_v : out_k;
        for (int e = lane; e < BN * (D / 8); e += 32) {  // 16-byte pieces, row-major
          const int r = e / (D / 8), pc = e % (D / 8), h = pc / 8, cc = pc % 8;
          const uint4 x = *reinterpret_cast<const uint4*>(ring + h * HALF + r * 128 + ((cc ^ (r & 7)) << 4));
          *reinterpret_cast<uint4*>(out + (static_cast<int64_t>(c) * BN + r) * D + pc * 8) = x;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&(kv ? bar.v_empty : bar.k_empty)[slot]);
        __syncwarp();
      }
    }
  }
}

}  // namespace

int launch_ring_probe(const AttnParams& p, int d, void* out_k, void* out_v, cudaStream_t stream) {
  const int smem = d == 64 ? WsSmem<64>::BYTES : WsSmem<128>::BYTES;
  const void* fn = d == 64 ? reinterpret_cast<const void*>(fga_ring_probe_kernel<64>)
                           : reinterpret_cast<const void*>(fga_ring_probe_kernel<128>);
  if (const int rc = smem_opt_in(fn, smem, "ring_probe"); rc != FGA_OK) return rc;
  auto* ok = static_cast<__nv_bfloat16*>(out_k);
  auto* ov = static_cast<__nv_bfloat16*>(out_v);
  if (d == 64)
    fga_ring_probe_kernel<64><<<1, 32 * NWARPS, smem, stream>>>(p, ok, ov);
  else
    fga_ring_probe_kernel<128><<<1, 32 * NWARPS, smem, stream>>>(p, ok, ov);
  return check_launch("fga_ring_probe_kernel");
}

int launch_attn_ws(const CUtensorMap* maps, const void* q, const AttnParams& p, int d, bool out_f32,
                   cudaStream_t stream) {
  if (d == 64) return out_f32 ? launch_ws<64, true>(maps, q, p, stream) : launch_ws<64, false>(maps, q, p, stream);
  return out_f32 ? launch_ws<128, true>(maps, q, p, stream) : launch_ws<128, false>(maps, q, p, stream);
}

}  // namespace fga
