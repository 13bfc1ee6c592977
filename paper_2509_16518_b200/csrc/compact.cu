// K1b: slice-mask compaction.  keep[row, :] (uint8) -> ascending kept key
// positions + count, bit-exact with
//   /root/reference/pkg/src/sliceattn/masks.py:75-91   (_lists_from_keep: np.nonzero,
//                                                        empty -> [argmax(scores)])
//   /root/reference/pkg/src/sliceattn/sparse.py:165-175 (export_padded: -1 tail)
//
// Two input formats: uint8 keep bytes (fga_compact) and bit-packed keep words
// (fga_compact_bits, 8x fewer bytes to read or to ship from the host).
//
// One 256-thread CTA per (b,h,g) row (keep bytes), or persistent CTAs looping over the rows
// with the next row's words prefetched (keep bits, FGA_CK_PERSIST); a row is walked in rounds of 8 warps x SPW steps
// of 1024 keys: warp w owns the contiguous steps [SPW*w, SPW*w + SPW) of the
// round, so every lane issues all SPW steps' loads before it needs any of
// them (keep bytes: lane l loads the 16-byte blocks at 16l and 512 + 16l of a
// step, two coalesced LDG.128; keep bits: word l of the step).  Per step a lane
// turns its bytes into two 16-bit occupancy masks with byte-SIMD arithmetic
// and ONE warp scan of the packed counts (low half: first 512 keys of the
// step, high half: last 512) gives its two offsets; the SPW scans are
// independent, so they overlap.  One __syncthreads per round exchanges the
// warp totals.  Each lane then emits its kept positions into its warp's
// shared-memory stage with an unrolled predicated loop (no divergence) and
// after a __syncwarp the warp writes the step's positions out coalesced (one
// 2 KB stage per warp and a second __syncwarp before the next step's emission:
// 16 KB per CTA and <= 48 registers give 5 CTAs per SM, faster than a
// double-buffered stage at 4 CTAs; FGA_CK_BUFS=2).
// Positions come out ascending, bit-exact with np.nonzero, with no sort.
// HBM-bound: read n bytes (n/8 for bits), write 4*count (+4*(n-count)).
// (Round-1 history: a block scan per 16 keys per thread was issue-bound at 80%
// issue-slot utilisation, 3.2 TB/s — ~270 instructions of per-round overhead
// per warp; one warp per row removed the barriers but left one serial step
// chain per warp with ~21 warps per SM: 2.5 TB/s.)
#include <type_traits>

#include "internal.h"
#include "ptx.cuh"

namespace fga {
namespace {

constexpr int STEP = 1024;  // keys per warp step
#ifndef FGA_CK_WARPS
#define FGA_CK_WARPS 8
#endif
#ifndef FGA_CK_SPW
#define FGA_CK_SPW 4
#endif
#ifndef FGA_CK_MINB
#define FGA_CK_MINB 5  // min CTAs per SM for __launch_bounds__ (caps registers at 48)
#endif
#ifndef FGA_CK_MINB_BYTES
#define FGA_CK_MINB_BYTES 4  // the keep-byte kernel: 4 CTAs per SM (64 registers) beat 5 / 6 (61.3 / 63.6 / 76.5 us back to back)
#endif
#ifndef FGA_CK_BUFS
#define FGA_CK_BUFS 1
#endif
#ifndef FGA_CK_BULK
#define FGA_CK_BULK 1  // stage absolute int32 keys and write each step's aligned body with one TMA bulk store
#endif
#ifndef FGA_CK_PERSIST
#define FGA_CK_PERSIST 1  // bits: persistent CTAs (FGA_CK_MINB per SM) that prefetch the next row's words
#endif
#ifndef FGA_CK_EMIT
#define FGA_CK_EMIT 1  // stage emission through a shared-memory address register (predicated STS + add per key)
#endif
constexpr int WARPS = FGA_CK_WARPS;
constexpr int SPW = FGA_CK_SPW;    // steps per warp per round: 8 x 4 steps = 32768 keys (c2's whole row)
constexpr int BUFS = FGA_CK_BUFS;  // stage buffers per warp (1: an extra __syncwarp per step)

// bit k of the result = (byte k of x != 0), k = 0..3
__device__ __forceinline__ uint32_t nz4(uint32_t x) {
  const uint32_t h = (((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;  // bit 7 of each nonzero byte
  return ((h >> 7) * 0x01020408u) >> 24;                                       // gather the 4 bits
}
__device__ __forceinline__ uint32_t nz16(const uint4& w) {
  return nz4(w.x) | (nz4(w.y) << 4) | (nz4(w.z) << 8) | (nz4(w.w) << 12);
}

// emit base-relative positions rel0 + e for the set bits e of a 16-bit mask
__device__ __forceinline__ void emit16(uint16_t* st, int off, uint32_t m, int rel0) {
#pragma unroll
  for (int e = 0; e < 16; ++e)
    if (m & (1u << e)) st[off++] = static_cast<uint16_t>(rel0 + e);
}

// the same for an int32 stage of absolute keys v0 + e
#if !FGA_CK_EMIT
__device__ __forceinline__ void emit16_i32(int32_t* st, int off, uint32_t m, int v0) {
#pragma unroll
  for (int e = 0; e < 16; ++e)
    if (m & (1u << e)) st[off++] = v0 + e;
}
#endif

// The same with the stage address carried in a register: per key slot one predicate test, the value,
// a predicated STS and a predicated add (the C loop above compiles to ~6 instructions per slot, the
// offset re-scaled into an address every time).  Returns the address past the last key written.
#define FGA_EMIT1(M)                                  \
  "and.b32 t, %2, " #M ";\n\t"                       \
  "setp.ne.b32 p, t, 0;\n\t"                         \
  "@p st.shared.b32 [%0], v;\n\t"                   \
  "@p add.u32 %0, %0, 4;\n\t"                        \
  "add.u32 v, v, 1;\n\t"
#define FGA_EMIT8(A, B, C, D, E, F, G, H) \
  FGA_EMIT1(A) FGA_EMIT1(B) FGA_EMIT1(C) FGA_EMIT1(D) FGA_EMIT1(E) FGA_EMIT1(F) FGA_EMIT1(G) FGA_EMIT1(H)
#define FGA_EMIT_LO16 FGA_EMIT8(0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40, 0x80) \
  FGA_EMIT8(0x100, 0x200, 0x400, 0x800, 0x1000, 0x2000, 0x4000, 0x8000)
#define FGA_EMIT_HI16 FGA_EMIT8(0x10000, 0x20000, 0x40000, 0x80000, 0x100000, 0x200000, 0x400000, 0x800000) \
  FGA_EMIT8(0x1000000, 0x2000000, 0x4000000, 0x8000000, 0x10000000, 0x20000000, 0x40000000, 0x80000000)

template <int NB>
__device__ __forceinline__ uint32_t emit_addr(uint32_t a, uint32_t m, int v0) {
  static_assert(NB == 16 || NB == 32, "16 or 32 key slots");
  if constexpr (NB == 16)
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t, v;\n\tmov.b32 v, %1;\n\t" FGA_EMIT_LO16 "}"
                 : "+r"(a) : "r"(v0), "r"(m) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t, v;\n\tmov.b32 v, %1;\n\t" FGA_EMIT_LO16 FGA_EMIT_HI16 "}"
                 : "+r"(a) : "r"(v0), "r"(m) : "memory");
  return a;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

struct Blk2 {
  uint4 a, b;
};

// keep bytes: one step's data for this lane
struct ByteSrc {
  const uint8_t* abase;  // 16-byte aligned start of the row's bytes
  int head, span;        // the row is abase[head, span)  (n < 2^31)
  int lane;
  __device__ __forceinline__ uint4 ld(int lo) const {
    return (lo >= head && lo + 16 <= span) ? __ldg(reinterpret_cast<const uint4*>(abase + lo))
                                           : make_uint4(0u, 0u, 0u, 0u);
  }
  __device__ __forceinline__ Blk2 load(int64_t s) const {
    const int lo = static_cast<int>(s) * STEP + lane * 16;
    return Blk2{ld(lo), ld(lo + STEP / 2)};
  }
  __device__ __noinline__ uint32_t mask_edge(int lo) const {  // the row's ragged ends
    uint32_t m = 0;
    for (int e = 0; e < 16; ++e) {
      const int pos = lo + e;
      if (pos >= head && pos < span && abase[pos] != 0) m |= 1u << e;
    }
    return m;
  }
  __device__ __forceinline__ uint32_t mask16(const uint4& w, int lo) const {
    if (lo >= head && lo + 16 <= span) return nz16(w);
    return (lo < span && lo + 16 > head) ? mask_edge(lo) : 0u;
  }
  // masks of the step's two 16-key blocks (half 0: keys 16l.., half 1: 512 + 16l..)
  __device__ __forceinline__ void masks(const Blk2& d, int64_t s, uint32_t& m0, uint32_t& m1) const {
    const int lo = static_cast<int>(s) * STEP + lane * 16;
    m0 = mask16(d.a, lo);
    m1 = mask16(d.b, lo + STEP / 2);
  }
  static constexpr bool kHalfMajor = true;  // all lanes' half 0, then all lanes' half 1
  __device__ __forceinline__ int key_base(int64_t s) const { return static_cast<int>(s) * STEP - head; }
};

// keep bits: word l of the step
struct BitSrc {
  const uint32_t* br;
  int64_t words, n;
  int lane;
  __device__ __forceinline__ uint32_t load(int64_t s) const {
    const int64_t w = s * 32 + lane;
    return w < words ? __ldg(br + w) : 0u;
  }
  __device__ __forceinline__ void masks(uint32_t v, int64_t s, uint32_t& m0, uint32_t& m1) const {
    const int64_t k0 = (s * 32 + lane) * 32;
    if (k0 + 32 > n) v &= (k0 >= n) ? 0u : ((1u << (n - k0)) - 1u);  // keys past n are not keys
    m0 = v & 0xFFFFu;
    m1 = v >> 16;
  }
  static constexpr bool kHalfMajor = false;  // lane-major: lane l's 32 keys are contiguous
  __device__ __forceinline__ int key_base(int64_t s) const { return static_cast<int>(s * STEP); }
};

// Stage element: uint16 positions relative to the step (flushed by coalesced stores), or with
// FGA_CK_BULK int32 absolute keys placed at (output position) mod 4, so that the step's run
// out[base .. base + tot) splits into <= 3 head keys, a 16-byte-aligned body written from shared
// memory by one `cp.async.bulk` (TMA) store, and <= 3 tail keys -- the per-key flush loads and
// stores (~10 instructions per 32 keys with their address arithmetic) become one instruction per step.
constexpr int STAGE_N = FGA_CK_BULK ? STEP + 4 : STEP;
using StageT = typename std::conditional<FGA_CK_BULK, int32_t, uint16_t>::type;

// Optional cross-row prefetch (persistent bit compaction): `pref` holds the first round's data of
// this row when `have_pref`, and receives the first round of `next` (if non-null) as soon as the last
// round's scan is done, so those loads are in flight while this row is emitted.  `pending` (lane 0: a
// bulk store may still be reading this warp's stage) carries across rows.
template <class Src, class D = decltype(Src{}.load(0))>
__device__ __forceinline__ int compact_row(const Src& src, int64_t nsteps, int32_t* __restrict__ out,
                                           int (*s_warp)[WARPS], StageT (*stage)[STAGE_N], bool& pending, int& rb,
                                           D* pref = nullptr, bool have_pref = false, const Src* next = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int running = 0;
  const bool bulk = FGA_CK_BULK && (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  for (int64_t r0 = 0; r0 < nsteps; r0 += WARPS * SPW, rb ^= 1) {
    const int64_t s0 = r0 + int64_t(warp) * SPW;
    D d[SPW];
    if (pref != nullptr && have_pref && r0 == 0) {
#pragma unroll
      for (int j = 0; j < SPW; ++j) d[j] = pref[j];
    } else {
#pragma unroll
      for (int j = 0; j < SPW; ++j) d[j] = src.load(s0 + j);  // all loads in flight first
    }
    uint32_t m0[SPW], m1[SPW];
    int o0[SPW], o1[SPW], tot[SPW], wsum = 0;
#pragma unroll
    for (int j = 0; j < SPW; ++j) {
      src.masks(d[j], s0 + j, m0[j], m1[j]);
      const int c0 = __popc(m0[j]), c1 = __popc(m1[j]);
      const int packed = Src::kHalfMajor ? (c0 | (c1 << 16)) : c0 + c1;  // a half's sum <= 512
      const int incl = warp_incl_scan(packed, lane);
      const int t = __shfl_sync(0xffffffffu, incl, 31);
      const int ex = incl - packed;
      if (Src::kHalfMajor) {
        o0[j] = ex & 0xFFFF;
        o1[j] = (t & 0xFFFF) + (ex >> 16);
        tot[j] = (t & 0xFFFF) + (t >> 16);
      } else {
        o0[j] = ex;
        o1[j] = ex + c0;
        tot[j] = t;
      }
      wsum += tot[j];
    }
    if (next != nullptr && r0 + WARPS * SPW >= nsteps) {
#pragma unroll
      for (int j = 0; j < SPW; ++j) pref[j] = next->load(int64_t(warp) * SPW + j);
    }
    if (lane == 0) s_warp[rb][warp] = wsum;
    __syncthreads();
    int base = running, rtotal = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const int v = s_warp[rb][w];
      rtotal += v;
      base += w < warp ? v : 0;
    }
    const int rel1 = Src::kHalfMajor ? STEP / 2 + lane * 16 : lane * 32 + 16;
    const int rel0 = Src::kHalfMajor ? lane * 16 : lane * 32;
#pragma unroll
    for (int j = 0; j < SPW; ++j) {
      StageT* st = stage[warp * BUFS + (j % BUFS)];
      const int kb = src.key_base(s0 + j);
      if constexpr (FGA_CK_BULK) {
        if (lane == 0 && pending) bulk_wait_read_all();  // the previous step's bulk store has read the stage
        __syncwarp();
        const int shift = base & 3, tj = tot[j];
#if FGA_CK_EMIT
        if constexpr (!Src::kHalfMajor) {  // lane-major: the lane's 32 keys in one run
          emit_addr<32>(static_cast<uint32_t>(__cvta_generic_to_shared(st + shift + o0[j])), m0[j] | (m1[j] << 16),
                        kb + rel0);
        } else {
          emit_addr<16>(static_cast<uint32_t>(__cvta_generic_to_shared(st + shift + o0[j])), m0[j], kb + rel0);
          emit_addr<16>(static_cast<uint32_t>(__cvta_generic_to_shared(st + shift + o1[j])), m1[j], kb + rel1);
        }
#else
        emit16_i32(st + shift, o0[j], m0[j], kb + rel0);
        emit16_i32(st + shift, o1[j], m1[j], kb + rel1);
#endif
        if (bulk) fence_proxy_async_smem();  // the stage's generic-proxy writes -> the bulk store
        __syncwarp();
        const int i0 = bulk ? min(tj, (4 - shift) & 3) : tj;  // aligned body [i0, i1)
        const int i1 = bulk ? i0 + ((tj - i0) & ~3) : tj;
        if (!bulk) {
          for (int i = lane; i < tj; i += 32) out[base + i] = st[shift + i];
        } else {
          if (lane < i0) out[base + lane] = st[shift + lane];
          if (lane < tj - i1) out[base + i1 + lane] = st[shift + i1 + lane];
          if (lane == 0 && i1 > i0) {
            bulk_s2g(out + base + i0, st + shift + i0, static_cast<uint32_t>(i1 - i0) * 4u);
            bulk_commit();
            pending = true;
          }
        }
      } else {
        if (BUFS == 1 && j > 0) __syncwarp();  // the previous step's flush has read the stage
        emit16(reinterpret_cast<uint16_t*>(st), o0[j], m0[j], rel0);
        emit16(reinterpret_cast<uint16_t*>(st), o1[j], m1[j], rel1);
        __syncwarp();
        for (int i = lane; i < tot[j]; i += 32) out[base + i] = kb + reinterpret_cast<uint16_t*>(st)[i];
      }
      base += tot[j];
    }
    running += rtotal;
  }
  return running;
}

__global__ void __launch_bounds__(WARPS * 32, FGA_CK_MINB_BYTES) fga_compact_kernel(const uint8_t* __restrict__ keep,
                                                                const float* __restrict__ scores, int64_t n,
                                                                int32_t* __restrict__ idx, int64_t stride,
                                                                int32_t* __restrict__ counts, int fill) {
  __shared__ int s_warp[2][WARPS];
  __shared__ float s_bv[WARPS];
  __shared__ int s_bi[WARPS];
  __shared__ __align__(16) StageT s_stage[WARPS * BUFS][STAGE_N];
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint8_t* kr = keep + row * n;
  int32_t* out = idx + row * stride;
  const int head = static_cast<int>(reinterpret_cast<uintptr_t>(kr) & 15u);
  const ByteSrc src{kr - head, head, head + static_cast<int>(n), lane};
  bool pending = false;
  int rb = 0;
  int running = compact_row(src, (head + n + STEP - 1) / STEP, out, s_warp, s_stage, pending, rb);
  if (FGA_CK_BULK && lane == 0 && pending) bulk_wait_all();  // stores complete before the CTA exits

  if (running == 0 && scores != nullptr) {
    // argmax fallback, first maximum (np.argmax semantics)
    const float* sr = scores + row * n;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int64_t i = tid; i < n; i += WARPS * 32) {
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
      for (int w = 1; w < WARPS; ++w)
        if (s_bv[w] > bv || (s_bv[w] == bv && s_bi[w] < bi)) { bv = s_bv[w]; bi = s_bi[w]; }
      out[0] = bi == 0x7fffffff ? 0 : bi;  // all -inf / NaN rows: index 0 like np.argmax
    }
    running = 1;
  }
  if (tid == 0) counts[row] = running;
  if (fill)
    for (int64_t i = running + tid; i < n; i += WARPS * 32) out[i] = -1;
}

// ---------------------------------------------------------------- bit-packed masks
// keep bits: uint32 words, bit b of word w = key 32w + b.  Packing: one warp
// ballot per 32 keys.  Compaction from bits: the same round schedule, lane l
// holding word l of each 1024-key step (keys 32l .. 32l + 31).
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

__global__ void __launch_bounds__(WARPS * 32, FGA_CK_MINB) fga_compact_bits_kernel(const uint32_t* __restrict__ bits, int64_t rows, int64_t words,
                                                                     int64_t n, int32_t* __restrict__ idx,
                                                                     int64_t stride, int32_t* __restrict__ counts,
                                                                     int fill, int32_t* __restrict__ fix_rows,
                                                                     int32_t* __restrict__ fix_count) {
  __shared__ int s_warp[2][WARPS];
  __shared__ __align__(16) StageT s_stage[WARPS * BUFS][STAGE_N];
  const int tid = threadIdx.x;
  const int64_t nsteps = (words + 31) / 32;
  bool pending = false;
  int rb = 0;
  uint32_t pref[SPW];
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    int32_t* out = idx + row * stride;
    const BitSrc src{bits + row * words, words, n, tid & 31};
    const int64_t nrow = row + gridDim.x;
    const BitSrc nsrc{bits + (nrow < rows ? nrow : row) * words, words, n, tid & 31};
    int running = compact_row(src, nsteps, out, s_warp, s_stage, pending, rb, pref, row != blockIdx.x,
                              nrow < rows ? &nsrc : nullptr);
    if (running == 0 && fix_rows != nullptr) {  // argmax fallback of a fused threshold pass (masks.py:86-87):
      if (tid == 0) fix_rows[atomicAdd(fix_count, 1)] = static_cast<int32_t>(row);  // out[0] by the fix-up
      running = 1;
    }
    if (tid == 0) counts[row] = running;
    if (fill)
      for (int64_t i = running + tid; i < n; i += WARPS * 32) out[i] = -1;
  }
  if (FGA_CK_BULK && (tid & 31) == 0 && pending) bulk_wait_all();  // stores complete before the CTA exits
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
                        int32_t* counts, int fill, cudaStream_t stream, int32_t* fix_rows, int32_t* fix_count) {
  if (rows < 0 || n <= 0 || idx_stride < n) return fail(FGA_EINVAL, "compact_bits: need rows >= 0, n > 0, idx_stride >= n");
  if (n >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact_bits: n must be < 2^31");
  if (rows == 0) return FGA_OK;
  if (rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact_bits: too many rows");
  const int64_t resident = int64_t(FGA_CK_MINB) * sm_count();
  const int64_t grid = FGA_CK_PERSIST && rows > resident ? resident : rows;
  fga_compact_bits_kernel<<<static_cast<unsigned>(grid), WARPS * 32, 0, stream>>>(bits, rows, (n + 31) / 32, n, idx,
                                                                                idx_stride, counts, fill, fix_rows,
                                                                                fix_count);
  return check_launch("fga_compact_bits_kernel");
}

int launch_compact(const uint8_t* keep, const float* scores, int64_t rows, int64_t n, int32_t* idx,
                   int64_t idx_stride, int32_t* counts, int fill, cudaStream_t stream) {
  if (rows < 0 || n <= 0 || idx_stride < n) return fail(FGA_EINVAL, "compact: need rows >= 0, n > 0, idx_stride >= n");
  if (n >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact: n must be < 2^31");
  if (rows == 0) return FGA_OK;
  if (rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "compact: too many rows");
  fga_compact_kernel<<<static_cast<unsigned>(rows), WARPS * 32, 0, stream>>>(keep, scores, n, idx, idx_stride, counts, fill);
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
