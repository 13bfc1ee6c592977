// K1a tail + K1b in one kernel for bf16-valued selection scores: threshold or top-k
// selection fused with the compaction into ascending key lists.
//
// Reference semantics (/root/reference/pkg/src/sliceattn/masks.py):
//   threshold (masks.py:131-132 + 75-91): keep j iff s_j >= tau, an empty row falls back to
//       [argmax(s)] (first maximum);
//   top-k (masks.py:133-147): the top_k largest s_j, ties toward the smaller index
//       (np.lexsort((arange(n), -s))[:top_k]); SparseIndexMask (sparse.py:45-55) stores every
//       list ascending.
// The scores are bf16 (the builders' analysis_scores rounding, precision='bf16'), so each row is
// a row of 16-bit keys: 2 bytes per score instead of 4 read from HBM, and the whole row fits in
// shared memory (n <= FGA_SELECT_MAX_N), where the top-k threshold is found by a bisection over
// key values -- one contention-free counting pass per bit of the occupied key range, each a
// packed bf16x2 compare over LDS.128 and a block sum -- instead of histogram atomics, which the
// clustered scores of the builders serialise on a few bins (maskbuild.cu topk_kernel).
//
// One 256-thread CTA per (b,h,g) row:
//   1. load: global bf16 -> SMEM (+ min / max of the order-preserving 16-bit keys),
//   2. top-k: thr = the largest value v with #{s >= v} >= k (interpolation steps alternating
//      with bisection steps over [min, max] keys),
//   3. count: warp w owns a contiguous range of 256-key blocks; its kept keys (> thr, == thr) are
//      the bisection's last per-warp counts (threshold: one counting pass); one block scan gives
//      every warp its output offset and the number of threshold ties before its range (ties are
//      kept in index order until k),
//   4. emit: each warp writes its kept positions in order (ballot ranks, coalesced stores).
// Output bit-exact with the reference lists for the same bf16 scores.  HBM-bound: 2n bytes read
// and 4*count (+ the -1 tail) written per row.
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace fga {
namespace {

#ifndef FGA_SEL_INTERP
#define FGA_SEL_INTERP 1  // top-k: interpolation steps between the bisection steps
#endif
#ifndef FGA_SEL_MINB
#define FGA_SEL_MINB 3  // CTAs per SM for __launch_bounds__ (a c2 row is 64 KB of SMEM: 3 rows per SM)
#endif
#ifndef FGA_SEL_THREADS
#define FGA_SEL_THREADS 256  // c2 top-k 188 -> 141 us, threshold 106 -> 92 us against 512 (128: 154 / 105, 1024: 334 / 197)
#endif
constexpr int SEL_THREADS = FGA_SEL_THREADS;
constexpr int SEL_WARPS = SEL_THREADS / 32;

// bf16 bits -> order-preserving unsigned key (negative values reversed below the positives)
__device__ __forceinline__ uint32_t okey2(uint32_t w) {  // two packed keys
  return w ^ ((((w >> 15) & 0x00010001u) * 0x7FFFu) | 0x80008000u);
}
__device__ __forceinline__ uint32_t okey_bits(uint32_t k) {  // inverse of okey2 for one key
  return (k & 0x8000u) ? (k & 0x7FFFu) : (~k & 0xFFFFu);
}
__device__ __forceinline__ float bf16_value(uint32_t b) { return __uint_as_float(b << 16); }
#ifndef FGA_SEL_HMASK
#define FGA_SEL_HMASK 1  // emission masks from bf16x2 compares (HSET2) packed to 8 bits
#endif
// four bf16x2 compare masks (0xFFFF per half that holds; m_j: keys 2j low, 2j + 1 high) -> bit i = key i
__device__ __forceinline__ uint32_t pack8(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
  const uint32_t t = (m0 & 0x00020001u) | (m1 & 0x00080004u) | (m2 & 0x00200010u) | (m3 & 0x00800040u);
  return (t | (t >> 16)) & 0xFFu;
}
__device__ __forceinline__ const __nv_bfloat162& as_b2(const uint32_t& w) {
  return *reinterpret_cast<const __nv_bfloat162*>(&w);
}

// sum over the block of the warps' partial sums (v: this warp's, the same in every lane); `red`
// holds two buffers of SEL_WARPS (the phase alternates, so one barrier per call suffices)
__device__ __forceinline__ int block_sum(int v, int* red, int& phase) {
  int* r = red + phase * SEL_WARPS;
  if ((threadIdx.x & 31) == 0) r[threadIdx.x >> 5] = v;
  __syncthreads();
  int s = 0;
#pragma unroll
  for (int w = 0; w < SEL_WARPS; ++w) s += r[w];
  phase ^= 1;
  return s;
}

template <bool TOPK>
__global__ void __launch_bounds__(SEL_THREADS, FGA_SEL_MINB)
    select_compact_kernel(const uint16_t* __restrict__ scores, int64_t n64, float tau, int64_t top_k,
                          int32_t* __restrict__ idx, int64_t stride, int32_t* __restrict__ counts, int fill) {
  extern __shared__ __align__(16) uint16_t s_key[];  // the row's bf16 bits, padded with -NaN to a multiple of 256
  __shared__ int s_red[2 * SEL_WARPS];
  __shared__ int s_cnt[2][SEL_WARPS];
  __shared__ unsigned long long s_best[SEL_WARPS];
  __shared__ __align__(8) uint64_t s_bar;
  const int n = static_cast<int>(n64);
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint16_t* src = scores + row * n64;
  int32_t* out = idx + row * stride;
  const int nv = (n + 7) / 8;  // 16-byte vectors of keys
  const int nvp = (nv + 31) / 32 * 32;  // padded to whole 256-key blocks: the block loops need no bound check
  uint4* sv = reinterpret_cast<uint4*>(s_key);
  for (int i = nv + tid; i < nvp; i += SEL_THREADS) sv[i] = make_uint4(~0u, ~0u, ~0u, ~0u);  // -NaN: never counted

  // ---- 1. load (+ range of the order-preserving keys for the bisection)
  uint32_t kmin2 = 0xFFFFFFFFu, kmax2 = 0u;
  if ((n & 7) == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
    // the whole row in one TMA bulk transfer (a few 32 KB copies on one mbarrier): the row
    // arrives at the SM's bulk-copy rate instead of one DRAM latency per strided LDG round
    if (tid == 0) {
      mbar_init(&s_bar, 1);
      fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0) {
      const uint32_t bytes = static_cast<uint32_t>(nv) * 16u;
      mbar_expect_tx(&s_bar, bytes);
      for (uint32_t off = 0; off < bytes; off += 32768u)
        bulk_g2s(s_key + off / 2, src + off / 2, min(32768u, bytes - off), &s_bar);
    }
    mbar_wait(&s_bar, 0);
    if (TOPK) {
      for (int i = tid; i < nv; i += SEL_THREADS) {
        const uint4 x = sv[i];
        const uint32_t a = okey2(x.x), b = okey2(x.y), c = okey2(x.z), d = okey2(x.w);
        kmin2 = __vminu2(kmin2, __vminu2(__vminu2(a, b), __vminu2(c, d)));
        kmax2 = __vmaxu2(kmax2, __vmaxu2(__vmaxu2(a, b), __vmaxu2(c, d)));
      }
    }
  } else {
    for (int i = tid; i < 8 * nv; i += SEL_THREADS) {
      uint32_t b = 0xFFFFu;  // pad: -NaN, which no comparison counts or keeps
      if (i < n) {
        b = __ldg(src + i);
        if (TOPK) {
          const uint32_t kk = okey2(b) & 0xFFFFu;
          kmin2 = __vminu2(kmin2, kk | 0xFFFF0000u);
          kmax2 = __vmaxu2(kmax2, kk);
        }
      }
      s_key[i] = static_cast<uint16_t>(b);
    }
  }

  int phase = 0;
  float thr = 0.f;  // top-k: the k-th largest value
  int need = 0;
  // warp w owns the contiguous 256-key blocks [b0, b1) (lane l: keys 8l..8l+7 of each) in every
  // pass below, so the bisection's per-warp counts double as the emission's per-warp counts
  const int nb = (nv + 31) / 32;
  const int bpw = (nb + SEL_WARPS - 1) / SEL_WARPS;
  const int b0 = min(nb, warp * bpw), b1 = min(nb, b0 + bpw);
  int warp_ge = 0, warp_gt = 0;  // top-k: this warp's #{s >= thr}, #{s > thr}
  if (TOPK) {
    // ---- 2. bisection over the order-preserving keys: thr = max { v : #{s >= value(v)} >= k },
    //      #{s >= value(kmin)} = n >= k.  Each pass counts with HSET2.BF16 (a 0xFFFF mask per
    //      half-word that holds) accumulated by a 16x2 add: 2 instructions per 2 scores.
    uint32_t lo = min(kmin2 & 0xFFFFu, kmin2 >> 16), hi = max(kmax2 & 0xFFFFu, kmax2 >> 16);
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) { s_red[warp] = static_cast<int>(lo); s_red[SEL_WARPS + warp] = static_cast<int>(hi); }
    __syncthreads();  // also publishes s_key
    lo = 0xFFFFu; hi = 0u;
#pragma unroll
    for (int w = 0; w < SEL_WARPS; ++w) {
      lo = min(lo, static_cast<uint32_t>(s_red[w]));
      hi = max(hi, static_cast<uint32_t>(s_red[SEL_WARPS + w]));
    }
    __syncthreads();  // s_red is reused by block_sum
    const int k = static_cast<int>(top_k);
    // this warp's #{s >= value(v)}
    auto count_ge = [&](uint32_t v) {
      const uint32_t pb = okey_bits(v) * 0x00010001u;
      const __nv_bfloat162 piv = *reinterpret_cast<const __nv_bfloat162*>(&pb);
      uint32_t acc = 0;  // two 16-bit counters of -1s (|count| <= n/16 per thread each)
      for (int b = b0; b < b1; ++b) {
        const uint4 x = sv[b * 32 + lane];
        acc = __vadd2(acc, __hge2_mask(*reinterpret_cast<const __nv_bfloat162*>(&x.x), piv));
        acc = __vadd2(acc, __hge2_mask(*reinterpret_cast<const __nv_bfloat162*>(&x.y), piv));
        acc = __vadd2(acc, __hge2_mask(*reinterpret_cast<const __nv_bfloat162*>(&x.z), piv));
        acc = __vadd2(acc, __hge2_mask(*reinterpret_cast<const __nv_bfloat162*>(&x.w), piv));
      }
      const int mine = static_cast<int>(((0x10000u - (acc & 0xFFFFu)) & 0xFFFFu) + ((0x10000u - (acc >> 16)) & 0xFFFFu));
      return __reduce_add_sync(0xffffffffu, mine);
    };
    // invariant: #{s >= value(lo)} >= k, #{s >= value(hi + 1)} < k; each pass's per-warp count is
    // kept for the side it moves, so at the end #{s >= thr} and #{s > thr} = #{s >= value(thr + 1)}
    // are known per warp without another pass (consecutive keys are consecutive bf16 values apart
    // from -0 / +0, which can never straddle the final interval)
    // Interpolation steps (the pivot where a straight line through (lo, #{>= lo}) and
    // (hi + 1, #{>= hi + 1}) crosses k) alternate with bisection steps: the builders' score
    // distributions are smooth, so the interpolated pivot lands close and the interval collapses
    // in a few passes, while the bisection steps bound the worst case at twice the bisection's.
    bool have_lo = false, interp = FGA_SEL_INTERP != 0;
    int c_lo = n, c_hi1 = 0;  // block-wide #{s >= value(lo)} (every non-NaN key at kmin), #{s >= value(hi + 1)}
    while (lo < hi) {  // block-uniform
      uint32_t mid = (lo + hi + 1) >> 1;
      if (interp && c_lo > c_hi1) {  // (a heuristic pivot: float arithmetic is plenty)
        const float span = static_cast<float>(hi + 1 - lo);
        const uint32_t step = static_cast<uint32_t>(static_cast<float>(c_lo - k) * span / static_cast<float>(c_lo - c_hi1));
        mid = lo + min(max(step, 1u), hi - lo);
      }
      const int wc = count_ge(mid);
      const int c = block_sum(wc, s_red, phase);
      if (c >= k) { lo = mid; warp_ge = wc; have_lo = true; c_lo = c; }
      else { hi = mid - 1; warp_gt = wc; c_hi1 = c; }
      // alternate (interpolating again whenever the last step halved the interval measured slower:
      // 241.7 vs 229.4 us at c2, the one-sided regula-falsi steps)
      interp = FGA_SEL_INTERP != 0 && !interp;
    }
    if (!have_lo) warp_ge = count_ge(lo);  // the k-th value is the row's minimum
    thr = bf16_value(okey_bits(lo));
    need = k;  // minus the keys above thr: the ties at thr kept in index order
  } else {
    __syncthreads();
  }

  // ---- 3. per-warp counts: top-k from the bisection (keys above thr, ties at thr); threshold:
  //      keys >= tau over the warp's blocks (a bf16 compare against tau rounded up to bf16 is
  //      exact), masks accumulated 16x2 as in the bisection
  if (TOPK) {
    if (lane == 0) { s_cnt[0][warp] = warp_gt; s_cnt[1][warp] = warp_ge - warp_gt; }
  } else {
    const uint32_t cut2b = __bfloat16_as_ushort(__float2bfloat16_ru(tau)) * 0x00010001u;
    const __nv_bfloat162 cut2 = *reinterpret_cast<const __nv_bfloat162*>(&cut2b);
    uint32_t ga = 0;
    for (int b = b0; b < b1; ++b) {
      const int vi = b * 32 + lane;
      if (vi < nv) {  // (measured faster than the unguarded loop here, unlike the top-k passes)
        const uint4 x = sv[vi];
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[j]);
          ga = __vadd2(ga, __hge2_mask(h, cut2));
        }
      }
    }
    const int g = static_cast<int>(((0x10000u - (ga & 0xFFFFu)) & 0xFFFFu) + ((0x10000u - (ga >> 16)) & 0xFFFFu));
    const int gs = __reduce_add_sync(0xffffffffu, g);
    if (lane == 0) { s_cnt[0][warp] = gs; s_cnt[1][warp] = 0; }
  }
  __syncthreads();
  int total_gt = 0, base = 0, eqrun = 0;
#pragma unroll
  for (int w = 0; w < SEL_WARPS; ++w) total_gt += s_cnt[0][w];
  if (TOPK) need -= total_gt;  // >= 1 by the choice of thr
  int total = total_gt;
  if (TOPK) {
    int er = 0;
#pragma unroll
    for (int w = 0; w < SEL_WARPS; ++w) {
      const int e = s_cnt[1][w];
      const int kept_e = max(0, min(e, need - er));
      if (w < warp) { base += s_cnt[0][w] + kept_e; eqrun += e; }
      er += e;
      total += kept_e;
    }
  } else {
#pragma unroll
    for (int w = 0; w < SEL_WARPS; ++w) base += w < warp ? s_cnt[0][w] : 0;
  }

  // ---- 4. emit, ascending: per 256-key block one packed warp scan of (kept-above, ties) counts;
  //      the ties kept before lane l are min(tie prefix, ties still needed), so a lane's kept keys
  //      are its above-cut keys plus its lowest few ties, written at consecutive positions.
  const uint32_t thr2b = __bfloat16_as_ushort(__float2bfloat16_rn(thr)) * 0x00010001u;  // thr is a bf16 value
  const uint32_t tau2b = __bfloat16_as_ushort(__float2bfloat16_ru(tau)) * 0x00010001u;
  const __nv_bfloat162 thr2 = as_b2(thr2b), tau2 = as_b2(tau2b);
#ifndef FGA_SEL_OUTREG
#define FGA_SEL_OUTREG 1  // keep the row's output pointer in a register (no per-store rematerialisation)
#endif
  int32_t* outr = out;
  if (FGA_SEL_OUTREG && TOPK) asm volatile("mov.b64 %0, %0;" : "+l"(outr));  // (threshold: measured slower)
  for (int b = b0; b < b1; ++b) {
    const int vi = b * 32 + lane;
    uint32_t gm = 0, em = 0;  // bit j: key 8*vi + j (the -NaN padding never holds)
    if (FGA_SEL_HMASK && (TOPK || vi < nv)) {
      const uint4 x = sv[vi];
      if (TOPK) {
        gm = pack8(__hgt2_mask(as_b2(x.x), thr2), __hgt2_mask(as_b2(x.y), thr2), __hgt2_mask(as_b2(x.z), thr2),
                   __hgt2_mask(as_b2(x.w), thr2));
        em = pack8(__heq2_mask(as_b2(x.x), thr2), __heq2_mask(as_b2(x.y), thr2), __heq2_mask(as_b2(x.z), thr2),
                   __heq2_mask(as_b2(x.w), thr2));
      } else {
        gm = pack8(__hge2_mask(as_b2(x.x), tau2), __hge2_mask(as_b2(x.y), tau2), __hge2_mask(as_b2(x.z), tau2),
                   __hge2_mask(as_b2(x.w), tau2));
      }
    } else if (TOPK || vi < nv) {
      const uint4 x = sv[vi];
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float v = bf16_value((w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
        if (TOPK) {
          gm |= static_cast<uint32_t>(v > thr) << j;
          em |= static_cast<uint32_t>(v == thr) << j;
        } else {
          gm |= static_cast<uint32_t>(v >= tau) << j;
        }
      }
    }
    const int gc = __popc(gm), ec = __popc(em);
    const int packed = gc | (ec << 16);  // block counts <= 256 per half
    int incl = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    const int ex = incl - packed;
    const int gpre = ex & 0xFFFF, epre = ex >> 16;
    uint32_t keep = gm;
    int at = base + gpre;  // this lane's kept keys go to out[at ...), ascending
    if (TOPK) {
      const int room = max(0, need - eqrun);  // ties still to be kept at the block start
      const int mine = max(0, min(epre + ec, room) - min(epre, room));
      at += min(epre, room);
      if (mine == ec) {
        keep |= em;
      } else {
        uint32_t m = em;
        for (int i = 0; i < mine; ++i) { keep |= m & (0u - m); m &= m - 1u; }
      }
      base += (tot & 0xFFFF) + min(tot >> 16, room);
      eqrun += tot >> 16;
    } else {
      base += tot & 0xFFFF;
    }
    // a running output pointer stepped by the keep bit: predicated stores, no per-slot address
    // arithmetic or branch
    int32_t* op = outr + at;
    const int key0 = vi * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t kj = (keep >> j) & 1u;
      if (kj) *op = key0 + j;
      op += kj;
    }
  }

  if (!TOPK && total == 0) {
    // argmax fallback (masks.py:86-87): the largest value, first index (np.argmax); a NaN-free row
    // of bf16 values orders like its order-preserving keys
    unsigned long long best = 0ull;
    for (int i = tid; i < n; i += SEL_THREADS) {
      const unsigned long long v = (static_cast<unsigned long long>(okey2(s_key[i]) & 0xFFFFu) << 32) |
                                   (0xFFFFFFFFu - static_cast<uint32_t>(i));
      best = v > best ? v : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
      best = v > best ? v : best;
    }
    if (lane == 0) s_best[warp] = best;
    __syncthreads();
    if (tid == 0) {
      for (int w = 0; w < SEL_WARPS; ++w) best = s_best[w] > best ? s_best[w] : best;
      out[0] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(best & 0xFFFFFFFFull));
    }
    total = 1;
  }
  if (tid == 0) counts[row] = total;
  if (fill)
    for (int i = total + tid; i < n; i += SEL_THREADS) out[i] = -1;
}

}  // namespace

int launch_select_compact(const uint16_t* scores, int64_t rows, int64_t n, int mode, float tau, int64_t top_k,
                          int32_t* idx, int64_t idx_stride, int32_t* counts, int fill, cudaStream_t st) {
  if (rows < 0 || n < 1 || idx_stride < n) return fail(FGA_EINVAL, "select_compact: need rows >= 0, n >= 1, idx_stride >= n");
  if (n > FGA_SELECT_MAX_N) return fail(FGA_EUNSUPPORTED, "select_compact: n exceeds FGA_SELECT_MAX_N (shared-memory row)");
  if (mode != FGA_SELECT_THRESHOLD && mode != FGA_SELECT_TOPK) return fail(FGA_EINVAL, "select_compact: bad mode");
  if (mode == FGA_SELECT_TOPK && (top_k < 1 || top_k > n)) return fail(FGA_EINVAL, "top_k must be in [1, n]");
  if (rows == 0) return FGA_OK;
  if (rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "select_compact: too many rows");
  const int smem = static_cast<int>(((n + 7) / 8 + 31) / 32 * 32 * 16);  // whole 256-key blocks
  int rc;
  if (mode == FGA_SELECT_TOPK) {
    if ((rc = smem_opt_in(reinterpret_cast<const void*>(select_compact_kernel<true>), smem, "select_compact")) != FGA_OK)
      return rc;
    select_compact_kernel<true><<<static_cast<unsigned>(rows), SEL_THREADS, smem, st>>>(scores, n, tau, top_k, idx,
                                                                                         idx_stride, counts, fill);
  } else {
    if ((rc = smem_opt_in(reinterpret_cast<const void*>(select_compact_kernel<false>), smem, "select_compact")) != FGA_OK)
      return rc;
    select_compact_kernel<false><<<static_cast<unsigned>(rows), SEL_THREADS, smem, st>>>(scores, n, tau, top_k, idx,
                                                                                          idx_stride, counts, fill);
  }
  return check_launch("select_compact_kernel");
}

}  // namespace fga
