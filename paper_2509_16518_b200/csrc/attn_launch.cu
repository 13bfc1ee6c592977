// Host launcher of the FG-Attn forward kernels (K2 gather + K3 tcgen05 consumer).
//
// Reference semantics: /root/reference/pkg/src/sliceattn/sparse.py:111-156 (per-(b,h,g) chunk
// loop) with the online softmax of tiled.py:48-77.  One work tile = <=128 query rows of one group
// (decode_tile, attn_common.cuh).  Dispatch:
//   * attn_dual.cu for groups of 129..256 rows (both tiles of a group share each gathered chunk),
//   * attn_ws.cu otherwise (and for the dense denominator, contiguous TMA boxes).
// Tiles are claimed dynamically from a per-launch counter slot (attn_ws.cu tile_scheduler), in an
// optional caller-supplied order.  Per call the host does: shape checks, at most two tensor-map
// encodes (only the maps the chosen kernel reads), and the launch; shared-memory opt-in and the SM
// count are cached per device.
#include <cuda_bf16.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "attn_common.cuh"
#include "internal.h"

namespace fga {

// Dynamic-scheduler counters.  Each launch takes the next slot (mod FGA_SCHED_SLOTS); the kernel
// leaves its slot at zero when it finishes, so slots are reused without host work.
constexpr int FGA_SCHED_SLOTS = 256;
__device__ unsigned int g_sched_counters[FGA_SCHED_SLOTS];

namespace {

unsigned int* sched_slot() {
  static unsigned int* base[64] = {};
  static std::atomic<unsigned> seq{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (base[dev] == nullptr) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_sched_counters) != cudaSuccess) return nullptr;
    base[dev] = static_cast<unsigned int*>(p);
  }
  return base[dev] + (seq.fetch_add(1, std::memory_order_relaxed) % FGA_SCHED_SLOTS);
}

// Development timeline (FGA_TRACE=<file>, trace builds only: -DFGA_TRACE_ON=1, scripts/trace_run.py).
const char* trace_file() {
  static const char* f = std::getenv("FGA_TRACE");
  return f;
}

void dump_trace(const long long* host, const char* path) {
  FILE* f = std::fopen(path, "w");
  if (f == nullptr) return;
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

int dispatch(const CUtensorMap* maps, const void* q, const void* k, const void* v, const AttnParams& p, int d,
             bool f32, int flags, cudaStream_t stream) {
  if (!(flags & FGA_ATTN_PER_TILE)) {
    const int rc = launch_attn_dual(maps, p, d, f32, stream);
    if (rc != FGA_EUNSUPPORTED) return rc;
  }
  return launch_attn_ws(maps, q, p, d, f32, stream);
}

}  // namespace

int launch_attn(const AttnLaunch& a, const fga_shape& s, cudaStream_t stream) {
  const int64_t B = s.batch, H = s.heads, N = s.seq_len, D = s.head_dim, M = s.group_size;
  if (D != 64 && D != 128) return fail(FGA_EUNSUPPORTED, "head_dim must be 64 or 128");
  const int64_t rows = B * H * N;
  if (rows >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "B*H*N must be < 2^31");
  const int64_t G = (N + M - 1) / M;
  const int64_t tpg = (M + BM - 1) / BM;
  const int64_t n_tiles = B * H * G * tpg;
  if (n_tiles >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "too many tiles");
  int64_t tile_begin = a.tile_begin, tile_end = a.tile_end < 0 ? n_tiles : a.tile_end;
  if (tile_begin < 0 || tile_begin > tile_end || tile_end > n_tiles)
    return fail(FGA_EINVAL, "tile range must satisfy 0 <= begin <= end <= B*H*G*ceil(M/128)");
  const bool dense = a.idx == nullptr;
  const bool dual = !dense && !(a.flags & FGA_ATTN_PER_TILE) && tpg == 2 && tile_begin % 2 == 0 &&
                    (tile_end - tile_begin) % 2 == 0;

  // maps: [0] Q 128-row box (attn_dual.cu), [3] / [4] K / V 128-row boxes (dense attn_ws.cu)
  CUtensorMap maps[5];
  int rc;
  if (dual && (rc = make_tmap_bf16_2d(&maps[0], a.q, rows, D, 64, BM)) != FGA_OK) return rc;
  if (dense) {
    if ((rc = make_tmap_bf16_2d(&maps[3], a.k, rows, D, 64, BN)) != FGA_OK) return rc;
    if ((rc = make_tmap_bf16_2d(&maps[4], a.v, rows, D, 64, BN)) != FGA_OK) return rc;
  }

  AttnParams p{};
  p.k = a.k;
  p.v = a.v;
  p.idx = a.idx;
  p.idx_group_stride = dense ? N : a.idx_group_stride;
  p.counts = a.counts;
  p.out = a.o;
  p.lse = a.lse;
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
  p.status = a.status;
  p.order = a.order;
  p.cta_ns = a.cta_ns;
  p.cta_ns_len = a.cta_ns != nullptr ? a.cta_ns_len : 0;
  if (!(a.flags & FGA_ATTN_STATIC) && !dual) {
    p.sched = sched_slot();
    if (p.sched == nullptr) return fail(FGA_ECUDA, "scheduler counters unavailable");
  }
  if (tile_end == tile_begin) return FGA_OK;

  const bool f32 = a.o_dtype == FGA_OUT_F32;
  if (FGA_TRACE_ON && trace_file() != nullptr) {
    if (cudaMalloc(&p.trace, FGA_TRACE_LEN * sizeof(long long)) != cudaSuccess) return check_launch("trace buffer");
    cudaMemsetAsync(p.trace, 0, FGA_TRACE_LEN * sizeof(long long), stream);
    if (const char* ti = std::getenv("FGA_TRACE_IT")) p.trace_it = std::atoi(ti);
    const int rc2 = dispatch(maps, a.q, a.k, a.v, p, static_cast<int>(D), f32, a.flags, stream);
    static long long host[FGA_TRACE_LEN];
    cudaMemcpyAsync(host, p.trace, sizeof(host), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    cudaFree(p.trace);
    dump_trace(host, trace_file());
    return rc2;
  }
  return dispatch(maps, a.q, a.k, a.v, p, static_cast<int>(D), f32, a.flags, stream);
}

int launch_gather_probe(const void* k, const void* v, int64_t n, int64_t d, const int32_t* idx, int64_t idx_stride,
                        const int32_t* count, void* out_k, void* out_v, cudaStream_t stream) {
  if (d != 64 && d != 128) return fail(FGA_EUNSUPPORTED, "gather probe: head_dim must be 64 or 128");
  if (n < 1 || n >= (int64_t(1) << 31) || idx_stride < 1) return fail(FGA_EINVAL, "gather probe: bad n / stride");
  AttnParams p{};
  p.k = k;
  p.v = v;
  p.idx = idx;
  p.idx_group_stride = idx_stride;
  p.counts = count;
  p.tile_begin = 0;
  p.n_tiles = 1;
  p.heads = 1;
  p.seq_len = static_cast<int>(n);
  p.group_size = static_cast<int>(n < BM ? n : BM);
  p.groups = static_cast<int>((n + p.group_size - 1) / p.group_size);
  p.tiles_per_group = 1;
  return launch_ring_probe(p, static_cast<int>(d), out_k, out_v, stream);
}

}  // namespace fga
