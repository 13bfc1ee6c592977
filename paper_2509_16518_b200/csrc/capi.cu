// C ABI of libfgattn.so (include/fgattn.h): argument validation, error
// codes, TMA descriptor construction, and dispatch to the kernel launchers.
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "internal.h"

namespace fga {

int launch_group_max_map(const float* map, int64_t bh, int64_t n, int64_t m, int round, float* gmax, cudaStream_t st);
int launch_random_keep(int64_t rows, int64_t n, int64_t count, uint64_t seed, uint8_t* keep, cudaStream_t st);
int launch_validate(const int32_t* idx, int64_t stride, const int32_t* counts, int64_t rows, int64_t n,
                    int check_order, int32_t* status, cudaStream_t stream);
int status_to_code(const int32_t* status, cudaStream_t stream, const char* what);
int launch_tile_order(const int32_t* counts, const fga_shape& s, int32_t* order, cudaStream_t stream);

namespace {
thread_local std::string g_last_error;

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

int check_shape(const fga_shape& s) {
  if (s.batch < 1 || s.heads < 1 || s.seq_len < 1 || s.head_dim < 1 || s.group_size < 1)
    return fail(FGA_EINVAL, "batch, heads, seq_len, head_dim and group_size must be positive");
  if (s.group_size > s.seq_len) return fail(FGA_EINVAL, "group_size exceeds seq_len");
  if (s.seq_len >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "seq_len must be < 2^31");
  return FGA_OK;
}
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }

int smem_opt_in(const void* fn, int bytes, const char* what) {
  // the attribute only ever grows per (kernel, device), so a smaller launch never lowers it under
  // a larger one that already passed this check
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> granted;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int& have = granted[{fn, dev}];
  if (bytes <= have) return FGA_OK;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return check_launch(what);
  have = bytes;
  return FGA_OK;
}

int sm_count() {
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    cache[dev] = sms;
  }
  return cache[dev];
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return FGA_OK;
  return fail(FGA_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                      uint32_t box_rows) {
  EncodeTiled enc = encode_fn();
  if (enc == nullptr) return fail(FGA_ECUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if ((reinterpret_cast<uintptr_t>(base) & 15u) != 0) return fail(FGA_EINVAL, "tensor base must be 16-byte aligned");
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FGA_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return FGA_OK;
}

}  // namespace fga

using namespace fga;

extern "C" {

int fga_version(void) { return 200; }

const char* fga_last_error(void) { return g_last_error.c_str(); }

int fga_device_supported(int device) {
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return prop.major == 10 && prop.minor == 0 ? 1 : 0;
}

int fga_compact(const uint8_t* keep, const float* scores, int64_t rows, int64_t n, int32_t* idx, int64_t idx_stride,
                int32_t* counts, int fill_sentinel, void* stream) {
  if ((keep == nullptr || idx == nullptr || counts == nullptr) && rows > 0) return fail(FGA_EINVAL, "null pointer");
  return launch_compact(keep, scores, rows, n, idx, idx_stride, counts, fill_sentinel,
                        static_cast<cudaStream_t>(stream));
}

int fga_pack_bits(const uint8_t* keep, int64_t rows, int64_t n, uint32_t* bits, void* stream) {
  if (rows > 0 && (!keep || !bits)) return fail(FGA_EINVAL, "null pointer");
  return launch_pack_bits(keep, rows, n, bits, static_cast<cudaStream_t>(stream));
}

int fga_compact_bits(const uint32_t* bits, int64_t rows, int64_t n, int32_t* idx, int64_t idx_stride, int32_t* counts,
                     int fill_sentinel, void* stream) {
  if (rows > 0 && (!bits || !idx || !counts)) return fail(FGA_EINVAL, "null pointer");
  return launch_compact_bits(bits, rows, n, idx, idx_stride, counts, fill_sentinel, static_cast<cudaStream_t>(stream));
}

int fga_fgm1_unpack(const int32_t* words, const int64_t* starts, int64_t rows, int64_t n, int32_t* idx,
                    int64_t idx_stride, int32_t* counts, int fill_sentinel, void* stream) {
  if (rows > 0 && (!words || !starts || !idx || !counts)) return fail(FGA_EINVAL, "null pointer");
  return launch_fgm1_unpack(words, starts, rows, n, idx, idx_stride, counts, fill_sentinel,
                            static_cast<cudaStream_t>(stream));
}

int fga_sparse_attn_fwd_ex(const void* q, const void* k, const void* v, const int32_t* idx, int64_t idx_group_stride,
                           const int32_t* counts, void* o, int o_dtype, float* lse, fga_shape shape, int64_t tile_begin,
                           int64_t tile_end, const int32_t* order, int32_t* status, int flags, void* stream) {
  return fga_sparse_attn_fwd_timed(q, k, v, idx, idx_group_stride, counts, o, o_dtype, lse, shape, tile_begin, tile_end,
                                   order, status, flags, nullptr, 0, stream);
}

int fga_sparse_attn_fwd_timed(const void* q, const void* k, const void* v, const int32_t* idx,
                              int64_t idx_group_stride, const int32_t* counts, void* o, int o_dtype, float* lse,
                              fga_shape shape, int64_t tile_begin, int64_t tile_end, const int32_t* order,
                              int32_t* status, int flags, long long* cta_ns, int64_t cta_ns_len, void* stream) {
  int rc = check_shape(shape);
  if (rc != FGA_OK) return rc;
  if (!q || !k || !v || !idx || !counts || !o) return fail(FGA_EINVAL, "null pointer");
  if (idx_group_stride < 1) return fail(FGA_EINVAL, "idx_group_stride must be >= 1");
  if (o_dtype != FGA_OUT_BF16 && o_dtype != FGA_OUT_F32) return fail(FGA_EINVAL, "o_dtype must be FGA_OUT_BF16 or FGA_OUT_F32");
  if ((flags & FGA_ATTN_CHECK) && status == nullptr) return fail(FGA_EINVAL, "FGA_ATTN_CHECK needs a status word");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (flags & FGA_ATTN_CHECK) {
    // counts and key ranges of the launch's groups (the kernel consumes lists in any order)
    const int64_t G = (shape.seq_len + shape.group_size - 1) / shape.group_size;
    const int64_t tpg = (shape.group_size + 127) / 128;
    const int64_t n_tiles = shape.batch * shape.heads * G * tpg;
    const int64_t tb = tile_begin < 0 ? 0 : tile_begin, te = tile_end < 0 ? n_tiles : tile_end;
    const int64_t g0 = tb / tpg, g1 = te > tb ? (te + tpg - 1) / tpg : g0;
    if (g1 > g0 && g1 <= shape.batch * shape.heads * G) {
      rc = launch_validate(idx + g0 * idx_group_stride, idx_group_stride, counts + g0, g1 - g0, shape.seq_len, 0,
                           status, st);
      if (rc != FGA_OK) return rc;
    }
  }
  AttnLaunch a;
  a.q = q;
  a.k = k;
  a.v = v;
  a.idx = idx;
  a.idx_group_stride = idx_group_stride;
  a.counts = counts;
  a.o = o;
  a.o_dtype = o_dtype;
  a.lse = lse;
  a.tile_begin = tile_begin;
  a.tile_end = tile_end;
  a.order = order;
  a.status = status;
  a.flags = flags;
  a.cta_ns = cta_ns;
  a.cta_ns_len = cta_ns_len;
  rc = launch_attn(a, shape, st);
  if (rc != FGA_OK || !(flags & FGA_ATTN_CHECK)) return rc;
  return status_to_code(status, st, "fga_sparse_attn_fwd_ex");
}

int fga_sparse_attn_fwd(const void* q, const void* k, const void* v, const int32_t* idx, int64_t idx_group_stride,
                        const int32_t* counts, void* o, int o_dtype, float* lse, fga_shape shape, void* stream) {
  return fga_sparse_attn_fwd_ex(q, k, v, idx, idx_group_stride, counts, o, o_dtype, lse, shape, 0, -1, nullptr,
                                nullptr, 0, stream);
}

int fga_sparse_attn_fwd_tiles(const void* q, const void* k, const void* v, const int32_t* idx,
                              int64_t idx_group_stride, const int32_t* counts, void* o, int o_dtype, float* lse,
                              fga_shape shape, int64_t tile_begin, int64_t tile_end, void* stream) {
  return fga_sparse_attn_fwd_ex(q, k, v, idx, idx_group_stride, counts, o, o_dtype, lse, shape, tile_begin, tile_end,
                                nullptr, nullptr, 0, stream);
}

int fga_validate_mask(const int32_t* idx, int64_t idx_group_stride, const int32_t* counts, int64_t rows, int64_t n,
                      int32_t* status, void* stream) {
  if (rows < 0 || n < 1 || idx_group_stride < 1) return fail(FGA_EINVAL, "rows >= 0, n >= 1 and stride >= 1 required");
  if (!status || (rows > 0 && (!idx || !counts))) return fail(FGA_EINVAL, "null pointer");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int rc = launch_validate(idx, idx_group_stride, counts, rows, n, 1, status, st);
  if (rc != FGA_OK) return rc;
  return status_to_code(status, st, "fga_validate_mask");
}

int fga_tile_order(const int32_t* counts, fga_shape shape, int32_t* order, void* stream) {
  int rc = check_shape(shape);
  if (rc != FGA_OK) return rc;
  if (!counts || !order) return fail(FGA_EINVAL, "null pointer");
  return launch_tile_order(counts, shape, order, static_cast<cudaStream_t>(stream));
}

int fga_dense_attn_fwd(const void* q, const void* k, const void* v, void* o, int o_dtype, float* lse,
                       fga_shape shape, void* stream) {
  int rc = check_shape(shape);
  if (rc != FGA_OK) return rc;
  if (!q || !k || !v || !o) return fail(FGA_EINVAL, "null pointer");
  if (o_dtype != FGA_OUT_BF16 && o_dtype != FGA_OUT_F32) return fail(FGA_EINVAL, "o_dtype must be FGA_OUT_BF16 or FGA_OUT_F32");
  AttnLaunch a;
  a.q = q;
  a.k = k;
  a.v = v;
  a.o = o;
  a.o_dtype = o_dtype;
  a.lse = lse;
  return launch_attn(a, shape, static_cast<cudaStream_t>(stream));
}

int fga_gather_rows(const void* matrix, int64_t rows, int64_t d, const int32_t* indices, int64_t n_idx, void* out,
                    void* stream) {
  if (n_idx > 0 && (!matrix || !indices || !out)) return fail(FGA_EINVAL, "null pointer");
  return launch_gather(matrix, rows, d, indices, n_idx, out, static_cast<cudaStream_t>(stream));
}

int64_t fga_workspace_bytes(int op, fga_shape shape, int round_bf16) {
  if (const int rc = check_shape(shape); rc != FGA_OK) return rc;
  const int64_t G = (shape.seq_len + shape.group_size - 1) / shape.group_size;
  const int64_t cells = shape.batch * shape.heads * G * shape.seq_len;  // [B, H, G, N]
  switch (op) {
    case FGA_WS_POOLED_SCORES:
      return static_cast<int64_t>(ws_pooled_bytes(shape));
    case FGA_WS_CACHED_GROUP_MAX:
      return static_cast<int64_t>(ws_cached_bytes(shape));
    case FGA_WS_BUILD_AVGQ: {
      // fused threshold (keep bits + the list of rows that kept nothing + its count), or bf16
      // scores for the selection kernel, or fp32 scores + keep bytes: the largest of the three
      const int64_t rows = shape.batch * shape.heads * G;
      const size_t fused = Workspace::align(4 * rows * ((shape.seq_len + 31) / 32)) + Workspace::align(4 * rows) +
                           Workspace::align(4);
      size_t rest = round_bf16 && shape.seq_len <= FGA_SELECT_MAX_N ? Workspace::align(2 * cells)
                                                                     : Workspace::align(4 * cells) + Workspace::align(cells);
      if (round_bf16 && fused > rest) rest = fused;
      return static_cast<int64_t>(ws_pooled_bytes(shape) + rest);
    }
    case FGA_WS_BUILD_CACHED:
      return static_cast<int64_t>(ws_cached_bytes(shape) + Workspace::align(4 * cells) + Workspace::align(cells));
    default:
      return fail(FGA_EINVAL, "fga_workspace_bytes: unknown op");
  }
}

namespace {
int check_ws(void* ws) {
  if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return fail(FGA_EINVAL, "workspace must be 256-byte aligned");
  return FGA_OK;
}
}  // namespace

int fga_pooled_scores(const void* q, const void* k, fga_shape shape, int round_bf16, float* scores, void* ws,
                      size_t ws_bytes, void* stream) {
  int rc = check_shape(shape);
  if (rc != FGA_OK) return rc;
  if (!q || !k || !scores) return fail(FGA_EINVAL, "null pointer");
  if ((rc = check_ws(ws)) != FGA_OK) return rc;
  Workspace w(ws, ws_bytes);
  PooledOut out;
  out.scores = scores;
  return launch_pooled_scores(q, k, shape, round_bf16, out, w, static_cast<cudaStream_t>(stream));
}

int fga_gather_ring_probe(const void* k, const void* v, int64_t n, int64_t d, const int32_t* idx, int64_t idx_stride,
                          const int32_t* count, void* out_k, void* out_v, void* stream) {
  if (!k || !v || !idx || !count || !out_k || !out_v) return fail(FGA_EINVAL, "null pointer");
  return launch_gather_probe(k, v, n, d, idx, idx_stride, count, out_k, out_v, static_cast<cudaStream_t>(stream));
}

int fga_pooled_scores_bf16(const void* q, const void* k, fga_shape shape, uint16_t* scores, void* ws,
                           size_t ws_bytes, void* stream) {
  int rc = check_shape(shape);
  if (rc != FGA_OK) return rc;
  if (!q || !k || !scores) return fail(FGA_EINVAL, "null pointer");
  if ((rc = check_ws(ws)) != FGA_OK) return rc;
  Workspace w(ws, ws_bytes);
  PooledOut out;
  out.scores16 = scores;
  return launch_pooled_scores(q, k, shape, 1, out, w, static_cast<cudaStream_t>(stream));
}

int fga_select_compact(const uint16_t* scores, int64_t rows, int64_t n, int mode, float tau, int64_t top_k,
                       int32_t* idx, int64_t idx_stride, int32_t* counts, int fill_sentinel, void* stream) {
  if (rows > 0 && (!scores || !idx || !counts)) return fail(FGA_EINVAL, "null pointer");
  return launch_select_compact(scores, rows, n, mode, tau, top_k, idx, idx_stride, counts, fill_sentinel,
                               static_cast<cudaStream_t>(stream));
}

int fga_build_mask_avgq(const void* q, const void* k, fga_shape shape, int strategy, float tau, int64_t top_k,
                        int round_bf16, int32_t* idx, int64_t idx_stride, int32_t* counts, int fill_sentinel,
                        void* ws, size_t ws_bytes, void* stream) {
  int rc = check_shape(shape);
  if (rc != FGA_OK) return rc;
  if (!q || !k || !idx || !counts) return fail(FGA_EINVAL, "null pointer");
  if (strategy == FGA_SELECT_THRESHOLD && !(tau > 0.f)) return fail(FGA_EINVAL, "threshold strategies need tau > 0");
  if (strategy == FGA_SELECT_TOPK && (top_k < 1 || top_k > shape.seq_len))
    return fail(FGA_EINVAL, "top_k must be in [1, seq_len]");
  if (strategy != FGA_SELECT_THRESHOLD && strategy != FGA_SELECT_TOPK) return fail(FGA_EINVAL, "unknown strategy");
  if (idx_stride < shape.seq_len) return fail(FGA_EINVAL, "idx_stride must be >= seq_len");
  if ((rc = check_ws(ws)) != FGA_OK) return rc;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t G = (shape.seq_len + shape.group_size - 1) / shape.group_size;
  const int64_t rows = shape.batch * shape.heads * G, n = shape.seq_len;
  Workspace w(ws, ws_bytes);
  if (round_bf16 && strategy == FGA_SELECT_THRESHOLD && (shape.head_dim == 64 || shape.head_dim == 128)) {
    // threshold decided in the tensor-core score epilogue: keep bits + argmax, no score tensor
    Workspace pw = w;
    pw.take<char>(static_cast<int64_t>(ws_pooled_bytes(shape)));
    const int64_t words = (n + 31) / 32;
    PooledOut out;
    out.keep_bits = pw.take<uint32_t>(rows * words);
    out.fix_rows = pw.take<int32_t>(rows);
    out.fix_count = pw.take<int32_t>(1);
    out.tau = tau;
    out.idx = idx;
    out.idx_stride = idx_stride;
    out.counts = counts;
    out.fill = fill_sentinel;
    if (out.keep_bits == nullptr || out.fix_rows == nullptr || out.fix_count == nullptr)
      return fail(FGA_EINVAL, "build_mask_avgq: workspace too small (fga_workspace_bytes)");
    // (fix_count is zeroed by the pooled-mean launch) scores -> keep bits -> lists -> argmax fix-up
    return launch_pooled_scores(q, k, shape, 1, out, w, st);
  }
  if (round_bf16 && n <= FGA_SELECT_MAX_N) {  // bf16 scores -> fused selection + compaction
    Workspace pw = w;
    pw.take<char>(static_cast<int64_t>(ws_pooled_bytes(shape)));
    uint16_t* s16 = pw.take<uint16_t>(rows * n);
    if (s16 == nullptr) return fail(FGA_EINVAL, "build_mask_avgq: workspace too small (fga_workspace_bytes)");
    PooledOut out;
    out.scores16 = s16;
    if ((rc = launch_pooled_scores(q, k, shape, 1, out, w, st)) != FGA_OK) return rc;
    return launch_select_compact(s16, rows, n, strategy, tau, top_k, idx, idx_stride, counts, fill_sentinel, st);
  }
  Workspace pw = w;
  pw.take<char>(static_cast<int64_t>(ws_pooled_bytes(shape)));
  float* sc = pw.take<float>(rows * n);
  uint8_t* keep = pw.take<uint8_t>(rows * n);
  if (sc == nullptr || keep == nullptr) return fail(FGA_EINVAL, "build_mask_avgq: workspace too small (fga_workspace_bytes)");
  PooledOut out;
  out.scores = sc;
  if ((rc = launch_pooled_scores(q, k, shape, round_bf16, out, w, st)) != FGA_OK) return rc;
  if (strategy == FGA_SELECT_THRESHOLD) {
    if ((rc = launch_threshold(sc, rows * n, tau, keep, st)) != FGA_OK) return rc;
    return launch_compact(keep, sc, rows, n, idx, idx_stride, counts, fill_sentinel, st);
  }
  if ((rc = launch_topk(sc, rows, n, top_k, keep, st)) != FGA_OK) return rc;
  return launch_compact(keep, nullptr, rows, n, idx, idx_stride, counts, fill_sentinel, st);
}

int fga_build_mask_cached(const void* q, const void* k, fga_shape shape, float tau, int round_bf16, int32_t* idx,
                          int64_t idx_stride, int32_t* counts, int fill_sentinel, void* ws, size_t ws_bytes,
                          void* stream) {
  int rc = check_shape(shape);
  if (rc != FGA_OK) return rc;
  if (!q || !k || !idx || !counts) return fail(FGA_EINVAL, "null pointer");
  if (!(tau > 0.f)) return fail(FGA_EINVAL, "tau must be positive");
  if (idx_stride < shape.seq_len) return fail(FGA_EINVAL, "idx_stride must be >= seq_len");
  if ((rc = check_ws(ws)) != FGA_OK) return rc;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t G = (shape.seq_len + shape.group_size - 1) / shape.group_size;
  const int64_t rows = shape.batch * shape.heads * G, n = shape.seq_len;
  Workspace w(ws, ws_bytes);
  Workspace pw = w;
  pw.take<char>(static_cast<int64_t>(ws_cached_bytes(shape)));
  float* gmax = pw.take<float>(rows * n);
  uint8_t* keep = pw.take<uint8_t>(rows * n);
  if (gmax == nullptr || keep == nullptr) return fail(FGA_EINVAL, "build_mask_cached: workspace too small (fga_workspace_bytes)");
  if ((rc = launch_cached_group_max(q, k, shape, round_bf16, gmax, w, st)) != FGA_OK) return rc;
  if ((rc = launch_threshold(gmax, rows * n, tau, keep, st)) != FGA_OK) return rc;
  return launch_compact(keep, gmax, rows, n, idx, idx_stride, counts, fill_sentinel, st);
}

int fga_threshold_keep(const float* scores, int64_t n_elems, float tau, uint8_t* keep, void* stream) {
  if (n_elems < 0) return fail(FGA_EINVAL, "n_elems must be >= 0");
  if (n_elems > 0 && (!scores || !keep)) return fail(FGA_EINVAL, "null pointer");
  return launch_threshold(scores, n_elems, tau, keep, static_cast<cudaStream_t>(stream));
}

int fga_topk_keep(const float* scores, int64_t rows, int64_t n, int64_t top_k, uint8_t* keep, void* stream) {
  if (rows < 0 || n < 1) return fail(FGA_EINVAL, "rows must be >= 0 and n >= 1");
  if (rows > 0 && (!scores || !keep)) return fail(FGA_EINVAL, "null pointer");
  return launch_topk(scores, rows, n, top_k, keep, static_cast<cudaStream_t>(stream));
}

int fga_group_max_map(const float* map, int64_t bh, int64_t n, int64_t group_size, int round_bf16, float* gmax,
                      void* stream) {
  if (!map || !gmax) return fail(FGA_EINVAL, "null pointer");
  return launch_group_max_map(map, bh, n, group_size, round_bf16, gmax, static_cast<cudaStream_t>(stream));
}

int fga_cached_group_max(const void* q, const void* k, fga_shape shape, int round_bf16, float* gmax, void* ws,
                         size_t ws_bytes, void* stream) {
  int rc = check_shape(shape);
  if (rc != FGA_OK) return rc;
  if (!q || !k || !gmax) return fail(FGA_EINVAL, "null pointer");
  if ((rc = check_ws(ws)) != FGA_OK) return rc;
  Workspace w(ws, ws_bytes);
  return launch_cached_group_max(q, k, shape, round_bf16, gmax, w, static_cast<cudaStream_t>(stream));
}

int fga_random_keep(int64_t rows, int64_t n, int64_t count, uint64_t seed, uint8_t* keep, void* stream) {
  if (rows < 0 || n < 1) return fail(FGA_EINVAL, "rows must be >= 0 and n >= 1");
  if (rows > 0 && !keep) return fail(FGA_EINVAL, "null pointer");
  return launch_random_keep(rows, n, count, seed, keep, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
