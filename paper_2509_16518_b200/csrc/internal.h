// Internal host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/fgattn.h"

namespace fga {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda,
// so the library loads on hosts without a driver).
// 2D bf16 map over [rows, cols] (cols innermost), box {box_cols, box_rows}, 128B swizzle.
int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                      uint32_t box_rows);

// Opt `fn` into `bytes` of dynamic shared memory (once per kernel and device).
int smem_opt_in(const void* fn, int bytes, const char* what);
// Multiprocessor count of the current device (cached).
int sm_count();

// One attention launch (attn_launch.cu).  idx == nullptr means dense (contiguous key chunks).
struct AttnLaunch {
  const void* q = nullptr;
  const void* k = nullptr;
  const void* v = nullptr;
  const int32_t* idx = nullptr;
  int64_t idx_group_stride = 0;
  const int32_t* counts = nullptr;
  void* o = nullptr;
  int o_dtype = FGA_OUT_BF16;
  float* lse = nullptr;
  int64_t tile_begin = 0;
  int64_t tile_end = -1;
  const int32_t* order = nullptr;
  int32_t* status = nullptr;
  int flags = 0;
  long long* cta_ns = nullptr;
  int64_t cta_ns_len = 0;
};

// Caller-provided device workspace (the C ABI never allocates): take() carves 256-byte aligned
// pieces and returns nullptr when the remaining bytes do not suffice.
struct Workspace {
  char* p = nullptr;
  size_t left = 0;
  Workspace() = default;
  Workspace(void* base, size_t bytes) : p(static_cast<char*>(base)), left(base ? bytes : 0) {}
  static constexpr size_t align(size_t b) { return (b + 255) & ~size_t(255); }
  template <class T>
  T* take(int64_t count) {
    const size_t bytes = align(static_cast<size_t>(count) * sizeof(T));
    if (p == nullptr || bytes > left) return nullptr;
    T* r = reinterpret_cast<T*>(p);
    p += bytes;
    left -= bytes;
    return r;
  }
};
// Workspace bytes per operation (fga_workspace_bytes), for a checked shape.
size_t ws_pooled_bytes(const fga_shape& s);
size_t ws_cached_bytes(const fga_shape& s);

// Launchers (attn_launch.cu / gather.cu / compact.cu / maskbuild.cu).
int launch_attn(const AttnLaunch& a, const fga_shape& s, cudaStream_t stream);
int launch_gather_probe(const void* k, const void* v, int64_t n, int64_t d, const int32_t* idx, int64_t idx_stride,
                        const int32_t* count, void* out_k, void* out_v, cudaStream_t stream);
int launch_gather(const void* matrix, int64_t rows, int64_t d, const int32_t* indices, int64_t n_idx, void* out,
                  cudaStream_t stream);
int launch_pack_bits(const uint8_t* keep, int64_t rows, int64_t n, uint32_t* bits, cudaStream_t stream);
// fix_rows / fix_count (nullable): rows with no bit set are listed there (count 1, idx[0] left to the
// caller's argmax pass) instead of getting count 0.
int launch_compact_bits(const uint32_t* bits, int64_t rows, int64_t n, int32_t* idx, int64_t idx_stride,
                        int32_t* counts, int fill, cudaStream_t stream, int32_t* fix_rows = nullptr,
                        int32_t* fix_count = nullptr);
int launch_fgm1_unpack(const int32_t* words, const int64_t* starts, int64_t rows, int64_t n, int32_t* idx,
                       int64_t idx_stride, int32_t* counts, int fill, cudaStream_t stream);
int launch_cached_group_max_tc(const void* q, const void* k, const fga_shape& s, int round, float* gmax,
                               float* row_max, float* row_rinv, cudaStream_t st);
// Outputs of the avg-query pooled-score pass (exactly one of scores / scores16 / keep_bits):
// fp32 scores, bf16 scores, or the threshold decision fused into the epilogue -- keep bits
// (bit b of word w of row r = key 32w + b), compacted into idx / counts, rows that keep nothing
// listed in fix_rows (fix_count zeroed by the caller) and given their argmax key by a fix-up pass.
struct PooledOut {
  float* scores = nullptr;
  uint16_t* scores16 = nullptr;
  uint32_t* keep_bits = nullptr;
  float tau = 0.f;
  int32_t* idx = nullptr;  // keep_bits: the compacted lists
  int64_t idx_stride = 0;
  int32_t* counts = nullptr;
  int fill = 0;
  int32_t* fix_rows = nullptr;   // [rows]
  int32_t* fix_count = nullptr;  // [1]
};
// parts_ready: the three bf16 parts of q̄ are already in parts (pooled_mean_bulk_kernel), else split here
int launch_pooled_scores_tc(const float* qbar, __nv_bfloat16* parts, bool parts_ready, const void* k,
                            const fga_shape& s, int round, const PooledOut& out, cudaStream_t st);
// q̄ value v -> parts[i], parts[n + i], parts[2n + i] (bf16, hi + mid + lo == v exactly)
__device__ __forceinline__ void split3(float v, __nv_bfloat16* parts, int64_t n, int64_t i) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(hi);
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
  parts[i] = hi;
  parts[n + i] = mid;
  parts[2 * n + i] = lo;
}
int launch_pooled_scores(const void* q, const void* k, const fga_shape& s, int round, const PooledOut& out,
                         Workspace& ws, cudaStream_t st);
int launch_cached_group_max(const void* q, const void* k, const fga_shape& s, int round, float* gmax, Workspace& ws,
                            cudaStream_t st);
int launch_threshold(const float* s, int64_t n, float tau, uint8_t* keep, cudaStream_t st);
int launch_topk(const float* s, int64_t rows, int64_t n, int64_t k, uint8_t* keep, cudaStream_t st);
int launch_select_compact(const uint16_t* scores, int64_t rows, int64_t n, int mode, float tau, int64_t top_k,
                          int32_t* idx, int64_t idx_stride, int32_t* counts, int fill, cudaStream_t st);
int launch_compact(const uint8_t* keep, const float* scores, int64_t rows, int64_t n, int32_t* idx,
                   int64_t idx_stride, int32_t* counts, int fill, cudaStream_t stream);

}  // namespace fga
