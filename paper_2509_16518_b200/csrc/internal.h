// Internal host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda.h>
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

// Launchers (attn_sm100.cu / gather.cu / compact.cu / maskbuild.cu).
int launch_attn(const void* q, const void* k, const void* v, const int32_t* idx, int64_t idx_group_stride,
                const int32_t* counts, void* o, int o_dtype, float* lse, const fga_shape& s, bool dense,
                cudaStream_t stream, int64_t tile_begin = 0, int64_t tile_end = -1);
int launch_gather(const void* matrix, int64_t rows, int64_t d, const int32_t* indices, int64_t n_idx, void* out,
                  cudaStream_t stream);
int launch_pack_bits(const uint8_t* keep, int64_t rows, int64_t n, uint32_t* bits, cudaStream_t stream);
int launch_compact_bits(const uint32_t* bits, int64_t rows, int64_t n, int32_t* idx, int64_t idx_stride,
                        int32_t* counts, int fill, cudaStream_t stream);
int launch_fgm1_unpack(const int32_t* words, const int64_t* starts, int64_t rows, int64_t n, int32_t* idx,
                       int64_t idx_stride, int32_t* counts, int fill, cudaStream_t stream);
int launch_cached_group_max_tc(const void* q, const void* k, const fga_shape& s, int round, float* gmax,
                               float* row_max, cudaStream_t st);
int launch_pooled_scores_tc(const float* qbar, const void* k, const fga_shape& s, int round, float* scores,
                            cudaStream_t st);
int launch_compact(const uint8_t* keep, const float* scores, int64_t rows, int64_t n, int32_t* idx,
                   int64_t idx_stride, int32_t* counts, int fill, cudaStream_t stream);

}  // namespace fga
