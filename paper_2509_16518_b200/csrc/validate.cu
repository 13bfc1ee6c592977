// Index-mask utilities around the attention launch.
//
// fga_validate_mask: the invariants SparseIndexMask enforces on the host
// (/root/reference/pkg/src/sliceattn/sparse.py:36-52): every (b,h,g) row has 1 <= count <= stride
// keys, each in [0, N), strictly ascending (sorted and deduplicated, as np.unique leaves them).
// One warp per row; HBM-bound (reads 4*count bytes per row once).
//
// fga_tile_order: the longest-first claim order for the dynamic tile scheduler (attn_ws.cu): one
// CTA per head bitonic-sorts the head's groups by list length in shared memory.
#include <climits>

#include "attn_common.cuh"
#include "internal.h"

namespace fga {
namespace {

__global__ void __launch_bounds__(256) fga_validate_kernel(const int32_t* __restrict__ idx, int64_t stride,
                                                           const int32_t* __restrict__ counts, int64_t rows, int n,
                                                           int check_order, int32_t* status) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int c = __ldg(counts + row);
  int32_t bad = (c < 1 ? FGA_STATUS_EMPTY : 0) | (c > stride ? FGA_STATUS_STRIDE : 0);
  const int live = static_cast<int>(min(static_cast<int64_t>(max(c, 0)), stride));
  const int32_t* list = idx + row * stride;
  bool oor = false, order = false;
  for (int j = lane; j < live; j += 32) {
    const int key = __ldg(list + j);
    oor |= static_cast<unsigned>(key) >= static_cast<unsigned>(n);
    if (check_order && j > 0) order |= __ldg(list + j - 1) >= key;
  }
  if (__any_sync(0xffffffffu, oor)) bad |= FGA_STATUS_RANGE;
  if (__any_sync(0xffffffffu, order)) bad |= FGA_STATUS_ORDER;
  if (lane == 0 && bad) {
    atomicOr(status, bad);
    atomicMin(status + 1, static_cast<int32_t>(min(row, static_cast<int64_t>(INT_MAX))));
  }
}

constexpr int ORDER_MAX_G = 16384;  // groups per head sorted in shared memory (128 KB of keys)

// keys: (count << 32) | ~g, sorted descending -> longest list first, ties by the smaller group
__global__ void __launch_bounds__(1024) fga_tile_order_kernel(const int32_t* __restrict__ counts, int G, int gpad,
                                                              int tpg, int32_t* __restrict__ order) {
  extern __shared__ unsigned long long keys[];
  const int64_t bh = blockIdx.x;
  for (int i = threadIdx.x; i < gpad; i += blockDim.x) {
    unsigned long long key = 0;
    if (i < G) {
      const int c = max(__ldg(counts + bh * G + i), 0);
      key = (static_cast<unsigned long long>(c) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(i));
    }
    keys[i] = key;
  }
  __syncthreads();
  for (int k = 2; k <= gpad; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < gpad; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = keys[i], b = keys[ixj];
          const bool desc = (i & k) == 0;  // descending runs become the final descending order
          if (desc ? a < b : a > b) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < G * tpg; i += blockDim.x) {
    const int rank = i / tpg, sub = i % tpg;
    const uint32_t g = ~static_cast<uint32_t>(keys[rank] & 0xffffffffull);
    order[bh * G * tpg + i] = static_cast<int32_t>((bh * G + g) * tpg + sub);
  }
}

__global__ void fga_identity_order_kernel(int64_t n, int32_t* order) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    order[i] = static_cast<int32_t>(i);
}

}  // namespace

int launch_tile_order(const int32_t* counts, const fga_shape& s, int32_t* order, cudaStream_t stream) {
  const int64_t G = (s.seq_len + s.group_size - 1) / s.group_size;
  const int64_t tpg = (s.group_size + BM - 1) / BM;
  const int64_t bh = s.batch * s.heads;
  if (bh * G * tpg >= (int64_t(1) << 31)) return fail(FGA_EINVAL, "too many tiles");
  if (G > ORDER_MAX_G) {  // too many groups to sort per head in shared memory: ascending order
    fga_identity_order_kernel<<<1184, 256, 0, stream>>>(bh * G * tpg, order);
    return check_launch("fga_identity_order_kernel");
  }
  int gpad = 1;
  while (gpad < G) gpad <<= 1;
  const int smem = gpad * 8;
  if (const int rc = smem_opt_in(reinterpret_cast<const void*>(fga_tile_order_kernel), ORDER_MAX_G * 8,
                                 "tile_order");
      rc != FGA_OK)
    return rc;
  fga_tile_order_kernel<<<static_cast<unsigned>(bh), 1024, smem, stream>>>(counts, static_cast<int>(G), gpad,
                                                                          static_cast<int>(tpg), order);
  return check_launch("fga_tile_order_kernel");
}

int launch_validate(const int32_t* idx, int64_t stride, const int32_t* counts, int64_t rows, int64_t n,
                    int check_order, int32_t* status, cudaStream_t stream) {
  if (cudaMemsetAsync(status, 0, sizeof(int32_t), stream) != cudaSuccess ||
      cudaMemsetAsync(status + 1, 0x7f, sizeof(int32_t), stream) != cudaSuccess)
    return check_launch("fga_validate_mask (status reset)");
  if (rows > 0) {
    const int64_t blocks = (rows + 7) / 8;
    fga_validate_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(idx, stride, counts, rows,
                                                                          static_cast<int>(n), check_order, status);
    if (const int rc = check_launch("fga_validate_kernel"); rc != FGA_OK) return rc;
  }
  return FGA_OK;
}

// Host side of the checked entry points: read the status word back (synchronising the stream) and
// turn it into the reference's error classes.  Count problems come first (sparse.py:47-48), then
// key ranges (:49-52), then ordering.
int status_to_code(const int32_t* status, cudaStream_t stream, const char* what) {
  int32_t host[2] = {0, INT_MAX};
  if (cudaMemcpyAsync(host, status, sizeof(host), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
      cudaStreamSynchronize(stream) != cudaSuccess)
    return check_launch(what);
  const int32_t bits = host[0];
  const std::string at = host[1] != INT_MAX && host[1] != 0x7f7f7f7f ? " (first at row " + std::to_string(host[1]) + ")" : "";
  if (bits & FGA_STATUS_EMPTY) return fail(FGA_EINVAL, std::string(what) + ": every group needs at least one key" + at);
  if (bits & FGA_STATUS_STRIDE) return fail(FGA_EINVAL, std::string(what) + ": a count exceeds the index row stride" + at);
  if (bits & FGA_STATUS_RANGE) return fail(FGA_ERANGE, std::string(what) + ": key index out of range" + at);
  if (bits & FGA_STATUS_ORDER)
    return fail(FGA_EINVAL, std::string(what) + ": key lists must be strictly ascending (sorted, no duplicates)" + at);
  return FGA_OK;
}

}  // namespace fga
