/*
 * fgattn.h -- C ABI of libfgattn.so, the B200 (sm_100a) FG-Attn hot path.
 *
 * Drop-in boundary for the reference package `sliceattn`
 * (/root/reference/pkg/src/sliceattn).  The reference is pure Python/NumPy
 * and has no FFI of its own; each entry point below is the native body of
 * one reference operator, and the Python mirror in
 * paper_2509_16518_b200/ binds them with ctypes exactly as a maintainer of
 * the reference would.
 *
 * Conventions
 *   - All pointers are DEVICE pointers owned by the caller (torch); the
 *     library never allocates or frees caller memory.
 *   - `stream` is a cudaStream_t passed as void*; every call is
 *     stream-ordered and asynchronous (no device synchronisation).
 *   - Q/K/V are bf16 [B, H, N, D] contiguous, D innermost.
 *   - A "group" is `group_size` (M) consecutive query rows; G = ceil(N/M)
 *     (core.py:69-76).  Masks are per (b, h, g) rows of N slots.
 *   - Return 0 on success, a negative FGA_E* code otherwise; the message is
 *     available from fga_last_error() (thread-local).
 */
#ifndef FGATTN_H_
#define FGATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FGA_OK 0
#define FGA_EINVAL (-1)        /* shape / config error   -> ShapeError / ValueError */
#define FGA_ERANGE (-2)        /* index out of range     -> IndexError / ValueError */
#define FGA_ECUDA (-3)         /* CUDA launch / driver   -> RuntimeError            */
#define FGA_EUNSUPPORTED (-4)  /* D not supported, not sm_100                         */

#define FGA_OUT_BF16 0
#define FGA_OUT_F32 1

/* Problem shape; mirrors AttnConfig (core.py:32-63).  scale <= 0 means 1/sqrt(D). */
typedef struct fga_shape {
  int64_t batch;
  int64_t heads;
  int64_t seq_len;
  int64_t head_dim;
  int64_t group_size;
  float scale;
} fga_shape;

/* Library version (major*10000 + minor*100 + patch). */
int fga_version(void);

/* Thread-local description of the last failure ("" when none). */
const char* fga_last_error(void);

/* 1 when `device` is an sm_100 part the kernels were built for, else 0. */
int fga_device_supported(int device);

/*
 * Slice-mask compaction (K1b).  Replaces masks.py:75-91 (_lists_from_keep)
 * followed by sparse.py:165-175 (export_padded).
 *   keep   : uint8 [rows, n], nonzero = keep key j for that (b,h,g) row.
 *   scores : optional fp32 [rows, n]; when given, an empty row falls back to
 *            the first position of its maximum (masks.py:86-87).  When NULL
 *            an empty row keeps count 0.
 *   idx    : int32 [rows, idx_stride]; receives the ascending kept positions.
 *   counts : int32 [rows].
 *   fill_sentinel : nonzero -> slots [count, n) of each row are set to -1
 *            (the export_padded layout); zero -> left untouched.
 */
int fga_compact(const uint8_t* keep, const float* scores, int64_t rows, int64_t n, int32_t* idx,
                int64_t idx_stride, int32_t* counts, int fill_sentinel, void* stream);

/*
 * Bit-packed slice masks: bit b of word w of a row is key 32w+b (8x fewer
 * bytes than uint8 keep, e.g. for shipping masks from the host).
 *   fga_pack_bits    : keep uint8 [rows, n] -> bits uint32 [rows, ceil(n/32)].
 *   fga_compact_bits : same output contract as fga_compact without the
 *                      argmax fallback (an empty row keeps count 0).
 */
int fga_pack_bits(const uint8_t* keep, int64_t rows, int64_t n, uint32_t* bits, void* stream);
int fga_compact_bits(const uint32_t* bits, int64_t rows, int64_t n, int32_t* idx, int64_t idx_stride, int32_t* counts,
                     int fill_sentinel, void* stream);

/*
 * FGM1 slice-mask files (paper_2509_16518_b200/io.py) decoded on the
 * device: the host parses the header and the per-row list starts (the lengths are
 * interleaved with the lists), uploads the u32 payload once, and this scatters it
 * into the fga_compact output layout.
 *   words  : int32 view of the payload after the 48-byte header.
 *   starts : int64 [rows]; row r's list is words[starts[r] .. starts[r] + words[starts[r]-1]).
 *   idx, counts, fill_sentinel : as fga_compact.
 */
int fga_fgm1_unpack(const int32_t* words, const int64_t* starts, int64_t rows, int64_t n, int32_t* idx,
                    int64_t idx_stride, int32_t* counts, int fill_sentinel, void* stream);

/*
 * FG-Attn forward (K2 gather producer + K3 tcgen05 consumer).
 * Replaces sparse.py:111-156 (sparse_attention), whose numerics are the
 * online softmax of tiled.py:48-77; equals oracle.py:55-82
 * (masked_dense_attention) within bf16 tolerance.
 *   idx    : int32, row (b,h,g) at idx + ((b*H+h)*G+g)*idx_group_stride,
 *            first counts[(b*H+h)*G+g] entries used (ascending, as
 *            SparseIndexMask keeps them).
 *   counts : int32 [B*H*G], each in [1, idx_group_stride].
 *   o      : [B, H, N, D], bf16 (o_dtype = FGA_OUT_BF16) or fp32 (FGA_OUT_F32).
 *   lse    : optional fp32 [B, H, N] natural-log softmax normaliser.
 * Supported: head_dim in {64, 128}; any group_size in [1, N].
 * Masks that break the invariants never make the kernels read out of bounds
 * (counts are clamped to [0, stride], keys to min(unsigned key, N-1)) but give
 * unspecified rows (a group with no key gets zeros); fga_validate_mask or the
 * FGA_ATTN_CHECK flag of fga_sparse_attn_fwd_ex report them as the reference
 * does (sparse.py:47-52).
 */
int fga_sparse_attn_fwd(const void* q, const void* k, const void* v, const int32_t* idx,
                        int64_t idx_group_stride, const int32_t* counts, void* o, int o_dtype, float* lse,
                        fga_shape shape, void* stream);

/*
 * fga_sparse_attn_fwd restricted to work tiles [tile_begin, tile_end).  A
 * tile is <=128 query rows of one group; tiles are numbered head-major,
 * tile = ((b*H + h)*G + g)*ceil(M/128) + sub, so a contiguous range is a run
 * of (head, group-range) units.  Multi-GPU shards call this with their own
 * range on full-size tensors; rows outside the range are not written.
 */
int fga_sparse_attn_fwd_tiles(const void* q, const void* k, const void* v, const int32_t* idx,
                              int64_t idx_group_stride, const int32_t* counts, void* o, int o_dtype, float* lse,
                              fga_shape shape, int64_t tile_begin, int64_t tile_end, void* stream);

/* Mask-violation bits written to a status word (int32[2] device workspace:
 * [0] = OR of the bits, [1] = first offending row when known). */
#define FGA_STATUS_EMPTY 1   /* a group with count < 1        (sparse.py:47-48) */
#define FGA_STATUS_RANGE 2   /* a key outside [0, N)          (sparse.py:49-52) */
#define FGA_STATUS_STRIDE 4  /* count > idx_group_stride                        */
#define FGA_STATUS_ORDER 8   /* list not strictly ascending (fga_validate_mask) */

/* fga_sparse_attn_fwd_ex flags */
#define FGA_ATTN_CHECK 1     /* validate counts + key ranges first (status reset), run, synchronise, return
                                FGA_EINVAL / FGA_ERANGE on violations (fga_validate_mask without the order check) */
#define FGA_ATTN_PER_TILE 2  /* per-tile kernel also for 129..256-row groups (no shared-gather dual kernel)  */
#define FGA_ATTN_STATIC 4    /* static tile stride instead of the dynamic tile scheduler                     */

/*
 * General form of the two entries above.
 *   order  : optional int32 [tile_end - tile_begin]: the k-th tile claimed is
 *            tile_begin + order[k] (a permutation; e.g. longest lists first
 *            within each head, see fga_tile_order).  NULL = ascending.
 *   status : optional int32[2] device word; the kernel ORs the count bits
 *            (FGA_STATUS_EMPTY / _STRIDE) of the tiles it runs into status[0]
 *            (the caller zeroes it, unless FGA_ATTN_CHECK, which also checks
 *            the key ranges before the launch).
 *   flags  : FGA_ATTN_* bits.
 */
int fga_sparse_attn_fwd_ex(const void* q, const void* k, const void* v, const int32_t* idx,
                           int64_t idx_group_stride, const int32_t* counts, void* o, int o_dtype, float* lse,
                           fga_shape shape, int64_t tile_begin, int64_t tile_end, const int32_t* order,
                           int32_t* status, int flags, void* stream);

/*
 * fga_sparse_attn_fwd_ex plus a per-CTA timeline of the persistent kernel
 * (load-balance measurement): cta_ns[2b] / cta_ns[2b + 1] = %globaltimer (ns)
 * when CTA b starts / finishes its tiles, for b < cta_ns_len / 2 (device
 * int64 buffer; the grid is at most one CTA per SM).
 */
int fga_sparse_attn_fwd_timed(const void* q, const void* k, const void* v, const int32_t* idx,
                              int64_t idx_group_stride, const int32_t* counts, void* o, int o_dtype, float* lse,
                              fga_shape shape, int64_t tile_begin, int64_t tile_end, const int32_t* order,
                              int32_t* status, int flags, long long* cta_ns, int64_t cta_ns_len, void* stream);

/*
 * Checks an index mask against the SparseIndexMask invariants
 * (sparse.py:36-52): 1 <= counts[r] <= idx_group_stride, keys in [0, n),
 * strictly ascending.  Synchronises `stream`; returns FGA_OK, FGA_EINVAL
 * (count or order) or FGA_ERANGE (key range).  status: int32[2] device
 * workspace (left holding the bits and the first offending row).
 */
int fga_validate_mask(const int32_t* idx, int64_t idx_group_stride, const int32_t* counts, int64_t rows, int64_t n,
                      int32_t* status, void* stream);

/*
 * Longest-first tile order for fga_sparse_attn_fwd_ex: within each head
 * (b,h), its groups' tiles sorted by list length, descending (ties by group
 * index); heads stay in order, so the K/V of about two heads are live in L2
 * at a time.  order: int32 [B*H*G*ceil(M/128)].
 */
int fga_tile_order(const int32_t* counts, fga_shape shape, int32_t* order, void* stream);

/*
 * Dense attention with the same kernel and contiguous key chunks (every group
 * lists all N keys).  Replaces tiled.py:80-114 (flash_attention) /
 * oracle.py:29-42 (dense_attention); the dense denominator of the speed-up.
 */
int fga_dense_attn_fwd(const void* q, const void* k, const void* v, void* o, int o_dtype, float* lse,
                       fga_shape shape, void* stream);

/*
 * Gather-load primitive (K2 in isolation, for bitwise parity).  Replaces
 * sparse.py:95-108 (gather_rows): out[i, :] = matrix[indices[i], :].
 *   matrix : bf16 [rows, d], d a multiple of 64, d <= 256.
 *   indices: int32 [n_idx], each in [0, rows) (duplicates allowed).
 *   out    : bf16 [n_idx, d].
 */
int fga_gather_rows(const void* matrix, int64_t rows, int64_t d, const int32_t* indices, int64_t n_idx,
                    void* out, void* stream);

/*
 * Device workspace.  The library never allocates device memory: operations
 * that need scratch space take (ws, ws_bytes), a caller-owned buffer of at
 * least fga_workspace_bytes(op, shape, round_bf16) bytes, 256-byte aligned,
 * used stream-ordered on `stream` (reusable once the stream passes the call).
 * Returns the byte count (>= 0), or a negative FGA_* code for a bad shape/op.
 */
#define FGA_WS_POOLED_SCORES 1    /* fga_pooled_scores, fga_pooled_scores_bf16 */
#define FGA_WS_CACHED_GROUP_MAX 2 /* fga_cached_group_max                      */
#define FGA_WS_BUILD_AVGQ 3       /* fga_build_mask_avgq                       */
#define FGA_WS_BUILD_CACHED 4     /* fga_build_mask_cached                     */
int64_t fga_workspace_bytes(int op, fga_shape shape, int round_bf16);

/*
 * K2 of the attention kernel in isolation (test hook).  Runs the hot path's
 * own gather producers (attn_ws.cu producer_half: 16-byte cp.async into the
 * 128B-swizzled K/V ring slots) for one key list and copies every ring slot
 * back out, un-swizzled, in chunk order: rows [0, c) of out_k / out_v equal
 * gather_rows(k, idx[:c]) (sparse.py:95-108) bitwise, with c = min(*count,
 * idx_stride); rows [c, 128*ceil(c/128)) are zero (the zero-filled tail of the
 * last chunk).  Keys are clamped like the kernel's (min(unsigned key, n-1)).
 *   k, v  : bf16 [n, d], d in {64, 128};  count : device int32[1];
 *   out_k, out_v : bf16 [128*ceil(c/128), d].
 */
int fga_gather_ring_probe(const void* k, const void* v, int64_t n, int64_t d, const int32_t* idx, int64_t idx_stride,
                          const int32_t* count, void* out_k, void* out_v, void* stream);

/*
 * Average-query pooled scores (K1a, avg-query builder).  Replaces
 * masks.py:108-118 (pooled_query_scores):
 *   scores[b,h,g,j] = exp((k_j . mean_{i in g} q_i) * scale) / D   (fp32),
 *   rounded to bf16 (RNE, widened) when round_bf16 != 0.
 *   scores : fp32 [B, H, G, N].
 */
int fga_pooled_scores(const void* q, const void* k, fga_shape shape, int round_bf16, float* scores, void* ws,
                      size_t ws_bytes, void* stream);

/* The same scores as bf16 bits (round_bf16 = 1 semantics, half the bytes):
 * the input of fga_select_compact.  scores : uint16 [B, H, G, N]. */
int fga_pooled_scores_bf16(const void* q, const void* k, fga_shape shape, uint16_t* scores, void* ws,
                           size_t ws_bytes, void* stream);

/*
 * Selection + compaction in one kernel for bf16 scores (K1a tail + K1b).
 * Replaces masks.py:131-147 followed by masks.py:75-91 / sparse.py:45-55:
 *   FGA_SELECT_THRESHOLD: keep s >= tau; an empty row keeps [argmax(s)];
 *   FGA_SELECT_TOPK     : the top_k largest, ties toward the smaller index;
 * lists ascending in idx[row * idx_stride ...], counts[row]; fill_sentinel
 * writes -1 up to n.  scores : uint16 bf16 bits [rows, n], n <= FGA_SELECT_MAX_N.
 */
#define FGA_SELECT_THRESHOLD 0
#define FGA_SELECT_TOPK 1
#define FGA_SELECT_MAX_N 114688
int fga_select_compact(const uint16_t* scores, int64_t rows, int64_t n, int mode, float tau, int64_t top_k,
                       int32_t* idx, int64_t idx_stride, int32_t* counts, int fill_sentinel, void* stream);

/*
 * Single-call mask builders (K1a -> K1b), lists straight into the device
 * index layout.  fga_build_mask_avgq replaces masks.py:121-150
 * (build_mask_avg_query; strategy FGA_SELECT_THRESHOLD with tau > 0, or
 * FGA_SELECT_TOPK with 1 <= top_k <= N); fga_build_mask_cached replaces
 * masks.py:94-105 on attention_map(q, k) (oracle.py:45-52) without the N x N
 * map.  idx : int32 [B*H*G, idx_stride >= N]; counts : int32 [B*H*G].
 */
int fga_build_mask_avgq(const void* q, const void* k, fga_shape shape, int strategy, float tau, int64_t top_k,
                        int round_bf16, int32_t* idx, int64_t idx_stride, int32_t* counts, int fill_sentinel,
                        void* ws, size_t ws_bytes, void* stream);
int fga_build_mask_cached(const void* q, const void* k, fga_shape shape, float tau, int round_bf16, int32_t* idx,
                          int64_t idx_stride, int32_t* counts, int fill_sentinel, void* ws, size_t ws_bytes,
                          void* stream);

/* keep[i] = scores[i] >= tau  (masks.py:132 / masks.py:104). */
int fga_threshold_keep(const float* scores, int64_t n_elems, float tau, uint8_t* keep, void* stream);

/*
 * Top-k keep bits per row (masks.py:133-147): the top_k largest scores of
 * each row, ties broken toward the smaller key index.
 *   scores : fp32 [rows, n]; keep : uint8 [rows, n].
 */
int fga_topk_keep(const float* scores, int64_t rows, int64_t n, int64_t top_k, uint8_t* keep, void* stream);

/*
 * Group maximum of an explicit post-softmax map (K1a, cached builder from a
 * materialised map).  Replaces masks.py:66-72 (_group_max) on
 * analysis_scores(map) as used by masks.py:94-105 (build_mask_cached):
 *   gmax[bh, g, j] = max_{i in group g} map[bh, i, j]   (bf16-rounded when round_bf16)
 *   map  : fp32 [BH, N, N];  gmax : fp32 [BH, G, N].
 */
int fga_group_max_map(const float* map, int64_t bh, int64_t n, int64_t group_size, int round_bf16, float* gmax,
                      void* stream);

/*
 * Cached-threshold statistics (K1a, cached builder) without materialising
 * the [B,H,N,N] map: pass 1 computes each query row's softmax normaliser,
 * pass 2 the per-group column maximum of the normalised map.  Replaces
 * oracle.py:45-52 (attention_map) + masks.py:66-72 (_group_max) as used by
 * masks.py:94-105 (build_mask_cached).
 *   gmax   : fp32 [B, H, G, N]; bf16-rounded when round_bf16 != 0.
 *   ws     : fga_workspace_bytes(FGA_WS_CACHED_GROUP_MAX, ...) bytes.
 */
int fga_cached_group_max(const void* q, const void* k, fga_shape shape, int round_bf16, float* gmax, void* ws,
                         size_t ws_bytes, void* stream);

/*
 * Benchmark masks: every row keeps exactly `count` distinct keys chosen
 * uniformly at random (the random_mask count rule, sparse.py:216-232, with
 * a counter-based device RNG -- not NumPy's Philox stream).
 */
int fga_random_keep(int64_t rows, int64_t n, int64_t count, uint64_t seed, uint8_t* keep, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FGATTN_H_ */
