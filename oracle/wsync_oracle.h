/*
 * wsync_oracle.h -- CPU restatement of the reference weight-sync data plane.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2605_06534_b200/, its C-ABI in include/wsync.h, or the Python
 * mirror) may link, load or call this code.  It is used by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline leg.
 *
 * Each function restates one reference function from
 * /root/reference/proj/src/transfer/ (cited per function in wsync_oracle.c)
 * and extends it where the B200 build needs more than the reference has:
 *   - dtype BF16 (code 2): 16-bit words compared by bit pattern, delta is the
 *     u16 wrap-around difference, apply is the u16 wrap-around add -- the
 *     reference's I32 semantics (codec.cpp:52-61, :80-91) on 16-bit words.
 *   - cross-dim reslicing: a box intersection when source and destination are
 *     sliced along different dims (the reference throws ShapeMismatch,
 *     codec.cpp:101-102); selectable so the same-dim behaviour stays pinned.
 *
 * Parity pinning: the F32/I32 paths are checked element for element against
 * the compiled reference (oracle/_ref/libref_capi.so) in tests/test_oracle.py;
 * BF16 has no reference counterpart and is pinned only through the I32 path
 * it generalises.
 */
#ifndef WSYNC_ORACLE_H
#define WSYNC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { WSO_F32 = 0, WSO_I32 = 1, WSO_BF16 = 2 };

/* Status codes: identical numbering to ws_status in include/wsync.h. */
enum {
  WSO_OK = 0,
  WSO_SHAPE_MISMATCH = 1,
  WSO_PAYLOAD_FORMAT = 2,
  WSO_INDEX_OUT_OF_SHARD = 3,
  WSO_INDIVISIBLE_SHAPE = 4,
  WSO_INVALID_ARGUMENT = 23,
};

int wso_dtype_size(int dtype);

/* codec.cpp:34-63 diff_shards over n elements (shape check is the caller's). */
int wso_diff_shards(int dtype, const void* prev, const void* next, uint64_t n,
                    uint64_t* out_idx, void* out_val, uint64_t* out_nnz);

/* codec.cpp:65-92 apply_delta; like the reference, an out-of-range index
 * stops the loop with WSO_INDEX_OUT_OF_SHARD after the earlier records were
 * applied. */
int wso_apply_delta(int dtype, void* target, uint64_t n, const uint64_t* idx,
                    const void* val, uint64_t nnz);

/* codec.cpp:94-138 reslice_delta.  A shard is (slice_dim, start, end) with
 * slice_dim < 0 meaning the full tensor (shard.hpp:32-45).  When
 * allow_cross_dim is 0, slices along different dims fail with
 * WSO_SHAPE_MISMATCH as in the reference; when 1, the box intersection is
 * used.  out_* must hold nnz records. */
int wso_reslice_delta(int dtype, const int64_t* full_shape, int ndims,
                      int src_dim, int64_t src_start, int64_t src_end,
                      int dst_dim, int64_t dst_start, int64_t dst_end,
                      int allow_cross_dim, const uint64_t* idx, const void* val,
                      uint64_t nnz, uint64_t* out_idx, void* out_val,
                      uint64_t* out_nnz);

/* shard.cpp:111-134 extract_shard (shard of a full tensor). */
int wso_extract_shard(int dtype, const int64_t* full_shape, int ndims,
                      int dim, int64_t start, int64_t end, const void* full,
                      void* out);

/* shard.cpp:136-170 copy_overlap generalised to boxes: copies the overlap of
 * the src shard into the dst shard, both shards of one tensor of full_shape.
 * Returns copied elements (>= 0) or a negative status. */
int64_t wso_copy_overlap_box(int dtype, const int64_t* full_shape, int ndims,
                             int dst_dim, int64_t dst_start, int64_t dst_end,
                             void* dst, int src_dim, int64_t src_start,
                             int64_t src_end, const void* src);

/* Sparse decision of engine.cpp:118-127: sparse iff nnz/n <= threshold. */
int wso_is_sparse(uint64_t nnz, uint64_t n, double threshold);

/* The synthetic bf16 weight-pair generator,
 * restated on the CPU so the device generator can be checked.  Fills the
 * elements of one shard (slice_dim/start/end of a tensor of full_shape).
 * Element g of the full tensor draws from splitmix64 counters keyed by
 * splitmix64(seed ^ fnv1a64(name)) (rng.hpp:73-87, :98) -- so the values do
 * not depend on the layout.  change_thr = floor(density * 2^32), at most 2^32. */
uint64_t wso_param_key(uint64_t seed, const char* name);
void wso_gen_pair_bf16(uint64_t key, const int64_t* full_shape, int ndims,
                       int dim, int64_t start, int64_t end,
                       uint64_t change_thr, uint16_t* prev, uint16_t* next);
/* Same with a threshold per index along dim 0 (per-expert densities). */
void wso_gen_pair_bf16_dim0(uint64_t key, const int64_t* full_shape, int ndims,
                            int dim, int64_t start, int64_t end,
                            const uint64_t* thr_dim0, uint16_t* prev, uint16_t* next);

/* Sparse wire payload, codec.cpp:145-183 (encode) and :196-263 (decode).
 * dtype 2 (BF16) uses magic "CWS2"/"CWD2" and 2-byte values (DESIGN.md
 * "Wire format"); F32/I32 keep CWS1/CWD1.  encode returns bytes written. */
uint64_t wso_sparse_payload_size(int dtype, int ndims, int index_width,
                                 uint64_t nnz);
int wso_encode_sparse(int dtype, const int64_t* shape, int ndims,
                      int index_width, const uint64_t* idx, const void* val,
                      uint64_t nnz, uint8_t* out, uint64_t* out_len);

#ifdef __cplusplus
}
#endif
#endif
