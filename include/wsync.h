/*
 * wsync.h -- C-ABI of the B200-native sparse weight-sync data plane
 * (libwsync.so, sm_100a).
 *
 * This is the drop-in boundary for the hot path of the reference's
 * cross-cluster weight-transfer engine (/root/reference/proj/include/
 * coserve/transfer).  Every entry point names the reference interface it
 * replaces; INTEGRATION.md shows the C++ shim that re-exposes the reference's
 * own signatures (HostTensor / SparseDelta) on top of these calls.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "dev" pointers are CUDA device
 *     pointers; "host" pointers are host memory.  No exception crosses the
 *     ABI: every call returns a ws_status whose numbering maps 1:1 onto the
 *     reference's TransferError hierarchy (tensor.hpp:16-24, codec.hpp:9-11,
 *     shard.hpp:9-14, plan.hpp:7-9, relay.hpp:17-22, key.hpp:10-12).
 *     ws_last_error() returns the message of the calling thread's last error.
 *   - Kernel entry points are asynchronous on the given stream.  Errors found
 *     on the device (an index outside the shard) are reported through a
 *     device word `err_dev` (bit flags WS_ERRBIT_*); the caller reads it
 *     after synchronising.  Unlike the reference (codec.cpp:73-79, which
 *     applies a prefix of the records before throwing) a device-detected
 *     error leaves the target untouched.
 *   - dtype codes 0/1 are the reference's DType (tensor.hpp:26); code 2 is
 *     the bf16 extension (16-bit words compared by bit pattern, u16
 *     wrap-around delta and apply -- the reference's I32 rule on 16-bit
 *     words, codec.cpp:52-61 / :80-91).
 *   - Delta streams (the reference's SparseDelta, codec.hpp:16-32) are SoA:
 *     ascending, unique u32 local flat indices + raw values of the dtype
 *     width.  (pick_index_width, codec.cpp:140-143, picks 4 bytes for every
 *     shard below 2^32 elements; shards beyond that are rejected with
 *     WS_INVALID_ARGUMENT.)
 *   - Threading: one stream per call; handles are not shared across threads
 *     without external synchronisation (engine.hpp:70-92's TransferEngine is
 *     likewise used by one caller at a time).
 */
#ifndef WSYNC_H
#define WSYNC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ws_stream_t; /* == cudaStream_t */

typedef enum ws_status {
  WS_OK = 0,
  WS_SHAPE_MISMATCH = 1,       /* ShapeMismatch        tensor.hpp:19-21 */
  WS_PAYLOAD_FORMAT = 2,       /* PayloadFormatError   tensor.hpp:22-24 */
  WS_INDEX_OUT_OF_SHARD = 3,   /* IndexOutOfShard      codec.hpp:9-11   */
  WS_INDIVISIBLE_SHAPE = 4,    /* IndivisibleShape     shard.hpp:9-11   */
  WS_UNKNOWN_MODULE_KIND = 5,  /* UnknownModuleKind    shard.hpp:12-14  */
  WS_INCOMPLETE_COVERAGE = 6,  /* IncompleteCoverage   plan.hpp:7-9     */
  WS_RELAY_TIMEOUT = 7,        /* RelayTimeout         relay.hpp:17-19  */
  WS_INTEGRITY = 8,            /* IntegrityError       relay.hpp:20-22  */
  WS_KEY_FORMAT = 9,           /* KeyFormatError       key.hpp:10-12    */
  WS_TRANSFER_ERROR = 10,      /* TransferError        tensor.hpp:16-18 */
  WS_CUDA = 20,
  WS_NCCL = 21,
  WS_CAPACITY = 22,
  WS_INVALID_ARGUMENT = 23
} ws_status;

typedef enum ws_dtype { WS_F32 = 0, WS_I32 = 1, WS_BF16 = 2 } ws_dtype;

/* ModuleKind (manifest.hpp:13-19) + WS_EXPERT: a stacked expert tensor
 * [E, ...] that is split along dim 0 (EP) by every layout. */
typedef enum ws_module_kind {
  WS_COLUMN_LINEAR = 0,
  WS_ROW_LINEAR = 1,
  WS_EMBEDDING = 2,
  WS_NORM = 3,
  WS_REPLICATED = 4,
  WS_EXPERT = 5
} ws_module_kind;

/* Device-side error bits written to err_dev. */
#define WS_ERRBIT_INDEX_OUT_OF_SHARD 0x1u
#define WS_ERRBIT_CAPACITY 0x2u

#define WS_MAX_DIMS 4

const char* ws_status_name(ws_status s);
const char* ws_last_error(void);
int ws_abi_version(void);

/* ------------------------------------------------------------------------ */
/* Codec kernels on one shard (raw device pointers)                          */
/* ------------------------------------------------------------------------ */

/* Workspace bytes needed by ws_diff_shards / ws_reslice_delta for n
 * elements (resp. nnz records). */
size_t ws_diff_workspace_bytes(uint64_t n);

/* K1, replaces diff_shards (codec.hpp:37, codec.cpp:34-63): every position
 * whose value changed between prev and next, ascending.  Records beyond
 * `cap` are counted but not written (nnz_dev still receives the full
 * count), so cap = threshold * n implements the density fallback of
 * engine.cpp:118-127 without a second pass. */
ws_status ws_diff_shards(ws_dtype dtype, const void* prev_dev,
                         const void* next_dev, uint64_t n, uint32_t* idx_dev,
                         void* val_dev, uint64_t cap, uint64_t* nnz_dev,
                         void* workspace_dev, size_t workspace_bytes,
                         ws_stream_t stream);

/* K4, replaces apply_delta (codec.hpp:41, codec.cpp:65-92): target[idx[k]]
 * += val[k] (F32 IEEE add; I32/BF16 wrap-around add).  The record count is
 * read from nnz_dev when non-null (nnz is then an upper bound that sizes the
 * launch; 0 = unknown, a full-device grid), else nnz.  All indices are validated
 * before any write; an index >= n sets WS_ERRBIT_INDEX_OUT_OF_SHARD in
 * err_dev and leaves target unchanged. */
ws_status ws_apply_delta(ws_dtype dtype, void* target_dev, uint64_t n,
                         const uint32_t* idx_dev, const void* val_dev,
                         uint64_t nnz, const uint64_t* nnz_dev, uint32_t* err_dev,
                         ws_stream_t stream);

/* One rank's slice of one parameter (ShardDescriptor, shard.hpp:32-45):
 * slice_dim < 0 means the full tensor. */
typedef struct ws_shard {
  int32_t slice_dim;
  int64_t start;
  int64_t end;
} ws_shard;

/* K3 (re-index part), replaces reslice_delta (codec.hpp:46-48,
 * codec.cpp:94-138): re-expresses a delta local to `src` as a delta local to
 * `dst`, dropping records outside dst, order preserving.  Extension: when
 * src and dst are sliced along different dims the box intersection is used
 * (the reference throws ShapeMismatch, codec.cpp:101-102); pass
 * allow_cross_dim = 0 for the reference's behaviour.  An index outside the
 * source shard sets WS_ERRBIT_INDEX_OUT_OF_SHARD and writes no output. */
ws_status ws_reslice_delta(ws_dtype dtype, const int64_t* full_shape, int ndims,
                           ws_shard src, ws_shard dst, int allow_cross_dim,
                           const uint32_t* idx_dev, const void* val_dev,
                           uint64_t nnz, const uint64_t* nnz_dev,
                           uint32_t* out_idx_dev, void* out_val_dev,
                           uint64_t* out_nnz_dev, uint32_t* err_dev,
                           void* workspace_dev, size_t workspace_bytes,
                           ws_stream_t stream);

/* Dense fallback apply, replaces copy_overlap (shard.hpp:62-63,
 * shard.cpp:136-170) generalised to two shards of one tensor (same-dim or
 * cross-dim): copies src's overlap with dst into dst.  *copied receives the
 * element count (host). */
ws_status ws_copy_overlap(ws_dtype dtype, const int64_t* full_shape, int ndims,
                          ws_shard dst, void* dst_dev, ws_shard src,
                          const void* src_dev, int64_t* copied,
                          ws_stream_t stream);

/* Replaces extract_shard (shard.hpp:57, shard.cpp:111-134) on the device. */
ws_status ws_extract_shard(ws_dtype dtype, const int64_t* full_shape, int ndims,
                           ws_shard desc, const void* full_dev, void* out_dev,
                           ws_stream_t stream);

/* Synthetic bf16 weight pair for one shard;
 * the device twin of random_weights/perturb_weights (manifest.cpp:47-89).
 * change_thr = floor(density * 2^32) (<= 2^32). */
ws_status ws_gen_pair_bf16(uint64_t seed, const char* param_name,
                           const int64_t* full_shape, int ndims, ws_shard desc,
                           uint64_t change_thr, uint16_t* prev_dev,
                           uint16_t* next_dev, ws_stream_t stream);

/* Same with a change threshold per index along dim 0 (thr_dim0_dev: device
 * array of full_shape[0] entries), e.g. per-expert densities of a stacked
 * [E, ...] expert tensor. */
ws_status ws_gen_pair_bf16_dim0(uint64_t seed, const char* param_name,
                                const int64_t* full_shape, int ndims, ws_shard desc,
                                const uint64_t* thr_dim0_dev, uint16_t* prev_dev,
                                uint16_t* next_dev, ws_stream_t stream);

/* Skewed per-expert change densities (BASELINE config 4): Zipf(zipf_s)
 * weights over the ranks 1..experts, normalised to mean 1, assigned to the
 * experts by a Fisher-Yates shuffle driven by splitmix64(perm_seed + k);
 * out[e] = floor(min(1, density * weight) * 2^32). */
ws_status ws_expert_thresholds(int experts, double density, double zipf_s,
                               uint64_t perm_seed, uint64_t* out);

/* ------------------------------------------------------------------------ */
/* Wire format on the device (codec.cpp:140-263, wire.cpp, key.cpp)          */
/* ------------------------------------------------------------------------ */

typedef struct ws_payload_info {
  char codec;             /* 'S' sparse delta, 'D' dense snapshot */
  int32_t dtype;          /* ws_dtype */
  int32_t ndims;
  int32_t index_width;    /* 4 or 8 (sparse), 0 (dense) */
  int64_t shape[8];
  uint64_t nnz;           /* sparse records */
  uint64_t header_bytes;  /* offset of the index (sparse) / value (dense) block */
  uint64_t total_bytes;
} ws_payload_info;

/* Bytes of a payload: count = records (codec 'S') or elements ('D'). */
uint64_t ws_payload_bytes(ws_dtype dtype, int ndims, char codec, int index_width,
                          uint64_t count);

/* encode_sparse / encode_dense (codec.cpp:145-183) into device memory
 * (8-byte aligned, ws_payload_bytes long).  F32/I32: "CWS1"/"CWD1"; BF16:
 * "CWS2"/"CWD2" with 2-byte values.  idx are u32 local indices, written
 * as index_width (4 or 8) bytes. */
ws_status ws_encode_sparse_dev(ws_dtype dtype, const int64_t* shape, int ndims,
                               int index_width, const uint32_t* idx_dev,
                               const void* val_dev, uint64_t nnz, void* out_dev,
                               ws_stream_t stream);
ws_status ws_encode_dense_dev(ws_dtype dtype, const int64_t* shape, int ndims,
                              const void* data_dev, void* out_dev, ws_stream_t stream);

/* decode_header + size checks of decode_payload (codec.cpp:196-263) on a
 * payload in device memory: PayloadFormatError exactly where the reference
 * throws. */
ws_status ws_peek_payload_dev(const void* payload_dev, uint64_t len,
                              ws_payload_info* info);

/* peek_payload_size (codec.hpp:66-67, codec.cpp:219-227): the full size of a
 * payload of which only the first `len` bytes (at least its header) are in
 * device memory; PayloadFormatError on a bad or truncated header. */
ws_status ws_peek_payload_size_dev(const void* payload_dev, uint64_t len, uint64_t* total);

/* The records of a sparse payload (after ws_peek_payload_dev): u32 indices
 * (PayloadFormatError unless strictly ascending, codec.cpp:257) and values.
 * Synchronises. */
ws_status ws_decode_sparse_dev(const void* payload_dev, const ws_payload_info* info,
                               uint32_t* idx_dev, void* val_dev, ws_stream_t stream);

/* frame_crc32 (wire.cpp:9-13, zlib polynomial) of n device byte ranges;
 * crc_out is host memory.  Synchronises. */
ws_status ws_crc32_dev(const void* const* data_dev, const uint64_t* len, int n,
                       uint32_t* crc_out, ws_stream_t stream);

/* The bucket frames of one payload (engine.cpp:136-148 + wire.cpp:35-47):
 * bucket k = payload[k*bucket_bytes, ...), at least one bucket; frame k =
 * [key_len u32][keys[k]][len u32][bucket][crc32 u32] at out + frame_off[k]
 * (frame_off has nbuckets + 1 entries, host).  Synchronises. */
ws_status ws_encode_bucket_frames_dev(const void* payload_dev, uint64_t payload_len,
                                      uint64_t bucket_bytes, const char* const* keys,
                                      const uint64_t* key_lens, int nbuckets,
                                      void* out_dev, uint64_t out_cap,
                                      uint64_t* frame_off, ws_stream_t stream);

/* BucketKey::encode (key.cpp:47-69): w|s<step>|p<param>|t<r>.<n>|g<stage>|
 * d<slice>|c<codec><iw>|q<seq>, '%' and '|' in the name escaped. */
ws_status ws_bucket_key(uint64_t step, const char* param, int tp_rank, int tp_size,
                        int pp_stage, ws_shard desc, char codec, int index_width,
                        uint32_t seq, char* out, uint64_t cap, uint64_t* out_len);

/* ------------------------------------------------------------------------ */
/* Planner (host, plan.hpp / shard.hpp)                                      */
/* ------------------------------------------------------------------------ */

typedef struct ws_param {
  const char* name;
  int32_t kind;  /* ws_module_kind */
  int32_t ndims;
  int64_t shape[WS_MAX_DIMS];
  int32_t layer; /* owning pipeline layer (manifest.hpp:28) */
} ws_param;

typedef enum ws_train_scheme {
  WS_TRAIN_TP = 0,  /* TrainConfig{tp,pp,dp} dealt by plan_pushes (plan.cpp:8-21) */
  WS_TRAIN_FSDP = 1 /* every parameter split along dim 0 over all ranks */
} ws_train_scheme;

typedef struct ws_train_layout {
  int32_t scheme;
  int32_t tp, pp, dp;
} ws_train_layout;

/* Which serving rank each GPU of the world hosts (trainer rank g and one
 * serving rank share GPU g). */
typedef enum ws_placement {
  WS_PLACE_RANK = 0,    /* serving rank g on GPU g (the reference's numbering) */
  WS_PLACE_OVERLAP = 1  /* serving ranks assigned to GPUs so that the elements each
                           GPU's trainer shards route to its own serving shards are
                           maximal in sum: fewest bytes over NVLink (FSDP-N -> TP2 x
                           N/2 puts coordinate 0 on GPUs 0..N/2-1) */
} ws_placement;

/* ServeConfig{tp,pp} (plan.hpp:17-21) times `replicas` identical copies.
 * Serving rank of (replica r, stage s, tp rank k) is r*tp*pp + s*tp + k.
 * WS_EXPERT parameters are split along dim 0 over the tp ranks (EP = TP
 * for experts, e.g. tp 8 gives EP8).  `placement` (ws_placement; 0 when
 * zero-initialised) maps serving ranks to GPUs. */
typedef struct ws_serve_layout {
  int32_t tp, pp, replicas;
  int32_t placement;
} ws_serve_layout;

typedef struct ws_plan ws_plan;

/* Builds the static plan of rank `rank` of `world` GPUs: which trainer
 * shards it encodes (plan_pushes), which serving shards it holds
 * (ServeState::init, engine.cpp:34-49), and the route from every trainer
 * shard to every serving shard that intersects it (plan_pulls,
 * plan.cpp:89-121, extended with box intersection across dims).
 * world == 1 with a multi-rank layout is a one-GPU plan of that layout: the
 * one GPU encodes every trainer rank's shards and holds every serving
 * coordinate's shards (one replica), all routes local -- the whole
 * TransferEngine::sync_step of engine.cpp:66-254 on one device.  Errors:
 * WS_INDIVISIBLE_SHAPE, WS_UNKNOWN_MODULE_KIND, WS_INCOMPLETE_COVERAGE,
 * WS_INVALID_ARGUMENT (world != layout sizes). */
ws_status ws_plan_create(const ws_param* params, int nparams, ws_dtype dtype,
                         const ws_train_layout* train,
                         const ws_serve_layout* serve, int world, int rank,
                         ws_plan** out);
void ws_plan_destroy(ws_plan* plan);

typedef struct ws_plan_info {
  int32_t num_segments;       /* trainer shards encoded on this rank */
  int32_t num_serve_shards;   /* serving shards resident on this rank */
  int32_t num_routes;         /* (segment, serving coordinate) pairs */
  int32_t serve_coord;        /* this rank's serving coordinate; -1 if none, or all of
                                 them (one-GPU plan of a multi-rank layout) */
  uint64_t train_arena_elems; /* prev/next arena sizes (elements) */
  uint64_t serve_arena_elems;
  uint64_t train_elems;       /* sum of segment sizes (dense-equivalent) */
  uint64_t model_elems;       /* whole model */
  int32_t serve_rank;         /* serving rank hosted on this GPU (replica * tp * pp +
                                 serve_coord; -1 when serve_coord is -1) */
  int32_t serve_replica;      /* its replica index, or -1 */
} ws_plan_info;
ws_status ws_plan_get_info(const ws_plan* plan, ws_plan_info* info);

/* Segment i of this rank: parameter index, shard descriptor, offset in the
 * trainer arena, element count. */
ws_status ws_plan_segment(const ws_plan* plan, int i, int32_t* param,
                          ws_shard* desc, uint64_t* offset, uint64_t* n);
/* Serving shard i of this rank. */
ws_status ws_plan_serve_shard(const ws_plan* plan, int i, int32_t* param,
                              ws_shard* desc, uint64_t* offset, uint64_t* n);
/* Serving coordinate (stage * tp + tp rank, plan.hpp:44) of serving shard i. */
ws_status ws_plan_serve_shard_coord(const ws_plan* plan, int i, int32_t* coord);

/* The ShardDescriptor fields of segment i that its bucket keys carry
 * (BucketKey::for_shard, key.hpp:55-67). */
ws_status ws_plan_segment_key_fields(const ws_plan* plan, int i, int32_t* tp_rank,
                                     int32_t* tp_size, int32_t* pp_stage);

/* Checks, on the host, the peer-memory exchange layouts every rank of this
 * plan would build with `rounds` exchange rounds (entries, rounds,
 * destinations vs expectations, mailbox size): WS_OK when consistent. */
ws_status ws_plan_check_exchange(const ws_plan* plan, int rounds);

/* Exchange rounds an engine of this plan uses (K1 overlapped with the
 * exchange when the layout's exchange is heavy: 3 when some rank stores at
 * least half an element into peers per element it encodes, else 1;
 * WSYNC_ROUNDS overrides). */
ws_status ws_plan_exchange_rounds(const ws_plan* plan, int32_t* rounds);

/* Route i: source segment, destination serving coordinate, number of
 * destination ranks (replicas of that coordinate) and the elements of the
 * box intersection. */
ws_status ws_plan_route(const ws_plan* plan, int i, int32_t* segment,
                        int32_t* coord, int32_t* num_dst_ranks,
                        uint64_t* overlap_elems);

/* Worst-case exchange sizes of this rank in records: what it may send to
 * each serving coordinate (tp*pp entries) and receive from each rank (world
 * entries).  The engine allocates its NVLink buffers from these. */
ws_status ws_plan_exchange_caps(const ws_plan* plan, uint64_t* send_cap_per_coord,
                                uint64_t* recv_cap_per_rank);

/* ------------------------------------------------------------------------ */
/* Engine: one weight sync (TransferEngine::sync_step, engine.cpp:66-254)     */
/* ------------------------------------------------------------------------ */

typedef struct ws_engine ws_engine;

typedef struct ws_sync_options { /* SyncOptions, engine.hpp:18-32 */
  int32_t sparse;           /* sparse deltas with dense fallback (default 1) */
  double density_threshold; /* inclusive, default 0.20 (engine.cpp:121) */
  int32_t reverse;          /* 1: sync next -> prev (swap snapshot roles) */
} ws_sync_options;

typedef struct ws_report { /* TransferReport, engine.hpp:34-42 */
  double wall_s;    /* device time from encode launch to last apply */
  double encode_s;  /* K1 */
  double route_s;   /* pack + exchange */
  double apply_s;   /* K4 (sparse scatter + dense copies) */
  uint64_t pushed_bytes;  /* record/dense bytes leaving this rank */
  uint64_t pulled_bytes;  /* record/dense bytes arriving at this rank */
  uint64_t nnz;           /* changed elements found on this rank */
  int32_t dense_shards, sparse_shards;
  uint32_t kernel_launches; /* kernels launched by this sync */
  int32_t streamed_apply;   /* K1 ran its streamed-apply instantiation */
} ws_report;

/* unique_id: 128-byte NCCL unique id (ws_nccl_unique_id on rank 0, then
 * broadcast by the caller), NULL when world == 1. */
ws_status ws_nccl_unique_id(uint8_t out[128]);
ws_status ws_engine_create(const ws_plan* plan, int device,
                           const uint8_t* unique_id, ws_engine** out);
void ws_engine_destroy(ws_engine* eng);

/* Binds the caller-owned device arenas (sizes from ws_plan_info). */
ws_status ws_engine_bind(ws_engine* eng, void* train_prev_dev,
                         void* train_next_dev, void* serve_dev);

/* Fills this rank's bound trainer arenas with the synthetic pair and its
 * serving arena with the matching `prev` values (ServeState::init). */
ws_status ws_engine_generate(ws_engine* eng, uint64_t seed, double density,
                             ws_stream_t stream);

/* Same, with the change density of every EXPERT-kind tensor skewed per
 * expert (ws_expert_thresholds(E, density, zipf_s, perm_seed)). */
ws_status ws_engine_generate_skewed(ws_engine* eng, uint64_t seed, double density,
                                   double zipf_s, uint64_t perm_seed, ws_stream_t stream);

/* One sync on `stream`.  When report is non-null the call synchronises and
 * fills it; otherwise it only enqueues (graph-capturable when world == 1). */
ws_status ws_engine_sync_step(ws_engine* eng, const ws_sync_options* opts,
                              ws_stream_t stream, ws_report* report);

/* A relay (relay.hpp:27-35) seen through C callbacks: the binding of the
 * reference's Relay / RelayFactory.  get_any returns the
 * length of the payload of the first of the n keys present (its index in
 * *hit), copying it to out when it fits in cap (call again with a larger
 * buffer otherwise); -1 = RelayTimeout, other negatives = errors. */
typedef struct ws_relay {
  void* ctx;
  int (*put)(void* ctx, const char* key, uint64_t key_len, const uint8_t* data,
             uint64_t len);
  int64_t (*get_any)(void* ctx, const char* const* keys, const uint64_t* key_lens, int n,
                     int timeout_ms, int* hit, uint8_t* out, uint64_t cap);
  /* Optional framed transport (both or neither; NULL: put/get_any above).
   * Every bucket then travels as the reference's bucket frame
   * [key_len u32][key][len u32][bucket][crc32 u32] (wire.cpp:35-47), built
   * and CRC-32'd on the GPU -- e.g. written as is after the PUT op byte of
   * the reference's TCP relay (tcp_relay.hpp:10-17).  put_frame returns 0,
   * or 3 when the receiver's CRC check failed (IntegrityError).
   * get_any_frame returns the length of the whole frame of the first key
   * present (copied to out when it fits in cap), -1 on timeout; the engine
   * checks its key and CRC on the GPU (IntegrityError on mismatch). */
  int (*put_frame)(void* ctx, const uint8_t* frame, uint64_t len);
  int64_t (*get_any_frame)(void* ctx, const char* const* keys, const uint64_t* key_lens, int n,
                           int timeout_ms, int* hit, uint8_t* out, uint64_t cap);
} ws_relay;

typedef struct ws_relay_options {
  uint64_t bucket_bytes;       /* SyncOptions::bucket_bytes (64 MiB) */
  uint64_t pull_batch_bytes;   /* SyncOptions::pull_batch_bytes */
  double push_bytes_per_s;     /* TokenBucket pacing per direction, 0 = unlimited */
  double pull_bytes_per_s;
  double burst_bytes;
  int32_t timeout_ms;          /* SyncOptions::relay_timeout_ms */
  int32_t async;               /* SyncMode::Async (1) or Batch (0) */
  int32_t force_wide_index;
  int32_t staging_buffers;     /* pinned staging depth per direction (>= 2) */
} ws_relay_options;

typedef struct ws_relay_report { /* TransferReport (engine.hpp:34-42) */
  double wall_s, push_s, pull_s, encode_s, apply_s;
  uint64_t pushed_bytes, pulled_bytes, push_buckets, pull_buckets;
  uint32_t dense_shards, sparse_shards;
} ws_relay_report;

/* TransferEngine::sync_step across clusters (engine.cpp:66-254), one call
 * per rank: this rank's pusher encodes on the GPU (K1 + payloads) and puts
 * its trainer shards' buckets (BucketKey keys, bucket_bytes) through pinned
 * double-buffered staging; its puller (one per serving rank, as
 * engine.cpp:233-238) fetches the buckets of every trainer shard of any rank
 * routed to its serving coordinate (plan_pulls; codec probed from the first
 * key as engine.cpp:164-171), stages them to the GPU, decodes, reslices and
 * applies there.  Async runs both sides concurrently, Batch pushes first.
 * With world > 1 every rank calls it for the same step on a relay the ranks
 * share; the NVLink exchange is not used. */
ws_status ws_engine_sync_relay(ws_engine* eng, uint64_t step, const ws_sync_options* opts,
                               const ws_relay_options* relay_opts, const ws_relay* relay,
                               ws_relay_report* report);

/* Frees what ws_engine_sync_relay keeps across calls (device and pinned
 * staging at the dense bound of the largest shard, the decode scratch pool);
 * the next relay sync allocates it again. */
ws_status ws_engine_release_staging(ws_engine* eng);

/* Segment i's payload from the last sync in the reference wire format
 * (sparse if it was sent sparse, else the dense `next` snapshot), written to
 * out_dev when non-null (8-byte aligned, info->total_bytes long).
 * force_wide_index: 8-byte indices (engine.cpp:122).  Synchronises. */
ws_status ws_engine_payload(ws_engine* eng, int i, int force_wide_index, void* out_dev,
                            ws_payload_info* info, ws_stream_t stream);

/* Same, with the new snapshot read from HOST memory (pinned for full
 * speed): copies it into the trainer arena that becomes `next` for this
 * step, syncs, and copies the per-segment change counts back to the host
 * (nnz_host, num_segments entries, may be NULL). */
ws_status ws_engine_sync_step_host(ws_engine* eng, const void* next_host,
                                   const ws_sync_options* opts,
                                   ws_stream_t stream, uint64_t* nnz_host,
                                   ws_report* report);

/* ------------------------------------------------------------------------ */
/* Process-local rank groups                                                  */
/* ------------------------------------------------------------------------ */

/* All `world` ranks of a layout as engines of ONE process on one GPU: the
 * ranks share mailboxes, receive regions and serving arenas as plain device
 * pointers instead of CUDA IPC, and a group sync runs every rank's kernels
 * (K1, local route, pack_kernel, apply_p2p_kernel -- the multi-GPU data path)
 * interleaved on one stream.  Used to run any multi-rank layout of the
 * reference (TrainConfig{tp,pp,dp} -> ServeConfig{tp,pp}, engine.cpp:66-254)
 * on a single device.  Order: ws_group_create; per rank
 * ws_engine_create_grouped + ws_engine_bind; ws_group_connect; then
 * ws_group_sync_step (ws_engine_sync_step refuses grouped engines).  Destroy
 * the engines before the group. */
typedef struct ws_group ws_group;
ws_status ws_group_create(int world, ws_group** out);
void ws_group_destroy(ws_group* group);
ws_status ws_engine_create_grouped(const ws_plan* plan, int device, ws_group* group,
                                   ws_engine** out);
ws_status ws_group_connect(ws_group* group);
/* One sync of every rank; reports: NULL or `world` entries (synchronises). */
ws_status ws_group_sync_step(ws_group* group, const ws_sync_options* opts, ws_stream_t stream,
                             ws_report* reports);

/* Device-time totals of the syncs since the last reset (the most recent 256
 * at most), summed from CUDA events recorded on each sync's stream -- so a
 * timed loop needs no per-step synchronisation.  Synchronises the engine's
 * last stream.  reset != 0 clears the totals after reading. */
typedef struct ws_timing {
  uint32_t steps;
  uint32_t kernel_launches; /* libwsync kernels launched by those syncs */
  double wall_s, encode_s, route_s, apply_s;
  /* the pack (NVLink stores) part of route_s, summed over the last
   * pack_steps syncs (single-round P2P exchange; 0 otherwise) */
  uint32_t pack_steps;
  double pack_s;
} ws_timing;
ws_status ws_engine_timing(ws_engine* eng, int reset, ws_timing* out);

/* NVLink traffic of the last sync on this rank (bytes): wire records stored
 * into the replicas' receive regions (one copy per replica), dense-fallback
 * boxes stored straight into their serving arenas, and the records other
 * ranks published into this rank's regions.  NCCL-fallback exchange: bytes
 * sent / received.  Zero at world 1.  Synchronises. */
ws_status ws_engine_exchange_bytes(ws_engine* eng, uint64_t* sent_record_bytes,
                                   uint64_t* sent_dense_bytes, uint64_t* recv_record_bytes);

/* Every segment's change count and codec ('S' sparse, 'D' dense) from the
 * last sync (num_segments entries each; either may be NULL).  Synchronises. */
ws_status ws_engine_segment_counts(ws_engine* eng, uint64_t* nnz, char* codec);

/* Segment i's delta stream from the last sync: device pointers into the
 * engine's record buffer, its record count (host, needs a synchronised
 * stream) and the codec chosen ('S' sparse, 'D' dense). */
ws_status ws_engine_segment_delta(ws_engine* eng, int i, const uint32_t** idx,
                                  const void** val, uint64_t* nnz, char* codec);

/* Segment i's record stream as K1 wrote it in the last sync (engine mode,
 * before any compaction): one run per super-tile of `*tile_elems` elements,
 * the runs in reservation order, ascending inside each; `*nrec` records
 * (min(count, capacity); 0 when the segment went dense).  Device pointers
 * into the engine's record buffer.  Synchronises. */
ws_status ws_engine_segment_stream(ws_engine* eng, int i, const uint32_t** idx,
                                   const void** val, uint64_t* nrec, uint64_t* tile_elems);

#ifdef __cplusplus
}
#endif
#endif /* WSYNC_H */
