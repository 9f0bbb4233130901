// kernels.h -- host-side launch interface of the libwsync device kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace wsync {

#ifndef WS_ENC_SUBTILES
#define WS_ENC_SUBTILES 4
#endif
#ifndef WS_ENC_RING
#define WS_ENC_RING 4
#endif
#ifndef WS_ENC_CONSUMERS
#define WS_ENC_CONSUMERS 512
#endif
#ifndef WS_ENC_BUFFERS
#define WS_ENC_BUFFERS 2
#endif
#ifndef WS_ENC_CAPDIV
#define WS_ENC_CAPDIV 16  // staged records per super-tile buffer: 3/CAPDIV of its elements
#endif
constexpr int kEncodeThreads = 256;                 // block size of the small codec kernels
constexpr int kEncodeVPT = 4;                       // their vectors per thread
constexpr int kEncConsumers = WS_ENC_CONSUMERS;     // K1 consumer threads (16 warps)
constexpr int kEncBuffers = WS_ENC_BUFFERS;         // record staging buffers (one resolver each)
constexpr int kEncodeBlock = kEncConsumers + 32 + kEncBuffers * 32;  // + producer + resolvers
constexpr int kEncodeSubTiles = WS_ENC_SUBTILES;    // sub-tiles (ring stages) per super-tile
constexpr int kRing = WS_ENC_RING;                  // shared-memory ring stages
constexpr uint32_t kStageBytes = 16384;             // per array per stage

// Elements per encode super-tile: 32768 for bf16, 16384 for 4-byte dtypes
// (64 KB of prev plus 64 KB of next).
inline uint32_t encode_tile_elems(int dtype) {
  return kStageBytes / (dtype == WS_BF16 ? 2 : 4) * kEncodeSubTiles;
}
inline uint32_t elems_per_vec(int dtype) { return dtype == WS_BF16 ? 8 : 4; }
inline int dtype_size(int dtype) { return dtype == WS_BF16 ? 2 : 4; }

// One encode segment: a trainer shard at `base` (elements, multiple of the
// vector width) in the prev/next arenas, its records written at
// [rec, rec + min(nnz, cap)) of the record arrays.
struct SegDev {
  uint64_t base, n, rec, cap;
};

// Fused apply of a segment's records into a serving shard resident on the
// same GPU (K1 writes each record once; applying it at that moment removes
// the separate read of the record stream).  mode 0: none, 1: flat shift with
// a keep window (dim-0 layouts), 2: general box remap.
struct FuseEntry {
  int32_t mode;
  uint32_t keep_lo, keep_hi;
  int64_t shift;
  uint64_t dst_base;
  Remap map;
};

// A route of a segment to another GPU as K1 sees it (engine, P2P, bf16):
// K1's flush re-indexes each record into the destination shard and stores it
// as a wire record straight into every replica's receive region over NVLink,
// so the transfer overlaps the encode tile by tile.
struct RemoteMap {
  int32_t identity;
  uint32_t keep_lo, keep_hi;     // identity: keep segment-local i in [keep_lo, keep_hi)
  int64_t shift;                 // identity: destination-local = i + shift
  uint64_t dst_base;             // destination shard offset in the serving arena
  Remap map;                     // general box re-index
  uint64_t cap;                  // region capacity (records)
  unsigned int* cnt;             // the route's slot counter (zeroed per sync)
  void* rec[8];                  // region at each replica (null-terminated)
};
struct RemoteEmit {
  const RemoteMap* maps;         // grouped by segment
  const uint32_t* seg_first;     // nseg + 1
  const unsigned long long* ack; // this rank's mailbox ack words (per peer)
  uint32_t ack_mask;             // peers whose ack of the previous step must be seen first
  uint32_t epoch;                // this step
};

struct EncodeArgs {
  const void* prev;
  const void* next;
  const SegDev* segs;     // null: the single segment seg0
  SegDev seg0;
  const uint32_t* tile0;  // nseg + 1 prefix of per-segment tile counts (null with seg0)
  const uint32_t* tile_seg;  // optional: segment of every super-tile (skips the search)
  int32_t nseg;
  uint32_t ntiles;
  uint32_t* out_idx;
  void* out_val;
  uint64_t* seg_nnz;
  unsigned long long* status;  // >= ntiles words
  uint32_t epoch;
  unsigned int* ticket;        // zeroed before launch
  uint32_t debug;              // perf experiments only (WSYNC_ENCODE_DEBUG): 1 no look-back, 2 no writes
  const FuseEntry* fuse;       // optional, per segment: apply records to `serve` as they are written
  const uint32_t* fuse_on;     // per segment: fuse this step (device-adapted from the last one)
  void* serve;
  // Unordered mode (the engine): a super-tile reserves its records' place in
  // its segment with one atomic on seg_nnz (zeroed before the launch) instead
  // of the look-back, so no super-tile waits on another.  Records stay
  // ascending inside a super-tile; (tile_base, tile_cnt) locate them, and
  // launch_compact restores the ascending segment stream when one is asked for.
  int32_t unordered;
  uint32_t* tile_cnt;          // per global super-tile
  uint32_t* tile_base;         // per global super-tile: first record in the segment stream
  // Changes past a thread's shared-memory slots go to its warp's region of
  // this scratch (encode_spill_bytes(dtype, spill_blocks)); the grid is
  // clamped to spill_blocks.
  void* spill;
  uint32_t spill_blocks;
  // Count-only super-tiles (engine): segments predicted dense (seg_mode[s]
  // = 1, from the previous sync) are only counted.  A second launch then
  // processes the tiles of those that turned out sparse: tile_list /
  // ntiles_dev give its super-tiles and `fill` (zeroed) their reservations.
  uint32_t tile_offset;           // this launch claims super-tiles [tile_offset, + ntiles)
  uint32_t max_grid;              // 0: one block per SM; else at most this many (SMs left free)
  const uint32_t* seg_mode;
  const uint32_t* tile_list;
  const uint32_t* ntiles_dev;
  unsigned long long* fill;
  RemoteEmit remote;             // maps == null: no fused remote emission
  // Streamed apply (bf16, fused identity routes, fuse_on == 2): the producer
  // also streams the serving sub-tile into a third ring, and consumers store
  // serve + (next - prev) for every changed 16-byte vector -- sequential
  // instead of one scattered read-modify-write per record.
  int32_t serve_stream;
};

// Between the two K1 launches of an engine sync: lists the super-tiles of
// the count-only segments that came out sparse, and sets every segment's
// mode for the next sync (dense now -> count-only next).
cudaError_t launch_fixup_plan(const uint32_t* tile0, int seg_begin, int seg_end,
                              const uint64_t* seg_nnz, const uint64_t* seg_cap, uint32_t* seg_mode,
                              uint32_t* tile_list, uint32_t* ntiles_dev, cudaStream_t s);

constexpr uint32_t kMaxEncodeGrid = 160;  // >= SMs of a B200 (148)
size_t encode_spill_bytes(int dtype, uint32_t blocks);

// Stream-ordered scratch from the library's own caching pool of the current
// device (wire.cu); release with cudaFreeAsync on the same stream.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s);

// Ascending segment stream from an unordered K1 output: the segment's
// super-tiles' records in tile order (API / wire / relay path, not the sync):
// an exclusive scan of the tile counts, then one warp per super-tile copies
// its records to their ascending place.
cudaError_t launch_compact(int dtype, const uint32_t* tile_cnt, const uint32_t* tile_base,
                           uint32_t ntiles, uint64_t cap, const uint32_t* in_idx,
                           const void* in_val, uint32_t* out_idx, void* out_val, cudaStream_t s);

// K1: fused compare + ballot/popc + block scan + decoupled look-back
// compaction over all segments.  Returns the persistent grid used.
cudaError_t launch_encode(int dtype, const EncodeArgs& a, cudaStream_t s, int* grid_out = nullptr);

// Record validation + in-place apply (ws_apply_delta).
cudaError_t launch_apply(int dtype, void* target, uint64_t n, const uint32_t* idx,
                         const void* val, uint64_t nnz, const uint64_t* nnz_dev,
                         uint32_t* err, cudaStream_t s);

// Order-preserving filter + re-index of one record stream (ws_reslice_delta).
struct ResliceArgs {
  Remap map;
  uint64_t src_elems;
  const uint32_t* idx;
  const void* val;
  uint64_t cap_in;            // upper bound on the record count
  const uint64_t* nnz_dev;    // actual count (device) or null
  uint64_t nnz;               // actual count when nnz_dev is null
  uint32_t* out_idx;
  void* out_val;
  uint64_t* out_nnz;
  uint32_t* err;
  unsigned long long* status;
  uint32_t epoch;
  unsigned int* ticket;
};
constexpr uint32_t kResliceTile = 256 * 4;
cudaError_t launch_reslice(int dtype, const ResliceArgs& a, cudaStream_t s);

// Dense box copy: the overlap of two shards of one tensor (copy_overlap).
struct BoxCopyArgs {
  void* dst;
  const void* src;
  uint64_t rows;          // rows of the overlap (product of outer dims)
  uint64_t run;           // contiguous elements per row
  int32_t nd_outer;       // dims enumerated by `rows`
  uint32_t outer_ext[WS_MAX_DIMS];
  uint64_t src_stride[WS_MAX_DIMS], dst_stride[WS_MAX_DIMS];  // elements
  uint64_t src_base, dst_base;                                // elements
  int vec;                // 1: 16-byte vectors are legal for every row
};
cudaError_t launch_box_copy(int dtype, const BoxCopyArgs& a, cudaStream_t s);

// Builds BoxCopyArgs for copying the overlap of `src` into `dst` (both
// shards of full_shape).  Returns the overlap element count (0: none).
uint64_t make_box_copy(int dtype, const int64_t* full, int nd, const ws_shard& dst,
                       const ws_shard& src, BoxCopyArgs* out);

// Synthetic bf16 pair for one shard; also used to initialise serving shards
// (prev only when next == nullptr).
cudaError_t launch_gen_bf16(uint64_t key, const int64_t* full, int nd, const ws_shard& desc,
                            uint64_t change_thr, uint16_t* prev, uint16_t* next, cudaStream_t s,
                            const uint64_t* thr_dim0 = nullptr);
// Per-expert change thresholds (ws_expert_thresholds).
void expert_thresholds(int experts, double density, double zipf_s, uint64_t perm_seed,
                       uint64_t* out);

// Host helpers.
uint64_t param_key(uint64_t seed, const char* name);
Box shard_box(const int64_t* full, int nd, const ws_shard& d);
Remap make_remap(const int64_t* full, int nd, const ws_shard& src, const ws_shard& dst);
int sm_count();

}  // namespace wsync
