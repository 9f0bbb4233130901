// route.h -- serving-side route tables shared by the engine and its kernels.
#pragma once

#include "kernels.h"

namespace wsync {

constexpr uint32_t kTilesPerUnit = 8;    // super-tiles of records per work unit (one per warp)
// A sparse segment with more than 1/kStreamDiv of its elements changed is
// cheaper to apply by streaming serve += next - prev over its box (8 B per
// element) than by scattered read-modify-writes (~100 B of DRAM per record, and
// partial-sector writes);
// the same bound decides whether K1 fuses the apply.
constexpr uint64_t kStreamDiv = 10;  // measured: fused RMW wins at 10%, streaming at 20%
constexpr uint64_t kCopyChunk = 65536;   // elements per dense-copy work unit

// SyncOptions::density_threshold's default (engine.hpp:27): what the P2P
// receive regions are sized for until a sync asks for more.
constexpr double kDefaultThreshold = 0.20;

// The largest record count k of an n-element shard with k / n <= t: one more
// change makes the shard dense (engine.cpp:121, inclusive).  This is a
// segment's record capacity, and the most records a sparse shard can send.
inline uint64_t sparse_capacity(uint64_t n, double t) {
  if (!n || !(t > 0.0)) return 0;
  if (t >= 1.0) return n;
  uint64_t c = (uint64_t)(t * (double)n);
  if (c > n) c = n;
  while (c < n && (double)(c + 1) / (double)n <= t) ++c;
  while (c > 0 && (double)c / (double)n > t) --c;
  return c;
}

// One (trainer segment -> serving shard) route whose destination is resident
// on this GPU.  Sparse records map through `identity` (flat shift with a keep
// window, the same-dim dim-0 case) or the general box `map`; dense segments
// copy `box` from the trainer `next` arena into the serving arena.
struct LocalEntry {
  int32_t seg;
  int32_t identity;
  int32_t coord;              // destination serving coordinate (pack region)
  int32_t fused_ok;           // the segment's only local route: K1 may apply it (fuse_on)
  uint32_t keep_lo, keep_hi;  // identity: keep src-local i in [keep_lo, keep_hi)
  int64_t shift;              // identity: dst-local = i + shift
  uint64_t dst_base;          // serving shard offset (elements)
  Remap map;
  BoxCopyArgs box;            // src/dst bases relative to the segment / shard
};

struct RouteSideArgs {
  const LocalEntry* entries;
  int32_t nentries;
  int32_t sparse;               // 0: every segment dense (SyncOptions::sparse)
  int32_t fused;                // 1: K1 applied the sparse records of segments with fuse_on set
  uint32_t* fuse_on;            // per segment; re-decided here for the next sync from this one
  const uint64_t* seg_nnz;
  const uint64_t* seg_cap;
  const uint64_t* seg_rec;
  const uint64_t* seg_base;     // segment offsets in the trainer arena
  const uint32_t* rec_idx;
  const void* rec_val;
  // K1's unordered record layout: super-tile t of a segment holds records
  // [tile_base[t], tile_base[t] + tile_cnt[t]) of the segment's region.
  const uint32_t* tile0;        // nseg + 1: first global super-tile of every segment
  const uint32_t* tile_cnt;
  const uint32_t* tile_base;
  uint32_t tile_elems;          // elements per super-tile
  const SegDev* segs;           // segment sizes
  int32_t stream_apply;         // local routes: dense-ish sparse segments apply by streaming
  uint32_t sa_div;              // K1 streamed apply: fuse_on = 2 for density in [1/sa_div, cap] (0: off)
  uint64_t* sa_elems;           // mapped host words: fused elements set to stream / to per-record RMW
  int32_t k1_emitted;           // pack: K1 already stored the sparse records remotely
  const void* train_prev;
  const void* train_next;
  void* serve;
  uint64_t* unit_off;           // nentries + 1
};

// Work list + fused reslice/apply/dense-copy for the local routes.
cudaError_t launch_local_route(int dtype, const RouteSideArgs& a, int grid, cudaStream_t s);

// Wire records of the NCCL-fallback exchange: self-describing (serving-arena
// index, value), so a receiver needs no route table and arrival order does
// not matter.  bf16: one u64 = set:1 | index:47 | value:16.  4-byte dtypes:
// {u64 set:1 | index:63, u32 value, u32 pad}.  "set" records carry dense-
// fallback values (overwrite, copy_overlap semantics); the others are deltas.
constexpr uint64_t kWireSet = 1ull << 63;
inline size_t wire_bytes(int dtype) { return dtype == WS_BF16 ? 8 : 16; }

// Records of the peer-memory exchange: every receive region belongs to one
// (source, route), so a record carries only its index local to the
// destination shard (u32: a shard has < 2^32 elements) and its value, as two
// arrays -- u32 idx[cap] | value[cap] -- 6 bytes per bf16 record, the
// algorithmic 4 + 2 of SURVEY §8(d).  The receiver adds the route's shard
// offset.  A region whose source segment went dense without direct box
// stores carries "set" records: its published count has bit 31 set.
inline size_t p2p_record_bytes(int dtype) { return 4 + (dtype == WS_BF16 ? 2 : 4); }
inline uint64_t p2p_region_bytes(int dtype, uint64_t cap) {
  return (cap * p2p_record_bytes(dtype) + 15) / 16 * 16;  // next region 16-byte aligned
}
constexpr uint32_t kCountSet = 0x80000000u;

// Packs the records of the routes to other GPUs into one region per serving
// coordinate (warp-aggregated atomic reservation; order inside a region is
// irrelevant).  Sparse segments are re-indexed (reslice) into the
// destination shard; dense-fallback segments emit set records for the box
// overlap.
constexpr int kMaxWorld = 8;      // GPUs of one box
constexpr int kMaxReplicas = 8;

// Mailbox words (u64, in every rank's own HBM, written by its peers) for a
// world of W ranks and R exchange rounds per sync:
//   [0, W)                      ready[g]: rank g reached step e (posted at the sync's start)
//   per round r, b = W + r(2W+2):
//     [b, b+W)                  flag[g]: source g published round r of step e
//     [b+W, b+2W)               ack[g]: destination g applied round r of step e
//     b+2W, b+2W+1              pack / apply blocks done (last-block detection)
// Round r of step e carries epoch R*e + r; ready[g] = R*e + R - 1.
constexpr int kMaxRounds = 4;
__host__ __device__ inline size_t mb_ready(int, int g) { return (size_t)g; }
__host__ __device__ inline size_t mb_flag(int W, int r, int g) { return (size_t)(W + r * (2 * W + 2) + g); }
__host__ __device__ inline size_t mb_ack(int W, int r, int g) { return (size_t)(W + r * (2 * W + 2) + W + g); }
__host__ __device__ inline size_t mb_pack_ctr(int W, int r) { return (size_t)(W + r * (2 * W + 2) + 2 * W); }
__host__ __device__ inline size_t mb_apply_ctr(int W, int r) { return mb_pack_ctr(W, r) + 1; }

// Peer-memory (P2P) exchange state shared by the pack and apply kernels.
// Mailbox of every rank (u64 words, in its own HBM, mapped by all peers):
//   [0, W) records sent by rank s this step   [W, 2W) step flag from s
//   [2W, 3W) ack of rank g for our last data   [3W] pack blocks done
//   [3W + 1] apply blocks done                 [4W, 5W) rank g reached step e
// The "reached" flag orders direct dense stores after everything the
// receiver's own stream did to its serving arena before the sync.
struct P2PArgs {
  int32_t on;                       // 0: NCCL mode (send region + host exchange)
  int32_t debug;                    // perf experiments (WSYNC_P2P_DEBUG): 1 no scatter, 2 no records
  int32_t world, rank;
  int32_t round;                    // exchange round of this launch (< kMaxRounds)
  uint32_t epoch;                   // R * step + round, equal on every rank
  uint32_t prev_epoch;              // the same round's epoch of the previous step (0: none)
  unsigned long long* mailbox;                        // local
  unsigned long long* peer_mailbox[kMaxWorld];        // mapped peers' mailboxes
  int32_t dest_rank[kMaxWorld][kMaxReplicas];         // -1 terminated
  // Dense-fallback boxes bypass the records: with dense_direct the pack
  // kernel copies them straight into every replica's (IPC-mapped) serving
  // arena, 2 bytes per bf16 element over NVLink instead of an 8-byte record.
  int32_t dense_direct;
  void* serve_dst[kMaxWorld][kMaxReplicas];           // per coordinate: replica serving arenas
  // sender side: one record region per (remote entry, replica) at the
  // replica, filled through per-entry counters; counts published at the end
  const struct EntryDest* edest;                      // per remote entry
  unsigned int* ent_cnt;                              // per remote entry, zeroed each step
  // receiver side: one region per (source, entry) that sends here
  const void* recv;                                   // local record area
  const struct RecvEntry* rentries;
  int32_t nrecv;
  const uint32_t* recv_cnt;                           // local count slots (written by the sources)
  uint64_t* recv_units;                               // nrecv + 1: apply units, prefix
  uint32_t expect_mask;                               // sources that send to this rank
  uint32_t* err;                                      // WS_ERRBIT_* (timeouts, capacity)
};

// Where one remote entry's records go at each replica of its coordinate.
struct EntryDest {
  void* rec[kMaxReplicas];      // record region at replica r (null-terminated)
  uint32_t* cnt[kMaxReplicas];  // its count slot at replica r
  uint64_t cap;                 // region capacity, records
};
// A region of this rank's receive area: `count` records (the source's
// published count) in the SoA layout of p2p_record_bytes at byte `off`.
struct RecvEntry {
  uint64_t off;                 // bytes from the start of the receive area
  uint64_t cap;                 // region capacity, records (the value array follows idx[cap])
  uint64_t dst_base;            // the destination shard's offset in the serving arena
  uint32_t cnt_idx;
  uint32_t src;
};
constexpr uint32_t kErrBitTimeout = 0x4u;
constexpr size_t kMailboxBytes = 4096;

struct PackArgs {
  RouteSideArgs r;                  // entries = the remote routes
  void* send;                       // NCCL mode: local send regions
  const uint64_t* region_off;       // per coordinate, in records (NCCL mode)
  const uint64_t* region_cap;       // per coordinate capacity (at the destination in P2P mode)
  unsigned long long* region_cnt;   // per coordinate, zeroed before the launch
  uint32_t* err;                    // WS_ERRBIT_CAPACITY on overflow
  P2PArgs p2p;
};
cudaError_t launch_pack(int dtype, const PackArgs& a, int grid, cudaStream_t s);

// Receiver side: applies nrec wire records to the serving arena in place.
cudaError_t launch_apply_wire(int dtype, const void* recv, uint64_t nrec, void* serve,
                             cudaStream_t s);

// P2P receiver, first thing in a sync: tells every source it may store into
// this rank's serving arena for step p.epoch.
cudaError_t launch_p2p_ready(const P2PArgs& p, cudaStream_t s);

// P2P receiver: waits for every expected source's step flag, applies the
// records of every (source, entry) region (its published count), acks.
cudaError_t launch_apply_p2p(int dtype, const P2PArgs& p, void* serve, int grid, cudaStream_t s);

// Fills a LocalEntry for the route src -> dst of a tensor of `full`.
LocalEntry make_local_entry(int dtype, const int64_t* full, int nd, int seg, const ws_shard& src,
                            const ws_shard& dst, uint64_t dst_base);

}  // namespace wsync
