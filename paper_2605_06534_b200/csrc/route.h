// route.h -- serving-side route tables shared by the engine and its kernels.
#pragma once

#include "kernels.h"

namespace wsync {

constexpr uint64_t kApplyChunk = 8192;   // records per apply work unit
constexpr uint64_t kCopyChunk = 65536;   // elements per dense-copy work unit

// One (trainer segment -> serving shard) route whose destination is resident
// on this GPU.  Sparse records map through `identity` (flat shift with a keep
// window, the same-dim dim-0 case) or the general box `map`; dense segments
// copy `box` from the trainer `next` arena into the serving arena.
struct LocalEntry {
  int32_t seg;
  int32_t identity;
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
  const uint64_t* seg_nnz;
  const uint64_t* seg_cap;
  const uint64_t* seg_rec;
  const uint64_t* seg_base;     // segment offsets in the trainer arena
  const uint32_t* rec_idx;
  const void* rec_val;
  const void* train_next;
  void* serve;
  uint64_t* unit_off;           // nentries + 1
};

// Work list + fused reslice/apply/dense-copy for the local routes.
cudaError_t launch_local_route(int dtype, const RouteSideArgs& a, int grid, cudaStream_t s);

// Fills a LocalEntry for the route src -> dst of a tensor of `full`.
LocalEntry make_local_entry(int dtype, const int64_t* full, int nd, int seg, const ws_shard& src,
                            const ws_shard& dst, uint64_t dst_base);

}  // namespace wsync
