// plan.h -- host control plane of one weight sync: shard geometry, push
// dealing and the trainer-shard -> serving-shard route (shard.hpp, plan.hpp).
#pragma once

#include <stdint.h>

#include <optional>
#include <string>
#include <vector>

#include "wsync.h"

namespace wsync {

struct PlanError {
  ws_status status;
  std::string msg;
};

struct ParamMeta {  // manifest.hpp:23-29
  std::string name;
  int kind = WS_REPLICATED;
  std::vector<int64_t> shape;
  int layer = 0;
};

struct ShardDesc {  // ShardDescriptor, shard.hpp:32-45 (+ owning param index)
  int param = -1;
  int tp_rank = 0, tp_size = 1, pp_stage = 0;
  ws_shard d{-1, 0, 0};
};

// shard.cpp:8-18 (+ WS_EXPERT -> dim 0).  Throws PlanError.
std::optional<int> tp_shard_dim(int kind);
// shard.cpp:20-30
std::pair<int64_t, int64_t> slice_range(int64_t extent, int rank, int size);
// shard.cpp:32-50
int pp_stage_of(int layer, int num_layers, int pp);
std::pair<int, int> pp_stage_layer_range(int stage, int num_layers, int pp);
// shard.cpp:52-79
std::vector<ShardDesc> param_shards(const std::vector<ParamMeta>& m, int p, int tp, int pp,
                                    int num_layers);
int manifest_num_layers(const std::vector<ParamMeta>& m);  // manifest.cpp:41-45
uint64_t shard_numel(const ParamMeta& p, const ws_shard& d);
uint64_t overlap_numel(const ParamMeta& p, const ws_shard& a, const ws_shard& b);

struct Segment {        // a trainer shard encoded on this rank
  ShardDesc shard;
  uint64_t offset = 0;  // element offset in the trainer arenas
  uint64_t n = 0;
};

struct ServeShard {     // a serving shard resident on this rank
  ShardDesc shard;
  uint64_t offset = 0;  // element offset in the serving arena
  uint64_t n = 0;
};

struct Route {          // trainer segment -> serving coordinate
  int seg = -1;         // index into segments (of the source rank)
  int coord = -1;       // serving coordinate (stage * tp + tp_rank)
  ShardDesc dst;        // the serving shard at that coordinate
  uint64_t dst_offset = 0;  // its offset in that coordinate's serving arena
  uint64_t overlap = 0;     // elements of the box intersection
};

class Plan {
 public:
  Plan(std::vector<ParamMeta> manifest, int dtype, const ws_train_layout& train,
       const ws_serve_layout& serve, int world, int rank);

  const std::vector<ParamMeta>& manifest() const { return manifest_; }
  int dtype() const { return dtype_; }
  int world() const { return world_; }
  int rank() const { return rank_; }
  int coords() const { return serve_.tp * serve_.pp; }
  int replicas() const { return serve_.replicas; }
  int coord_of_rank(int r) const;            // -1 when rank r holds no serving shard
  // serving rank (replica * coords + coord) hosted on GPU r (ws_placement)
  int serve_rank_of(int r) const { return collapsed_ || r < 0 || r >= world_ ? -1 : serve_rank_[r]; }
  // One GPU hosts every rank of a multi-rank layout (world 1 with trainer
  // ranks or serving coordinates > 1): all logical trainer ranks' shards are
  // its segments, all coordinates' serving shards its serving arena, and
  // every route is local.
  bool collapsed() const { return collapsed_; }
  bool route_is_local(const Route& r) const { return collapsed_ || r.coord == my_coord(); }

  // This rank's view.
  const std::vector<Segment>& segments() const { return segments_[rank_]; }
  const std::vector<ServeShard>& serve_shards() const {
    return collapsed_ ? serve_all_ : serve_by_coord_[my_coord()];
  }
  // serving coordinate of serve_shards()[i]
  int serve_shard_coord(int i) const { return collapsed_ ? serve_all_coord_[i] : my_coord(); }
  const std::vector<Route>& routes() const { return routes_[rank_]; }
  int my_coord() const { return collapsed_ ? -1 : coord_of_rank(rank_); }
  uint64_t train_arena_elems() const { return train_arena_[rank_]; }
  uint64_t serve_arena_elems() const;

  // Any rank's view (the route is static: every rank computes all of it).
  const std::vector<Segment>& segments_of(int r) const { return segments_[r]; }
  const std::vector<Route>& routes_of(int r) const { return routes_[r]; }
  const std::vector<ServeShard>& serve_of_coord(int c) const { return serve_by_coord_[c]; }
  uint64_t model_elems() const { return model_elems_; }
  uint64_t train_elems() const;

 private:
  std::vector<ParamMeta> manifest_;
  int dtype_;
  ws_train_layout train_;
  ws_serve_layout serve_;
  int world_, rank_;
  bool collapsed_ = false;
  std::vector<ServeShard> serve_all_;      // collapsed: every coordinate's shards
  std::vector<int> serve_all_coord_;
  uint64_t serve_all_elems_ = 0;
  uint64_t model_elems_ = 0;
  std::vector<std::vector<Segment>> segments_;        // per rank
  std::vector<uint64_t> train_arena_;                 // per rank
  std::vector<std::vector<ServeShard>> serve_by_coord_;
  std::vector<uint64_t> serve_arena_by_coord_;
  std::vector<std::vector<Route>> routes_;            // per source rank
  std::vector<int> serve_rank_;                       // per GPU: hosted serving rank

  void place();
};

// Minimum-cost perfect assignment of n rows to n columns (cost row-major,
// n x n): col[row].  O(n^3) shortest augmenting paths with potentials.
std::vector<int> assign_min_cost(const std::vector<int64_t>& cost, int n);

constexpr uint64_t kArenaAlign = 64;  // elements; keeps 16-B vectors aligned for every dtype

// Static exchange sizes of rank `me` in records (worst case: every routed
// element sent): send capacity per serving coordinate, receive capacity
// from every rank.  Defined in exchange.cu.
void exchange_caps(const Plan& plan, int me, std::vector<uint64_t>* send_cap,
                   std::vector<uint64_t>* recv_cap);

}  // namespace wsync
