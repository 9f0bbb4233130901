// plan.cpp -- shard geometry, push dealing and routes (host control plane).
//
// Restates the reference's shard.cpp:8-79 and plan.cpp:8-121 for the B200
// engine and extends them in two ways: (1) an FSDP trainer layout (every
// parameter split along dim 0 over all ranks), (2) routes are box
// intersections, so a trainer shard sliced along one dim can feed a serving
// shard sliced along another (the reference's cover_slice drops such
// sources and reports IncompleteCoverage, plan.cpp:51-55).
#include "plan.h"

#include <algorithm>
#include <limits>
#include <map>

namespace wsync {

std::optional<int> tp_shard_dim(int kind) {
  switch (kind) {
    case WS_COLUMN_LINEAR: return 0;
    case WS_ROW_LINEAR: return 1;
    case WS_EMBEDDING: return 0;
    case WS_EXPERT: return 0;
    case WS_NORM:
    case WS_REPLICATED: return std::nullopt;
  }
  throw PlanError{WS_UNKNOWN_MODULE_KIND, "unknown module kind ordinal " + std::to_string(kind)};
}

std::pair<int64_t, int64_t> slice_range(int64_t extent, int rank, int size) {
  if (size <= 0 || rank < 0 || rank >= size)
    throw PlanError{WS_TRANSFER_ERROR,
                    "slice_range: rank " + std::to_string(rank) + " of " + std::to_string(size)};
  if (extent % size != 0)
    throw PlanError{WS_INDIVISIBLE_SHAPE, "extent " + std::to_string(extent) +
                                              " not divisible by tp size " + std::to_string(size)};
  const int64_t per = extent / size;
  return {per * rank, per * (rank + 1)};
}

std::pair<int, int> pp_stage_layer_range(int stage, int num_layers, int pp) {
  if (pp <= 0 || stage < 0 || stage >= pp)
    throw PlanError{WS_TRANSFER_ERROR,
                    "pp stage " + std::to_string(stage) + " of " + std::to_string(pp)};
  const int base = num_layers / pp, rem = num_layers % pp;
  const int lo = stage * base + std::min(stage, rem);
  return {lo, lo + base + (stage < rem ? 1 : 0)};
}

int pp_stage_of(int layer, int num_layers, int pp) {
  for (int s = 0; s < pp; ++s) {
    const auto [lo, hi] = pp_stage_layer_range(s, num_layers, pp);
    if (layer >= lo && layer < hi) return s;
  }
  throw PlanError{WS_TRANSFER_ERROR, "layer " + std::to_string(layer) + " outside 0.." +
                                         std::to_string(num_layers - 1)};
}

int manifest_num_layers(const std::vector<ParamMeta>& m) {
  int n = 0;
  for (const auto& p : m) n = std::max(n, p.layer + 1);
  return n;
}

std::vector<ShardDesc> param_shards(const std::vector<ParamMeta>& m, int p, int tp, int pp,
                                    int num_layers) {
  const ParamMeta& meta = m[p];
  const int stage = pp_stage_of(meta.layer, num_layers, pp);
  const auto dim = tp_shard_dim(meta.kind);
  std::vector<ShardDesc> out;
  if (!dim || tp == 1) {
    ShardDesc d;
    d.param = p;
    d.pp_stage = stage;
    out.push_back(d);
    return out;
  }
  if (*dim >= (int)meta.shape.size())
    throw PlanError{WS_SHAPE_MISMATCH, "parameter '" + meta.name + "' has no dim " +
                                           std::to_string(*dim)};
  for (int r = 0; r < tp; ++r) {
    const auto [lo, hi] = slice_range(meta.shape[*dim], r, tp);
    ShardDesc d;
    d.param = p;
    d.tp_rank = r;
    d.tp_size = tp;
    d.pp_stage = stage;
    d.d = ws_shard{*dim, lo, hi};
    out.push_back(d);
  }
  return out;
}

uint64_t shard_numel(const ParamMeta& p, const ws_shard& d) {
  uint64_t n = 1;
  for (size_t i = 0; i < p.shape.size(); ++i)
    n *= (uint64_t)((int)i == d.slice_dim ? d.end - d.start : p.shape[i]);
  return n;
}

uint64_t overlap_numel(const ParamMeta& p, const ws_shard& a, const ws_shard& b) {
  uint64_t n = 1;
  for (size_t i = 0; i < p.shape.size(); ++i) {
    int64_t lo = 0, hi = p.shape[i];
    if ((int)i == a.slice_dim) {
      lo = std::max(lo, a.start);
      hi = std::min(hi, a.end);
    }
    if ((int)i == b.slice_dim) {
      lo = std::max(lo, b.start);
      hi = std::min(hi, b.end);
    }
    if (hi <= lo) return 0;
    n *= (uint64_t)(hi - lo);
  }
  return n;
}

static uint64_t align_up(uint64_t x) { return (x + kArenaAlign - 1) / kArenaAlign * kArenaAlign; }

Plan::Plan(std::vector<ParamMeta> manifest, int dtype, const ws_train_layout& train,
           const ws_serve_layout& serve, int world, int rank)
    : manifest_(std::move(manifest)), dtype_(dtype), train_(train), serve_(serve),
      world_(world), rank_(rank) {
  if (world <= 0 || rank < 0 || rank >= world)
    throw PlanError{WS_INVALID_ARGUMENT, "rank " + std::to_string(rank) + " of " +
                                             std::to_string(world)};
  if (serve.tp <= 0 || serve.pp <= 0 || serve.replicas <= 0)
    throw PlanError{WS_INVALID_ARGUMENT, "serve tp, pp and replicas must be positive"};
  if (serve.placement != WS_PLACE_RANK && serve.placement != WS_PLACE_OVERLAP)
    throw PlanError{WS_INVALID_ARGUMENT, "unknown serve placement"};
  const int train_ranks =
      train.scheme == WS_TRAIN_TP ? train.tp * train.pp * train.dp : world;
  // world 1 with a multi-rank layout: one GPU hosts every rank
  collapsed_ = world == 1 && (train_ranks > 1 || serve.tp * serve.pp > 1);
  if (collapsed_ && serve.replicas != 1)
    throw PlanError{WS_INVALID_ARGUMENT, "a one-GPU plan of a multi-rank layout has one replica"};
  if (!collapsed_ && serve.tp * serve.pp * serve.replicas != world)
    throw PlanError{WS_INVALID_ARGUMENT, "serve tp*pp*replicas must equal the world size"};
  if (manifest_.empty()) throw PlanError{WS_INVALID_ARGUMENT, "empty manifest"};
  for (const auto& p : manifest_) {
    if (p.shape.empty() || p.shape.size() > WS_MAX_DIMS)
      throw PlanError{WS_INVALID_ARGUMENT, "parameter '" + p.name + "': rank out of range"};
    uint64_t n = 1;
    for (auto d : p.shape) {
      if (d <= 0) throw PlanError{WS_SHAPE_MISMATCH, "parameter '" + p.name + "': bad dim"};
      n *= (uint64_t)d;
    }
    if (n >= (1ull << 32))
      throw PlanError{WS_INVALID_ARGUMENT, "parameter '" + p.name + "' has 2^32 elements or more"};
    model_elems_ += n;
    tp_shard_dim(p.kind);  // UnknownModuleKind
  }
  const int L = manifest_num_layers(manifest_);
  const int P = (int)manifest_.size();

  // ---- trainer shards per rank --------------------------------------------
  segments_.assign(world, {});
  if (train.scheme == WS_TRAIN_TP) {
    // plan.cpp:8-21: every shard dealt round-robin over dp; the dealt rank's
    // GPU at (stage, tp_rank) encodes it (rank 0 when collapsed).
    if (train.tp <= 0 || train.pp <= 0 || train.dp <= 0 ||
        (!collapsed_ && train.tp * train.pp * train.dp != world))
      throw PlanError{WS_INVALID_ARGUMENT, "train tp*pp*dp must equal the world size"};
    size_t next = 0;
    for (int p = 0; p < P; ++p) {
      for (auto& d : param_shards(manifest_, p, train.tp, train.pp, L)) {
        const int dp_rank = (int)(next++ % (size_t)train.dp);
        const int g = dp_rank * train.pp * train.tp + d.pp_stage * train.tp + d.tp_rank;
        Segment s;
        s.shard = d;
        segments_[collapsed_ ? 0 : g].push_back(s);
      }
    }
  } else if (train.scheme == WS_TRAIN_FSDP) {
    for (int p = 0; p < P; ++p) {
      for (int r = 0; r < world; ++r) {
        ShardDesc d;
        d.param = p;
        if (world > 1) {
          const auto [lo, hi] = slice_range(manifest_[p].shape[0], r, world);
          d.tp_rank = r;
          d.tp_size = world;
          d.d = ws_shard{0, lo, hi};
        }
        Segment s;
        s.shard = d;
        segments_[r].push_back(s);
      }
    }
  } else {
    throw PlanError{WS_INVALID_ARGUMENT, "unknown train scheme"};
  }
  train_arena_.assign(world, 0);
  for (int r = 0; r < world; ++r) {
    uint64_t off = 0;
    for (auto& s : segments_[r]) {
      s.n = shard_numel(manifest_[s.shard.param], s.shard.d);
      s.offset = off;
      off = align_up(off + s.n);
    }
    train_arena_[r] = off;
  }

  // ---- serving shards per coordinate (ServeState::init, engine.cpp:34-49) --
  const int C = serve.tp * serve.pp;
  serve_by_coord_.assign(C, {});
  serve_arena_by_coord_.assign(C, 0);
  for (int c = 0; c < C; ++c) {
    const int stage = c / serve.tp, k = c % serve.tp;
    uint64_t off = 0;
    for (int p = 0; p < P; ++p) {
      const auto shards = param_shards(manifest_, p, serve.tp, serve.pp, L);
      if (shards[0].pp_stage != stage) continue;  // ServeState::owns, engine.cpp:51-54
      ServeShard ss;
      ss.shard = shards.size() == 1 ? shards[0] : shards[k];  // plan.cpp:34-39
      ss.n = shard_numel(manifest_[p], ss.shard.d);
      ss.offset = off;
      off = align_up(off + ss.n);
      serve_by_coord_[c].push_back(ss);
    }
    serve_arena_by_coord_[c] = off;
  }
  if (collapsed_) {  // every coordinate's arena, one after the other
    for (int c = 0; c < C; ++c) {
      for (ServeShard ss : serve_by_coord_[c]) {
        ss.offset += serve_all_elems_;
        serve_all_.push_back(ss);
        serve_all_coord_.push_back(c);
      }
      serve_all_elems_ += serve_arena_by_coord_[c];
    }
  }

  // ---- routes: box intersections (plan_pulls, plan.cpp:89-121, extended) ---
  routes_.assign(world, {});
  std::vector<uint64_t> coord_base(C, 0);  // collapsed: coordinate c's arena offset
  for (int c = 1; c < C; ++c) coord_base[c] = coord_base[c - 1] + serve_arena_by_coord_[c - 1];
  std::map<std::pair<int, int>, uint64_t> covered;  // (coord, param) -> elements
  for (int r = 0; r < world; ++r) {
    const auto& segs = segments_[r];
    for (int si = 0; si < (int)segs.size(); ++si) {
      const ShardDesc& src = segs[si].shard;
      for (int c = 0; c < C; ++c) {
        for (const auto& ss : serve_by_coord_[c]) {
          if (ss.shard.param != src.param) continue;
          const uint64_t ov = overlap_numel(manifest_[src.param], src.d, ss.shard.d);
          if (!ov) continue;
          Route rt;
          rt.seg = si;
          rt.coord = c;
          rt.dst = ss.shard;
          rt.dst_offset = ss.offset + (collapsed_ ? coord_base[c] : 0);
          rt.overlap = ov;
          routes_[r].push_back(rt);
          covered[{c, src.param}] += ov;
        }
      }
    }
  }
  place();
  for (int c = 0; c < C; ++c)
    for (const auto& ss : serve_by_coord_[c]) {
      const uint64_t got = covered[{c, ss.shard.param}];
      if (got != ss.n)
        throw PlanError{WS_INCOMPLETE_COVERAGE,
                        "parameter '" + manifest_[ss.shard.param].name + "': serving coordinate " +
                            std::to_string(c) + " covered " + std::to_string(got) + " of " +
                            std::to_string(ss.n) + " elements"};
    }
}

int Plan::coord_of_rank(int r) const {
  if (collapsed_ || r < 0 || r >= world_) return -1;
  return serve_rank_[r] % coords();
}

std::vector<int> assign_min_cost(const std::vector<int64_t>& cost, int n) {
  // rows are added one at a time; each grows a shortest-path tree over the
  // columns (reduced costs stay >= 0 thanks to the potentials u, v)
  const int64_t INF = std::numeric_limits<int64_t>::max() / 4;
  std::vector<int64_t> u(n + 1, 0), v(n + 1, 0);
  std::vector<int> row_of(n + 1, 0), way(n + 1, 0);  // column j (1-based) -> row (1-based)
  for (int i = 1; i <= n; ++i) {
    row_of[0] = i;
    int j0 = 0;
    std::vector<int64_t> minv(n + 1, INF);
    std::vector<char> used(n + 1, 0);
    do {
      used[j0] = 1;
      const int i0 = row_of[j0];
      int64_t delta = INF;
      int j1 = 0;
      for (int j = 1; j <= n; ++j) {
        if (used[j]) continue;
        const int64_t cur = cost[(size_t)(i0 - 1) * n + (j - 1)] - u[i0] - v[j];
        if (cur < minv[j]) minv[j] = cur, way[j] = j0;
        if (minv[j] < delta) delta = minv[j], j1 = j;
      }
      for (int j = 0; j <= n; ++j) {
        if (used[j]) u[row_of[j]] += delta, v[j] -= delta;
        else minv[j] -= delta;
      }
      j0 = j1;
    } while (row_of[j0] != 0);
    do {  // flip the augmenting path
      const int j1 = way[j0];
      row_of[j0] = row_of[j1];
      j0 = j1;
    } while (j0);
  }
  std::vector<int> col(n, -1);
  for (int j = 1; j <= n; ++j) col[row_of[j] - 1] = j - 1;
  return col;
}

// Serving rank of every GPU.  WS_PLACE_OVERLAP: GPU g hosting serving rank j
// (coordinate j % C) keeps local the elements its trainer shards route to
// that coordinate; the assignment maximises their sum (ties: rank order).
void Plan::place() {
  const int W = world_, C = coords();
  serve_rank_.resize(W);
  for (int g = 0; g < W; ++g) serve_rank_[g] = g;
  if (collapsed_ || serve_.placement == WS_PLACE_RANK) return;
  std::vector<uint64_t> w((size_t)W * C, 0);  // elements GPU g's shards route to coord c
  for (int g = 0; g < W; ++g)
    for (const Route& r : routes_[g]) w[(size_t)g * C + r.coord] += r.overlap;
  const int64_t tie = W + 1;  // any weight difference outranks every tie-break
  std::vector<int64_t> cost((size_t)W * W);
  for (int g = 0; g < W; ++g)
    for (int j = 0; j < W; ++j)
      cost[(size_t)g * W + j] = -(int64_t)w[(size_t)g * C + j % C] * tie + (j != g ? 1 : 0);
  serve_rank_ = assign_min_cost(cost, W);
}

uint64_t Plan::serve_arena_elems() const {
  return collapsed_ ? serve_all_elems_ : serve_arena_by_coord_[my_coord()];
}

uint64_t Plan::train_elems() const {
  uint64_t n = 0;
  for (const auto& s : segments()) n += s.n;
  return n;
}

}  // namespace wsync
