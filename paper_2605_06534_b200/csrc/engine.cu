// engine.cu -- planner and engine entry points of include/wsync.h.
//
// ws_engine_sync_step is the B200 counterpart of TransferEngine::sync_step
// (engine.cpp:66-254): the reference's pusher thread (extract + diff +
// encode per shard, :107-156) becomes ONE K1 launch over every trainer shard
// of this GPU, and its puller threads (decode + reslice + apply, :158-231)
// become the route/apply kernels; shards bound for other GPUs travel over
// NVLink (exchange.cu).
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "capi_util.h"
#include "engine.h"

using namespace wsync;

namespace wsync {

LocalEntry make_local_entry(int dtype, const int64_t* full, int nd, int seg, const ws_shard& src,
                            const ws_shard& dst, uint64_t dst_base) {
  LocalEntry e{};
  e.seg = seg;
  e.dst_base = dst_base;
  const Box S = shard_box(full, nd, src), D = shard_box(full, nd, dst);
  bool only_dim0 = true;
  for (int d = 1; d < nd; ++d)
    only_dim0 = only_dim0 && S.lo[d] == 0 && D.lo[d] == 0 && S.ext[d] == (uint32_t)full[d] &&
                D.ext[d] == (uint32_t)full[d];
  if (only_dim0) {
    uint64_t inner = 1;
    for (int d = 1; d < nd; ++d) inner *= (uint64_t)full[d];
    const int64_t lo0 = std::max<int64_t>(S.lo[0], D.lo[0]);
    const int64_t hi0 = std::min<int64_t>((int64_t)S.lo[0] + S.ext[0], (int64_t)D.lo[0] + D.ext[0]);
    e.identity = 1;
    e.keep_lo = (uint32_t)((lo0 - S.lo[0]) * (int64_t)inner);
    e.keep_hi = (uint32_t)(std::max<int64_t>(hi0 - S.lo[0], 0) * (int64_t)inner);
    e.shift = ((int64_t)S.lo[0] - (int64_t)D.lo[0]) * (int64_t)inner;
  }
  e.map = make_remap(full, nd, src, dst);
  make_box_copy(dtype, full, nd, dst, src, &e.box);
  return e;
}

}  // namespace wsync


static ws_status plan_guard(const std::function<void()>& f) {
  try {
    f();
    return WS_OK;
  } catch (const PlanError& e) {
    return set_error(e.status, e.msg);
  } catch (const std::exception& e) {
    return set_error(WS_TRANSFER_ERROR, e.what());
  }
}

extern "C" {

ws_status ws_plan_create(const ws_param* params, int nparams, ws_dtype dtype,
                         const ws_train_layout* train, const ws_serve_layout* serve, int world,
                         int rank, ws_plan** out) {
  if (!params || nparams <= 0 || !train || !serve || !out)
    return set_error(WS_INVALID_ARGUMENT, "ws_plan_create: null argument");
  if (!valid_dtype(dtype)) return set_error(WS_INVALID_ARGUMENT, "ws_plan_create: bad dtype");
  *out = nullptr;
  return plan_guard([&] {
    std::vector<ParamMeta> m;
    for (int i = 0; i < nparams; ++i) {
      ParamMeta pm;
      pm.name = params[i].name ? params[i].name : "";
      pm.kind = params[i].kind;
      if (params[i].ndims < 1 || params[i].ndims > WS_MAX_DIMS)
        throw PlanError{WS_INVALID_ARGUMENT, "parameter '" + pm.name + "': ndims out of range"};
      pm.shape.assign(params[i].shape, params[i].shape + params[i].ndims);
      pm.layer = params[i].layer;
      m.push_back(std::move(pm));
    }
    auto* h = new ws_plan;
    h->p = std::make_unique<Plan>(std::move(m), dtype, *train, *serve, world, rank);
    *out = h;
  });
}

void ws_plan_destroy(ws_plan* plan) { delete plan; }

ws_status ws_plan_get_info(const ws_plan* plan, ws_plan_info* info) {
  if (!plan || !info) return set_error(WS_INVALID_ARGUMENT, "ws_plan_get_info: null argument");
  const Plan& p = *plan->p;
  info->num_segments = (int32_t)p.segments().size();
  info->num_serve_shards = (int32_t)p.serve_shards().size();
  info->num_routes = (int32_t)p.routes().size();
  info->serve_coord = p.my_coord();
  info->train_arena_elems = p.train_arena_elems();
  info->serve_arena_elems = p.serve_arena_elems();
  info->train_elems = p.train_elems();
  info->model_elems = p.model_elems();
  info->serve_rank = p.serve_rank_of(p.rank());
  info->serve_replica = info->serve_rank < 0 ? -1 : info->serve_rank / p.coords();
  return WS_OK;
}

ws_status ws_plan_segment(const ws_plan* plan, int i, int32_t* param, ws_shard* desc,
                          uint64_t* offset, uint64_t* n) {
  if (!plan || i < 0 || i >= (int)plan->p->segments().size())
    return set_error(WS_INVALID_ARGUMENT, "ws_plan_segment: index out of range");
  const Segment& s = plan->p->segments()[i];
  if (param) *param = s.shard.param;
  if (desc) *desc = s.shard.d;
  if (offset) *offset = s.offset;
  if (n) *n = s.n;
  return WS_OK;
}

ws_status ws_plan_serve_shard_coord(const ws_plan* plan, int i, int32_t* coord) {
  if (!plan || !coord || i < 0 || i >= (int)plan->p->serve_shards().size())
    return set_error(WS_INVALID_ARGUMENT, "ws_plan_serve_shard_coord: index out of range");
  *coord = plan->p->serve_shard_coord(i);
  return WS_OK;
}

ws_status ws_plan_segment_key_fields(const ws_plan* plan, int i, int32_t* tp_rank,
                                     int32_t* tp_size, int32_t* pp_stage) {
  if (!plan || i < 0 || i >= (int)plan->p->segments().size())
    return set_error(WS_INVALID_ARGUMENT, "ws_plan_segment_key_fields: index out of range");
  const Segment& s = plan->p->segments()[i];
  if (tp_rank) *tp_rank = s.shard.tp_rank;
  if (tp_size) *tp_size = s.shard.tp_size;
  if (pp_stage) *pp_stage = s.shard.pp_stage;
  return WS_OK;
}

ws_status ws_plan_serve_shard(const ws_plan* plan, int i, int32_t* param, ws_shard* desc,
                              uint64_t* offset, uint64_t* n) {
  if (!plan || i < 0 || i >= (int)plan->p->serve_shards().size())
    return set_error(WS_INVALID_ARGUMENT, "ws_plan_serve_shard: index out of range");
  const ServeShard& s = plan->p->serve_shards()[i];
  if (param) *param = s.shard.param;
  if (desc) *desc = s.shard.d;
  if (offset) *offset = s.offset;
  if (n) *n = s.n;
  return WS_OK;
}

ws_status ws_plan_route(const ws_plan* plan, int i, int32_t* segment, int32_t* coord,
                        int32_t* num_dst_ranks, uint64_t* overlap_elems) {
  if (!plan || i < 0 || i >= (int)plan->p->routes().size())
    return set_error(WS_INVALID_ARGUMENT, "ws_plan_route: index out of range");
  const Route& r = plan->p->routes()[i];
  if (segment) *segment = r.seg;
  if (coord) *coord = r.coord;
  if (num_dst_ranks) *num_dst_ranks = plan->p->replicas();
  if (overlap_elems) *overlap_elems = r.overlap;
  return WS_OK;
}

ws_status ws_plan_exchange_caps(const ws_plan* plan, uint64_t* send_cap_per_coord,
                                uint64_t* recv_cap_per_rank) {
  if (!plan) return set_error(WS_INVALID_ARGUMENT, "ws_plan_exchange_caps: null plan");
  std::vector<uint64_t> s, r;
  exchange_caps(*plan->p, plan->p->rank(), &s, &r);
  if (send_cap_per_coord) std::memcpy(send_cap_per_coord, s.data(), s.size() * 8);
  if (recv_cap_per_rank) std::memcpy(recv_cap_per_rank, r.data(), r.size() * 8);
  return WS_OK;
}

ws_status ws_engine_create(const ws_plan* plan, int device, const uint8_t* unique_id,
                           ws_engine** out) {
  DeviceGuard device_guard;
  if (!plan || !out) return set_error(WS_INVALID_ARGUMENT, "ws_engine_create: null argument");
  *out = nullptr;
  try {
    auto* e = new ws_engine(*plan->p, device);
    ws_status st = e->init(unique_id);
    if (st != WS_OK) {
      delete e;
      return st;
    }
    *out = e;
    return WS_OK;
  } catch (const PlanError& e) {
    return set_error(e.status, e.msg);
  } catch (const std::exception& e) {
    return set_error(WS_TRANSFER_ERROR, e.what());
  }
}

void ws_engine_destroy(ws_engine* eng) { delete eng; }

ws_status ws_engine_bind(ws_engine* eng, void* train_prev_dev, void* train_next_dev,
                         void* serve_dev) {
  DeviceGuard device_guard;
  if (!eng) return set_error(WS_INVALID_ARGUMENT, "ws_engine_bind: null engine");
  const uintptr_t a = (uintptr_t)train_prev_dev | (uintptr_t)train_next_dev | (uintptr_t)serve_dev;
  if (a & 15) return set_error(WS_INVALID_ARGUMENT, "ws_engine_bind: arenas must be 16-byte aligned");
  if (eng->grouped() && eng->connected())
    return set_error(WS_INVALID_ARGUMENT, "ws_engine_bind: engine of a connected ws_group");
  eng->arena[0] = train_prev_dev;
  eng->arena[1] = train_next_dev;
  eng->serve = serve_dev;
  return eng->map_serve();
}

ws_status ws_engine_generate(ws_engine* eng, uint64_t seed, double density, ws_stream_t stream) {
  DeviceGuard device_guard;
  if (!eng) return set_error(WS_INVALID_ARGUMENT, "ws_engine_generate: null engine");
  return eng->generate(seed, density, reinterpret_cast<cudaStream_t>(stream));
}

ws_status ws_engine_payload(ws_engine* eng, int i, int force_wide_index, void* out_dev,
                            ws_payload_info* info, ws_stream_t stream) {
  DeviceGuard device_guard;
  if (!eng || !info) return set_error(WS_INVALID_ARGUMENT, "ws_engine_payload: null argument");
  return eng->payload(i, force_wide_index != 0, out_dev, info,
                      reinterpret_cast<cudaStream_t>(stream));
}

ws_status ws_engine_generate_skewed(ws_engine* eng, uint64_t seed, double density, double zipf_s,
                                   uint64_t perm_seed, ws_stream_t stream) {
  DeviceGuard device_guard;
  if (!eng) return set_error(WS_INVALID_ARGUMENT, "ws_engine_generate_skewed: null engine");
  if (!(zipf_s >= 0.0)) return set_error(WS_INVALID_ARGUMENT, "zipf_s must be >= 0");
  return eng->generate(seed, density, reinterpret_cast<cudaStream_t>(stream), zipf_s, perm_seed);
}

ws_status ws_engine_sync_step(ws_engine* eng, const ws_sync_options* opts, ws_stream_t stream,
                              ws_report* report) {
  DeviceGuard device_guard;
  if (!eng || !opts) return set_error(WS_INVALID_ARGUMENT, "ws_engine_sync_step: null argument");
  return eng->sync_step(*opts, reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr, report);
}

ws_status ws_engine_sync_step_host(ws_engine* eng, const void* next_host,
                                   const ws_sync_options* opts, ws_stream_t stream,
                                   uint64_t* nnz_host, ws_report* report) {
  DeviceGuard device_guard;
  if (!eng || !opts || !next_host)
    return set_error(WS_INVALID_ARGUMENT, "ws_engine_sync_step_host: null argument");
  return eng->sync_step(*opts, reinterpret_cast<cudaStream_t>(stream), next_host, nnz_host,
                        report);
}

ws_status ws_engine_timing(ws_engine* eng, int reset, ws_timing* out) {
  DeviceGuard device_guard;
  if (!eng) return set_error(WS_INVALID_ARGUMENT, "ws_engine_timing: null engine");
  return eng->timing(reset, out);
}

ws_status ws_engine_segment_counts(ws_engine* eng, uint64_t* nnz, char* codec) {
  DeviceGuard device_guard;
  if (!eng) return set_error(WS_INVALID_ARGUMENT, "ws_engine_segment_counts: null engine");
  return eng->segment_counts(nnz, codec);
}

ws_status ws_engine_segment_stream(ws_engine* eng, int i, const uint32_t** idx, const void** val,
                                   uint64_t* nrec, uint64_t* tile_elems) {
  DeviceGuard device_guard;
  if (!eng || !idx || !val || !nrec || !tile_elems)
    return set_error(WS_INVALID_ARGUMENT, "ws_engine_segment_stream: null argument");
  return eng->segment_stream(i, idx, val, nrec, tile_elems);
}

ws_status ws_engine_segment_delta(ws_engine* eng, int i, const uint32_t** idx, const void** val,
                                  uint64_t* nnz, char* codec) {
  DeviceGuard device_guard;
  if (!eng) return set_error(WS_INVALID_ARGUMENT, "ws_engine_segment_delta: null engine");
  return eng->segment_delta(i, idx, val, nnz, codec);
}

}  // extern "C"
