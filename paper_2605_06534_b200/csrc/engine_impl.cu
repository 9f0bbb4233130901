// engine_impl.cu -- ws_engine: device tables, K1 launch, local route/apply.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdint>
#include <vector>

#include "capi_util.h"
#include "engine.h"

using namespace wsync;

#define WS_CUDA_TRY(expr, what)                        \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return cuda_status(_e, what); \
  } while (0)

ws_engine::ws_engine(const Plan& plan, int device)
    : plan_(plan), device_(device), dtype_(plan.dtype()),
      nseg_((int)plan.segments().size()) {}

ws_engine::~ws_engine() {
  cudaSetDevice(device_);
  cudaFree(d_segs_);
  cudaFree(d_tile0_);
  cudaFree(d_tile_seg_);
  cudaFree(d_spill_);
  cudaFree(d_seg_mode_);
  cudaFree(d_fill_);
  cudaFree(d_fix_list_);
  cudaFree(d_fix_n_);
  cudaFree(d_tile_cnt_);
  cudaFree(d_tile_base_);
  cudaFree(d_seq_idx_);
  cudaFree(d_seq_val_);
  cudaFree(d_status_);
  cudaFree(d_ticket_);
  cudaFree(d_nnz_);
  cudaFree(d_cap_);
  cudaFree(d_rec_);
  cudaFree(d_base_);
  cudaFree(d_idx_);
  cudaFree(d_val_);
  cudaFree(d_local_);
  cudaFree(d_fuse_);
  cudaFree(d_fuse_on_);
  cudaFree(d_unit_off_);
  if (h_nnz_pinned_) cudaFreeHost(h_nnz_pinned_);
  if (h_sa_) cudaFreeHost(h_sa_);
  for (auto& e : relay_dev_) cudaFree(e.first);
  for (auto& e : relay_host_) cudaFreeHost(e.first);
  for (cudaStream_t st : relay_streams_)
    if (st) cudaStreamDestroy(st);
  if (ring_) {
    for (int i = 0; i < kRing; ++i)
      for (auto& e : ring_[i])
        if (e) cudaEventDestroy(e);
    delete[] ring_;
  }
  destroy_comm();
}

uint32_t ws_engine::next_epoch() {
  epoch_ = (epoch_ + 1) & 0x3fffffffu;
  if (epoch_ == 0) epoch_ = 1;
  return epoch_;
}

ws_status ws_engine::init(const uint8_t* unique_id, bool grouped) {
  grouped_ = grouped;
  WS_CUDA_TRY(cudaSetDevice(device_), "cudaSetDevice");
  const auto& segs = plan_.segments();
  // Encode tiles: one look-back chain per segment.
  std::vector<uint32_t> tile0(nseg_ + 1, 0);
  const uint32_t tile = encode_tile_elems(dtype_);
  uint64_t t = 0;
  for (int i = 0; i < nseg_; ++i) {
    tile0[i] = (uint32_t)t;
    t += (segs[i].n + tile - 1) / tile;
  }
  tile0[nseg_] = (uint32_t)t;
  if (t >= (1ull << 31)) return set_error(WS_CAPACITY, "too many encode tiles");
  ntiles_ = (uint32_t)t;
  tile_elems_ = tile;
  segs_.resize(nseg_);
  std::vector<uint64_t> base(nseg_);
  for (int i = 0; i < nseg_; ++i) {
    segs_[i] = SegDev{segs[i].offset, segs[i].n, 0, 0};
    base[i] = segs[i].offset;
  }
  const size_t ns = std::max(1, nseg_);
  WS_CUDA_TRY(cudaMalloc(&d_segs_, ns * sizeof(SegDev)), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&d_tile0_, (ns + 1) * sizeof(uint32_t)), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&d_status_, std::max<size_t>(1, ntiles_) * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMemset(d_status_, 0, std::max<size_t>(1, ntiles_) * 8), "cudaMemset");
  WS_CUDA_TRY(cudaMalloc(&d_ticket_, 256), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&d_seg_mode_, ns * 4), "cudaMalloc");
  WS_CUDA_TRY(cudaMemset(d_seg_mode_, 0, ns * 4), "cudaMemset");
  WS_CUDA_TRY(cudaMalloc(&d_fill_, ns * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&d_fix_list_, std::max<size_t>(1, ntiles_) * 4), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&d_fix_n_, 4), "cudaMalloc");
  if (const char* f = ablation_env("WSYNC_COUNT_ONLY")) count_only_ = atoi(f) != 0;
  spill_blocks_ = std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)sm_count(), ntiles_));
  WS_CUDA_TRY(cudaMalloc(&d_spill_, encode_spill_bytes(dtype_, spill_blocks_)), "cudaMalloc spill");
  WS_CUDA_TRY(cudaMalloc(&d_tile_cnt_, std::max<size_t>(1, ntiles_) * 4), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&d_tile_base_, std::max<size_t>(1, ntiles_) * 4), "cudaMalloc");
  WS_CUDA_TRY(cudaMemset(d_tile_cnt_, 0, std::max<size_t>(1, ntiles_) * 4), "cudaMemset");
  WS_CUDA_TRY(cudaMemset(d_tile_base_, 0, std::max<size_t>(1, ntiles_) * 4), "cudaMemset");
  WS_CUDA_TRY(cudaMalloc(&d_nnz_, ns * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMemset(d_nnz_, 0, ns * 8), "cudaMemset");
  WS_CUDA_TRY(cudaMalloc(&d_cap_, ns * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&d_rec_, ns * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&d_base_, ns * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMemcpy(d_tile0_, tile0.data(), (nseg_ + 1) * 4, cudaMemcpyHostToDevice), "H2D");
  plan_tile0_ = tile0;
  {  // segment of every super-tile: one load instead of a search in K1's producer
    std::vector<uint32_t> tile_seg(std::max<uint32_t>(1, ntiles_));
    for (int i = 0; i < nseg_; ++i)
      for (uint32_t tt = tile0[i]; tt < tile0[i + 1]; ++tt) tile_seg[tt] = (uint32_t)i;
    WS_CUDA_TRY(cudaMalloc(&d_tile_seg_, tile_seg.size() * 4), "cudaMalloc");
    WS_CUDA_TRY(cudaMemcpy(d_tile_seg_, tile_seg.data(), tile_seg.size() * 4,
                           cudaMemcpyHostToDevice), "H2D");
  }
  if (nseg_)
    WS_CUDA_TRY(cudaMemcpy(d_base_, base.data(), nseg_ * 8, cudaMemcpyHostToDevice), "H2D");
  WS_CUDA_TRY(cudaMallocHost(&h_nnz_pinned_, ns * 8), "cudaMallocHost");
  h_nnz_.assign(nseg_, 0);

  // Local routes: destinations on this GPU's serving coordinate.
  std::vector<LocalEntry> local;
  std::vector<int> local_per_seg(std::max(1, nseg_), 0);
  for (const Route& r : plan_.routes()) {
    if (!plan_.route_is_local(r)) continue;
    const ParamMeta& p = plan_.manifest()[r.dst.param];
    local.push_back(make_local_entry(dtype_, p.shape.data(), (int)p.shape.size(), r.seg,
                                     segs[r.seg].shard.d, r.dst.d, r.dst_offset));
    ++local_per_seg[r.seg];
  }
  nlocal_ = (int)local.size();
  // Per-segment fused-apply entries for K1: a segment feeding exactly one
  // serving shard of this GPU (one shard per parameter per coordinate; a
  // one-GPU plan of a multi-rank layout can hold several) has it applied by
  // K1; the others go through the local route.
  std::vector<FuseEntry> fuse(std::max(1, nseg_));
  for (auto& f : fuse) f = FuseEntry{};
  for (LocalEntry& e : local) {
    if (local_per_seg[e.seg] != 1) continue;
    e.fused_ok = 1;
    FuseEntry& f = fuse[e.seg];
    f.mode = e.identity ? 1 : 2;
    f.keep_lo = e.keep_lo;
    f.keep_hi = e.keep_hi;
    f.shift = e.shift;
    f.dst_base = e.dst_base;
    f.map = e.map;
  }
  WS_CUDA_TRY(cudaMalloc(&d_fuse_, fuse.size() * sizeof(FuseEntry)), "cudaMalloc");
  {
    std::vector<uint32_t> on(fuse.size(), 1u);  // fuse until a sync says a segment runs dense
    WS_CUDA_TRY(cudaMalloc(&d_fuse_on_, on.size() * 4), "cudaMalloc");
    WS_CUDA_TRY(cudaMemcpy(d_fuse_on_, on.data(), on.size() * 4, cudaMemcpyHostToDevice), "H2D");
  }
  WS_CUDA_TRY(cudaMemcpy(d_fuse_, fuse.data(), fuse.size() * sizeof(FuseEntry),
                         cudaMemcpyHostToDevice), "H2D");
  if (const char* f = ablation_env("WSYNC_NO_FUSED_APPLY")) fuse_apply_ = atoi(f) == 0;
  sa_div_ = dtype_ == WS_BF16 ? 250u : 0u;  // K1 streamed apply from 0.4% density
  if (const char* f = ablation_env("WSYNC_SA_DIV")) {
    sa_div_ = dtype_ == WS_BF16 ? (uint32_t)atoi(f) : 0u;
    sa_env_ = true;
  }
  if (sa_div_) {
    WS_CUDA_TRY(cudaHostAlloc(&h_sa_, 16, cudaHostAllocMapped), "cudaHostAlloc");
    h_sa_[0] = h_sa_[1] = 0;
    WS_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_sa_), h_sa_, 0), "mapped");
    if (const char* f = ablation_env("WSYNC_SA_FORCE")) sa_force_ = atoi(f) != 0;
  }
  WS_CUDA_TRY(cudaMalloc(&d_local_, std::max<size_t>(1, local.size()) * sizeof(LocalEntry)),
              "cudaMalloc");
  if (nlocal_)
    WS_CUDA_TRY(cudaMemcpy(d_local_, local.data(), local.size() * sizeof(LocalEntry),
                           cudaMemcpyHostToDevice),
                "H2D");
  WS_CUDA_TRY(cudaMalloc(&d_unit_off_, (local.size() + 1) * 8), "cudaMalloc");
  route_grid_ = sm_count() * 8;
  ring_ = new cudaEvent_t[kRing][7]();
  for (int i = 0; i < kRing; ++i)
    for (auto& e : ring_[i]) WS_CUDA_TRY(cudaEventCreate(&e), "cudaEventCreate");
  // a group wires the exchange of all its ranks at once (ws_group_connect)
  return grouped ? WS_OK : init_comm(unique_id, nullptr);
}

ws_status ws_engine::ensure_records(double threshold, int sparse) {
  if (threshold == cur_threshold_ && sparse == cur_sparse_) return WS_OK;
  if (!(threshold >= 0.0)) return set_error(WS_INVALID_ARGUMENT, "density_threshold must be >= 0");
  // The largest record count k with k/n <= threshold (engine.cpp:121) is
  // the capacity of a segment: one more change makes it dense.
  uint64_t total = 0;
  std::vector<uint64_t> cap(nseg_), rec(nseg_);
  for (int i = 0; i < nseg_; ++i) {
    const uint64_t c = sparse ? sparse_capacity(segs_[i].n, threshold) : 0;
    cap[i] = c;
    rec[i] = total;
    total += (c + 63) / 64 * 64;
    segs_[i].cap = c;
    segs_[i].rec = rec[i];
  }
  WS_CUDA_TRY(cudaDeviceSynchronize(), "sync before record realloc");
  if (total > rec_alloc_) {
    cudaFree(d_idx_);
    cudaFree(d_val_);
    d_idx_ = nullptr;
    d_val_ = nullptr;
    WS_CUDA_TRY(cudaMalloc(&d_idx_, total * 4), "cudaMalloc records");
    WS_CUDA_TRY(cudaMalloc(&d_val_, total * dtype_size(dtype_)), "cudaMalloc records");
    rec_alloc_ = total;
  }
  if (nseg_) {
    WS_CUDA_TRY(cudaMemcpy(d_segs_, segs_.data(), nseg_ * sizeof(SegDev), cudaMemcpyHostToDevice),
                "H2D");
    WS_CUDA_TRY(cudaMemcpy(d_cap_, cap.data(), nseg_ * 8, cudaMemcpyHostToDevice), "H2D");
    WS_CUDA_TRY(cudaMemcpy(d_rec_, rec.data(), nseg_ * 8, cudaMemcpyHostToDevice), "H2D");
  }
  cur_threshold_ = threshold;
  cur_sparse_ = sparse;
  return WS_OK;
}

ws_status ws_engine::generate(uint64_t seed, double density, cudaStream_t s, double zipf_s,
                              uint64_t perm_seed) {
  if (dtype_ != WS_BF16) return set_error(WS_INVALID_ARGUMENT, "generate: bf16 engines only");
  if (!arena[0] || !arena[1] || !serve) return set_error(WS_INVALID_ARGUMENT, "generate: unbound");
  WS_CUDA_TRY(cudaSetDevice(device_), "cudaSetDevice");
  const double d = std::min(std::max(density, 0.0), 1.0);
  const uint64_t thr = (uint64_t)(d * 4294967296.0);
  // skewed mode: one threshold table per EXPERT tensor (dim 0 = expert)
  std::vector<uint64_t> tab;
  std::vector<size_t> tab_off(plan_.manifest().size(), SIZE_MAX);
  if (zipf_s >= 0.0) {
    for (size_t i = 0; i < plan_.manifest().size(); ++i) {
      const ParamMeta& p = plan_.manifest()[i];
      if (p.kind != WS_EXPERT || p.shape.empty()) continue;
      tab_off[i] = tab.size();
      tab.resize(tab.size() + p.shape[0]);
      expert_thresholds((int)p.shape[0], d, zipf_s, perm_seed, tab.data() + tab_off[i]);
    }
  }
  uint64_t* d_tab = nullptr;
  if (!tab.empty()) {
    WS_CUDA_TRY(cudaMalloc(&d_tab, tab.size() * 8), "cudaMalloc");
    WS_CUDA_TRY(cudaMemcpy(d_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice), "H2D");
  }
  auto table = [&](int param) -> const uint64_t* {
    return tab_off[param] == SIZE_MAX ? nullptr : d_tab + tab_off[param];
  };
  ws_status st = WS_OK;
  for (const Segment& sg : plan_.segments()) {
    const ParamMeta& p = plan_.manifest()[sg.shard.param];
    cudaError_t e = launch_gen_bf16(param_key(seed, p.name.c_str()), p.shape.data(),
                                    (int)p.shape.size(), sg.shard.d, thr,
                                    (uint16_t*)arena[0] + sg.offset,
                                    (uint16_t*)arena[1] + sg.offset, s, table(sg.shard.param));
    if (e != cudaSuccess && st == WS_OK) st = cuda_status(e, "generate");
  }
  for (const ServeShard& ss : plan_.serve_shards()) {
    const ParamMeta& p = plan_.manifest()[ss.shard.param];
    cudaError_t e = launch_gen_bf16(param_key(seed, p.name.c_str()), p.shape.data(),
                                    (int)p.shape.size(), ss.shard.d, thr,
                                    (uint16_t*)serve + ss.offset, nullptr, s,
                                    table(ss.shard.param));
    if (e != cudaSuccess && st == WS_OK) st = cuda_status(e, "generate");
  }
  if (d_tab) {
    cudaStreamSynchronize(s);
    cudaFree(d_tab);
  }
  return st;
}

EncodeArgs ws_engine::encode_args(int pa, int na) {
  EncodeArgs a{};
  a.unordered = 1;
  a.spill = d_spill_;
  a.spill_blocks = spill_blocks_;
  a.tile_cnt = d_tile_cnt_;
  a.tile_base = d_tile_base_;
  a.prev = arena[pa];
  a.next = arena[na];
  a.segs = d_segs_;
  a.tile0 = d_tile0_;
  a.tile_seg = d_tile_seg_;
  if (fuse_apply_ && !encode_only_) {
    a.fuse = d_fuse_;
    a.fuse_on = d_fuse_on_;
    a.serve = serve;
    // the streamed-apply instantiation when more fused elements stream than
    // take the per-record RMW (from the last sync whose worklist has run; a
    // stale answer only costs speed -- either instantiation is exact for any
    // fuse_on)
    const volatile uint64_t* sa = h_sa_;
    a.serve_stream = (sa_div() && (sa_force_ || (sa[0] && sa[0] >= sa[1]))) ? 1 : 0;
  }
  a.nseg = nseg_;
  a.ntiles = ntiles_;
  a.out_idx = d_idx_;
  a.out_val = d_val_;
  a.seg_nnz = d_nnz_;
  a.status = d_status_;
  a.epoch = next_epoch();
  a.ticket = d_ticket_;
  if (count_only_) a.seg_mode = d_seg_mode_;
  return a;
}

// Super-tiles of predicted-dense segments in [seg_begin, seg_end) that came
// out sparse, then K1 over just those (an empty list costs two near-empty
// launches).
ws_status ws_engine::launch_fixup(const EncodeArgs& a, int seg_begin, int seg_end, cudaStream_t s,
                                  uint32_t* launches) {
  WS_CUDA_TRY(launch_fixup_plan(d_tile0_, seg_begin, seg_end, d_nnz_, d_cap_, d_seg_mode_,
                                d_fix_list_, d_fix_n_, s),
              "fixup plan");
  EncodeArgs f = a;
  f.seg_mode = nullptr;
  f.tile_list = d_fix_list_;
  f.ntiles_dev = d_fix_n_;
  f.tile_offset = 0;
  f.ntiles = ntiles_;
  f.fill = d_fill_;
  WS_CUDA_TRY(launch_encode(dtype_, f, s), "encode fixup");
  *launches += 2;
  return WS_OK;
}

ws_status ws_engine::local_route(const ws_sync_options& o, int pa, int na, cudaStream_t s,
                                 uint32_t* launches) {
  RouteSideArgs r{};
  r.entries = d_local_;
  r.nentries = nlocal_;
  r.sparse = o.sparse ? 1 : 0;
  r.seg_nnz = d_nnz_;
  r.seg_cap = d_cap_;
  r.seg_rec = d_rec_;
  r.seg_base = d_base_;
  r.rec_idx = d_idx_;
  r.rec_val = d_val_;
  fill_tiles(r);
  r.segs = d_segs_;
  r.stream_apply = 1;
  r.train_prev = arena[pa];
  r.train_next = arena[na];
  r.serve = serve;
  r.unit_off = d_unit_off_;
  r.fused = (fuse_apply_ && o.sparse && ntiles_) ? 1 : 0;
  r.fuse_on = d_fuse_on_;
  r.sa_div = sa_div();
  r.sa_elems = d_sa_;
  WS_CUDA_TRY(launch_local_route(dtype_, r, route_grid_, s), "local route");
  if (nlocal_) *launches += 2;
  return WS_OK;
}

ws_status ws_engine::sync_begin(SyncCtx& x, const ws_sync_options& o, cudaStream_t s,
                                const void* next_host) {
  if (!bound()) return set_error(WS_INVALID_ARGUMENT, "sync: unbound");
  WS_CUDA_TRY(cudaSetDevice(device_), "cudaSetDevice");
  if (!(o.density_threshold >= 0.0))
    return set_error(WS_INVALID_ARGUMENT, "density_threshold must be >= 0");
  // larger receive regions for a higher threshold (collective; a group has
  // done this for all its ranks already)
  ws_status st = exchange_prepare(o);
  if (st != WS_OK) return st;
  st = ensure_records(o.density_threshold, o.sparse ? 1 : 0);
  if (st != WS_OK) return st;
  x.o = o;
  x.pa = o.reverse ? 1 : 0;
  x.na = 1 - x.pa;
  x.launches = 0;
  x.ev = ring_[ring_head_];
  pack_ev_ = false;
  ring_head_ = (ring_head_ + 1) % kRing;
  ring_steps_ = std::min<uint32_t>(ring_steps_ + 1, kRing);
  last_stream_ = s;
  WS_CUDA_TRY(cudaEventRecord(x.ev[0], s), "event");
  if (plan_.world() > 1 && !encode_only_) {  // (the relay path exchanges nothing here)
    st = exchange_begin(s, &x.launches);
    if (st != WS_OK) return st;
  }
  if (next_host) {
    WS_CUDA_TRY(cudaMemcpyAsync(arena[x.na], next_host,
                                plan_.train_arena_elems() * dtype_size(dtype_),
                                cudaMemcpyHostToDevice, s),
                "H2D next snapshot");
  }
  WS_CUDA_TRY(cudaEventRecord(x.ev[1], s), "event");
  last_sparse_ = o.sparse != 0;
  last_next_arena_ = x.na;
  return WS_OK;
}

ws_status ws_engine::sync_encode(SyncCtx& x, cudaStream_t s, bool run_local) {
  const ws_sync_options& o = x.o;
  if (o.sparse && ntiles_) {
    // K1 reserves each super-tile's records with an atomic on its segment's count
    WS_CUDA_TRY(cudaMemsetAsync(d_nnz_, 0, nseg_ * 8, s), "memset counts");
    if (count_only_) WS_CUDA_TRY(cudaMemsetAsync(d_fill_, 0, nseg_ * 8, s), "memset fill");
    EncodeArgs a = encode_args(x.pa, x.na);
    if (plan_.world() > 1 && !encode_only_ && !grouped_) {
      ws_status st = exchange_fuse_k1(a, s);
      if (st != WS_OK) return st;
    }
    WS_CUDA_TRY(launch_encode(dtype_, a, s), "encode");
    ++x.launches;
    x.streamed_apply = a.serve_stream != 0;
    if (count_only_) {
      ws_status st = launch_fixup(a, 0, nseg_, s, &x.launches);
      if (st != WS_OK) return st;
    }
  }
  WS_CUDA_TRY(cudaEventRecord(x.ev[2], s), "event");
  if (!run_local) return WS_OK;  // the caller runs the local route (and ev[3])
  if (!encode_only_) {  // relay pusher: the serving side applies what it pulls
    ws_status st = local_route(o, x.pa, x.na, s, &x.launches);
    if (st != WS_OK) return st;
  }
  WS_CUDA_TRY(cudaEventRecord(x.ev[3], s), "event");
  return WS_OK;
}

ws_status ws_engine::sync_finish(SyncCtx& x, cudaStream_t s, uint64_t* nnz_host,
                                 ws_report* report) {
  cudaEvent_t* ev_ = x.ev;
  WS_CUDA_TRY(cudaEventRecord(ev_[4], s), "event");
  if ((nnz_host || report) && nseg_)
    WS_CUDA_TRY(cudaMemcpyAsync(h_nnz_pinned_, d_nnz_, nseg_ * 8, cudaMemcpyDeviceToHost, s),
                "D2H counts");
  WS_CUDA_TRY(cudaEventRecord(ev_[5], s), "event");
  launch_total_ += x.launches;
  last_launches_ = x.launches;
  last_streamed_apply_ = x.streamed_apply;
  pack_steps_ = pack_ev_ ? pack_steps_ + 1 : 0;  // the most recent run of steps with one
  if (!nnz_host && !report) return WS_OK;
  WS_CUDA_TRY(cudaStreamSynchronize(s), "sync");
  if (nnz_host && nseg_) std::memcpy(nnz_host, h_nnz_pinned_, nseg_ * 8);
  return report_of(x, report);
}

// Fills `report` (if any) from the synchronised sync x (counts in
// h_nnz_pinned_, stage events in x.ev) and surfaces exchange faults.
ws_status ws_engine::report_of(const SyncCtx& x, ws_report* report) {
  const ws_sync_options& o = x.o;
  cudaEvent_t* ev_ = x.ev;
  ws_status st = exchange_status();
  if (st != WS_OK) return st;
  std::memcpy(h_nnz_.data(), h_nnz_pinned_, nseg_ * 8);
  if (report) {
    const int esz = dtype_size(dtype_);
    std::memset(report, 0, sizeof(*report));
    float ms = 0;
    cudaEventElapsedTime(&ms, ev_[0], ev_[5]);
    report->wall_s = ms * 1e-3;
    cudaEventElapsedTime(&ms, ev_[1], ev_[2]);
    report->encode_s = ms * 1e-3;
    cudaEventElapsedTime(&ms, ev_[2], ev_[3]);
    report->apply_s = ms * 1e-3;
    cudaEventElapsedTime(&ms, ev_[3], ev_[4]);
    report->route_s = ms * 1e-3;
    // Wire accounting of the reference payloads (transfer_cases.hpp:187-194),
    // with the dtype's value width.
    for (int i = 0; i < nseg_; ++i) {
      const auto& sg = plan_.segments()[i];
      const uint64_t nd = plan_.manifest()[sg.shard.param].shape.size();
      const bool sparse = o.sparse && (!ntiles_ || h_nnz_[i] <= segs_[i].cap);
      if (sparse) {
        report->sparse_shards++;
        report->pushed_bytes += 8 + 8 * nd + 8 + h_nnz_[i] * (4 + esz);
      } else {
        report->dense_shards++;
        report->pushed_bytes += 8 + 8 * nd + sg.n * esz;
      }
      report->nnz += o.sparse ? h_nnz_[i] : 0;
    }
    report->pulled_bytes = pulled_bytes_;
    report->kernel_launches = x.launches;
    report->streamed_apply = x.streamed_apply ? 1 : 0;
  }
  return WS_OK;
}

ws_status ws_engine::sync_step(const ws_sync_options& o, cudaStream_t s, const void* next_host,
                               uint64_t* nnz_host, ws_report* report) {
  if (grouped_)
    return set_error(WS_INVALID_ARGUMENT, "engine of a ws_group: sync through ws_group_sync_step");
  return sync_step_impl(o, s, next_host, nnz_host, report);
}

ws_status ws_engine::sync_step_impl(const ws_sync_options& o, cudaStream_t s,
                                    const void* next_host, uint64_t* nnz_host,
                                    ws_report* report) {
  SyncCtx x;
  ws_status st = sync_begin(x, o, s, next_host);
  if (st != WS_OK) return st;
  const bool rounds = plan_.world() > 1 && o.sparse && ntiles_ && !encode_only_ &&
                      exchange_rounds() > 1;
  if (rounds) {
    st = sync_rounds(o, x.pa, x.na, s, &x.launches, x.ev);
    if (st != WS_OK) return st;
  } else {
    // no overlapped rounds: the local route runs on a side stream beside the
    // pack and the receive-side apply (disjoint serving boxes; it overlaps
    // the NVLink transfer with this GPU's own HBM copy / apply)
    cudaStream_t side = exchange_side_stream();
    const bool fork = side && plan_.world() > 1 && !encode_only_;
    st = sync_encode(x, s, !fork);
    if (st != WS_OK) return st;
    if (fork) {
      st = exchange_fork(s, side);
      if (st == WS_OK) st = local_route(o, x.pa, x.na, side, &x.launches);
      if (st != WS_OK) return st;
      WS_CUDA_TRY(cudaEventRecord(x.ev[3], side), "event");
    }
    if (plan_.world() > 1 && !encode_only_) {
      st = exchange(o, x.na, s, &x.launches);
      if (st != WS_OK) return st;
    }
    if (fork) {
      st = exchange_join(s, side);
      if (st != WS_OK) return st;
    }
  }
  return sync_finish(x, s, nnz_host, report);
}

ws_status ws_engine::segment_counts(uint64_t* nnz, char* codec) {
  WS_CUDA_TRY(cudaSetDevice(device_), "cudaSetDevice");
  WS_CUDA_TRY(cudaDeviceSynchronize(), "sync");
  std::vector<uint64_t> n(std::max(1, nseg_), 0);
  if (nseg_) WS_CUDA_TRY(cudaMemcpy(n.data(), d_nnz_, nseg_ * 8, cudaMemcpyDeviceToHost), "D2H");
  for (int i = 0; i < nseg_; ++i) {
    if (nnz) nnz[i] = n[i];
    if (codec) codec[i] = (last_sparse_ && (!ntiles_ || n[i] <= segs_[i].cap)) ? 'S' : 'D';
  }
  return WS_OK;
}

ws_status ws_engine::segment_stream(int i, const uint32_t** idx, const void** val,
                                    uint64_t* nrec, uint64_t* tile_elems) {
  if (i < 0 || i >= nseg_) return set_error(WS_INVALID_ARGUMENT, "segment index out of range");
  WS_CUDA_TRY(cudaSetDevice(device_), "cudaSetDevice");
  WS_CUDA_TRY(cudaDeviceSynchronize(), "sync");
  uint64_t n = 0;
  WS_CUDA_TRY(cudaMemcpy(&n, d_nnz_ + i, 8, cudaMemcpyDeviceToHost), "D2H nnz");
  const bool sparse = last_sparse_ && n <= segs_[i].cap;
  *idx = d_idx_ + segs_[i].rec;
  *val = static_cast<const char*>(d_val_) + segs_[i].rec * dtype_size(dtype_);
  *nrec = sparse ? n : 0;
  *tile_elems = encode_tile_elems(dtype_);
  return WS_OK;
}

ws_status ws_engine::segment_delta(int i, const uint32_t** idx, const void** val, uint64_t* nnz,
                                   char* codec) {
  if (i < 0 || i >= nseg_) return set_error(WS_INVALID_ARGUMENT, "segment index out of range");
  WS_CUDA_TRY(cudaSetDevice(device_), "cudaSetDevice");
  WS_CUDA_TRY(cudaDeviceSynchronize(), "sync");
  uint64_t n = 0;
  WS_CUDA_TRY(cudaMemcpy(&n, d_nnz_ + i, 8, cudaMemcpyDeviceToHost), "D2H nnz");
  const bool sparse = last_sparse_ && n <= segs_[i].cap;
  const size_t esz = dtype_size(dtype_);
  // K1 left the records grouped by super-tile in reservation order; hand
  // out the ascending stream (codec.cpp:48-49 order), compacted here.
  const uint64_t need = std::max<uint64_t>(1, segs_[i].cap);
  if (need > seq_alloc_) {
    cudaFree(d_seq_idx_);
    cudaFree(d_seq_val_);
    d_seq_idx_ = nullptr;
    d_seq_val_ = nullptr;
    WS_CUDA_TRY(cudaMalloc(&d_seq_idx_, need * 4), "cudaMalloc");
    WS_CUDA_TRY(cudaMalloc(&d_seq_val_, need * esz), "cudaMalloc");
    seq_alloc_ = need;
  }
  if (sparse && n) {
    const uint32_t t0 = plan_tile0_[i], nt = plan_tile0_[i + 1] - t0;
    WS_CUDA_TRY(launch_compact(dtype_, d_tile_cnt_ + t0, d_tile_base_ + t0, nt, segs_[i].cap,
                               d_idx_ + segs_[i].rec, (const char*)d_val_ + segs_[i].rec * esz,
                               d_seq_idx_, d_seq_val_, nullptr),
                "compact");
    WS_CUDA_TRY(cudaDeviceSynchronize(), "sync");
  }
  if (idx) *idx = d_seq_idx_;
  if (val) *val = d_seq_val_;
  if (nnz) *nnz = n;
  if (codec) *codec = sparse ? 'S' : 'D';
  return WS_OK;
}

ws_status ws_engine::payload(int i, bool wide, void* out_dev, ws_payload_info* info,
                             cudaStream_t s) {
  if (i < 0 || i >= nseg_) return set_error(WS_INVALID_ARGUMENT, "segment index out of range");
  const uint32_t* idx = nullptr;
  const void* val = nullptr;
  uint64_t nnz = 0;
  char codec = 'D';
  ws_status st = segment_delta(i, &idx, &val, &nnz, &codec);  // ascending stream
  if (st != WS_OK) return st;
  return payload_from(i, wide, idx, val, nnz, codec, out_dev, info, s);
}

ws_status ws_engine::compact_segment(int i, uint32_t* out_idx, void* out_val, cudaStream_t s) {
  const size_t esz = dtype_size(dtype_);
  const uint32_t t0 = plan_tile0_[i], nt = plan_tile0_[i + 1] - t0;
  WS_CUDA_TRY(launch_compact(dtype_, d_tile_cnt_ + t0, d_tile_base_ + t0, nt, segs_[i].cap,
                             d_idx_ + segs_[i].rec, (const char*)d_val_ + segs_[i].rec * esz,
                             out_idx, out_val, s),
              "compact");
  return WS_OK;
}

ws_status ws_engine::payload_from(int i, bool wide, const uint32_t* idx, const void* val,
                                  uint64_t nnz, char codec, void* out_dev,
                                  ws_payload_info* info, cudaStream_t s) {
  const Segment& sg = plan_.segments()[i];
  const ParamMeta& p = plan_.manifest()[sg.shard.param];
  int64_t shape[8];
  const int nd = (int)p.shape.size();
  for (int d = 0; d < nd; ++d) shape[d] = p.shape[d];
  if (sg.shard.d.slice_dim >= 0) shape[sg.shard.d.slice_dim] = sg.shard.d.end - sg.shard.d.start;
  // pick_index_width (codec.cpp:140-143): local indices of a shard < 2^32 -> 4
  const int iw = codec == 'S' ? (wide ? 8 : 4) : 0;
  std::memset(info, 0, sizeof(*info));
  info->codec = codec;
  info->dtype = dtype_;
  info->ndims = nd;
  info->index_width = iw;
  for (int d = 0; d < nd; ++d) info->shape[d] = shape[d];
  info->nnz = codec == 'S' ? nnz : 0;
  info->header_bytes = 8 + 8 * (uint64_t)nd + (codec == 'S' ? 8 : 0);
  info->total_bytes = ws_payload_bytes((ws_dtype)dtype_, nd, codec, iw,
                                       codec == 'S' ? nnz : sg.n);
  if (!out_dev) return WS_OK;
  const ws_stream_t ss = reinterpret_cast<ws_stream_t>(s);
  ws_status st;
  if (codec == 'S')
    st = ws_encode_sparse_dev((ws_dtype)dtype_, shape, nd, iw, idx, val, nnz, out_dev, ss);
  else
    st = ws_encode_dense_dev((ws_dtype)dtype_, shape, nd,
                             (const char*)arena[last_next_arena_] + sg.offset * dtype_size(dtype_),
                             out_dev, ss);
  if (st != WS_OK) return st;
  WS_CUDA_TRY(cudaStreamSynchronize(s), "payload");
  return WS_OK;
}

ws_status ws_engine::timing(int reset, ws_timing* out) {
  WS_CUDA_TRY(cudaSetDevice(device_), "cudaSetDevice");
  if (last_stream_) WS_CUDA_TRY(cudaStreamSynchronize(last_stream_), "sync");
  WS_CUDA_TRY(cudaDeviceSynchronize(), "sync");
  ws_status st = exchange_status();  // timed syncs must not hide an exchange fault
  if (st != WS_OK) return st;
  ws_timing t{};
  t.steps = ring_steps_;
  t.kernel_launches = launch_total_;
  t.pack_steps = std::min(pack_steps_, ring_steps_);
  for (uint32_t k = 0; k < ring_steps_; ++k) {
    const cudaEvent_t* e = ring_[(ring_head_ + kRing - 1 - k) % kRing];
    float ms = 0;
    cudaEventElapsedTime(&ms, e[0], e[5]);
    t.wall_s += ms * 1e-3;
    cudaEventElapsedTime(&ms, e[1], e[2]);
    t.encode_s += ms * 1e-3;
    cudaEventElapsedTime(&ms, e[2], e[3]);
    t.apply_s += ms * 1e-3;
    cudaEventElapsedTime(&ms, e[3], e[4]);
    t.route_s += ms * 1e-3;
    if (k < pack_steps_ && cudaEventElapsedTime(&ms, e[3], e[6]) == cudaSuccess)
      t.pack_s += ms * 1e-3;
  }
  if (out) *out = t;
  if (reset) {
    ring_steps_ = 0;
    pack_steps_ = 0;
    launch_total_ = 0;
  }
  return WS_OK;
}
