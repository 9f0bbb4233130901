// engine.h -- the per-GPU weight-sync engine behind ws_engine_*.
#pragma once

#include <functional>
#include <vector>

#include "fabric.h"
#include "plan.h"
#include "route.h"

#include <memory>

struct ws_plan {  // the C-ABI plan handle
  std::unique_ptr<wsync::Plan> p;
};

struct ws_engine {
  ws_engine(const wsync::Plan& plan, int device);
  ~ws_engine();

  // group: the engine is one rank of a process-local ws_group (its exchange
  // is wired by ws_group_connect); otherwise unique_id (world > 1)
  ws_status init(const uint8_t* unique_id, bool grouped = false);
  ws_status generate(uint64_t seed, double density, cudaStream_t s, double zipf_s = -1.0,
                     uint64_t perm_seed = 0);
  ws_status sync_step(const ws_sync_options& o, cudaStream_t s, const void* next_host,
                      uint64_t* nnz_host, ws_report* report);
  ws_status segment_stream(int i, const uint32_t** idx, const void** val, uint64_t* nrec,
                           uint64_t* tile_elems);
  ws_status segment_delta(int i, const uint32_t** idx, const void** val, uint64_t* nnz,
                          char* codec);
  ws_status segment_counts(uint64_t* nnz, char* codec);
  ws_status timing(int reset, ws_timing* out);
  ws_status payload(int i, bool wide, void* out_dev, ws_payload_info* info, cudaStream_t s);
  // payload of segment i from its ascending stream (idx, val, nnz, codec);
  // out_dev == null: sizes only.  Synchronises stream s only.
  ws_status payload_from(int i, bool wide, const uint32_t* idx, const void* val, uint64_t nnz,
                         char codec, void* out_dev, ws_payload_info* info, cudaStream_t s);
  // segment i's ascending record stream into (out_idx, out_val), on stream s
  ws_status compact_segment(int i, uint32_t* out_idx, void* out_val, cudaStream_t s);
  // cross-cluster sync through a relay (relay.cpp)
  ws_status sync_relay(uint64_t step, const ws_sync_options& o, const ws_relay_options& ro,
                       const ws_relay& relay, ws_relay_report* rep);
  // frees sync_relay's staging and the cached wire scratch (ws_engine_release_staging)
  ws_status release_staging();
  bool encode_only_ = false;  // sync_step: K1 only (no fused apply, no routes)
  // sync_relay's staging (device / pinned host) and streams, kept across calls
  std::vector<std::pair<void*, size_t>> relay_dev_, relay_host_;
  cudaStream_t relay_streams_[3] = {nullptr, nullptr, nullptr};

  // caller-owned arenas (ws_engine_bind)
  void* arena[2] = {nullptr, nullptr};
  void* serve = nullptr;
  // Multi-GPU P2P: maps every replica's serving arena for direct dense
  // copies.  Collective: every rank binds (ws_engine_bind) in the same order.
  ws_status map_serve();

  // One sync in phases (sync_step runs them back to back; ws_group_sync_step
  // interleaves the phases of all ranks of a group on one stream, so every
  // flag a kernel waits for was published by an earlier launch).
  struct SyncCtx {
    ws_sync_options o{};
    int pa = 0, na = 1;
    cudaEvent_t* ev = nullptr;
    uint32_t launches = 0;
    bool streamed_apply = false;  // K1's streamed-apply instantiation ran
  };
  ws_status sync_begin(SyncCtx& x, const ws_sync_options& o, cudaStream_t s,
                       const void* next_host);
  // K1 (every exchange round's segments back to back) + local route
  ws_status sync_encode(SyncCtx& x, cudaStream_t s, bool run_local = true);
  ws_status sync_finish(SyncCtx& x, cudaStream_t s, uint64_t* nnz_host, ws_report* report);
  // sync_step without the grouped-engine check
  ws_status sync_step_impl(const ws_sync_options& o, cudaStream_t s, const void* next_host,
                           uint64_t* nnz_host, ws_report* report);
  int exchange_rounds() const;
  // P2P syncs without overlapped rounds (one round, or sparse=False): the
  // stream the local route runs on beside the exchange (null when there is
  // none), and the fork / join around it
  cudaStream_t exchange_side_stream() const;
  ws_status exchange_fork(cudaStream_t s, cudaStream_t side);
  ws_status exchange_join(cudaStream_t s, cudaStream_t side);
  ws_status exchange_pack(const ws_sync_options& o, int next_arena, int round, cudaStream_t s,
                          uint32_t* launches);
  ws_status exchange_apply(int round, cudaStream_t s, uint32_t* launches);
  ws_status exchange_end(cudaStream_t s);
  ws_status exchange_mark_pack(cudaStream_t s);
  ws_status exchange_bytes(uint64_t* sent_record_bytes, uint64_t* sent_dense_bytes,
                           uint64_t* recv_record_bytes);
  bool exchange_needs_resize(const ws_sync_options& o) const;
  // grows the P2P receive regions for o.density_threshold (collective)
  ws_status exchange_prepare(const ws_sync_options& o);
  ws_status init_comm(const uint8_t* unique_id, wsync::GroupShared* group);  // exchange.cu
  int device() const { return device_; }
  int world() const { return plan_.world(); }
  int rank() const { return plan_.rank(); }
  bool grouped() const { return grouped_; }
  bool connected() const { return comm_ != nullptr; }
  bool bound() const { return arena[0] && arena[1] && serve; }

 private:
  bool grouped_ = false;
  uint32_t last_launches_ = 0;
  bool last_streamed_apply_ = false;
  ws_status report_of(const SyncCtx& x, ws_report* report);
  ws_status ensure_records(double threshold, int sparse);
  ws_status init_p2p();
  ws_status p2p_size(double t);  // receive regions for syncs with threshold <= t
  ws_status size_send(const std::vector<uint64_t>& region_cap);
  ws_status size_recv(uint64_t records);
  void destroy_comm();
  ws_status exchange_begin(cudaStream_t s, uint32_t* launches);  // P2P "reached step" flags
  ws_status exchange_status() const;                             // faults seen by the kernels
  wsync::P2PArgs round_args(int round) const;
  // R > 1 (P2P): K1 round by round on a high-priority stream, round r's
  // exchange on a low-priority stream overlapping the encode of round r + 1
  ws_status sync_rounds(const ws_sync_options& o, int pa, int na, cudaStream_t s,
                        uint32_t* launches, cudaEvent_t* ev);
  wsync::EncodeArgs encode_args(int pa, int na);
  ws_status launch_fixup(const wsync::EncodeArgs& a, int seg_begin, int seg_end, cudaStream_t s,
                         uint32_t* launches);
  ws_status local_route(const ws_sync_options& o, int pa, int na, cudaStream_t s,
                        uint32_t* launches);
  bool overlap_ = true;  // WSYNC_OVERLAP=0 runs the rounds back to back
  ws_status exchange_round(const ws_sync_options& o, int next_arena, int round, cudaStream_t s,
                           uint32_t* launches);
  // P2P + bf16 + direct dense: K1 stores the remote records itself (fills a.remote)
  ws_status exchange_fuse_k1(wsync::EncodeArgs& a, cudaStream_t s);
  ws_status exchange(const ws_sync_options& o, int next_arena, cudaStream_t s, uint32_t* launches);
  uint32_t next_epoch();

  wsync::Plan plan_;
  int device_;
  int dtype_;
  int nseg_;
  uint32_t ntiles_ = 0;
  uint32_t epoch_ = 0;
  int route_grid_ = 0;

  // encode tables (device)
  wsync::SegDev* d_segs_ = nullptr;
  uint32_t* d_tile0_ = nullptr;
  uint32_t* d_tile_seg_ = nullptr;
  uint32_t* d_seg_mode_ = nullptr;   // 1: counted only this sync (dense the last one)
  unsigned long long* d_fill_ = nullptr;
  uint32_t* d_fix_list_ = nullptr;   // fixup pass super-tiles
  uint32_t* d_fix_n_ = nullptr;
  bool count_only_ = true;           // WSYNC_COUNT_ONLY=0 disables the prediction
  void* d_spill_ = nullptr;          // K1 spill scratch (encode_spill_bytes)
  uint32_t spill_blocks_ = 0;
  uint32_t* d_tile_cnt_ = nullptr;   // K1's unordered layout (see EncodeArgs)
  uint32_t* d_tile_base_ = nullptr;
  uint32_t tile_elems_ = 0;
  std::vector<uint32_t> plan_tile0_;
  // ascending stream of one segment, compacted on demand (segment_delta)
  uint32_t* d_seq_idx_ = nullptr;
  void* d_seq_val_ = nullptr;
  uint64_t seq_alloc_ = 0;
  void fill_tiles(wsync::RouteSideArgs& r) const {
    r.tile0 = d_tile0_;
    r.tile_cnt = d_tile_cnt_;
    r.tile_base = d_tile_base_;
    r.tile_elems = tile_elems_;
  }
  unsigned long long* d_status_ = nullptr;
  unsigned int* d_ticket_ = nullptr;
  uint64_t* d_nnz_ = nullptr;
  uint64_t* d_cap_ = nullptr;
  uint64_t* d_rec_ = nullptr;
  uint64_t* d_base_ = nullptr;
  std::vector<wsync::SegDev> segs_;
  double cur_threshold_ = -1.0;
  int cur_sparse_ = -1;

  // record buffers
  uint32_t* d_idx_ = nullptr;
  void* d_val_ = nullptr;
  uint64_t rec_alloc_ = 0;

  // local routes
  wsync::LocalEntry* d_local_ = nullptr;
  wsync::FuseEntry* d_fuse_ = nullptr;
  uint32_t* d_fuse_on_ = nullptr;
  uint32_t sa_div_ = 0;  // K1 streamed apply for fused bf16 segments denser than 1/sa_div_ (0: off)
  uint64_t* h_sa_ = nullptr;  // mapped [2]: fused elements set to stream / RMW by the last worklist
  uint64_t* d_sa_ = nullptr;
  bool sa_force_ = false;     // ablation: always the streamed-apply instantiation
  bool sa_env_ = false;       // WSYNC_SA_DIV given explicitly
  // Off by default under overlapped exchange rounds: the serving stream then
  // competes with the receive scatter for HBM (measured at N = 4: 3.77 ->
  // 3.92 ms in round 1; final build 3.21 -> 3.24 ms config 2, 10.26 -> 10.29
  // ms config 3, profiles/r02_sa_under_rounds_n4.jsonl).
  uint32_t sa_div() const { return (sa_env_ || exchange_rounds() <= 1) ? sa_div_ : 0u; }
  bool fuse_apply_ = true;  // K1 applies local sparse records (WSYNC_NO_FUSED_APPLY=1 disables)
  int nlocal_ = 0;
  uint64_t* d_unit_off_ = nullptr;

  // per-step stage events: [start, after H2D, after encode, after local
  // apply, after exchange, end, after the pack (single-round exchange)]; a
  // ring so timed loops need no sync.
  static constexpr int kRing = 256;
  cudaEvent_t (*ring_)[7] = nullptr;
  uint32_t ring_steps_ = 0;    // steps recorded since reset
  uint32_t ring_head_ = 0;     // next slot
  uint32_t launch_total_ = 0;
  uint32_t pack_steps_ = 0;    // steps since reset whose pack event was recorded
  bool pack_ev_ = false;       // this step recorded ring slot 6
  cudaStream_t last_stream_ = nullptr;
  bool last_sparse_ = true;
  int last_next_arena_ = 1;
  std::vector<uint64_t> h_nnz_;
  uint64_t* h_nnz_pinned_ = nullptr;

  // multi-GPU state (exchange.cu)
  struct Comm;
  Comm* comm_ = nullptr;
  uint64_t pulled_bytes_ = 0;
  uint64_t pushed_wire_bytes_ = 0;
};
