// exchange.cu -- the cross-GPU part of a sync (K3 over NVLink / NVSwitch).
//
// The reference moves every pushed shard through a relay: the pusher puts
// encoded buckets (engine.cpp:136-148) and each puller fetches the shards its
// serving rank needs (plan_pulls, engine.cpp:158-197), then reslices and
// applies them (:209-218).  On one box the relay is replaced by one exchange
// per sync:
//   1. pack (kernels_route.cu): the records of every route to a serving
//      coordinate held by another GPU are re-indexed into that coordinate's
//      serving arena and appended to the coordinate's send region as
//      self-describing wire records (set records for dense-fallback shards);
//   2. the per-coordinate record counts are all-gathered (8 bytes per
//      coordinate per rank), so every rank knows what it will receive;
//   3. one grouped ncclSend/ncclRecv moves each region to every replica of
//      its coordinate (the same region goes to all replicas);
//   4. the receiver scatters the records into its serving arena in place.
// Region and receive capacities are sized from the static plan for the
// worst case (every element of every route sent dense), so no step can
// overflow.
#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "capi_util.h"
#include "engine.h"
#include "fabric.h"

using namespace wsync;

#define WS_CUDA_TRY(expr, what)                          \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_status(_e, what); \
  } while (0)

#define WS_NCCL_TRY(expr, what)                                                          \
  do {                                                                                   \
    ncclResult_t _r = (expr);                                                            \
    if (_r != ncclSuccess)                                                               \
      return set_error(WS_NCCL, std::string(what) + ": " + ncclGetErrorString(_r));      \
  } while (0)

struct ws_engine::Comm {
  ncclComm_t comm = nullptr;                     // one process per GPU (not in a ws_group)
  std::unique_ptr<Fabric> fab;                   // how peers map each other's memory
  int world = 1, rank = 0, coords = 1;
  // remote routes (this rank as a sender)
  LocalEntry* d_entries = nullptr;
  int nentries = 0;
  uint64_t* d_unit_off = nullptr;
  // NCCL-fallback exchange (no CUDA IPC between the GPUs)
  std::vector<uint64_t> region_off, region_cap;  // per coordinate, records
  uint64_t* d_region_off = nullptr;
  uint64_t* d_region_cap = nullptr;
  unsigned long long* d_region_cnt = nullptr;
  uint64_t* d_allcnt = nullptr;                  // [world][coords]
  uint64_t* h_allcnt = nullptr;                  // pinned copy
  uint32_t* d_err = nullptr;
  uint32_t* h_err = nullptr;                     // pinned copy, refreshed every sync
  void* d_send = nullptr;
  void* d_recv = nullptr;
  uint64_t send_cap = 0, recv_cap = 0;           // records
  std::vector<std::vector<int>> dests;           // per coordinate: receiving ranks != me
  // peer-memory mode
  bool p2p = false;
  void* d_head = nullptr;                        // [mailbox | count slots], fixed size
  void* d_rec = nullptr;                         // receive regions, sized by the threshold
  std::vector<void*> peer_head, peer_rec, peer_serve;  // every rank's, mapped here
  double sized_t = -1.0;                         // density threshold the regions hold
  double want_t = kDefaultThreshold;             // the largest a sync has asked for
  P2PArgs pargs{};
  std::vector<int> mine;                         // my remote routes (indices into routes())
  std::vector<EntryDest> edest;                  // host copy of d_edest
  std::vector<RemoteMap> rmaps;                  // K1's view of them, grouped by segment
  std::vector<int> rmap_entry;                   // remote entry of every rmaps element
  uint32_t epoch = 0;
  RemoteMap* d_rmaps = nullptr;
  uint32_t* d_rseg_first = nullptr;
  bool k1_emit = false;                          // this sync's records went out from K1
  EntryDest* d_edest = nullptr;
  unsigned int* d_ent_cnt = nullptr;
  int nsend_entries = 0;
  // exchange rounds (P2P): K1 encodes segment runs round by round and round
  // r's pack/apply overlap the encode of round r + 1
  int R = 1;
  int overlap_sms = 28;                          // SMs left to the exchange beside K1
  uint64_t step = 0;                             // syncs so far (epochs derive from it)
  std::vector<int> ent_first;                    // R + 1: my remote entries per round
  std::vector<int> seg_first;                    // R + 1: my segments per round
  std::vector<uint32_t> tile_first;              // R + 1: my super-tiles per round
  struct RoundRecv {
    RecvEntry* d_rentries = nullptr;
    uint64_t* d_units = nullptr;
    int n = 0;
    uint32_t mask = 0;                           // sources with entries in this round
    int32_t dest_rank[kMaxWorld][kMaxReplicas];  // where my round-r entries go
  };
  std::vector<RoundRecv> rr;
  cudaStream_t s_enc = nullptr, s_xchg = nullptr;  // high / low priority (R > 1)
  std::vector<cudaEvent_t> ev_round;               // K1 round r done
  cudaEvent_t ev_start = nullptr, ev_xdone = nullptr, ev_encdone = nullptr;
  // syncs without exchange rounds: the local route's stream beside the exchange
  cudaStream_t s_side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

  void release_peers(std::vector<void*>& v) {
    for (int g = 0; g < (int)v.size(); ++g)
      if (g != rank && v[g] && fab) fab->release(v[g]);
    v.clear();
  }
  ~Comm() {
    release_peers(peer_head);
    release_peers(peer_rec);
    release_peers(peer_serve);
    cudaFree(d_head);
    cudaFree(d_rec);
    cudaFree(d_edest);
    cudaFree(d_rmaps);
    cudaFree(d_rseg_first);
    cudaFree(d_ent_cnt);
    for (auto& x : rr) {
      cudaFree(x.d_rentries);
      cudaFree(x.d_units);
    }
    for (auto& e : ev_round) cudaEventDestroy(e);
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_xdone) cudaEventDestroy(ev_xdone);
    if (ev_encdone) cudaEventDestroy(ev_encdone);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (s_side) cudaStreamDestroy(s_side);
    if (s_enc) cudaStreamDestroy(s_enc);
    if (s_xchg) cudaStreamDestroy(s_xchg);
    cudaFree(d_entries);
    cudaFree(d_unit_off);
    cudaFree(d_region_off);
    cudaFree(d_region_cap);
    cudaFree(d_region_cnt);
    cudaFree(d_allcnt);
    cudaFree(d_err);
    if (h_err) cudaFreeHost(h_err);
    cudaFree(d_send);
    cudaFree(d_recv);
    if (h_allcnt) cudaFreeHost(h_allcnt);
    fab.reset();
    if (comm) ncclCommDestroy(comm);
  }
};

namespace wsync {

// Static exchange sizes of rank `me` (records): send capacity per serving
// coordinate and receive capacity from every other rank.
void exchange_caps(const Plan& plan, int me, std::vector<uint64_t>* send_cap,
                   std::vector<uint64_t>* recv_cap) {
  const int C = plan.coords(), W = plan.world();
  send_cap->assign(C, 0);
  recv_cap->assign(W, 0);
  const int my_coord = plan.coord_of_rank(me);
  for (int r = 0; r < W; ++r) {
    for (const Route& rt : plan.routes_of(r)) {
      const bool remote_dest = plan.replicas() > 1 || rt.coord != plan.coord_of_rank(r);
      if (!remote_dest) continue;  // only the sender itself holds that coordinate
      if (r == me) (*send_cap)[rt.coord] += rt.overlap;
      else if (rt.coord == my_coord) (*recv_cap)[r] += rt.overlap;
    }
  }
}

// ---- fabrics ------------------------------------------------------------------

namespace {
// Base of the allocation holding `p` (driver entry point; the library does
// not link libcuda).  IPC handles are per allocation, and the serving arena
// may be a view into a larger caller allocation.
bool allocation_base(void* p, void** base) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<Fn>(f);
  }();
  if (!fn) return false;
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return false;
  *base = reinterpret_cast<void*>(b);
  return true;
}

struct IpcEntry {
  cudaIpcMemHandle_t h;
  uint64_t offset;
  uint32_t ok, present;
};
}  // namespace

ws_status NcclFabric::share(void* p, std::vector<void*>* out) {
  const int W = world_, me = rank_;
  IpcEntry mine{};
  if (p) {
    mine.present = 1;
    void* base = nullptr;
    if (allocation_base(p, &base) && cudaIpcGetMemHandle(&mine.h, base) == cudaSuccess) {
      mine.offset = static_cast<char*>(p) - static_cast<char*>(base);
      mine.ok = 1;
    }
    cudaGetLastError();
  } else {
    mine.ok = 1;
  }
  IpcEntry* d = nullptr;
  if (cudaMalloc(&d, (size_t)W * sizeof(IpcEntry)) != cudaSuccess)
    return set_error(WS_CUDA, "fabric: cudaMalloc");
  cudaMemcpy(d + me, &mine, sizeof(mine), cudaMemcpyHostToDevice);
  cudaStream_t s0;
  cudaStreamCreate(&s0);
  ncclResult_t nr = ncclAllGather(d + me, d, sizeof(IpcEntry), ncclUint8, comm_, s0);
  cudaStreamSynchronize(s0);
  cudaStreamDestroy(s0);
  std::vector<IpcEntry> all(W);
  cudaMemcpy(all.data(), d, (size_t)W * sizeof(IpcEntry), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (nr != ncclSuccess) return set_error(WS_NCCL, "fabric: handle all-gather failed");
  out->assign(W, nullptr);
  int ok = 1;
  for (int g = 0; g < W; ++g) ok &= all[g].ok ? 1 : 0;
  for (int g = 0; g < W && ok; ++g) {
    if (!all[g].present) continue;
    if (g == me) {
      (*out)[g] = p;
      continue;
    }
    void* q = nullptr;
    if (cudaIpcOpenMemHandle(&q, all[g].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    (*out)[g] = static_cast<char*>(q) + all[g].offset;
  }
  ws_status st = all_min(&ok);  // every rank must agree, or one would wait forever for a flag
  if (st == WS_OK && ok) return WS_OK;
  for (int g = 0; g < W; ++g)
    if (g != me && (*out)[g]) release((*out)[g]);
  out->assign(W, nullptr);
  return st != WS_OK ? st : set_error(WS_CUDA, "fabric: CUDA IPC unavailable between the ranks");
}

void NcclFabric::release(void* p) {
  void* base = nullptr;
  if (allocation_base(p, &base)) cudaIpcCloseMemHandle(base);
  cudaGetLastError();
}

ws_status NcclFabric::all_min(int* v) {
  int* d = nullptr;
  if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) return set_error(WS_CUDA, "fabric: cudaMalloc");
  cudaMemcpy(d, v, sizeof(int), cudaMemcpyHostToDevice);
  cudaStream_t s0;
  cudaStreamCreate(&s0);
  ncclResult_t nr = ncclAllReduce(d, d, 1, ncclInt32, ncclMin, comm_, s0);
  cudaStreamSynchronize(s0);
  cudaStreamDestroy(s0);
  cudaMemcpy(v, d, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return nr == ncclSuccess ? WS_OK : set_error(WS_NCCL, "fabric: all-reduce failed");
}

void GroupShared::barrier() {
  std::unique_lock<std::mutex> lk(m);
  const unsigned gen = generation;
  if (++arrived == world) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return generation != gen; });
  }
}

ws_status GroupFabric::share(void* p, std::vector<void*>* out) {
  g_->slots[rank_] = p;
  g_->barrier();
  *out = g_->slots;
  g_->barrier();
  return WS_OK;
}

ws_status GroupFabric::all_min(int* v) {
  g_->ints[rank_] = *v;
  g_->barrier();
  int m = *v;
  for (int x : g_->ints) m = std::min(m, x);
  g_->barrier();
  *v = m;
  return WS_OK;
}

}  // namespace wsync

namespace {
// Remote routes of rank g (their coordinate has a replica other than g),
// ordered by segment: the order of g's remote entries on every rank.
std::vector<int> remote_routes(const Plan& plan, int g) {
  std::vector<int> out;
  const auto& rs = plan.routes_of(g);
  for (int i = 0; i < (int)rs.size(); ++i)
    if (plan.replicas() > 1 || rs[i].coord != plan.coord_of_rank(g)) out.push_back(i);
  std::stable_sort(out.begin(), out.end(), [&](int x, int y) { return rs[x].seg < rs[y].seg; });
  return out;
}
// Exchange round of each of rank g's segments: R contiguous runs of segments
// with about equal super-tile counts (K1 encodes them round by round).
std::vector<int> segment_rounds(const Plan& plan, int g, int R, uint32_t tile) {
  const auto& segs = plan.segments_of(g);
  uint64_t total = 0, acc = 0;
  for (const Segment& sg : segs) total += (sg.n + tile - 1) / tile;
  std::vector<int> out(segs.size(), 0);
  for (size_t i = 0; i < segs.size(); ++i) {
    out[i] = (int)std::min<uint64_t>(R - 1, acc * R / std::max<uint64_t>(1, total));
    acc += (segs[i].n + tile - 1) / tile;
  }
  return out;
}
struct RecvLayout {
  std::vector<std::pair<int, int>> entries;  // (source rank, its remote-entry index)
  std::vector<uint64_t> off, cap;            // bytes (p2p_region_bytes), records
  std::vector<uint64_t> dst_base;            // the route's destination shard offset
  std::vector<int> round;
  uint64_t records = 0;
  uint64_t bytes = 0;                        // receive area
  size_t head = 0;                           // mailbox + count slots, bytes
};
// Records one remote entry (route r of rank g) can carry in a sync whose
// density threshold is at most t: a sparse source segment holds at most
// sparse_capacity(n, t) records, and with direct dense boxes a dense one
// sends none -- so the region needs min(overlap, that), not the worst case
// of every routed element as a record (t >= 1).
uint64_t entry_capacity(const Plan& plan, int g, const Route& r, double t) {
  if (t >= 1.0) return r.overlap;
  const uint64_t n = plan.segments_of(g)[r.seg].n;
  return std::min<uint64_t>(r.overlap, sparse_capacity(n, t));
}
RecvLayout recv_layout(const Plan& plan, int q, int R, uint32_t tile, double t) {
  RecvLayout L;
  const int k = plan.coord_of_rank(q);
  for (int g = 0; g < plan.world(); ++g) {
    if (g == q) continue;
    const std::vector<int> rr = remote_routes(plan, g);
    const std::vector<int> sr = segment_rounds(plan, g, R, tile);
    for (int e = 0; e < (int)rr.size(); ++e) {
      const Route& r = plan.routes_of(g)[rr[e]];
      if (r.coord != k) continue;
      const uint64_t cap = entry_capacity(plan, g, r, t);
      L.entries.emplace_back(g, e);
      L.off.push_back(L.bytes);
      L.cap.push_back(cap);
      L.dst_base.push_back(r.dst_offset);
      L.round.push_back(sr[r.seg]);
      L.records += cap;
      L.bytes += p2p_region_bytes(plan.dtype(), cap);
    }
  }
  L.head = kMailboxBytes + ((L.entries.size() * 4 + 255) / 256) * 256;
  return L;
}
// Exchange rounds of a plan: overlapping the exchange with K1 pays only when
// the exchange is heavy, because K1 gives up SMs to it in every round after
// the first.  The measure is the largest "remote share" over the ranks:
// elements a rank stores into peers per element it encodes (every route once
// per replica, minus the copy its own serving shard holds).  Measured (1%
// unless noted): config 2 (share 0.15 at N = 2, 1.15 at N = 4) gains from 3
// rounds only at N = 4 (4.10 -> 3.74 ms); config 3 (share 1.0, 0.5%) gains
// at N = 2 too (20.89 -> 20.35 ms); config 4 (expert-sharded, share 0.005
// at N = 4) loses 18% with them (7.67 vs 9.38 ms).
double remote_share(const Plan& plan) {
  double worst = 0;
  for (int g = 0; g < plan.world(); ++g) {
    uint64_t train = 0, remote = 0;
    for (const Segment& sg : plan.segments_of(g)) train += sg.n;
    for (const Route& r : plan.routes_of(g))
      remote += r.overlap * (uint64_t)plan.replicas() -
                (r.coord == plan.coord_of_rank(g) ? r.overlap : 0);
    if (train) worst = std::max(worst, (double)remote / (double)train);
  }
  return worst;
}
int default_rounds(const Plan& plan) {
  int R = remote_share(plan) >= 0.5 ? 3 : 1;
  if (const char* e = getenv("WSYNC_ROUNDS")) R = std::max(1, std::min(kMaxRounds, atoi(e)));
  return R;
}
// SMs K1 leaves to the exchange kernels in rounds after the first: 28 at a
// remote share near 1 (config 2 at N = 4: 16/20/28/36 SMs -> 3.41/3.28/3.20/
// 3.36 ms), 40 from a share of 2 (FSDP4 -> TP1 x 4, share 3, the stand-in
// for config 2 at N = 8: 4.61 ms with 28, 4.54 with 40, 4.75 with 56).
int overlap_sms(const Plan& plan) {
  return remote_share(plan) >= 2.0 ? 40 : 28;
}
}  // namespace

ws_status ws_engine::init_comm(const uint8_t* unique_id, GroupShared* group) {
  if (plan_.world() == 1) return WS_OK;
  if (!unique_id && !group)
    return set_error(WS_INVALID_ARGUMENT, "multi-GPU engine needs an NCCL unique id");
  auto* c = new Comm;
  comm_ = c;
  c->world = plan_.world();
  c->rank = plan_.rank();
  c->coords = plan_.coords();
  if (group) {
    c->fab.reset(new GroupFabric(c->world, c->rank, group));
  } else {
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    WS_NCCL_TRY(ncclCommInitRank(&c->comm, c->world, id, c->rank), "ncclCommInitRank");
    c->fab.reset(new NcclFabric(c->world, c->rank, c->comm));
  }

  // remote routes: every route whose coordinate has a replica other than me
  const int me = plan_.rank();
  std::vector<LocalEntry> remote;
  const auto& segs = plan_.segments();
  for (int ri : remote_routes(plan_, me)) {
    const Route& r = plan_.routes()[ri];
    const ParamMeta& p = plan_.manifest()[r.dst.param];
    LocalEntry e = make_local_entry(dtype_, p.shape.data(), (int)p.shape.size(), r.seg,
                                    segs[r.seg].shard.d, r.dst.d, r.dst_offset);
    e.coord = r.coord;
    remote.push_back(e);
  }
  c->nentries = (int)remote.size();
  WS_CUDA_TRY(cudaMalloc(&c->d_entries, std::max<size_t>(1, remote.size()) * sizeof(LocalEntry)),
              "cudaMalloc");
  if (!remote.empty())
    WS_CUDA_TRY(cudaMemcpy(c->d_entries, remote.data(), remote.size() * sizeof(LocalEntry),
                           cudaMemcpyHostToDevice),
                "H2D");
  WS_CUDA_TRY(cudaMalloc(&c->d_unit_off, (remote.size() + kMaxRounds + 1) * 8), "cudaMalloc");
  c->dests.assign(c->coords, {});
  for (int g = 0; g < c->world; ++g)
    if (g != me) c->dests[plan_.coord_of_rank(g)].push_back(g);
  WS_CUDA_TRY(cudaMalloc(&c->d_region_off, c->coords * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&c->d_region_cap, c->coords * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&c->d_region_cnt, c->coords * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&c->d_allcnt, (size_t)c->world * c->coords * 8), "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&c->d_err, 4), "cudaMalloc");
  WS_CUDA_TRY(cudaMemset(c->d_err, 0, 4), "cudaMemset");
  WS_CUDA_TRY(cudaMallocHost(&c->h_err, 4), "cudaMallocHost");
  *c->h_err = 0;
  WS_CUDA_TRY(cudaMallocHost(&c->h_allcnt, (size_t)c->world * c->coords * 8), "cudaMallocHost");
  const char* mode = getenv("WSYNC_EXCHANGE");
  const bool fits = c->world <= kMaxWorld && c->coords <= kMaxWorld &&
                    plan_.replicas() <= kMaxReplicas;
  if (group && !fits) return set_error(WS_INVALID_ARGUMENT, "group: world beyond kMaxWorld");
  if (group || (fits && !(mode && std::string(mode) == "nccl"))) {
    ws_status st = init_p2p();
    if (st == WS_OK || group) return st;
    c->p2p = false;  // fall back to the NCCL exchange (e.g. no CUDA IPC between these GPUs)
  }
  // NCCL exchange: buffers start at a fraction of the worst case (every routed
  // element sent dense) and grow on demand: the all-gathered counts tell every
  // rank what it must send and receive before any byte moves (see exchange()).
  std::vector<uint64_t> send_full, recv_full;
  exchange_caps(plan_, me, &send_full, &recv_full);
  double frac = 0.25;
  if (const char* f = ablation_env("WSYNC_EXCHANGE_FRACTION")) frac = atof(f);
  std::vector<uint64_t> region_cap(c->coords);
  for (int k = 0; k < c->coords; ++k)
    region_cap[k] = send_full[k] ? std::max<uint64_t>(4096, (uint64_t)(frac * send_full[k])) : 0;
  uint64_t recv_full_total = 0;
  for (auto v : recv_full) recv_full_total += v;
  ws_status st = size_send(region_cap);
  if (st != WS_OK) return st;
  return size_recv(recv_full_total ? std::max<uint64_t>(4096, (uint64_t)(frac * recv_full_total)) : 0);
}

// Peer-memory exchange.  Every rank owns two shared allocations: the head
// [mailbox | one count slot per receive region], fixed for the plan, and
// the receive area, one region per (source rank, remote entry of that
// source) whose coordinate is this rank's -- sized by p2p_size for a density
// threshold.  The layouts of all ranks follow from the static plan, so the
// only data exchanged is the fabric's handles.  This sets up the head and
// the static tables; regions are sized when the serving arena is bound.
ws_status ws_engine::init_p2p() {
  Comm* c = comm_;
  const int me = c->rank, W = c->world;
  const int R = default_rounds(plan_);
  c->R = R;
  c->overlap_sms = overlap_sms(plan_);
  const uint32_t tile = encode_tile_elems(dtype_);
  const RecvLayout L = recv_layout(plan_, me, R, tile, 1.0);
  int ok = cudaMalloc(&c->d_head, L.head) == cudaSuccess &&
           cudaMemset(c->d_head, 0, L.head) == cudaSuccess;
  cudaGetLastError();
  ws_status st = c->fab->all_min(&ok);
  if (st != WS_OK || !ok) {
    cudaFree(c->d_head);
    c->d_head = nullptr;
    return st != WS_OK ? st : set_error(WS_CUDA, "p2p: mailbox allocation failed");
  }
  st = c->fab->share(c->d_head, &c->peer_head);
  if (st != WS_OK) {
    cudaFree(c->d_head);
    c->d_head = nullptr;
    return st;
  }

  P2PArgs& P = c->pargs;
  P = P2PArgs{};
  P.on = 1;
  P.world = W;
  P.rank = me;
  P.mailbox = static_cast<unsigned long long*>(c->d_head);
  for (int g = 0; g < W; ++g)
    P.peer_mailbox[g] = static_cast<unsigned long long*>(c->peer_head[g]);
  for (int k = 0; k < kMaxWorld; ++k)
    for (int r = 0; r < kMaxReplicas; ++r) P.dest_rank[k][r] = -1;
  // sender: only the coordinates I send to get destinations (their ranks ack
  // exactly the sources they expect)
  c->mine = remote_routes(plan_, me);
  const std::vector<int>& mine = c->mine;
  std::vector<char> sends_to(c->coords, 0);
  for (int e : mine) sends_to[plan_.routes_of(me)[e].coord] = 1;
  for (int k = 0; k < c->coords; ++k) {
    if (!sends_to[k]) continue;
    int r = 0;
    for (int g : c->dests[k]) P.dest_rank[k][r++] = g;
  }
  WS_CUDA_TRY(cudaMalloc(&c->d_edest, std::max<size_t>(1, mine.size()) * sizeof(EntryDest)),
              "cudaMalloc");
  WS_CUDA_TRY(cudaMalloc(&c->d_ent_cnt, std::max<size_t>(1, mine.size()) * 4), "cudaMalloc");
  {  // the same routes as K1 sees them, grouped by segment (regions filled by p2p_size)
    const auto& segs = plan_.segments();
    std::vector<std::vector<std::pair<RemoteMap, int>>> by_seg(segs.size());
    for (int e = 0; e < (int)mine.size(); ++e) {
      const Route& rt = plan_.routes_of(me)[mine[e]];
      const ParamMeta& p = plan_.manifest()[rt.dst.param];
      const LocalEntry le = make_local_entry(dtype_, p.shape.data(), (int)p.shape.size(), rt.seg,
                                             segs[rt.seg].shard.d, rt.dst.d, rt.dst_offset);
      RemoteMap m;
      std::memset(&m, 0, sizeof(m));
      m.identity = le.identity;
      m.keep_lo = le.keep_lo;
      m.keep_hi = le.keep_hi;
      m.shift = le.shift;
      m.dst_base = le.dst_base;
      m.map = le.map;
      m.cnt = c->d_ent_cnt + e;
      by_seg[rt.seg].emplace_back(m, e);
    }
    std::vector<uint32_t> first(segs.size() + 1, 0);
    for (size_t sg = 0; sg < segs.size(); ++sg) {
      first[sg] = (uint32_t)c->rmaps.size();
      for (auto& me_ : by_seg[sg]) {
        c->rmaps.push_back(me_.first);
        c->rmap_entry.push_back(me_.second);
      }
    }
    first[segs.size()] = (uint32_t)c->rmaps.size();
    WS_CUDA_TRY(cudaMalloc(&c->d_rmaps, std::max<size_t>(1, c->rmaps.size()) * sizeof(RemoteMap)),
                "cudaMalloc");
    WS_CUDA_TRY(cudaMalloc(&c->d_rseg_first, first.size() * 4), "cudaMalloc");
    WS_CUDA_TRY(cudaMemcpy(c->d_rseg_first, first.data(), first.size() * 4,
                           cudaMemcpyHostToDevice), "H2D");
  }
  // rounds of my segments / entries (sender side)
  {
    const std::vector<int> sr = segment_rounds(plan_, me, R, tile);
    const auto& segs = plan_.segments();
    c->seg_first.assign(R + 1, (int)segs.size());
    c->tile_first.assign(R + 1, 0);
    c->ent_first.assign(R + 1, (int)mine.size());
    uint32_t t = 0;
    for (int r = R - 1; r >= 0; --r)
      for (int i = (int)segs.size() - 1; i >= 0; --i)
        if (sr[i] >= r) c->seg_first[r] = i;
    for (size_t i = 0; i < segs.size(); ++i) {
      for (int r = 0; r <= R; ++r)
        if (c->seg_first[r] == (int)i) c->tile_first[r] = t;
      t += (uint32_t)((segs[i].n + tile - 1) / tile);
    }
    for (int r = 0; r <= R; ++r)
      if (c->seg_first[r] == (int)segs.size()) c->tile_first[r] = t;
    for (int r = R - 1; r >= 0; --r)
      for (int e = (int)mine.size() - 1; e >= 0; --e)
        if (sr[plan_.routes_of(me)[mine[e]].seg] >= r) c->ent_first[r] = e;
  }
  // receiver: which sources send in which round (region offsets: p2p_size)
  c->rr.assign(R, Comm::RoundRecv{});
  for (int r = 0; r < R; ++r) {
    Comm::RoundRecv& X = c->rr[r];
    for (int k = 0; k < kMaxWorld; ++k)
      for (int q = 0; q < kMaxReplicas; ++q) X.dest_rank[k][q] = -1;
    std::vector<char> to(c->coords, 0);
    for (int e = c->ent_first[r]; e < c->ent_first[r + 1]; ++e)
      to[plan_.routes_of(me)[mine[e]].coord] = 1;
    for (int k = 0; k < c->coords; ++k) {
      if (!to[k]) continue;
      int q = 0;
      for (int g : c->dests[k]) X.dest_rank[k][q++] = g;
    }
    for (int j = 0; j < (int)L.entries.size(); ++j)
      if (L.round[j] == r) {
        ++X.n;
        X.mask |= 1u << L.entries[j].first;
      }
    P.expect_mask |= X.mask;
    WS_CUDA_TRY(cudaMalloc(&X.d_rentries, std::max<size_t>(1, X.n) * sizeof(RecvEntry)),
                "cudaMalloc");
    WS_CUDA_TRY(cudaMalloc(&X.d_units, (X.n + 1) * 8), "cudaMalloc");
  }
  if (R > 1) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    WS_CUDA_TRY(cudaStreamCreateWithPriority(&c->s_enc, cudaStreamNonBlocking, hi), "stream");
    WS_CUDA_TRY(cudaStreamCreateWithPriority(&c->s_xchg, cudaStreamNonBlocking, lo), "stream");
    c->ev_round.resize(R);
    for (auto& e : c->ev_round) WS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "ev");
    WS_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming), "ev");
    WS_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_xdone, cudaEventDisableTiming), "ev");
    WS_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_encdone, cudaEventDisableTiming), "ev");
  }
  if (!grouped_) {  // syncs without rounds (one round, or sparse=False)
    WS_CUDA_TRY(cudaStreamCreateWithFlags(&c->s_side, cudaStreamNonBlocking), "stream");
    WS_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "ev");
    WS_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "ev");
  }
  P.edest = c->d_edest;
  P.ent_cnt = c->d_ent_cnt;
  P.recv_cnt = reinterpret_cast<const uint32_t*>(static_cast<char*>(c->d_head) + kMailboxBytes);
  P.err = c->d_err;
  if (const char* d = ablation_env("WSYNC_P2P_DEBUG")) P.debug = atoi(d);
  c->nsend_entries = (int)mine.size();
  WS_CUDA_TRY(cudaMemset(c->d_err, 0, 4), "memset");
  c->p2p = true;
  return WS_OK;
}

// (Re)sizes every rank's receive regions for syncs with density threshold
// <= t (t >= 1: the worst case, every routed element a record) and rebuilds
// the tables that point into them.  Collective; every rank's earlier syncs
// are complete before any region is freed.
ws_status ws_engine::p2p_size(double t) {
  Comm* c = comm_;
  const int me = c->rank, W = c->world, R = c->R;
  const uint32_t tile = encode_tile_elems(dtype_);
  int ok = cudaDeviceSynchronize() == cudaSuccess;
  ws_status st = c->fab->all_min(&ok);  // every rank's syncs so far are done
  if (st != WS_OK) return st;
  if (!ok) return set_error(WS_CUDA, "p2p: a rank failed before resizing its receive regions");
  c->release_peers(c->peer_rec);
  cudaFree(c->d_rec);
  c->d_rec = nullptr;
  c->sized_t = -1.0;
  std::vector<RecvLayout> lay(W);
  for (int q = 0; q < W; ++q) lay[q] = recv_layout(plan_, q, R, tile, t);
  const size_t bytes = std::max<uint64_t>(16, lay[me].bytes);
  ok = cudaMalloc(&c->d_rec, bytes) == cudaSuccess;
  cudaGetLastError();
  st = c->fab->all_min(&ok);
  if (st != WS_OK || !ok) {
    cudaFree(c->d_rec);
    c->d_rec = nullptr;
    return st != WS_OK ? st
                       : set_error(WS_CAPACITY, "p2p: receive regions for density_threshold " +
                                                    std::to_string(t) + " do not fit (" +
                                                    std::to_string(bytes) + " bytes on rank " +
                                                    std::to_string(me) + ")");
  }
  st = c->fab->share(c->d_rec, &c->peer_rec);
  if (st != WS_OK) return st;
  // sender: each of my remote entries' region at every replica of its coordinate
  const std::vector<int>& mine = c->mine;
  std::vector<EntryDest> ed(std::max<size_t>(1, mine.size()));
  for (int e = 0; e < (int)mine.size(); ++e) {
    EntryDest& D = ed[e];
    std::memset(&D, 0, sizeof(D));
    const Route& rt = plan_.routes_of(me)[mine[e]];
    D.cap = entry_capacity(plan_, me, rt, t);
    int r = 0;
    for (int q : c->dests[rt.coord]) {
      const RecvLayout& Lq = lay[q];
      int pos = -1;
      for (int j = 0; j < (int)Lq.entries.size(); ++j)
        if (Lq.entries[j].first == me && Lq.entries[j].second == e) pos = j;
      if (pos < 0) return set_error(WS_TRANSFER_ERROR, "p2p: entry missing from a receiver layout");
      D.rec[r] = static_cast<char*>(c->peer_rec[q]) + Lq.off[pos];
      D.cnt[r] = reinterpret_cast<uint32_t*>(static_cast<char*>(c->peer_head[q]) + kMailboxBytes) +
                 pos;
      ++r;
    }
  }
  WS_CUDA_TRY(cudaMemcpy(c->d_edest, ed.data(), ed.size() * sizeof(EntryDest),
                         cudaMemcpyHostToDevice), "H2D");
  c->edest = ed;
  for (size_t i = 0; i < c->rmaps.size(); ++i) {
    const EntryDest& D = ed[c->rmap_entry[i]];
    c->rmaps[i].cap = D.cap;
    for (int r = 0; r < kMaxReplicas && r < 8; ++r) c->rmaps[i].rec[r] = D.rec[r];
  }
  if (!c->rmaps.empty())
    WS_CUDA_TRY(cudaMemcpy(c->d_rmaps, c->rmaps.data(), c->rmaps.size() * sizeof(RemoteMap),
                           cudaMemcpyHostToDevice), "H2D");
  // receiver: my regions, per round
  const RecvLayout& L = lay[me];
  for (int r = 0; r < R; ++r) {
    std::vector<RecvEntry> re;
    for (int j = 0; j < (int)L.entries.size(); ++j)
      if (L.round[j] == r)
        re.push_back(RecvEntry{L.off[j], L.cap[j], L.dst_base[j], (uint32_t)j,
                               (uint32_t)L.entries[j].first});
    if (!re.empty())
      WS_CUDA_TRY(cudaMemcpy(c->rr[r].d_rentries, re.data(), re.size() * sizeof(RecvEntry),
                             cudaMemcpyHostToDevice), "H2D");
  }
  c->pargs.recv = c->d_rec;
  c->sized_t = t;
  return WS_OK;
}

// Maps the serving arena of every replica of the coordinates this rank sends
// to, so dense-fallback boxes are stored straight into them (pack kernel),
// then sizes the receive regions: for the density threshold when dense boxes
// go direct (records only for sparse shards), for the worst case otherwise.
// Any rank failing (e.g. a virtual-memory allocation without an IPC handle)
// turns the direct path off everywhere.  Collective.
ws_status ws_engine::map_serve() {
  Comm* c = comm_;
  if (!c || !c->p2p || !serve) return WS_OK;
  c->release_peers(c->peer_serve);
  P2PArgs& P = c->pargs;
  for (int k = 0; k < kMaxWorld; ++k)
    for (int r = 0; r < kMaxReplicas; ++r) P.serve_dst[k][r] = nullptr;
  P.dense_direct = 0;
  std::vector<void*> ps;
  const bool ok = c->fab->share(serve, &ps) == WS_OK;
  const char* env = ablation_env("WSYNC_DENSE_DIRECT");
  if (ok) {
    c->peer_serve = ps;
    if (!(env && env[0] == '0')) {
      for (int k = 0; k < c->coords; ++k) {
        int r = 0;
        for (int g : c->dests[k]) P.serve_dst[k][r++] = c->peer_serve[g];
      }
      P.dense_direct = 1;
    }
  }
  return p2p_size(P.dense_direct ? c->want_t : 1.0);
}

// (Re)allocates the send regions with the given per-coordinate capacities.
ws_status ws_engine::size_send(const std::vector<uint64_t>& region_cap) {
  Comm* c = comm_;
  c->region_cap = region_cap;
  c->region_off.assign(c->coords, 0);
  c->send_cap = 0;
  for (int k = 0; k < c->coords; ++k) {
    c->region_off[k] = c->send_cap;
    c->send_cap += region_cap[k];
  }
  cudaFree(c->d_send);
  c->d_send = nullptr;
  WS_CUDA_TRY(cudaMalloc(&c->d_send, std::max<uint64_t>(1, c->send_cap) * wire_bytes(dtype_)),
              "cudaMalloc send");
  WS_CUDA_TRY(cudaMemcpy(c->d_region_off, c->region_off.data(), c->coords * 8,
                         cudaMemcpyHostToDevice), "H2D");
  WS_CUDA_TRY(cudaMemcpy(c->d_region_cap, c->region_cap.data(), c->coords * 8,
                         cudaMemcpyHostToDevice), "H2D");
  return WS_OK;
}

ws_status ws_engine::size_recv(uint64_t records) {
  Comm* c = comm_;
  cudaFree(c->d_recv);
  c->d_recv = nullptr;
  c->recv_cap = records;
  WS_CUDA_TRY(cudaMalloc(&c->d_recv, std::max<uint64_t>(1, records) * wire_bytes(dtype_)),
              "cudaMalloc recv");
  return WS_OK;
}

void ws_engine::destroy_comm() {
  delete comm_;
  comm_ = nullptr;
}

// True when a sync with these options needs larger receive regions.
bool ws_engine::exchange_needs_resize(const ws_sync_options& o) const {
  const Comm* c = comm_;
  return c && c->p2p && c->pargs.dense_direct && o.sparse &&
         std::min(1.0, o.density_threshold) > c->sized_t;
}

// Grows the receive regions (collectively) before a sync whose density
// threshold exceeds what they were sized for.  Every rank calls this with
// the same options (as every rank passes the same SyncOptions).
ws_status ws_engine::exchange_prepare(const ws_sync_options& o) {
  if (!exchange_needs_resize(o)) return WS_OK;
  Comm* c = comm_;
  c->want_t = std::min(1.0, std::max(c->want_t, o.density_threshold));
  return p2p_size(c->want_t);
}

ws_status ws_engine::exchange_begin(cudaStream_t s, uint32_t* launches) {
  Comm* c = comm_;
  if (!c) return WS_OK;
  c->k1_emit = false;  // set again by exchange_fuse_k1 when K1 emits this sync
  if (!c->p2p) return WS_OK;
  ++c->step;  // this sync's rounds carry epochs R * step + r
  if (!c->pargs.dense_direct || !c->pargs.expect_mask) return WS_OK;
  P2PArgs p = c->pargs;
  p.epoch = (uint32_t)(c->R * c->step + c->R - 1);  // reached every round of this step
  WS_CUDA_TRY(launch_p2p_ready(p, s), "p2p ready");
  *launches += 1;
  return WS_OK;
}

cudaStream_t ws_engine::exchange_side_stream() const {
  static const bool on = [] {
    const char* e = ablation_env("WSYNC_SIDE_LOCAL");
    return !(e && e[0] == '0');
  }();
  return on && comm_ && comm_->p2p ? comm_->s_side : nullptr;
}

ws_status ws_engine::exchange_fork(cudaStream_t s, cudaStream_t side) {
  WS_CUDA_TRY(cudaEventRecord(comm_->ev_fork, s), "event");
  WS_CUDA_TRY(cudaStreamWaitEvent(side, comm_->ev_fork, 0), "wait");
  return WS_OK;
}

ws_status ws_engine::exchange_join(cudaStream_t s, cudaStream_t side) {
  WS_CUDA_TRY(cudaEventRecord(comm_->ev_join, side), "event");
  WS_CUDA_TRY(cudaStreamWaitEvent(s, comm_->ev_join, 0), "wait");
  return WS_OK;
}

int ws_engine::exchange_rounds() const {
  return comm_ && comm_->p2p ? comm_->R : 1;
}

ws_status ws_engine::exchange_fuse_k1(EncodeArgs& a, cudaStream_t s) {
  Comm* c = comm_;
  if (c) c->k1_emit = false;
  // Opt-in (WSYNC_FUSED_REMOTE=1, single round).  Measured on 2 and 4 B200s
  // it is slower than the separate pack: the ballots, counters and NVLink
  // stores sit on K1's issue-bound critical path (+0.4 ms at 1%), and
  // waiting for the previous step's acks inside K1 couples the ranks' start
  // times; the pack it replaces costs 0.2-0.5 ms.  See DESIGN.md §6.
  static const bool enabled = [] {
    const char* e = ablation_env("WSYNC_FUSED_REMOTE");
    return e && e[0] == '1';
  }();
  // Only with direct dense boxes: a segment that comes out dense after K1
  // emitted some of its records then reports 0 of them (pack_kernel).
  if (!c || !c->p2p || c->R != 1 || !c->pargs.dense_direct || dtype_ != WS_BF16 || !enabled ||
      !c->nsend_entries)
    return WS_OK;
  WS_CUDA_TRY(cudaMemsetAsync(c->d_ent_cnt, 0, c->nsend_entries * 4, s), "memset");
  a.remote.maps = c->d_rmaps;
  a.remote.seg_first = c->d_rseg_first;
  a.remote.ack = c->pargs.mailbox + mb_ack(c->world, 0, 0);
  a.remote.ack_mask = 0;
  for (int k = 0; k < kMaxWorld; ++k)
    for (int r = 0; r < kMaxReplicas && c->rr[0].dest_rank[k][r] >= 0; ++r)
      a.remote.ack_mask |= 1u << c->rr[0].dest_rank[k][r];
  a.remote.epoch = (uint32_t)c->step;  // waits for acks >= epoch - 1 (the previous step)
  c->k1_emit = true;
  return WS_OK;
}

// One P2P exchange round, sender side: pack this round's remote entries
// (records into the replicas' regions, dense boxes into their serving
// arenas) and publish.  No host synchronisation.
ws_status ws_engine::exchange_pack(const ws_sync_options& o, int next_arena, int round,
                                   cudaStream_t s, uint32_t* launches) {
  Comm* c = comm_;
  const int e0 = c->ent_first[round], ne = c->ent_first[round + 1] - e0;
  const P2PArgs P = round_args(round);
  if (ne && !c->k1_emit)
    WS_CUDA_TRY(cudaMemsetAsync(c->d_ent_cnt + e0, 0, ne * 4, s), "memset");
  PackArgs pa{};
  pa.r.entries = c->d_entries + e0;
  pa.r.nentries = ne;
  pa.r.sparse = o.sparse ? 1 : 0;
  pa.r.k1_emitted = c->k1_emit && o.sparse ? 1 : 0;
  pa.r.seg_nnz = d_nnz_;
  pa.r.seg_cap = d_cap_;
  pa.r.seg_rec = d_rec_;
  pa.r.seg_base = d_base_;
  pa.r.rec_idx = d_idx_;
  pa.r.rec_val = d_val_;
  fill_tiles(pa.r);
  pa.r.segs = d_segs_;
  pa.r.train_next = arena[next_arena];
  pa.r.serve = serve;
  pa.r.unit_off = c->d_unit_off + e0 + round;
  pa.region_off = c->d_region_off;
  pa.region_cap = c->d_region_cap;
  pa.region_cnt = c->d_region_cnt;
  pa.err = c->d_err;
  pa.p2p = P;
  WS_CUDA_TRY(launch_pack(dtype_, pa, route_grid_, s), "pack (p2p)");
  if (ne) *launches += 2;
  return WS_OK;
}

// Marks the end of the last round's pack on this sync's stage events (the
// pack's share of the route stage, ws_timing::pack_s).
ws_status ws_engine::exchange_mark_pack(cudaStream_t s) {
  WS_CUDA_TRY(cudaEventRecord(ring_[(ring_head_ + kRing - 1) % kRing][6], s), "event");
  pack_ev_ = true;
  return WS_OK;
}

// Receiver side of a round: apply what the sources sent for it, then ack.
ws_status ws_engine::exchange_apply(int round, cudaStream_t s, uint32_t* launches) {
  Comm* c = comm_;
  if (!c->rr[round].mask) return WS_OK;
  WS_CUDA_TRY(launch_apply_p2p(dtype_, round_args(round), serve, sm_count() * 8, s),
              "apply (p2p)");
  *launches += 2;
  return WS_OK;
}

P2PArgs ws_engine::round_args(int round) const {
  const Comm* c = comm_;
  const Comm::RoundRecv& X = c->rr[round];
  const int e0 = c->ent_first[round];
  P2PArgs P = c->pargs;
  P.round = round;
  P.epoch = (uint32_t)(c->R * c->step + round);
  P.prev_epoch = c->step > 1 ? (uint32_t)(c->R * (c->step - 1) + round) : 0u;
  for (int k = 0; k < kMaxWorld; ++k)
    for (int q = 0; q < kMaxReplicas; ++q) P.dest_rank[k][q] = X.dest_rank[k][q];
  P.edest = c->d_edest + e0;
  P.ent_cnt = c->d_ent_cnt + e0;
  P.rentries = X.d_rentries;
  P.nrecv = X.n;
  P.recv_units = X.d_units;
  P.expect_mask = X.mask;
  return P;
}

ws_status ws_engine::exchange_round(const ws_sync_options& o, int next_arena, int round,
                                    cudaStream_t s, uint32_t* launches) {
  ws_status st = exchange_pack(o, next_arena, round, s, launches);
  return st != WS_OK ? st : exchange_apply(round, s, launches);
}

// Queues the read-back of the exchange's device fault word (checked by the
// next synchronising call).
ws_status ws_engine::exchange_end(cudaStream_t s) {
  Comm* c = comm_;
  if (!c) return WS_OK;
  if (c->p2p) pulled_bytes_ = 0;
  WS_CUDA_TRY(cudaMemcpyAsync(c->h_err, c->d_err, 4, cudaMemcpyDeviceToHost, s), "D2H err");
  return WS_OK;
}

// A sync whose exchange is split in R rounds (P2P): round r's segments are
// encoded on a high-priority stream; their pack/apply run on a low-priority
// stream while K1 encodes round r + 1 on all but kOverlapSMs SMs (which the
// exchange kernels then occupy).  The last round's exchange follows the local
// route on the encode stream; the caller's stream joins both at the end.
ws_status ws_engine::sync_rounds(const ws_sync_options& o, int pa, int na, cudaStream_t s,
                                 uint32_t* launches, cudaEvent_t* ev) {
  Comm* c = comm_;
  const int R = c->R;
  static const int overlap_sms_env = [] {
    const char* e = ablation_env("WSYNC_OVERLAP_SMS");
    return e ? std::max(0, atoi(e)) : -1;
  }();
  const int overlap_sms = overlap_sms_env >= 0 ? overlap_sms_env : c->overlap_sms;
  static const bool overlap = [] {
    const char* e = ablation_env("WSYNC_OVERLAP");
    return !(e && e[0] == '0');
  }();
  cudaStream_t ks = c->s_enc, xs = overlap ? c->s_xchg : c->s_enc;
  // ablation build: WSYNC_TIMELINE=1 prints each sync's stage timeline (ms from
  // the start: every K1 round, pack and receive-side apply, the local route)
  static const bool timeline = ablation_env("WSYNC_TIMELINE") != nullptr;
  thread_local std::map<int, std::vector<cudaEvent_t>> tl_events;  // per device
  std::vector<cudaEvent_t>& tl_ev = tl_events[device_];
  std::vector<std::string> tl_name;
  auto mark = [&](const std::string& name, cudaStream_t st) -> ws_status {
    if (!timeline) return WS_OK;
    if (tl_name.size() == tl_ev.size()) {
      tl_ev.emplace_back();
      WS_CUDA_TRY(cudaEventCreate(&tl_ev.back()), "event");
    }
    WS_CUDA_TRY(cudaEventRecord(tl_ev[tl_name.size()], st), "event");
    tl_name.push_back(name);
    return WS_OK;
  };
  WS_CUDA_TRY(cudaEventRecord(c->ev_start, s), "event");
  WS_CUDA_TRY(cudaStreamWaitEvent(ks, c->ev_start, 0), "wait");
  if (xs != ks) WS_CUDA_TRY(cudaStreamWaitEvent(xs, c->ev_start, 0), "wait");
  WS_CUDA_TRY(cudaMemsetAsync(d_nnz_, 0, nseg_ * 8, ks), "memset counts");
  if (count_only_) WS_CUDA_TRY(cudaMemsetAsync(d_fill_, 0, nseg_ * 8, ks), "memset fill");
  const EncodeArgs a = encode_args(pa, na);
  const int sms = sm_count();
  ws_status st0 = mark("start", ks);
  if (st0 != WS_OK) return st0;
  for (int r = 0; r < R; ++r) {
    EncodeArgs ar = a;
    ar.tile_offset = c->tile_first[r];
    ar.ntiles = c->tile_first[r + 1] - c->tile_first[r];
    if (overlap && r > 0 && sms > overlap_sms + 8) ar.max_grid = (uint32_t)(sms - overlap_sms);
    if (ar.ntiles) {
      WS_CUDA_TRY(launch_encode(dtype_, ar, ks), "encode (round)");
      ++*launches;
    }
    if (count_only_) {
      ws_status st = launch_fixup(a, c->seg_first[r], c->seg_first[r + 1], ks, launches);
      if (st != WS_OK) return st;
    }
    ws_status st = mark("k1." + std::to_string(r), ks);
    if (st != WS_OK) return st;
    if (r < R - 1) {
      WS_CUDA_TRY(cudaEventRecord(c->ev_round[r], ks), "event");
      if (xs != ks) WS_CUDA_TRY(cudaStreamWaitEvent(xs, c->ev_round[r], 0), "wait");
      st = exchange_pack(o, na, r, xs, launches);
      if (st == WS_OK) st = mark("pack." + std::to_string(r), xs);
      if (st == WS_OK) st = exchange_apply(r, xs, launches);
      if (st == WS_OK) st = mark("apply." + std::to_string(r), xs);
      if (st != WS_OK) return st;
    }
  }
  WS_CUDA_TRY(cudaEventRecord(ev[2], ks), "event");
  ws_status st = local_route(o, pa, na, ks, launches);
  if (st != WS_OK) return st;
  WS_CUDA_TRY(cudaEventRecord(ev[3], ks), "event");
  st = mark("local", ks);
  if (st == WS_OK) st = exchange_pack(o, na, R - 1, ks, launches);
  if (st == WS_OK) st = mark("pack." + std::to_string(R - 1), ks);
  if (st == WS_OK) st = exchange_apply(R - 1, ks, launches);
  if (st == WS_OK) st = mark("apply." + std::to_string(R - 1), ks);
  if (st != WS_OK) return st;
  if (xs != ks) {
    WS_CUDA_TRY(cudaEventRecord(c->ev_xdone, xs), "event");
    WS_CUDA_TRY(cudaStreamWaitEvent(ks, c->ev_xdone, 0), "wait");
  }
  st = exchange_end(ks);
  if (st != WS_OK) return st;
  if (timeline) {
    st = mark("end", ks);
    if (st != WS_OK) return st;
    WS_CUDA_TRY(cudaEventSynchronize(tl_ev[tl_name.size() - 1]), "sync");
    std::string line = "{\"rank\": " + std::to_string(c->rank);
    for (size_t i = 1; i < tl_name.size(); ++i) {
      float ms = 0;
      WS_CUDA_TRY(cudaEventElapsedTime(&ms, tl_ev[0], tl_ev[i]), "elapsed");
      line += ", \"" + tl_name[i] + "\": " + std::to_string(ms);
    }
    fprintf(stderr, "%s}\n", line.c_str());
  }
  WS_CUDA_TRY(cudaEventRecord(c->ev_encdone, ks), "event");
  WS_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_encdone, 0), "wait");
  return WS_OK;
}

ws_status ws_engine::exchange(const ws_sync_options& o, int next_arena, cudaStream_t s,
                              uint32_t* launches) {
  Comm* c = comm_;
  if (!c) return set_error(WS_INVALID_ARGUMENT, "exchange without a communicator");
  const size_t wb = wire_bytes(dtype_);
  if (c->p2p) {
    for (int r = 0; r < c->R; ++r) {
      ws_status st = exchange_pack(o, next_arena, r, s, launches);
      if (st == WS_OK && r == c->R - 1) st = exchange_mark_pack(s);
      if (st == WS_OK) st = exchange_apply(r, s, launches);
      if (st != WS_OK) return st;
    }
    return exchange_end(s);
  }
  // 1. pack
  WS_CUDA_TRY(cudaMemsetAsync(c->d_region_cnt, 0, c->coords * 8, s), "memset");
  WS_CUDA_TRY(cudaMemsetAsync(c->d_err, 0, 4, s), "memset");
  PackArgs pa{};
  pa.r.entries = c->d_entries;
  pa.r.nentries = c->nentries;
  pa.r.sparse = o.sparse ? 1 : 0;
  pa.r.seg_nnz = d_nnz_;
  pa.r.seg_cap = d_cap_;
  pa.r.seg_rec = d_rec_;
  pa.r.seg_base = d_base_;
  pa.r.rec_idx = d_idx_;
  pa.r.rec_val = d_val_;
  fill_tiles(pa.r);
  pa.r.segs = d_segs_;
  pa.r.train_next = arena[next_arena];
  pa.r.serve = serve;
  pa.r.unit_off = c->d_unit_off;
  pa.send = c->d_send;
  pa.region_off = c->d_region_off;
  pa.region_cap = c->d_region_cap;
  pa.region_cnt = c->d_region_cnt;
  pa.err = c->d_err;
  WS_CUDA_TRY(launch_pack(dtype_, pa, route_grid_, s), "pack");
  if (c->nentries) *launches += 2;
  // 2. counts (a region that overflowed still counts every record it needs)
  WS_NCCL_TRY(ncclAllGather(c->d_region_cnt, c->d_allcnt, c->coords, ncclUint64, c->comm, s),
              "ncclAllGather");
  WS_CUDA_TRY(cudaMemcpyAsync(c->h_allcnt, c->d_allcnt, (size_t)c->world * c->coords * 8,
                              cudaMemcpyDeviceToHost, s),
              "D2H counts");
  WS_CUDA_TRY(cudaStreamSynchronize(s), "sync");
  const int me = c->rank, my_coord = plan_.my_coord();
  // grow what is too small (decided from global knowledge, no extra round)
  bool grow_send = false;
  std::vector<uint64_t> need(c->coords);
  for (int k = 0; k < c->coords; ++k) {
    need[k] = c->h_allcnt[(size_t)me * c->coords + k];
    grow_send |= need[k] > c->region_cap[k];
  }
  uint64_t recv_need = 0;
  for (int g = 0; g < c->world; ++g)
    if (g != me) recv_need += c->h_allcnt[(size_t)g * c->coords + my_coord];
  if (recv_need > c->recv_cap) {
    ws_status st = size_recv(recv_need + recv_need / 4);
    if (st != WS_OK) return st;
  }
  if (grow_send) {
    for (int k = 0; k < c->coords; ++k)
      need[k] = std::max(c->region_cap[k], need[k] + need[k] / 4);
    ws_status st = size_send(need);
    if (st != WS_OK) return st;
    pa.send = c->d_send;
    WS_CUDA_TRY(cudaMemsetAsync(c->d_region_cnt, 0, c->coords * 8, s), "memset");
    // the first pack's overflow was the signal to grow, not a fault
    WS_CUDA_TRY(cudaMemsetAsync(c->d_err, 0, 4, s), "memset");
    WS_CUDA_TRY(launch_pack(dtype_, pa, route_grid_, s), "pack (grown)");
    *launches += 2;
  }
  // 3. one grouped send/recv
  uint64_t recv_total = 0, sent = 0;
  WS_NCCL_TRY(ncclGroupStart(), "ncclGroupStart");
  for (int k = 0; k < c->coords; ++k) {
    const uint64_t n = c->h_allcnt[(size_t)me * c->coords + k];
    if (!n) continue;
    for (int g : c->dests[k]) {
      WS_NCCL_TRY(ncclSend(static_cast<const char*>(c->d_send) + c->region_off[k] * wb, n * wb,
                           ncclUint8, g, c->comm, s),
                  "ncclSend");
      sent += n * wb;
    }
  }
  for (int g = 0; g < c->world; ++g) {
    if (g == me) continue;
    const uint64_t n = c->h_allcnt[(size_t)g * c->coords + my_coord];
    if (!n) continue;
    if (recv_total + n > c->recv_cap) {
      ncclGroupEnd();
      return set_error(WS_CAPACITY, "exchange: receive buffer overflow");
    }
    WS_NCCL_TRY(ncclRecv(static_cast<char*>(c->d_recv) + recv_total * wb, n * wb, ncclUint8, g,
                         c->comm, s),
                "ncclRecv");
    recv_total += n;
  }
  WS_NCCL_TRY(ncclGroupEnd(), "ncclGroupEnd");
  // 4. apply what arrived
  WS_CUDA_TRY(launch_apply_wire(dtype_, c->d_recv, recv_total, serve, s), "apply wire");
  if (recv_total) *launches += 1;
  pulled_bytes_ = recv_total * wb;
  pushed_wire_bytes_ = sent;
  return exchange_end(s);
}

// Device-side exchange faults of the syncs so far (sticky in P2P mode), read
// after a synchronising call.
ws_status ws_engine::exchange_status() const {
  const Comm* c = comm_;
  if (!c || !c->h_err) return WS_OK;
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(c->h_err);
  if (e & kErrBitTimeout)
    return set_error(WS_RELAY_TIMEOUT, "exchange: a peer did not reach, send or ack a step in time");
  if (e & WS_ERRBIT_CAPACITY) return set_error(WS_CAPACITY, "exchange: region capacity exceeded");
  return WS_OK;
}

// Host-only consistency check of the P2P exchange layouts of every rank of
// a plan (what init_p2p builds per rank): each remote entry of every sender
// appears exactly once in the layout of each replica of its coordinate, in
// the round of its segment; a receiver expects a source in round r exactly
// when that source sends it something in round r; the mailbox fits.
static ws_status check_exchange(const Plan& plan, int rounds, double t);

extern "C" ws_status ws_plan_exchange_rounds(const ws_plan* plan_h, int32_t* rounds) {
  if (!plan_h || !rounds) return set_error(WS_INVALID_ARGUMENT, "ws_plan_exchange_rounds: null");
  *rounds = plan_h->p->world() > 1 ? default_rounds(*plan_h->p) : 1;
  return WS_OK;
}

extern "C" ws_status ws_plan_check_exchange(const ws_plan* plan_h, int rounds) {
  if (!plan_h || rounds < 1 || rounds > kMaxRounds)
    return set_error(WS_INVALID_ARGUMENT, "ws_plan_check_exchange: bad argument");
  // the worst-case regions and the ones bounded by the default threshold
  for (double t : {1.0, kDefaultThreshold}) {
    ws_status st = check_exchange(*plan_h->p, rounds, t);
    if (st != WS_OK) return st;
  }
  return WS_OK;
}

static ws_status check_exchange(const Plan& plan, int rounds, double t) {
  const int W = plan.world(), R = rounds;
  if (W > kMaxWorld) return set_error(WS_INVALID_ARGUMENT, "world beyond kMaxWorld");
  if ((size_t)(W + R * (2 * W + 2)) * 8 > kMailboxBytes)
    return set_error(WS_CAPACITY, "mailbox too small for this world and round count");
  const uint32_t tile = encode_tile_elems(plan.dtype());
  std::vector<RecvLayout> lay(W);
  for (int q = 0; q < W; ++q) lay[q] = recv_layout(plan, q, R, tile, t);
  // expectation per (receiver, round) from the layouts
  std::vector<std::vector<uint32_t>> expect(W, std::vector<uint32_t>(R, 0));
  for (int q = 0; q < W; ++q)
    for (size_t j = 0; j < lay[q].entries.size(); ++j)
      expect[q][lay[q].round[j]] |= 1u << lay[q].entries[j].first;
  std::vector<std::vector<uint32_t>> sends(W, std::vector<uint32_t>(R, 0));
  for (int g = 0; g < W; ++g) {
    const std::vector<int> rr = remote_routes(plan, g);
    const std::vector<int> sr = segment_rounds(plan, g, R, tile);
    int prev_round = 0;
    for (int e = 0; e < (int)rr.size(); ++e) {
      const Route& rt = plan.routes_of(g)[rr[e]];
      const int round = sr[rt.seg];
      if (round < prev_round) return set_error(WS_TRANSFER_ERROR, "entry rounds not monotonic");
      prev_round = round;
      for (int q = 0; q < W; ++q) {
        if (q == g || plan.coord_of_rank(q) != rt.coord) continue;
        int hits = 0;
        for (size_t j = 0; j < lay[q].entries.size(); ++j)
          if (lay[q].entries[j].first == g && lay[q].entries[j].second == e) {
            ++hits;
            if (lay[q].round[j] != round)
              return set_error(WS_TRANSFER_ERROR, "entry round differs at a receiver");
            if (lay[q].cap[j] != entry_capacity(plan, g, rt, t))
              return set_error(WS_TRANSFER_ERROR, "entry capacity differs at a receiver");
          }
        if (hits != 1) return set_error(WS_TRANSFER_ERROR, "entry missing or duplicated at a receiver");
        sends[g][round] |= 1u << q;
      }
    }
  }
  for (int q = 0; q < W; ++q)
    for (int r = 0; r < R; ++r)
      for (int g = 0; g < W; ++g)
        if (((expect[q][r] >> g) & 1u) != ((sends[g][r] >> q) & 1u))
          return set_error(WS_TRANSFER_ERROR, "expectation and destinations disagree");
  return WS_OK;
}

// Bytes of the last sync that crossed to / arrived from other GPUs: wire
// records stored into the replicas' receive regions (one copy per replica),
// dense boxes stored straight into their serving arenas, and the records
// the sources published into this rank's regions.  Synchronises.
ws_status ws_engine::exchange_bytes(uint64_t* sent_record_bytes, uint64_t* sent_dense_bytes,
                                    uint64_t* recv_record_bytes) {
  *sent_record_bytes = *sent_dense_bytes = *recv_record_bytes = 0;
  Comm* c = comm_;
  if (!c) return WS_OK;
  WS_CUDA_TRY(cudaSetDevice(device_), "cudaSetDevice");
  WS_CUDA_TRY(cudaDeviceSynchronize(), "sync");
  if (!c->p2p) {
    *sent_record_bytes = pushed_wire_bytes_;
    *recv_record_bytes = pulled_bytes_;
    return WS_OK;
  }
  const size_t wb = p2p_record_bytes(dtype_), esz = dtype_size(dtype_);
  const int ne = (int)c->mine.size();
  std::vector<uint32_t> cnt(std::max(1, ne));
  std::vector<uint64_t> nnz(std::max(1, nseg_)), cap(std::max(1, nseg_));
  if (ne) WS_CUDA_TRY(cudaMemcpy(cnt.data(), c->d_ent_cnt, ne * 4, cudaMemcpyDeviceToHost), "D2H");
  if (nseg_) {
    WS_CUDA_TRY(cudaMemcpy(nnz.data(), d_nnz_, nseg_ * 8, cudaMemcpyDeviceToHost), "D2H");
    WS_CUDA_TRY(cudaMemcpy(cap.data(), d_cap_, nseg_ * 8, cudaMemcpyDeviceToHost), "D2H");
  }
  for (int e = 0; e < ne; ++e) {
    const Route& rt = plan_.routes()[c->mine[e]];
    int nrep = 0;
    while (nrep < kMaxReplicas && c->edest[e].rec[nrep]) ++nrep;
    const bool dense = !last_sparse_ || nnz[rt.seg] > cap[rt.seg];
    if (dense && c->pargs.dense_direct)
      *sent_dense_bytes += rt.overlap * esz * nrep;
    else
      *sent_record_bytes += (uint64_t)std::min<uint64_t>(cnt[e], c->edest[e].cap) * wb * nrep;
  }
  const RecvLayout L = recv_layout(plan_, c->rank, c->R, encode_tile_elems(dtype_), c->sized_t);
  std::vector<uint32_t> rc(std::max<size_t>(1, L.entries.size()));
  if (!L.entries.empty())
    WS_CUDA_TRY(cudaMemcpy(rc.data(), static_cast<char*>(c->d_head) + kMailboxBytes,
                           L.entries.size() * 4, cudaMemcpyDeviceToHost), "D2H");
  for (size_t j = 0; j < L.entries.size(); ++j)
    *recv_record_bytes += (uint64_t)(rc[j] & ~kCountSet) * wb;
  return WS_OK;
}

extern "C" ws_status ws_engine_exchange_bytes(ws_engine* eng, uint64_t* sent_record_bytes,
                                              uint64_t* sent_dense_bytes, uint64_t* recv_record_bytes) {
  DeviceGuard device_guard;
  if (!eng || !sent_record_bytes || !sent_dense_bytes || !recv_record_bytes)
    return set_error(WS_INVALID_ARGUMENT, "ws_engine_exchange_bytes: null argument");
  return eng->exchange_bytes(sent_record_bytes, sent_dense_bytes, recv_record_bytes);
}

extern "C" ws_status ws_nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  WS_NCCL_TRY(ncclGetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "NCCL unique id size");
  std::memcpy(out, &id, sizeof(id));
  return WS_OK;
}



