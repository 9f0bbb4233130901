// group.cu -- every rank of a sync as an engine of ONE process (ws_group).
//
// The deployment runs one process per GPU and wires the NVLink exchange
// with CUDA IPC over NCCL (exchange.cu).  A ws_group instead holds all
// `world` ranks of a layout in one process, on one GPU: the ranks share
// their mailboxes, receive regions and serving arenas as plain device
// pointers (GroupFabric), and ws_group_sync_step interleaves the phases of
// all ranks on ONE stream -- every rank's "reached step" flag, then every
// K1 + local route, then per exchange round every pack (the same
// pack_kernel that stores over NVLink) and every receive-side apply
// (apply_p2p_kernel) -- so each flag a kernel waits for was published by an
// earlier launch of that stream.  It runs the multi-GPU data path of any
// layout (TrainConfig{tp,pp,dp}, FSDP-N, serving TP x PP x replicas, EP) on
// a single device, which is how the parity tests cover it on one B200.
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "capi_util.h"
#include "engine.h"

using namespace wsync;

struct ws_group {
  explicit ws_group(int w) : shared(w), eng(w, nullptr) {}
  GroupShared shared;
  std::vector<ws_engine*> eng;
  bool connected = false;
};

namespace {
// Runs fn(rank) on one host thread per rank (the group's collectives are
// host barriers between those threads); the first failure is returned with
// its message.
template <typename F>
ws_status run_ranks(ws_group* g, F fn) {
  const int W = g->shared.world;
  std::vector<ws_status> st(W, WS_OK);
  std::vector<std::string> msg(W);
  std::vector<std::thread> th;
  for (int r = 0; r < W; ++r)
    th.emplace_back([&, r] {
      cudaSetDevice(g->eng[r]->device());
      st[r] = fn(r);
      if (st[r] != WS_OK) msg[r] = ws_last_error();
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < W; ++r)
    if (st[r] != WS_OK) return set_error(st[r], "group rank " + std::to_string(r) + ": " + msg[r]);
  return WS_OK;
}
}  // namespace

extern "C" {

ws_status ws_group_create(int world, ws_group** out) {
  if (!out || world < 1 || world > kMaxWorld)
    return set_error(WS_INVALID_ARGUMENT, "ws_group_create: world must be in [1, 8]");
  *out = new ws_group(world);
  return WS_OK;
}

void ws_group_destroy(ws_group* g) { delete g; }

ws_status ws_engine_create_grouped(const ws_plan* plan, int device, ws_group* g,
                                   ws_engine** out) {
  if (!plan || !g || !out)
    return set_error(WS_INVALID_ARGUMENT, "ws_engine_create_grouped: null argument");
  *out = nullptr;
  const Plan& p = *plan->p;
  if (p.world() != g->shared.world)
    return set_error(WS_INVALID_ARGUMENT, "ws_engine_create_grouped: plan world != group world");
  if (g->connected || g->eng[p.rank()])
    return set_error(WS_INVALID_ARGUMENT, "ws_engine_create_grouped: rank already joined");
  try {
    auto* e = new ws_engine(p, device);
    ws_status st = e->init(nullptr, true);
    if (st != WS_OK) {
      delete e;
      return st;
    }
    g->eng[p.rank()] = e;
    *out = e;
    return WS_OK;
  } catch (const std::exception& e) {
    return set_error(WS_TRANSFER_ERROR, e.what());
  }
}

ws_status ws_group_connect(ws_group* g) {
  if (!g) return set_error(WS_INVALID_ARGUMENT, "ws_group_connect: null group");
  if (g->connected) return WS_OK;
  const int W = g->shared.world;
  for (int r = 0; r < W; ++r) {
    if (!g->eng[r]) return set_error(WS_INVALID_ARGUMENT, "ws_group_connect: a rank has not joined");
    if (!g->eng[r]->bound())
      return set_error(WS_INVALID_ARGUMENT, "ws_group_connect: a rank is not bound");
    if (g->eng[r]->device() != g->eng[0]->device())
      return set_error(WS_INVALID_ARGUMENT, "ws_group_connect: ranks on different devices");
  }
  ws_status st = run_ranks(g, [&](int r) {
    ws_engine* e = g->eng[r];
    ws_status s = e->init_comm(nullptr, &g->shared);
    return s != WS_OK ? s : e->map_serve();
  });
  if (st == WS_OK) g->connected = true;
  return st;
}

ws_status ws_group_sync_step(ws_group* g, const ws_sync_options* opts, ws_stream_t stream,
                             ws_report* reports) {
  if (!g || !opts) return set_error(WS_INVALID_ARGUMENT, "ws_group_sync_step: null argument");
  if (!g->connected) return set_error(WS_INVALID_ARGUMENT, "ws_group_sync_step: not connected");
  const int W = g->shared.world;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto& E = g->eng;
  if (E[0]->exchange_needs_resize(*opts)) {  // collective: every rank on its own thread
    ws_status st = run_ranks(g, [&](int r) { return E[r]->exchange_prepare(*opts); });
    if (st != WS_OK) return st;
  }
  std::vector<ws_engine::SyncCtx> x(W);
  ws_status st = WS_OK;
  for (int r = 0; r < W && st == WS_OK; ++r) st = E[r]->sync_begin(x[r], *opts, s, nullptr);
  for (int r = 0; r < W && st == WS_OK; ++r) st = E[r]->sync_encode(x[r], s);
  if (W > 1)
    for (int round = 0; round < E[0]->exchange_rounds() && st == WS_OK; ++round) {
      for (int r = 0; r < W && st == WS_OK; ++r)
        st = E[r]->exchange_pack(x[r].o, x[r].na, round, s, &x[r].launches);
      for (int r = 0; r < W && st == WS_OK; ++r) st = E[r]->exchange_apply(round, s, &x[r].launches);
    }
  for (int r = 0; r < W && st == WS_OK && W > 1; ++r) st = E[r]->exchange_end(s);
  for (int r = 0; r < W && st == WS_OK; ++r)
    st = E[r]->sync_finish(x[r], s, nullptr, reports ? reports + r : nullptr);
  return st;
}

}  // extern "C"
