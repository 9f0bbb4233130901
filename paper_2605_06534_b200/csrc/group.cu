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
//
// A group may instead hold one rank per GPU of the process (peer access over
// NVLink, pointers shared the same way): every rank then runs its whole sync
// concurrently on its own GPU, exactly the deployment's kernels, driven by
// one process (e.g. for ncu, which profiles one process).
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "capi_util.h"
#include "engine.h"

using namespace wsync;

struct ws_group {
  explicit ws_group(int w) : shared(w), eng(w, nullptr) {}
  ~ws_group() {
    for (size_t r = 0; r < streams.size(); ++r)
      if (streams[r]) {
        cudaSetDevice(eng[r] ? eng[r]->device() : 0);
        cudaStreamDestroy(streams[r]);
      }
  }
  GroupShared shared;
  std::vector<ws_engine*> eng;
  bool connected = false;
  bool multi_device = false;           // ranks on several GPUs of this process
  std::vector<cudaStream_t> streams;   // multi-device: one per rank, on its GPU
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
  DeviceGuard device_guard;
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
  DeviceGuard device_guard;
  if (!g) return set_error(WS_INVALID_ARGUMENT, "ws_group_connect: null group");
  if (g->connected) return WS_OK;
  const int W = g->shared.world;
  for (int r = 0; r < W; ++r) {
    if (!g->eng[r]) return set_error(WS_INVALID_ARGUMENT, "ws_group_connect: a rank has not joined");
    if (!g->eng[r]->bound())
      return set_error(WS_INVALID_ARGUMENT, "ws_group_connect: a rank is not bound");
  }
  std::vector<int> devs;
  for (int r = 0; r < W; ++r)
    if (std::find(devs.begin(), devs.end(), g->eng[r]->device()) == devs.end())
      devs.push_back(g->eng[r]->device());
  g->multi_device = devs.size() > 1;
  if (g->multi_device && (int)devs.size() != W)
    return set_error(WS_INVALID_ARGUMENT,
                     "ws_group_connect: ranks share either one GPU or one GPU each");
  ws_status st = run_ranks(g, [&](int r) {
    ws_engine* e = g->eng[r];
    // peers' memory on other GPUs is reached over NVLink (peer access)
    for (int d : devs) {
      if (d == e->device()) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, e->device(), d);
      if (!can) return set_error(WS_CUDA, "ws_group_connect: no peer access between the GPUs");
      const cudaError_t pe = cudaDeviceEnablePeerAccess(d, 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
        return cuda_status(pe, "cudaDeviceEnablePeerAccess");
      cudaGetLastError();
    }
    ws_status s = e->init_comm(nullptr, &g->shared);
    return s != WS_OK ? s : e->map_serve();
  });
  if (st != WS_OK) return st;
  if (g->multi_device) {
    g->streams.assign(W, nullptr);
    for (int r = 0; r < W; ++r) {
      cudaSetDevice(g->eng[r]->device());
      if (cudaStreamCreateWithFlags(&g->streams[r], cudaStreamNonBlocking) != cudaSuccess)
        return set_error(WS_CUDA, "ws_group_connect: stream");
    }
  }
  g->connected = true;
  return WS_OK;
}

ws_status ws_group_sync_step(ws_group* g, const ws_sync_options* opts, ws_stream_t stream,
                             ws_report* reports) {
  DeviceGuard device_guard;
  if (!g || !opts) return set_error(WS_INVALID_ARGUMENT, "ws_group_sync_step: null argument");
  if (!g->connected) return set_error(WS_INVALID_ARGUMENT, "ws_group_sync_step: not connected");
  const int W = g->shared.world;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto& E = g->eng;
  if (E[0]->exchange_needs_resize(*opts)) {  // collective: every rank on its own thread
    ws_status st = run_ranks(g, [&](int r) { return E[r]->exchange_prepare(*opts); });
    if (st != WS_OK) return st;
  }
  // Single GPU: every rank on the caller's stream.  One GPU per rank: each
  // rank on its own GPU's stream; the phases still go out in this order, so
  // a tool that serialises every launch of the process (ncu) runs them in an
  // order where each wait is already satisfied, and without one the GPUs run
  // concurrently, ordered only by the exchange's flags.
  int cur = 0;
  cudaGetDevice(&cur);
  auto on = [&](int r) {
    if (g->multi_device) cudaSetDevice(E[r]->device());
    return g->multi_device ? g->streams[r] : s;
  };
  std::vector<ws_engine::SyncCtx> x(W);
  ws_status st = WS_OK;
  for (int r = 0; r < W && st == WS_OK; ++r) st = E[r]->sync_begin(x[r], *opts, on(r), nullptr);
  for (int r = 0; r < W && st == WS_OK; ++r) st = E[r]->sync_encode(x[r], on(r));
  if (W > 1)
    for (int round = 0; round < E[0]->exchange_rounds() && st == WS_OK; ++round) {
      for (int r = 0; r < W && st == WS_OK; ++r) {
        st = E[r]->exchange_pack(x[r].o, x[r].na, round, on(r), &x[r].launches);
        if (st == WS_OK && round == E[r]->exchange_rounds() - 1) st = E[r]->exchange_mark_pack(on(r));
      }
      for (int r = 0; r < W && st == WS_OK; ++r)
        st = E[r]->exchange_apply(round, on(r), &x[r].launches);
    }
  for (int r = 0; r < W && st == WS_OK && W > 1; ++r) st = E[r]->exchange_end(on(r));
  for (int r = 0; r < W && st == WS_OK; ++r)
    st = E[r]->sync_finish(x[r], on(r), nullptr, reports ? reports + r : nullptr);
  if (g->multi_device)  // the call returns with every rank's sync complete
    for (int r = 0; r < W; ++r) {
      const cudaError_t e = cudaStreamSynchronize(on(r));
      if (st == WS_OK && e != cudaSuccess) st = cuda_status(e, "group sync");
    }
  cudaSetDevice(cur);
  return st;
}

}  // extern "C"
