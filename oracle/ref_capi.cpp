// ref_capi.cpp -- extern "C" access to the UNMODIFIED reference transfer
// engine, compiled from /root/reference/proj/src/transfer/*.cpp by
// oracle/Makefile into oracle/_ref/libref_capi.so.
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/ (as the parity checker) and by
// bench.py's cpu_baseline / --impl reference legs (as the timed CPU
// reference).  The product library never links it.
//
// Exceptions are mapped onto the ws_status numbering of include/wsync.h.

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "coserve/transfer/bench.hpp"
#include "coserve/transfer/codec.hpp"
#include "coserve/transfer/engine.hpp"
#include "coserve/transfer/key.hpp"
#include "coserve/transfer/plan.hpp"
#include "coserve/transfer/relay.hpp"
#include "coserve/transfer/tcp_relay.hpp"
#include "coserve/transfer/wire.hpp"

#include <arpa/inet.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <map>
#include <mutex>
#include <thread>

using namespace coserve;
using namespace coserve::transfer;

namespace {

thread_local std::string g_err;

int map_exception() {
  try {
    throw;
  } catch (const IndexOutOfShard& e) {
    g_err = e.what();
    return 3;
  } catch (const ShapeMismatch& e) {
    g_err = e.what();
    return 1;
  } catch (const PayloadFormatError& e) {
    g_err = e.what();
    return 2;
  } catch (const IndivisibleShape& e) {
    g_err = e.what();
    return 4;
  } catch (const UnknownModuleKind& e) {
    g_err = e.what();
    return 5;
  } catch (const IncompleteCoverage& e) {
    g_err = e.what();
    return 6;
  } catch (const RelayTimeout& e) {
    g_err = e.what();
    return 7;
  } catch (const IntegrityError& e) {
    g_err = e.what();
    return 8;
  } catch (const TransferError& e) {
    g_err = e.what();
    return 10;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

HostTensor make_tensor(int dt, const std::int64_t* shape, int nd, const void* data) {
  HostTensor t = HostTensor::zeros(static_cast<DType>(dt),
                                   std::vector<std::int64_t>(shape, shape + nd));
  if (data) std::memcpy(t.data.data(), data, t.data.size());
  return t;
}

ShardDescriptor make_desc(int dim, std::int64_t s, std::int64_t e) {
  ShardDescriptor d;
  d.param = "p";
  d.slice_dim = dim;
  d.start = dim < 0 ? 0 : s;
  d.end = dim < 0 ? 0 : e;
  return d;
}

}  // namespace

struct RefParam {
  const char* name;
  int kind;
  int ndims;
  std::int64_t shape[4];
  int layer;
};

struct RefState {
  TrainState train;
  ServeState serve;
  ServeConfig scfg;
  std::vector<std::pair<ShardDescriptor, char>> codecs;
  std::uint64_t step = 1;
  double model_bytes = 0;
  bool serve_ready = false;  // ref_state_prepare ran: the next run keeps `serve`
};

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// codec.cpp:34-63
int ref_diff_shards(int dt, const std::int64_t* shape, int nd, const void* prev,
                    const void* next, std::uint64_t* idx, void* val,
                    std::uint64_t* nnz) {
  try {
    const HostTensor a = make_tensor(dt, shape, nd, prev);
    const HostTensor b = make_tensor(dt, shape, nd, next);
    const SparseDelta d = diff_shards(a, b);
    std::memcpy(idx, d.indices.data(), d.indices.size() * 8);
    std::memcpy(val, d.values.data(), d.values.size());
    *nnz = d.nnz();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// codec.cpp:65-92 (target updated in place, partial on error like the ref)
int ref_apply_delta(int dt, const std::int64_t* shape, int nd, void* target,
                    const std::int64_t* dshape, int dnd, const std::uint64_t* idx,
                    const void* val, std::uint64_t nnz) {
  HostTensor t = make_tensor(dt, shape, nd, target);
  int rc = 0;
  try {
    SparseDelta d;
    d.dtype = static_cast<DType>(dt);
    d.shape.assign(dshape, dshape + dnd);
    d.indices.assign(idx, idx + nnz);
    d.values.assign(static_cast<const std::uint8_t*>(val),
                    static_cast<const std::uint8_t*>(val) + nnz * 4);
    apply_delta(t, d);
  } catch (...) {
    rc = map_exception();
  }
  std::memcpy(target, t.data.data(), t.data.size());
  return rc;
}

// codec.cpp:94-138
int ref_reslice_delta(int dt, const std::int64_t* full_shape, int nd, int sdim,
                      std::int64_t s0, std::int64_t s1, int ddim, std::int64_t d0,
                      std::int64_t d1, const std::int64_t* dshape, int dnd,
                      const std::uint64_t* idx, const void* val, std::uint64_t nnz,
                      std::uint64_t* out_idx, void* out_val, std::uint64_t* out_nnz,
                      std::int64_t* out_shape) {
  try {
    SparseDelta d;
    d.dtype = static_cast<DType>(dt);
    d.shape.assign(dshape, dshape + dnd);
    d.indices.assign(idx, idx + nnz);
    d.values.assign(static_cast<const std::uint8_t*>(val),
                    static_cast<const std::uint8_t*>(val) + nnz * 4);
    const std::vector<std::int64_t> full(full_shape, full_shape + nd);
    const SparseDelta o = reslice_delta(d, make_desc(sdim, s0, s1), make_desc(ddim, d0, d1), full);
    std::memcpy(out_idx, o.indices.data(), o.indices.size() * 8);
    std::memcpy(out_val, o.values.data(), o.values.size());
    *out_nnz = o.nnz();
    for (std::size_t i = 0; i < o.shape.size(); ++i) out_shape[i] = o.shape[i];
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// shard.cpp:111-134
int ref_extract_shard(int dt, const std::int64_t* shape, int nd, int dim,
                      std::int64_t s, std::int64_t e, const void* full, void* out) {
  try {
    const HostTensor t = make_tensor(dt, shape, nd, full);
    const HostTensor o = extract_shard(t, make_desc(dim, s, e));
    std::memcpy(out, o.data.data(), o.data.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// shard.cpp:136-170; returns copied elements or -status
std::int64_t ref_copy_overlap(int dt, const std::int64_t* dshape, int nd, void* dst,
                              std::int64_t dst_start, const std::int64_t* sshape,
                              const void* src, std::int64_t src_start, int dim) {
  try {
    HostTensor d = make_tensor(dt, dshape, nd, dst);
    const HostTensor s = make_tensor(dt, sshape, nd, src);
    const std::int64_t n = copy_overlap(d, dst_start, s, src_start, dim);
    std::memcpy(dst, d.data.data(), d.data.size());
    return n;
  } catch (...) {
    return -map_exception();
  }
}

// codec.cpp:140-183
int ref_encode_sparse(int dt, const std::int64_t* shape, int nd,
                      const std::uint64_t* idx, const void* val, std::uint64_t nnz,
                      int iw, std::uint8_t* out, std::uint64_t cap,
                      std::uint64_t* out_len) {
  try {
    SparseDelta d;
    d.dtype = static_cast<DType>(dt);
    d.shape.assign(shape, shape + nd);
    d.indices.assign(idx, idx + nnz);
    d.values.assign(static_cast<const std::uint8_t*>(val),
                    static_cast<const std::uint8_t*>(val) + nnz * 4);
    if (iw == 0) iw = pick_index_width(d);
    const auto bytes = encode_sparse(d, iw);
    *out_len = bytes.size();
    if (bytes.size() > cap) return 22;
    std::memcpy(out, bytes.data(), bytes.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_encode_dense(int dt, const std::int64_t* shape, int nd, const void* data,
                     std::uint8_t* out, std::uint64_t cap, std::uint64_t* out_len) {
  try {
    const auto bytes = encode_dense(make_tensor(dt, shape, nd, data));
    *out_len = bytes.size();
    if (bytes.size() > cap) return 22;
    std::memcpy(out, bytes.data(), bytes.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// key.cpp:47-69: BucketKey::encode of one bucket.
int ref_bucket_key(std::uint64_t step, const char* param, int tp_rank, int tp_size, int pp_stage,
                   int slice_dim, std::int64_t start, std::int64_t end, char codec, int iw,
                   std::uint32_t seq, char* out, std::uint64_t cap, std::uint64_t* out_len) {
  try {
    BucketKey k;
    k.step = step;
    k.param = param;
    k.tp_rank = tp_rank;
    k.tp_size = tp_size;
    k.pp_stage = pp_stage;
    k.slice_dim = slice_dim;
    k.start = start;
    k.end = end;
    k.codec = codec;
    k.index_width = iw;
    k.seq = seq;
    const std::string e = k.encode();
    *out_len = e.size();
    if (e.size() > cap) return 22;
    std::memcpy(out, e.data(), e.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// wire.cpp:35-47: one bucket frame (lengths, key, payload, zlib crc32).
int ref_encode_bucket_frame(const char* key, std::uint64_t key_len, const std::uint8_t* payload,
                            std::uint64_t payload_len, std::uint8_t* out, std::uint64_t cap,
                            std::uint64_t* out_len) {
  try {
    const auto f = encode_bucket_frame(std::string(key, key_len),
                                       std::vector<std::uint8_t>(payload, payload + payload_len));
    *out_len = f.size();
    if (f.size() > cap) return 22;
    std::memcpy(out, f.data(), f.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// relay.cpp:7-59: the reference's MemoryRelay behind the ws_relay callbacks
// (test harness for ws_engine_sync_relay).
void* ref_memrelay_create() { return new MemoryRelay(); }
void ref_memrelay_destroy(void* r) { delete static_cast<MemoryRelay*>(r); }
std::uint64_t ref_memrelay_size(void* r) { return static_cast<MemoryRelay*>(r)->size(); }

int ref_memrelay_put(void* ctx, const char* key, std::uint64_t klen, const std::uint8_t* data,
                     std::uint64_t len) {
  try {
    static_cast<MemoryRelay*>(ctx)->put(std::string(key, klen),
                                        std::vector<std::uint8_t>(data, data + len));
    return 0;
  } catch (...) {
    return -2;
  }
}

std::int64_t ref_memrelay_get_any(void* ctx, const char* const* keys, const std::uint64_t* lens,
                                  int n, int timeout_ms, int* hit, std::uint8_t* out,
                                  std::uint64_t cap) {
  try {
    std::vector<std::string> ks;
    for (int i = 0; i < n; ++i) ks.emplace_back(keys[i], lens[i]);
    auto kv = static_cast<MemoryRelay*>(ctx)->get_any(ks, timeout_ms);
    for (int i = 0; i < n; ++i)
      if (ks[i] == kv.first) *hit = i;
    if (kv.second.size() <= cap) std::memcpy(out, kv.second.data(), kv.second.size());
    return static_cast<std::int64_t>(kv.second.size());
  } catch (const RelayTimeout&) {
    return -1;
  } catch (...) {
    return -2;
  }
}

// keys under `prefix`, '\n'-separated; returns the bytes needed
std::uint64_t ref_memrelay_list(void* ctx, const char* prefix, char* out, std::uint64_t cap) {
  std::string all;
  for (const auto& k : static_cast<MemoryRelay*>(ctx)->list(prefix)) all += k + "\n";
  if (all.size() <= cap) std::memcpy(out, all.data(), all.size());
  return all.size();
}

std::int64_t ref_memrelay_get(void* ctx, const char* key, std::uint64_t klen, std::uint8_t* out,
                              std::uint64_t cap) {
  try {
    auto v = static_cast<MemoryRelay*>(ctx)->get(std::string(key, klen), 0);
    if (v.size() <= cap) std::memcpy(out, v.data(), v.size());
    return static_cast<std::int64_t>(v.size());
  } catch (...) {
    return -1;
  }
}

// ---- the reference's TCP relay server (tcp_relay.hpp), and a client for
// the engine's framed transport (ws_relay put_frame / get_any_frame): it
// writes the GPU-built frame after the PUT op byte and hands back the whole
// frame a GET_ANY returns, so the CRC the reference server checks on PUT was
// computed on the GPU, and the engine checks the one it gets back.  The
// protocol is the documented one of tcp_relay.hpp:10-17 (test harness).
void* ref_tcp_server_create() {
  try {
    return new TcpRelayServer(0);
  } catch (...) {
    map_exception();
    return nullptr;
  }
}
int ref_tcp_server_port(void* s) { return static_cast<TcpRelayServer*>(s)->port(); }
std::uint64_t ref_tcp_server_buckets(void* s) {
  return static_cast<TcpRelayServer*>(s)->stored_buckets();
}
void ref_tcp_server_destroy(void* s) { delete static_cast<TcpRelayServer*>(s); }

// The reference's own client (for reading back what the server stored).
void* ref_tcp_client_create(int port) {
  try {
    return new TcpRelayClient("127.0.0.1", static_cast<std::uint16_t>(port));
  } catch (...) {
    map_exception();
    return nullptr;
  }
}
void ref_tcp_client_destroy(void* c) { delete static_cast<TcpRelayClient*>(c); }
std::int64_t ref_tcp_client_get(void* c, const char* key, std::uint64_t klen, std::uint8_t* out,
                                std::uint64_t cap) {
  try {
    auto v = static_cast<TcpRelayClient*>(c)->get(std::string(key, klen), 2000);
    if (v.size() <= cap) std::memcpy(out, v.data(), v.size());
    return static_cast<std::int64_t>(v.size());
  } catch (...) {
    return -1;
  }
}

struct FramedClient {
  int port = 0;
  int flip_put = 0, flip_get = 0;  // corrupt one byte of every n-th frame (tests)
  std::mutex mu;
  std::map<std::thread::id, int> fds;  // one connection per calling thread
  std::uint64_t puts = 0, gets = 0;
  int fd() {
    std::lock_guard<std::mutex> lk(mu);
    auto it = fds.find(std::this_thread::get_id());
    if (it != fds.end()) return it->second;
    const int f = ::socket(AF_INET, SOCK_STREAM, 0);
    if (f < 0) return -1;
    sockaddr_in a{};
    a.sin_family = AF_INET;
    a.sin_port = htons(static_cast<std::uint16_t>(port));
    a.sin_addr.s_addr = htonl(INADDR_LOOPBACK);
    if (::connect(f, reinterpret_cast<sockaddr*>(&a), sizeof(a)) != 0) {
      ::close(f);
      return -1;
    }
    int one = 1;
    ::setsockopt(f, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
    fds[std::this_thread::get_id()] = f;
    return f;
  }
  ~FramedClient() {
    for (auto& kv : fds) ::close(kv.second);
  }
};

static bool send_all(int fd, const void* p, std::size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t k = ::send(fd, c, n, MSG_NOSIGNAL);
    if (k <= 0) return false;
    c += k;
    n -= static_cast<std::size_t>(k);
  }
  return true;
}
static bool recv_all(int fd, void* p, std::size_t n) {
  char* c = static_cast<char*>(p);
  while (n) {
    const ssize_t k = ::recv(fd, c, n, 0);
    if (k <= 0) return false;
    c += k;
    n -= static_cast<std::size_t>(k);
  }
  return true;
}

void* ref_framed_client_create(int port, int flip_put, int flip_get) {
  auto* c = new FramedClient;
  c->port = port;
  c->flip_put = flip_put;
  c->flip_get = flip_get;
  return c;
}
void ref_framed_client_destroy(void* c) { delete static_cast<FramedClient*>(c); }

int ref_framed_put(void* ctx, const std::uint8_t* frame, std::uint64_t len) {
  auto* c = static_cast<FramedClient*>(ctx);
  const int fd = c->fd();
  if (fd < 0) return -2;
  std::vector<std::uint8_t> msg(1 + len);
  msg[0] = 0x01;  // PUT
  std::memcpy(msg.data() + 1, frame, len);
  {
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->flip_put && ++c->puts % static_cast<std::uint64_t>(c->flip_put) == 0 && len > 16)
      msg[1 + len / 2] ^= 0x10;  // a flipped bit in transit
  }
  std::uint8_t status = 0xff;
  if (!send_all(fd, msg.data(), msg.size()) || !recv_all(fd, &status, 1)) return -2;
  return status;  // 0 ok, 3 integrity failure (tcp_relay.hpp:17)
}

std::int64_t ref_framed_get_any(void* ctx, const char* const* keys, const std::uint64_t* lens,
                                int n, int timeout_ms, int* hit, std::uint8_t* out,
                                std::uint64_t cap) {
  auto* c = static_cast<FramedClient*>(ctx);
  const int fd = c->fd();
  if (fd < 0) return -2;
  std::vector<std::uint8_t> req{0x03};  // GET_ANY
  auto u32 = [&](std::uint32_t v) {
    const auto* b = reinterpret_cast<const std::uint8_t*>(&v);
    req.insert(req.end(), b, b + 4);
  };
  u32(static_cast<std::uint32_t>(n));
  for (int i = 0; i < n; ++i) {
    u32(static_cast<std::uint32_t>(lens[i]));
    req.insert(req.end(), keys[i], keys[i] + lens[i]);
  }
  u32(static_cast<std::uint32_t>(timeout_ms));
  std::uint8_t status = 0xff;
  if (!send_all(fd, req.data(), req.size()) || !recv_all(fd, &status, 1)) return -2;
  if (status == 1) return -1;  // timeout
  if (status != 0) return -2;
  std::uint32_t klen = 0, plen = 0;
  if (!recv_all(fd, &klen, 4) || klen > kMaxKeyLen) return -2;
  std::vector<std::uint8_t> f(4 + klen + 4);
  std::memcpy(f.data(), &klen, 4);
  if (!recv_all(fd, f.data() + 4, klen) || !recv_all(fd, &plen, 4) || plen > kMaxPayloadLen)
    return -2;
  std::memcpy(f.data() + 4 + klen, &plen, 4);
  f.resize(f.size() + plen + 4);
  if (!recv_all(fd, f.data() + 8 + klen, plen + 4)) return -2;
  const std::string key(reinterpret_cast<const char*>(f.data()) + 4, klen);
  *hit = -1;
  for (int i = 0; i < n; ++i)
    if (key == std::string(keys[i], lens[i])) *hit = i;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->flip_get && ++c->gets % static_cast<std::uint64_t>(c->flip_get) == 0 && plen > 4)
      f[8 + klen + plen / 2] ^= 0x01;
  }
  if (f.size() <= cap) std::memcpy(out, f.data(), f.size());
  return static_cast<std::int64_t>(f.size());
}

// wire.cpp:9-13
std::uint32_t ref_frame_crc32(const std::uint8_t* data, std::uint64_t len) {
  return frame_crc32(data, len);
}

// codec.cpp:196-263: returns 0 and fills is_sparse/ndims/shape/nnz; the
// idx/val (or dense data) buffers must be large enough (caller peeks first).
int ref_decode_payload(const std::uint8_t* bytes, std::uint64_t len, int* is_sparse,
                       int* nd, std::int64_t* shape, std::uint64_t* nnz,
                       std::uint64_t* idx, void* val) {
  try {
    const std::vector<std::uint8_t> v(bytes, bytes + len);
    DecodedPayload p = decode_payload(v);
    *is_sparse = p.is_sparse();
    if (p.is_sparse()) {
      const auto& d = std::get<SparseDelta>(p.value);
      *nd = static_cast<int>(d.shape.size());
      for (std::size_t i = 0; i < d.shape.size(); ++i) shape[i] = d.shape[i];
      *nnz = d.nnz();
      if (idx) std::memcpy(idx, d.indices.data(), d.indices.size() * 8);
      if (val) std::memcpy(val, d.values.data(), d.values.size());
    } else {
      const auto& t = std::get<HostTensor>(p.value);
      *nd = static_cast<int>(t.shape.size());
      for (std::size_t i = 0; i < t.shape.size(); ++i) shape[i] = t.shape[i];
      *nnz = static_cast<std::uint64_t>(t.elems());
      if (val) std::memcpy(val, t.data.data(), t.data.size());
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

std::int64_t ref_peek_payload_size(const std::uint8_t* data, std::uint64_t len) {
  try {
    return static_cast<std::int64_t>(peek_payload_size(data, len));
  } catch (...) {
    return -map_exception();
  }
}

// --- planner (plan.cpp) ------------------------------------------------------
static std::vector<ParamMeta> to_manifest(const RefParam* p, int n, int dt) {
  std::vector<ParamMeta> m;
  for (int i = 0; i < n; ++i) {
    ParamMeta pm;
    pm.name = p[i].name;
    pm.kind = static_cast<ModuleKind>(p[i].kind);
    pm.shape.assign(p[i].shape, p[i].shape + p[i].ndims);
    pm.dtype = static_cast<DType>(dt);
    pm.layer = p[i].layer;
    m.push_back(std::move(pm));
  }
  return m;
}

static int param_index(const std::vector<ParamMeta>& m, const std::string& name) {
  for (std::size_t i = 0; i < m.size(); ++i)
    if (m[i].name == name) return static_cast<int>(i);
  return -1;
}

static void put_desc(std::int64_t* out, const std::vector<ParamMeta>& m,
                     const ShardDescriptor& d) {
  out[0] = param_index(m, d.param);
  out[1] = d.tp_rank;
  out[2] = d.tp_size;
  out[3] = d.pp_stage;
  out[4] = d.slice_dim;
  out[5] = d.start;
  out[6] = d.end;
}

// plan.cpp:8-32 (interleaved push order) and :89-121 (pulls).  Each shard is
// 7 int64 (param, tp_rank, tp_size, pp_stage, slice_dim, start, end); pulls
// are prefixed with the serving rank (8 int64 per entry).
int ref_plan(const RefParam* params, int n, int ttp, int tpp, int tdp, int stp,
             int spp, std::int64_t* push_out, int* npush, std::int64_t* pull_out,
             int* npull, int cap) {
  try {
    const auto m = to_manifest(params, n, 1);
    const auto order = interleave_pushes(plan_pushes(TrainConfig{ttp, tpp, tdp}, m));
    *npush = static_cast<int>(order.size());
    if (static_cast<int>(order.size()) > cap) return 22;
    for (std::size_t i = 0; i < order.size(); ++i) put_desc(push_out + 7 * i, m, order[i]);
    const auto pulls = plan_pulls(ServeConfig{stp, spp}, m, order);
    int k = 0;
    for (std::size_t r = 0; r < pulls.size(); ++r)
      for (const auto& d : pulls[r]) {
        if (k >= cap) return 22;
        pull_out[8 * k] = static_cast<std::int64_t>(r);
        put_desc(pull_out + 8 * k + 1, m, d);
        ++k;
      }
    *npull = k;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// --- sync state (bench.cpp:5-43 with a caller-supplied manifest) ------------
void* ref_state_create(const RefParam* params, int n, int dt, int ttp, int tpp,
                       int tdp, int stp, int spp, double density, std::uint64_t seed) {
  try {
    auto* s = new RefState;
    sim::RngHub hub(seed);  // bench.cpp:6-9
    s->train.cfg = TrainConfig{ttp, tpp, tdp};
    s->train.manifest = to_manifest(params, n, dt);
    s->train.prev = random_weights(s->train.manifest, hub.stream("weights.base"));
    s->train.next = perturb_weights(s->train.prev, density, hub.stream("weights.step"));
    s->scfg = ServeConfig{stp, spp};
    for (const auto& [name, t] : s->train.prev) s->model_bytes += static_cast<double>(t.byte_size());
    return s;
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

// The toy manifest of manifest.cpp:18-39, generated exactly like BenchHarness.
void* ref_state_create_toy(int layers, int hidden, int vocab, int dt, int ttp,
                           int tpp, int tdp, int stp, int spp, double density,
                           std::uint64_t seed) {
  try {
    const auto m = toy_transformer_manifest(
        ModelSpec{layers, hidden, vocab, static_cast<DType>(dt)});
    std::vector<RefParam> ps;
    for (const auto& p : m) {
      RefParam rp{p.name.c_str(), static_cast<int>(p.kind), static_cast<int>(p.shape.size()), {0, 0, 0, 0}, p.layer};
      for (std::size_t i = 0; i < p.shape.size(); ++i) rp.shape[i] = p.shape[i];
      ps.push_back(rp);
    }
    return ref_state_create(ps.data(), static_cast<int>(ps.size()), dt, ttp, tpp, tdp,
                            stp, spp, density, seed);
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

void ref_state_destroy(void* h) { delete static_cast<RefState*>(h); }

int ref_state_nparams(void* h) {
  return static_cast<int>(static_cast<RefState*>(h)->train.manifest.size());
}

const char* ref_state_param(void* h, int i, int* kind, int* ndims,
                            std::int64_t* shape, int* layer) {
  const auto& p = static_cast<RefState*>(h)->train.manifest[static_cast<std::size_t>(i)];
  *kind = static_cast<int>(p.kind);
  *ndims = static_cast<int>(p.shape.size());
  for (std::size_t k = 0; k < p.shape.size(); ++k) shape[k] = p.shape[k];
  *layer = p.layer;
  return p.name.c_str();
}

const void* ref_state_weights(void* h, int i, int which) {
  auto* s = static_cast<RefState*>(h);
  const auto& name = s->train.manifest[static_cast<std::size_t>(i)].name;
  return (which == 0 ? s->train.prev : s->train.next).at(name).data.data();
}

// bench.cpp:21-43 (MemoryRelay, unthrottled).  rep: wall, push, pull, encode,
// apply (s), pushed, pulled bytes, push/pull buckets, dense, sparse shards.
// ServeState::init (engine.cpp:34-49) ahead of the next run, so a timed
// run covers TransferEngine::sync_step alone (as bench.cpp:21-43 times it).
int ref_state_prepare(void* h) {
  auto* s = static_cast<RefState*>(h);
  try {
    s->serve = ServeState::init(s->scfg, s->train.manifest, s->train.prev);
    s->serve_ready = true;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_state_run(void* h, int mode, int shard_aware, int sparse, double threshold,
                  std::uint64_t bucket_bytes, int force_wide, double* rep) {
  auto* s = static_cast<RefState*>(h);
  try {
    if (!s->serve_ready) s->serve = ServeState::init(s->scfg, s->train.manifest, s->train.prev);
    s->serve_ready = false;
    auto mem = std::make_shared<MemoryRelay>();
    TransferEngine eng([mem]() -> std::shared_ptr<Relay> { return mem; }, nullptr, nullptr);
    SyncOptions o;
    o.mode = mode ? SyncMode::Async : SyncMode::Batch;
    o.shard_aware = shard_aware != 0;
    o.sparse = sparse != 0;
    o.density_threshold = threshold;
    o.bucket_bytes = bucket_bytes;
    o.force_wide_index = force_wide != 0;
    const TransferReport r = eng.sync_step(s->step++, s->train, s->serve, o);
    s->codecs = eng.last_codecs();
    const double v[] = {r.wall_s, r.push_s, r.pull_s, r.encode_s, r.apply_s,
                        static_cast<double>(r.pushed_bytes), static_cast<double>(r.pulled_bytes),
                        static_cast<double>(r.push_buckets), static_cast<double>(r.pull_buckets),
                        static_cast<double>(r.dense_shards), static_cast<double>(r.sparse_shards)};
    std::memcpy(rep, v, sizeof(v));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

double ref_state_model_bytes(void* h) { return static_cast<RefState*>(h)->model_bytes; }

// Serving shard of parameter i on serve rank `rank` (nullptr if not owned).
const void* ref_state_serve(void* h, int rank, int i, std::uint64_t* bytes) {
  auto* s = static_cast<RefState*>(h);
  const auto& name = s->train.manifest[static_cast<std::size_t>(i)].name;
  auto& m = s->serve.rank_weights[static_cast<std::size_t>(rank)];
  auto it = m.find(name);
  if (it == m.end()) return nullptr;
  *bytes = it->second.byte_size();
  return it->second.data.data();
}

int ref_state_ncodecs(void* h) {
  return static_cast<int>(static_cast<RefState*>(h)->codecs.size());
}

// 7 int64 descriptor (see put_desc) + codec char.
int ref_state_codec(void* h, int k, std::int64_t* desc) {
  auto* s = static_cast<RefState*>(h);
  const auto& [d, c] = s->codecs[static_cast<std::size_t>(k)];
  put_desc(desc, s->train.manifest, d);
  return c;
}

}  // extern "C"
