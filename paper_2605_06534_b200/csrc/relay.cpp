// relay.cpp -- the engine's cross-cluster sync through a relay (SURVEY.md
// 8(f) rank 4): TransferEngine::sync_step's pusher and puller
// (engine.cpp:109-238) with the encode, payloads, decode, reslice and apply on
// the GPU, and the relay reached through the C callbacks of ws_relay (the
// binding of the reference's Relay, relay.hpp:27-35).
//   pusher  K1 (encode only) -> per shard: device payload -> bucket D2H into
//           pinned staging on a copy stream, bucket k+1 in flight while bucket
//           k is paced (TokenBucket, relay.cpp:69-84) and put;
//   puller  (one per serving rank) per source, on any rank, of every
//           serving shard of this rank's coordinate (plan_pulls): probe the codec
//           with get_any over the D0/S4/S8 keys (engine.cpp:164-171), fetch
//           the remaining buckets, stage the payload to the GPU, decode,
//           reslice and apply (or copy the dense overlap) there.
//   modes   Async runs both sides concurrently, Batch pushes first
//           (engine.cpp:231-238).
#include <algorithm>
#include <cmath>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "capi_util.h"
#include "engine.h"

using namespace wsync;

namespace {

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

// TokenBucket (relay.cpp:69-84): a byte stream paced at `rate` against the
// wall clock; callers may overdraw and sleep the debt off.
class Pacer {
 public:
  Pacer(double rate, double burst) : rate_(rate), burst_(burst), tokens_(burst), last_(Clock::now()) {}
  void acquire(uint64_t bytes) {
    if (rate_ <= 0.0 || bytes == 0) return;
    double wait = 0;
    {
      std::lock_guard<std::mutex> lk(mu_);
      const auto now = Clock::now();
      tokens_ = std::min(burst_, tokens_ + secs(last_, now) * rate_);
      last_ = now;
      tokens_ -= (double)bytes;
      if (tokens_ < 0) wait = -tokens_ / rate_;
    }
    if (wait > 0) std::this_thread::sleep_for(std::chrono::duration<double>(wait));
  }

 private:
  double rate_, burst_, tokens_;
  Clock::time_point last_;
  std::mutex mu_;
};

// peek_payload_size (codec.cpp:219-227) on the first bucket, host side.
bool payload_total(const uint8_t* d, uint64_t n, uint64_t* total) {
  if (n < 8) return false;
  uint32_t magic;
  std::memcpy(&magic, d, 4);
  const bool sparse = magic == 0x31535743u || magic == 0x32535743u;
  const bool dense = magic == 0x31445743u || magic == 0x32445743u;
  if (!sparse && !dense) return false;
  const uint64_t esz = (magic >> 24) == '2' ? 2 : 4;
  const int nd = d[5], iw = d[6];
  uint64_t pos = 8 + 8 * (uint64_t)nd, elems = 1;
  if (n < pos) return false;
  constexpr uint64_t kMax = 1ull << 62;  // no payload is larger; keeps the products exact
  for (int k = 0; k < nd; ++k) {
    int64_t v;
    std::memcpy(&v, d + 8 + 8 * k, 8);
    if (v <= 0 || (uint64_t)v > kMax / elems) return false;
    elems *= (uint64_t)v;
  }
  if (dense) {
    if (elems > kMax / esz) return false;
    *total = pos + elems * esz;
    return true;
  }
  if (n < pos + 8 || (iw != 4 && iw != 8)) return false;
  uint64_t nnz;
  std::memcpy(&nnz, d + pos, 8);
  if (nnz > kMax / ((uint64_t)iw + esz)) return false;
  *total = pos + 8 + nnz * ((uint64_t)iw + esz);
  return true;
}

std::string key_of(uint64_t step, const std::string& param, const ShardDesc& d, char codec,
                   int iw, uint32_t seq) {
  char buf[8192];
  uint64_t n = 0;
  if (ws_bucket_key(step, param.c_str(), d.tp_rank, d.tp_size, d.pp_stage, d.d, codec, iw, seq,
                    buf, sizeof(buf), &n) != WS_OK)
    return std::string();
  return std::string(buf, n);
}

struct RelayError {
  ws_status st;
  std::string msg;
};

}  // namespace

ws_status ws_engine::sync_relay(uint64_t step, const ws_sync_options& o,
                                const ws_relay_options& ro, const ws_relay& relay,
                                ws_relay_report* rep) {
  if (!(relay.put && relay.get_any) && !(relay.put_frame && relay.get_any_frame))
    return set_error(WS_INVALID_ARGUMENT, "ws_engine_sync_relay: relay callbacks missing");
  if (ro.bucket_bytes == 0) return set_error(WS_INVALID_ARGUMENT, "bucket_bytes must be > 0");
  if (cudaSetDevice(device_) != cudaSuccess) return set_error(WS_CUDA, "cudaSetDevice");
  const int esz = dtype_size(dtype_);
  const int depth = std::max(2, ro.staging_buffers);
  const int timeout = ro.timeout_ms > 0 ? ro.timeout_ms : 10000;
  // streams and staging live in the engine across calls: pinning and
  // allocating hundreds of MB per sync would dominate it
  for (cudaStream_t& st : relay_streams_)
    if (!st) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaStream_t s_enc = relay_streams_[0], s_push = relay_streams_[1], s_pull = relay_streams_[2];
  auto cleanup = [] {};
  size_t dslot = 0, hslot = 0;  // the same allocation order every call
  auto dev_alloc = [&](size_t bytes) -> void* {
    bytes = std::max<size_t>(16, bytes);
    if (dslot == relay_dev_.size()) relay_dev_.push_back({nullptr, 0});
    auto& e = relay_dev_[dslot++];
    if (e.second < bytes) {
      cudaFree(e.first);
      e = {nullptr, 0};
      if (cudaMalloc(&e.first, bytes) != cudaSuccess) return nullptr;
      e.second = bytes;
    }
    return e.first;
  };
  auto host_alloc = [&](size_t bytes) -> uint8_t* {
    bytes = std::max<size_t>(16, bytes);
    if (hslot == relay_host_.size()) relay_host_.push_back({nullptr, 0});
    auto& e = relay_host_[hslot++];
    if (e.second < bytes) {
      cudaFreeHost(e.first);
      e = {nullptr, 0};
      if (cudaMallocHost(&e.first, bytes) != cudaSuccess) return nullptr;
      e.second = bytes;
    }
    return static_cast<uint8_t*>(e.first);
  };

  std::memset(rep, 0, sizeof(*rep));
  const auto wall0 = Clock::now();

  // ---- encode (K1 only: no fused apply, no routes) ------------------------
  encode_only_ = true;
  ws_status st = sync_step(o, s_enc, nullptr, nullptr, nullptr);
  encode_only_ = false;
  if (st != WS_OK) {
    cleanup();
    return st;
  }
  if (cudaStreamSynchronize(s_enc) != cudaSuccess) {
    cleanup();
    return set_error(WS_CUDA, "sync_relay: encode");
  }
  rep->encode_s = secs(wall0, Clock::now());
  // per-shard counts once (the pusher then never synchronises the device)
  std::vector<uint64_t> nnz_h(std::max(1, nseg_));
  if (nseg_ && cudaMemcpy(nnz_h.data(), d_nnz_, nseg_ * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
    cleanup();
    return set_error(WS_CUDA, "sync_relay: counts");
  }

  // What this rank pulls: every trainer shard, of any rank, with a route to
  // its serving coordinate (plan_pulls, one puller per serving rank as
  // engine.cpp:233-238; replicas of a coordinate pull independently).
  const auto& segs = plan_.segments();
  struct Pull {
    const Segment* src;
    const Route* route;
  };
  std::vector<Pull> pulls;
  for (int g = 0; g < plan_.world(); ++g)
    for (const Route& r : plan_.routes_of(g))
      if (g == plan_.rank() ? plan_.route_is_local(r) : r.coord == plan_.my_coord())
        pulls.push_back(Pull{&plan_.segments_of(g)[r.seg], &r});
  // sizes: the largest payload (dense bound) and record count of a shard
  // pushed or pulled here (a sparse payload holds at most threshold x n + 1)
  uint64_t max_payload = 64, max_n = 1, max_cap = 1;
  auto size_for = [&](const Segment& sg) {
    const int nd = (int)plan_.manifest()[sg.shard.param].shape.size();
    const uint64_t cap = std::min<uint64_t>(
        sg.n, (uint64_t)std::floor(std::max(0.0, o.density_threshold) * (double)sg.n) + 1);
    max_payload = std::max<uint64_t>(
        max_payload, std::max(ws_payload_bytes((ws_dtype)dtype_, nd, 'D', 0, sg.n),
                              ws_payload_bytes((ws_dtype)dtype_, nd, 'S', 8, cap)));
    max_n = std::max<uint64_t>(max_n, sg.n);
    max_cap = std::max<uint64_t>(max_cap, cap);
  };
  for (const Segment& sg : segs) size_for(sg);
  for (const Pull& pl : pulls) size_for(*pl.src);
  const uint64_t B = ro.bucket_bytes;

  Pacer push_pacer(ro.push_bytes_per_s, ro.burst_bytes > 0 ? ro.burst_bytes : (double)B);
  Pacer pull_pacer(ro.pull_bytes_per_s, ro.burst_bytes > 0 ? ro.burst_bytes : (double)B);
  std::mutex err_mu;
  RelayError first_err{WS_OK, ""};
  auto fail = [&](ws_status e, const std::string& m) {
    std::lock_guard<std::mutex> lk(err_mu);
    if (first_err.st == WS_OK) first_err = RelayError{e, m};
  };
  std::atomic<uint64_t> pushed{0}, pulled{0}, pbk{0}, lbk{0};
  std::atomic<uint32_t> dense_n{0}, sparse_n{0};
  double push_s = 0, pull_s = 0, apply_s = 0;

  // ---- pusher --------------------------------------------------------------
  // Framed transport (put_frame / get_any_frame): every bucket travels as the
  // frame of wire.cpp:35-47, built and CRC-32'd on the GPU; a frame adds
  // 12 bytes and its key to the bucket.
  const bool framed = relay.put_frame && relay.get_any_frame;
  if ((relay.put_frame != nullptr) != (relay.get_any_frame != nullptr))
    return set_error(WS_INVALID_ARGUMENT, "ws_relay: put_frame and get_any_frame go together");
  constexpr uint64_t kKeyRoom = 8192;  // key_of's buffer
  const uint64_t max_buckets = (max_payload + B - 1) / B + 1;
  const uint64_t frame_cap = std::min<uint64_t>(B, max_payload) + 12 + kKeyRoom;
  void* d_payload = dev_alloc(max_payload);
  uint32_t* d_seq_idx = static_cast<uint32_t*>(dev_alloc(max_cap * 4));
  void* d_seq_val = dev_alloc(max_cap * esz);
  void* d_frames = framed ? dev_alloc(max_payload + max_buckets * (12 + kKeyRoom)) : nullptr;
  std::vector<uint8_t*> stage(depth);
  for (auto& p : stage) p = host_alloc(framed ? frame_cap : std::min<uint64_t>(B, max_payload));
  std::vector<cudaEvent_t> ev(depth);
  for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  bool staged = d_payload && d_seq_idx && d_seq_val && (!framed || d_frames);
  for (auto* p : stage) staged = staged && p;
  auto pusher = [&] {
    // (a fresh std::thread in Async mode: its current device is 0)
    if (cudaSetDevice(device_) != cudaSuccess) {
      fail(WS_CUDA, "sync_relay: pusher cudaSetDevice");
      return;
    }
    const auto t0 = Clock::now();
    for (size_t i = 0; i < segs.size() && first_err.st == WS_OK; ++i) {
      ws_payload_info info;
      // the shard's ascending stream on the pusher's stream (codec.cpp:48-49
      // order), then its payload (engine.cpp:118-128)
      const uint64_t n = nnz_h[i];
      const bool sparse = o.sparse && n <= segs_[i].cap;
      ws_status e = WS_OK;
      if (sparse && n) e = compact_segment((int)i, d_seq_idx, d_seq_val, s_push);
      if (e == WS_OK)
        e = payload_from((int)i, ro.force_wide_index != 0, d_seq_idx, d_seq_val, n,
                         sparse ? 'S' : 'D', d_payload, &info, s_push);
      if (e != WS_OK) {
        fail(e, "sync_relay: payload");
        return;
      }
      (info.codec == 'S' ? sparse_n : dense_n)++;
      const std::string& name = plan_.manifest()[segs[i].shard.param].name;
      const uint64_t total = info.total_bytes;
      const uint64_t nb = total ? (total + B - 1) / B : 1;  // engine.cpp:139
      std::vector<std::string> keys(nb);
      for (uint64_t k = 0; k < nb; ++k)
        keys[k] = key_of(step, name, segs[i].shard, info.codec, info.index_width, (uint32_t)k);
      std::vector<uint64_t> frame_off(nb + 1, 0);
      if (framed) {  // every bucket's frame, CRC included, built on the GPU
        std::vector<const char*> kp(nb);
        std::vector<uint64_t> kl(nb);
        for (uint64_t k = 0; k < nb; ++k) {
          kp[k] = keys[k].data();
          kl[k] = keys[k].size();
        }
        e = ws_encode_bucket_frames_dev(d_payload, total, B, kp.data(), kl.data(), (int)nb,
                                        d_frames, max_payload + max_buckets * (12 + kKeyRoom),
                                        frame_off.data(), reinterpret_cast<ws_stream_t>(s_push));
        if (e != WS_OK) {
          fail(e, std::string("sync_relay: frames: ") + ws_last_error());
          return;
        }
      }
      auto issue = [&](uint64_t k) {
        if (framed) {
          cudaMemcpyAsync(stage[k % depth], static_cast<char*>(d_frames) + frame_off[k],
                          frame_off[k + 1] - frame_off[k], cudaMemcpyDeviceToHost, s_push);
        } else {
          const uint64_t n = std::min(B, total - std::min(total, k * B));
          cudaMemcpyAsync(stage[k % depth], static_cast<char*>(d_payload) + k * B, n,
                          cudaMemcpyDeviceToHost, s_push);
        }
        cudaEventRecord(ev[k % depth], s_push);
      };
      for (uint64_t k = 0; k < std::min<uint64_t>(nb, depth - 1); ++k) issue(k);
      for (uint64_t k = 0; k < nb; ++k) {
        if (k + depth - 1 < nb) issue(k + depth - 1);  // overlaps this bucket's put
        cudaEventSynchronize(ev[k % depth]);
        const uint64_t n = std::min(B, total - std::min(total, k * B));
        push_pacer.acquire(n);
        const std::string& key = keys[k];
        if (framed) {
          const int rc = relay.put_frame(relay.ctx, stage[k % depth], frame_off[k + 1] - frame_off[k]);
          if (rc != 0) {  // 3: the receiver's CRC check failed (tcp_relay.hpp status 3)
            fail(rc == 3 ? WS_INTEGRITY : WS_TRANSFER_ERROR,
                 (rc == 3 ? "relay rejected the frame of '" : "relay put failed for '") + key + "'");
            return;
          }
        } else if (relay.put(relay.ctx, key.data(), key.size(), stage[k % depth], n) != 0) {
          fail(WS_TRANSFER_ERROR, "relay put failed for '" + key + "'");
          return;
        }
        pushed += n;
        ++pbk;
      }
    }
    push_s = secs(t0, Clock::now());
  };

  // ---- puller --------------------------------------------------------------
  uint8_t* h_payload = host_alloc(framed ? frame_cap : max_payload);
  void* d_in = dev_alloc(max_payload);
  void* d_frame = framed ? dev_alloc(frame_cap) : nullptr;
  uint32_t* d_one = framed ? static_cast<uint32_t*>(dev_alloc(8)) : nullptr;
  uint32_t* d_idx = static_cast<uint32_t*>(dev_alloc(max_cap * 4));
  void* d_val = dev_alloc(max_cap * 4);
  uint32_t* d_ridx = static_cast<uint32_t*>(dev_alloc(max_cap * 4));
  void* d_rval = dev_alloc(max_cap * 4);
  uint64_t* d_rnnz = static_cast<uint64_t*>(dev_alloc(8));
  uint32_t* d_err = static_cast<uint32_t*>(dev_alloc(8));
  uint32_t* d_rerr = d_err ? d_err + 1 : nullptr;  // reslice's own error word
  size_t ws_bytes = ws_diff_workspace_bytes(max_cap);
  void* d_ws = dev_alloc(ws_bytes);
  staged = staged && (!framed || (d_frame && d_one)) && h_payload && d_in && d_idx && d_val && d_ridx && d_rval && d_rnnz && d_err &&
           d_ws;
  if (!staged) {
    for (auto& e : ev) cudaEventDestroy(e);
    return set_error(WS_CUDA, "sync_relay: staging allocation failed");
  }
  // Record scratch beyond max_cap: a pusher with a higher density threshold
  // than ours sends sparse payloads with more records (the reference decodes
  // any size); grown per payload, freed at the end of the call.
  struct Grown {
    void* p[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    uint64_t cap = 0;
    ~Grown() {
      for (void* q : p) cudaFree(q);
    }
  } grown;
  auto records_for = [&](uint64_t nnz) -> bool {
    if (nnz <= max_cap) return true;
    if (nnz > grown.cap) {
      for (void*& q : grown.p) {
        cudaFree(q);
        q = nullptr;
      }
      grown.cap = 0;
      const size_t sz[5] = {nnz * 4, nnz * 4, nnz * 4, nnz * 4, ws_diff_workspace_bytes(nnz)};
      for (int k = 0; k < 5; ++k)
        if (cudaMalloc(&grown.p[k], std::max<size_t>(16, sz[k])) != cudaSuccess) {
          cudaGetLastError();
          return false;
        }
      grown.cap = nnz;
    }
    d_idx = static_cast<uint32_t*>(grown.p[0]);
    d_val = grown.p[1];
    d_ridx = static_cast<uint32_t*>(grown.p[2]);
    d_rval = grown.p[3];
    d_ws = grown.p[4];
    ws_bytes = ws_diff_workspace_bytes(grown.cap);
    return true;
  };
  const bool dbg = ablation_env("WSYNC_RELAY_DEBUG") != nullptr;
  double dt[5] = {0, 0, 0, 0, 0};  // debug: h2d, peek, decode, reslice, apply
  // Framed pull of one bucket: the frame (in h_payload) is checked on the
  // GPU -- its CRC-32 over every preceding byte (wire.cpp:45, IntegrityError
  // on mismatch) and its key -- and its bucket lands at d_in + at.  Returns
  // the bucket length, or -1 after fail().
  auto take_frame = [&](int64_t n, const std::string& want_key, uint64_t at,
                        uint64_t room) -> int64_t {
    if (n < 12 || (uint64_t)n > frame_cap) {
      fail(WS_PAYLOAD_FORMAT, "relay frame of '" + want_key + "' is truncated or oversized");
      return -1;
    }
    uint32_t klen = 0, plen = 0, crc = 0;
    std::memcpy(&klen, h_payload, 4);
    if ((uint64_t)klen + 12 > (uint64_t)n) {
      fail(WS_PAYLOAD_FORMAT, "relay frame of '" + want_key + "': key length");
      return -1;
    }
    std::memcpy(&plen, h_payload + 4 + klen, 4);
    if ((uint64_t)klen + plen + 12 != (uint64_t)n || plen > room) {
      fail(WS_PAYLOAD_FORMAT, "relay frame of '" + want_key + "': payload length");
      return -1;
    }
    if (std::string(reinterpret_cast<const char*>(h_payload) + 4, klen) != want_key) {
      fail(WS_PAYLOAD_FORMAT, "relay frame carries another key than '" + want_key + "'");
      return -1;
    }
    std::memcpy(&crc, h_payload + 8 + klen + plen, 4);
    cudaMemcpyAsync(d_frame, h_payload, (uint64_t)n, cudaMemcpyHostToDevice, s_pull);
    const void* fp = d_frame;
    const uint64_t covered = 8 + (uint64_t)klen + plen;
    uint32_t got = 0;
    ws_status e = ws_crc32_dev(&fp, &covered, 1, &got, reinterpret_cast<ws_stream_t>(s_pull));
    if (e != WS_OK) {
      fail(e, std::string("sync_relay: frame crc: ") + ws_last_error());
      return -1;
    }
    if (got != crc) {
      fail(WS_INTEGRITY, "frame CRC mismatch for '" + want_key + "'");
      return -1;
    }
    cudaMemcpyAsync(static_cast<char*>(d_in) + at, static_cast<const char*>(d_frame) + 8 + klen,
                    plen, cudaMemcpyDeviceToDevice, s_pull);
    return plen;
  };
  auto puller = [&] {
    const auto t0 = Clock::now();
    double apply_acc = 0;
    for (const Pull& pl : pulls) {
      if (first_err.st != WS_OK) return;
      const Route& r = *pl.route;
      const Segment& src = *pl.src;
      const ParamMeta& p = plan_.manifest()[src.shard.param];
      std::string cand[3] = {key_of(step, p.name, src.shard, 'D', 0, 0),
                             key_of(step, p.name, src.shard, 'S', 4, 0),
                             key_of(step, p.name, src.shard, 'S', 8, 0)};
      const char* kp[3] = {cand[0].data(), cand[1].data(), cand[2].data()};
      const uint64_t kl[3] = {cand[0].size(), cand[1].size(), cand[2].size()};
      int hit = -1;
      int64_t n0 = framed ? relay.get_any_frame(relay.ctx, kp, kl, 3, timeout, &hit, h_payload,
                                                frame_cap)
                          : relay.get_any(relay.ctx, kp, kl, 3, timeout, &hit, h_payload,
                                          max_payload);
      if (n0 < 0 || hit < 0 || hit > 2) {
        fail(n0 == -1 ? WS_RELAY_TIMEOUT : WS_TRANSFER_ERROR,
             "relay get_any for '" + cand[1] + "' failed");
        return;
      }
      const uint8_t* head0 = h_payload;
      if (framed) {  // bucket 0 to d_in; its payload header read from the host copy
        uint32_t klen0 = 0;
        if (n0 >= 12) std::memcpy(&klen0, h_payload, 4);
        head0 = h_payload + 8 + klen0;
        n0 = take_frame(n0, cand[hit], 0, max_payload);
        if (n0 < 0) return;
      }
      pull_pacer.acquire((uint64_t)n0);
      uint64_t total = 0;
      if (!payload_total(head0, (uint64_t)n0, &total) || total > max_payload) {
        fail(WS_PAYLOAD_FORMAT, "bad first bucket for '" + cand[hit] + "'");
        return;
      }
      if ((uint64_t)n0 != std::min(total, B)) {
        fail(WS_PAYLOAD_FORMAT, "bucket 0 of '" + cand[hit] + "' has a wrong size");
        return;
      }
      const char codec = hit == 0 ? 'D' : 'S';
      const int iw = hit == 0 ? 0 : (hit == 1 ? 4 : 8);
      const uint64_t nb = total ? (total + B - 1) / B : 1;
      uint64_t have = (uint64_t)n0;
      pulled += have;
      ++lbk;
      for (uint64_t k = 1; k < nb; ++k) {
        const std::string kk = key_of(step, p.name, src.shard, codec, iw, (uint32_t)k);
        const char* kkp = kk.data();
        const uint64_t kkl = kk.size();
        int h = -1;
        int64_t nk = framed ? relay.get_any_frame(relay.ctx, &kkp, &kkl, 1, timeout, &h,
                                                  h_payload, frame_cap)
                            : relay.get_any(relay.ctx, &kkp, &kkl, 1, timeout, &h,
                                            h_payload + have, max_payload - have);
        if (framed && nk >= 0) {
          nk = take_frame(nk, kk, have, total - have);
          if (nk < 0) return;
        }
        if (nk < 0 || have + (uint64_t)nk > total) {
          fail(nk == -1 ? WS_RELAY_TIMEOUT : WS_PAYLOAD_FORMAT, "relay get for '" + kk + "' failed");
          return;
        }
        pull_pacer.acquire((uint64_t)nk);
        have += (uint64_t)nk;
        pulled += (uint64_t)nk;
        ++lbk;
      }
      if (have != total) {
        fail(WS_PAYLOAD_FORMAT, "reassembled payload has the wrong size");
        return;
      }
      const auto ta = Clock::now();
      if (!framed) cudaMemcpyAsync(d_in, h_payload, total, cudaMemcpyHostToDevice, s_pull);
      cudaStreamSynchronize(s_pull);
      auto tk = Clock::now();
      auto lap = [&](int q) {
        if (!dbg) return;
        cudaStreamSynchronize(s_pull);
        const auto now = Clock::now();
        dt[q] += secs(tk, now);
        tk = now;
      };
      dt[0] += dbg ? secs(ta, tk) : 0.0;
      ws_payload_info info;
      ws_status e = ws_peek_payload_dev(d_in, total, &info);
      lap(1);
      if (e != WS_OK) {
        fail(e, std::string(ws_last_error()));
        return;
      }
      const int nd = (int)p.shape.size();
      // the payload must be the planned source shard (codec.cpp:98-100:
      // ShapeMismatch), or its records would land at remapped positions
      bool shape_ok = info.ndims == nd && info.dtype == dtype_;
      for (int dd = 0; shape_ok && dd < nd; ++dd)
        shape_ok = info.shape[dd] == (src.shard.d.slice_dim == dd
                                          ? src.shard.d.end - src.shard.d.start
                                          : p.shape[dd]);
      if (!shape_ok) {
        fail(WS_SHAPE_MISMATCH, "sync_relay: payload of '" + cand[hit] +
                                    "' does not have the source shard's dtype and shape");
        return;
      }
      if (info.codec == 'S' && !records_for(info.nnz)) {
        fail(WS_CUDA, "sync_relay: record scratch allocation failed");
        return;
      }
      const ws_stream_t ps = reinterpret_cast<ws_stream_t>(s_pull);
      char* tgt = static_cast<char*>(serve) + r.dst_offset * esz;
      if (info.codec == 'S') {
        e = ws_decode_sparse_dev(d_in, &info, d_idx, d_val, ps);
        lap(2);
        if (e == WS_OK)
          e = ws_reslice_delta((ws_dtype)dtype_, p.shape.data(), nd, src.shard.d, r.dst.d, 1,
                               d_idx, d_val, info.nnz, nullptr, d_ridx, d_rval, d_rnnz, d_rerr,
                               d_ws, ws_bytes, ps);
        uint64_t dn = 1;
        for (int dd = 0; dd < nd; ++dd)
          dn *= (uint64_t)(r.dst.d.slice_dim == dd ? r.dst.d.end - r.dst.d.start : p.shape[dd]);
        lap(3);
        if (e == WS_OK)
          e = ws_apply_delta((ws_dtype)dtype_, tgt, dn, d_ridx, d_rval, info.nnz /* bound */,
                             d_rnnz, d_err, ps);
        lap(4);
        uint32_t herr[2] = {0, 0};  // apply's and reslice's error words
        cudaMemcpyAsync(herr, d_err, 8, cudaMemcpyDeviceToHost, s_pull);
        cudaStreamSynchronize(s_pull);
        if (e == WS_OK && herr[1])  // reslice_delta throws IndexOutOfShard (codec.cpp:120-122)
          e = set_error(WS_INDEX_OUT_OF_SHARD, "sync_relay: reslice: index outside the source shard");
        if (e == WS_OK && herr[0]) e = set_error(WS_INDEX_OUT_OF_SHARD, "sync_relay: apply");
      } else {
        int64_t copied = 0;
        e = ws_copy_overlap((ws_dtype)dtype_, p.shape.data(), nd, r.dst.d, tgt, src.shard.d,
                            static_cast<char*>(d_in) + info.header_bytes, &copied, ps);
        cudaStreamSynchronize(s_pull);
      }
      if (e != WS_OK) {
        fail(e, std::string(ws_last_error()));
        return;
      }
      apply_acc += secs(ta, Clock::now());
    }
    pull_s = secs(t0, Clock::now());
    apply_s = apply_acc;
  };

  const auto t_net = Clock::now();
  if (ro.async) {
    std::thread pt(pusher);
    puller();
    pt.join();
  } else {
    pusher();
    if (first_err.st == WS_OK) puller();
  }
  (void)t_net;
  for (auto& e : ev) cudaEventDestroy(e);
  if (dbg)
    fprintf(stderr, "relay puller: h2d %.4f peek %.4f decode %.4f reslice %.4f apply %.4f s\n",
            dt[0], dt[1], dt[2], dt[3], dt[4]);
  cleanup();
  rep->wall_s = secs(wall0, Clock::now());
  rep->push_s = push_s;
  rep->pull_s = pull_s;
  rep->apply_s = apply_s;
  rep->pushed_bytes = pushed;
  rep->pulled_bytes = pulled;
  rep->push_buckets = pbk;
  rep->pull_buckets = lbk;
  rep->dense_shards = dense_n;
  rep->sparse_shards = sparse_n;
  if (first_err.st != WS_OK) return set_error(first_err.st, first_err.msg);
  return WS_OK;
}

namespace wsync {
void scratch_trim(int dev);  // wire.cu
}

ws_status ws_engine::release_staging() {
  if (cudaSetDevice(device_) != cudaSuccess) return set_error(WS_CUDA, "cudaSetDevice");
  for (cudaStream_t st : relay_streams_)
    if (st) cudaStreamSynchronize(st);
  for (auto& e : relay_dev_) cudaFree(e.first);
  for (auto& e : relay_host_) cudaFreeHost(e.first);
  relay_dev_.clear();
  relay_host_.clear();
  cudaDeviceSynchronize();
  scratch_trim(device_);
  return cudaGetLastError() == cudaSuccess ? WS_OK : set_error(WS_CUDA, "release_staging");
}

extern "C" ws_status ws_engine_release_staging(ws_engine* eng) {
  DeviceGuard device_guard;
  if (!eng) return set_error(WS_INVALID_ARGUMENT, "ws_engine_release_staging: null engine");
  return eng->release_staging();
}

extern "C" ws_status ws_engine_sync_relay(ws_engine* eng, uint64_t step,
                                          const ws_sync_options* opts,
                                          const ws_relay_options* relay_opts,
                                          const ws_relay* relay, ws_relay_report* report) {
  DeviceGuard device_guard;
  if (!eng || !opts || !relay_opts || !relay || !report)
    return set_error(WS_INVALID_ARGUMENT, "ws_engine_sync_relay: null argument");
  try {
    return eng->sync_relay(step, *opts, *relay_opts, *relay, report);
  } catch (const std::exception& e) {
    return set_error(WS_TRANSFER_ERROR, e.what());
  }
}
