// codec_shim.cpp -- the reference's codec API (coserve/transfer/codec.hpp),
// implemented on top of libwsync's C-ABI (include/wsync.h).
//
// Compiled against the reference's own headers and linked INSTEAD of the
// reference's codec.cpp, it turns the unmodified reference engine
// (engine.cpp's sync_step pusher/puller threads, bench.cpp, plan.cpp ...) into
// a client of the B200 kernels: diff_shards -> K1 (ws_diff_shards),
// apply_delta -> K4 (ws_apply_delta), reslice_delta -> ws_reslice_delta.
// The payload functions (encode_dense / encode_sparse / pick_index_width /
// decode_payload / peek_payload_size) restate the wire format of
// codec.hpp:50-70 on the host.  See INTEGRATION.md.
//
// Each calling thread gets its own CUDA stream and device scratch (the
// reference runs one pusher and several puller threads concurrently,
// engine.cpp:233-238).
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "coserve/transfer/codec.hpp"
#include "wsync.h"

namespace coserve::transfer {

namespace {

struct DeviceScratch {
  cudaStream_t stream = nullptr;
  std::vector<std::pair<void*, size_t>> bufs;  // grown on demand
  DeviceScratch() {
    if (cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) != cudaSuccess)
      throw TransferError("codec shim: no CUDA device");
    bufs.assign(8, {nullptr, 0});
  }
  ~DeviceScratch() {
    for (auto& b : bufs) cudaFree(b.first);
    if (stream) cudaStreamDestroy(stream);
  }
  void* get(int slot, size_t bytes) {
    auto& b = bufs[static_cast<size_t>(slot)];
    if (b.second < bytes || !b.first) {
      cudaFree(b.first);
      b.first = nullptr;
      const size_t want = bytes < 256 ? 256 : bytes;
      if (cudaMalloc(&b.first, want) != cudaSuccess) throw TransferError("codec shim: cudaMalloc");
      b.second = want;
    }
    return b.first;
  }
};

DeviceScratch& scratch() {
  thread_local DeviceScratch s;
  return s;
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw TransferError(std::string(what) + ": " + cudaGetErrorString(e));
}

void ws_ok(ws_status st) {
  switch (st) {
    case WS_OK: return;
    case WS_SHAPE_MISMATCH: throw ShapeMismatch(ws_last_error());
    case WS_PAYLOAD_FORMAT: throw PayloadFormatError(ws_last_error());
    case WS_INDEX_OUT_OF_SHARD: throw IndexOutOfShard(ws_last_error());
    default: throw TransferError(std::string(ws_status_name(st)) + ": " + ws_last_error());
  }
}

ws_dtype wdt(DType d) { return d == DType::F32 ? WS_F32 : WS_I32; }

template <typename T>
void put(std::vector<std::uint8_t>& out, T v) {
  const std::size_t at = out.size();
  out.resize(at + sizeof(T));
  std::memcpy(out.data() + at, &v, sizeof(T));
}

template <typename T>
T get(const std::uint8_t* data, std::size_t len, std::size_t& pos, const char* what) {
  if (pos + sizeof(T) > len) throw PayloadFormatError(std::string("payload truncated reading ") + what);
  T v;
  std::memcpy(&v, data + pos, sizeof(T));
  pos += sizeof(T);
  return v;
}

constexpr std::uint32_t kDense = 0x31445743u;   // "CWD1"
constexpr std::uint32_t kSparse = 0x31535743u;  // "CWS1"

struct Head {
  std::uint32_t magic;
  DType dtype;
  int iw;
  std::vector<std::int64_t> shape;
  std::size_t pos;
};

Head read_head(const std::uint8_t* data, std::size_t len) {
  Head h;
  std::size_t pos = 0;
  h.magic = get<std::uint32_t>(data, len, pos, "magic");
  if (h.magic != kDense && h.magic != kSparse) throw PayloadFormatError("bad payload magic");
  const auto dt = get<std::uint8_t>(data, len, pos, "dtype");
  if (dt > 1) throw PayloadFormatError("bad dtype " + std::to_string(dt));
  h.dtype = static_cast<DType>(dt);
  const int nd = get<std::uint8_t>(data, len, pos, "ndims");
  h.iw = get<std::uint8_t>(data, len, pos, "index width");
  (void)get<std::uint8_t>(data, len, pos, "pad");
  for (int i = 0; i < nd; ++i) {
    const auto d = get<std::int64_t>(data, len, pos, "dim");
    if (d <= 0) throw PayloadFormatError("non-positive dim");
    h.shape.push_back(d);
  }
  h.pos = pos;
  return h;
}

void write_head(std::vector<std::uint8_t>& out, std::uint32_t magic, DType dt,
                const std::vector<std::int64_t>& shape, std::uint8_t iw) {
  put(out, magic);
  put(out, static_cast<std::uint8_t>(dt));
  put(out, static_cast<std::uint8_t>(shape.size()));
  put(out, iw);
  put(out, std::uint8_t{0});
  for (auto d : shape) put(out, d);
}

}  // namespace

SparseDelta diff_shards(const HostTensor& prev, const HostTensor& next) {
  if (!prev.same_layout(next))
    throw ShapeMismatch("diff_shards: " + shape_str(prev.shape) + " vs " + shape_str(next.shape));
  SparseDelta d;
  d.dtype = prev.dtype;
  d.shape = prev.shape;
  const std::uint64_t n = static_cast<std::uint64_t>(prev.elems());
  if (n == 0) return d;
  DeviceScratch& s = scratch();
  const size_t bytes = prev.data.size();
  void* a = s.get(0, bytes);
  void* b = s.get(1, bytes);
  auto* idx = static_cast<std::uint32_t*>(s.get(2, n * 4));
  void* val = s.get(3, n * 4);
  auto* cnt = static_cast<std::uint64_t*>(s.get(4, 8));
  const size_t wsb = ws_diff_workspace_bytes(n);
  void* wsp = s.get(5, wsb);
  cuda_ok(cudaMemcpyAsync(a, prev.data.data(), bytes, cudaMemcpyHostToDevice, s.stream), "H2D");
  cuda_ok(cudaMemcpyAsync(b, next.data.data(), bytes, cudaMemcpyHostToDevice, s.stream), "H2D");
  ws_ok(ws_diff_shards(wdt(prev.dtype), a, b, n, idx, val, n, cnt, wsp, wsb,
                       reinterpret_cast<ws_stream_t>(s.stream)));
  std::uint64_t nnz = 0;
  cuda_ok(cudaMemcpyAsync(&nnz, cnt, 8, cudaMemcpyDeviceToHost, s.stream), "D2H");
  cuda_ok(cudaStreamSynchronize(s.stream), "sync");
  std::vector<std::uint32_t> i32(nnz);
  d.values.resize(nnz * 4);
  cuda_ok(cudaMemcpyAsync(i32.data(), idx, nnz * 4, cudaMemcpyDeviceToHost, s.stream), "D2H");
  cuda_ok(cudaMemcpyAsync(d.values.data(), val, nnz * 4, cudaMemcpyDeviceToHost, s.stream), "D2H");
  cuda_ok(cudaStreamSynchronize(s.stream), "sync");
  d.indices.assign(i32.begin(), i32.end());
  return d;
}

void apply_delta(HostTensor& target, const SparseDelta& delta) {
  if (target.dtype != delta.dtype || target.shape != delta.shape)
    throw ShapeMismatch("apply_delta: target " + shape_str(target.shape) + " vs delta " +
                        shape_str(delta.shape));
  const std::uint64_t n = static_cast<std::uint64_t>(target.elems());
  const std::uint64_t nnz = delta.indices.size();
  if (nnz == 0) return;
  std::vector<std::uint32_t> i32(nnz);
  for (std::uint64_t k = 0; k < nnz; ++k) {
    if (delta.indices[k] >= n)  // validated before any write (tightens codec.cpp:73-79)
      throw IndexOutOfShard("delta index " + std::to_string(delta.indices[k]) + " >= " +
                            std::to_string(n));
    i32[k] = static_cast<std::uint32_t>(delta.indices[k]);
  }
  DeviceScratch& s = scratch();
  void* t = s.get(0, target.data.size());
  auto* idx = static_cast<std::uint32_t*>(s.get(2, nnz * 4));
  void* val = s.get(3, nnz * 4);
  auto* err = static_cast<std::uint32_t*>(s.get(4, 8));
  cuda_ok(cudaMemcpyAsync(t, target.data.data(), target.data.size(), cudaMemcpyHostToDevice,
                          s.stream), "H2D");
  cuda_ok(cudaMemcpyAsync(idx, i32.data(), nnz * 4, cudaMemcpyHostToDevice, s.stream), "H2D");
  cuda_ok(cudaMemcpyAsync(val, delta.values.data(), nnz * 4, cudaMemcpyHostToDevice, s.stream),
          "H2D");
  ws_ok(ws_apply_delta(wdt(target.dtype), t, n, idx, val, nnz, nullptr, err,
                       reinterpret_cast<ws_stream_t>(s.stream)));
  std::uint32_t bits = 0;
  cuda_ok(cudaMemcpyAsync(&bits, err, 4, cudaMemcpyDeviceToHost, s.stream), "D2H");
  cuda_ok(cudaMemcpyAsync(target.data.data(), t, target.data.size(), cudaMemcpyDeviceToHost,
                          s.stream), "D2H");
  cuda_ok(cudaStreamSynchronize(s.stream), "sync");
  if (bits & WS_ERRBIT_INDEX_OUT_OF_SHARD) throw IndexOutOfShard("delta index outside the shard");
}

SparseDelta reslice_delta(const SparseDelta& delta, const ShardDescriptor& src,
                          const ShardDescriptor& dst,
                          const std::vector<std::int64_t>& full_shape) {
  const auto src_shape = shard_shape(src, full_shape);
  if (delta.shape != src_shape)
    throw ShapeMismatch("reslice_delta: delta " + shape_str(delta.shape) +
                        " does not match source shard " + shape_str(src_shape));
  if (!src.full() && !dst.full() && src.slice_dim != dst.slice_dim)
    throw ShapeMismatch("reslice_delta: slices along different dims");
  SparseDelta out;
  out.dtype = delta.dtype;
  out.shape = shard_shape(dst, full_shape);
  const std::uint64_t nnz = delta.indices.size();
  std::uint64_t src_elems = 1;
  for (auto d : src_shape) src_elems *= static_cast<std::uint64_t>(d);
  std::vector<std::uint32_t> i32(nnz);
  for (std::uint64_t k = 0; k < nnz; ++k) {
    if (delta.indices[k] >= src_elems)  // codec.cpp:121-124
      throw IndexOutOfShard("delta index " + std::to_string(delta.indices[k]) +
                            " outside source shard of " + std::to_string(src_elems));
    i32[k] = static_cast<std::uint32_t>(delta.indices[k]);
  }
  if (nnz == 0) return out;
  DeviceScratch& s = scratch();
  auto* idx = static_cast<std::uint32_t*>(s.get(0, nnz * 4));
  void* val = s.get(1, nnz * 4);
  auto* oidx = static_cast<std::uint32_t*>(s.get(2, nnz * 4));
  void* oval = s.get(3, nnz * 4);
  auto* cnt = static_cast<std::uint64_t*>(s.get(4, 16));
  auto* err = cnt + 1;
  const size_t wsb = ws_diff_workspace_bytes(nnz);
  void* wsp = s.get(5, wsb);
  cuda_ok(cudaMemcpyAsync(idx, i32.data(), nnz * 4, cudaMemcpyHostToDevice, s.stream), "H2D");
  cuda_ok(cudaMemcpyAsync(val, delta.values.data(), nnz * 4, cudaMemcpyHostToDevice, s.stream),
          "H2D");
  const ws_shard ws_src{src.slice_dim, src.full() ? 0 : src.start, src.full() ? 0 : src.end};
  const ws_shard ws_dst{dst.slice_dim, dst.full() ? 0 : dst.start, dst.full() ? 0 : dst.end};
  ws_ok(ws_reslice_delta(wdt(delta.dtype), full_shape.data(), static_cast<int>(full_shape.size()),
                         ws_src, ws_dst, /*allow_cross_dim=*/0, idx, val, nnz, nullptr, oidx,
                         oval, cnt, reinterpret_cast<std::uint32_t*>(err), wsp, wsb,
                         reinterpret_cast<ws_stream_t>(s.stream)));
  std::uint64_t n_out = 0;
  cuda_ok(cudaMemcpyAsync(&n_out, cnt, 8, cudaMemcpyDeviceToHost, s.stream), "D2H");
  cuda_ok(cudaStreamSynchronize(s.stream), "sync");
  std::vector<std::uint32_t> o32(n_out);
  out.values.resize(n_out * 4);
  cuda_ok(cudaMemcpyAsync(o32.data(), oidx, n_out * 4, cudaMemcpyDeviceToHost, s.stream), "D2H");
  cuda_ok(cudaMemcpyAsync(out.values.data(), oval, n_out * 4, cudaMemcpyDeviceToHost, s.stream),
          "D2H");
  cuda_ok(cudaStreamSynchronize(s.stream), "sync");
  out.indices.assign(o32.begin(), o32.end());
  return out;
}

// ---- wire payloads (codec.hpp:50-70) ------------------------------------------

int pick_index_width(const SparseDelta& d) {
  const std::uint64_t top = d.indices.empty() ? 0 : d.indices.back();
  return top <= 0xFFFFFFFFull ? 4 : 8;
}

std::vector<std::uint8_t> encode_dense(const HostTensor& t) {
  std::vector<std::uint8_t> out;
  out.reserve(32 + t.data.size());
  write_head(out, kDense, t.dtype, t.shape, 0);
  out.insert(out.end(), t.data.begin(), t.data.end());
  return out;
}

std::vector<std::uint8_t> encode_sparse(const SparseDelta& d, int index_width) {
  if (index_width != 4 && index_width != 8) throw PayloadFormatError("index width must be 4 or 8");
  std::vector<std::uint8_t> out;
  out.reserve(40 + d.indices.size() * static_cast<std::size_t>(index_width + 4));
  write_head(out, kSparse, d.dtype, d.shape, static_cast<std::uint8_t>(index_width));
  put(out, static_cast<std::uint64_t>(d.indices.size()));
  for (auto i : d.indices) {
    if (index_width == 8) {
      put(out, i);
    } else {
      if (i > 0xFFFFFFFFull) throw PayloadFormatError("index " + std::to_string(i) + " exceeds u32");
      put(out, static_cast<std::uint32_t>(i));
    }
  }
  out.insert(out.end(), d.values.begin(), d.values.end());
  return out;
}

std::size_t peek_payload_size(const std::uint8_t* data, std::size_t len) {
  const Head h = read_head(data, len);
  std::uint64_t elems = 1;
  for (auto d : h.shape) elems *= static_cast<std::uint64_t>(d);
  if (h.magic == kDense) return h.pos + elems * 4;
  std::size_t pos = h.pos;
  const auto nnz = get<std::uint64_t>(data, len, pos, "nnz");
  return pos + nnz * (static_cast<std::size_t>(h.iw) + 4);
}

DecodedPayload decode_payload(const std::vector<std::uint8_t>& bytes) {
  const std::uint8_t* data = bytes.data();
  const std::size_t len = bytes.size();
  const Head h = read_head(data, len);
  std::size_t pos = h.pos;
  if (h.magic == kDense) {
    HostTensor t = HostTensor::zeros(h.dtype, h.shape);
    if (pos + t.data.size() != len)
      throw PayloadFormatError("dense payload size mismatch: header implies " +
                               std::to_string(pos + t.data.size()) + ", got " + std::to_string(len));
    std::memcpy(t.data.data(), data + pos, t.data.size());
    return DecodedPayload{std::move(t)};
  }
  if (h.iw != 4 && h.iw != 8) throw PayloadFormatError("sparse index width");
  SparseDelta d;
  d.dtype = h.dtype;
  d.shape = h.shape;
  const auto nnz = get<std::uint64_t>(data, len, pos, "nnz");
  const std::size_t want = pos + nnz * (static_cast<std::size_t>(h.iw) + 4);
  if (want != len)
    throw PayloadFormatError("sparse payload size mismatch: header implies " +
                             std::to_string(want) + ", got " + std::to_string(len));
  d.indices.reserve(nnz);
  for (std::uint64_t k = 0; k < nnz; ++k) {
    const std::uint64_t i = h.iw == 4 ? get<std::uint32_t>(data, len, pos, "index")
                                      : get<std::uint64_t>(data, len, pos, "index");
    if (k > 0 && i <= d.indices.back()) throw PayloadFormatError("indices not strictly ascending");
    d.indices.push_back(i);
  }
  d.values.assign(data + pos, data + len);
  return DecodedPayload{std::move(d)};
}

}  // namespace coserve::transfer
