// codec_shim.cpp -- the reference's codec API (coserve/transfer/codec.hpp),
// implemented on top of libwsync's C-ABI (include/wsync.h).
//
// Compiled against the reference's own headers and linked INSTEAD of the
// reference's codec.cpp, it turns the unmodified reference engine
// (engine.cpp's sync_step pusher/puller threads, bench.cpp, plan.cpp ...) into
// a client of the B200 kernels: diff_shards -> K1 (ws_diff_shards),
// apply_delta -> K4 (ws_apply_delta), reslice_delta -> ws_reslice_delta.
// The payload functions (encode_dense / encode_sparse / decode_payload /
// peek_payload_size) run on libwsync's device wire kernels (wire.cu), the
// code the engine's relay sync uses.  See INTEGRATION.md.
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

// Host bytes -> device scratch slot, and back, on the thread's stream.
void* upload(DeviceScratch& s, int slot, const void* host, std::size_t bytes) {
  void* dev = s.get(slot, bytes < 8 ? 8 : bytes);
  if (bytes) cuda_ok(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s.stream), "H2D");
  return dev;
}

void download(DeviceScratch& s, void* host, const void* dev, std::size_t bytes) {
  if (bytes) cuda_ok(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s.stream), "D2H");
  cuda_ok(cudaStreamSynchronize(s.stream), "sync");
}

// The reference's DType holds F32/I32 only: a bf16 payload ("CWS2"/"CWD2",
// dtype code 2) is foreign to this API, as the reference decoder says.
DType host_dtype(int code) {
  if (code != WS_F32 && code != WS_I32) throw PayloadFormatError("bad dtype " + std::to_string(code));
  return code == WS_F32 ? DType::F32 : DType::I32;
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

// ---- wire payloads (codec.hpp:50-70), built and parsed on the device ----------
// by libwsync's wire kernels (ws_encode_*_dev, ws_peek_*_dev,
// ws_decode_sparse_dev): the same code path the engine's relay sync uses.

int pick_index_width(const SparseDelta& d) {
  // indices ascend, so the last one decides whether 32 bits are enough
  return (!d.indices.empty() && (d.indices.back() >> 32) != 0) ? 8 : 4;
}

std::vector<std::uint8_t> encode_dense(const HostTensor& t) {
  DeviceScratch& s = scratch();
  const int nd = static_cast<int>(t.shape.size());
  const std::uint64_t total =
      ws_payload_bytes(wdt(t.dtype), nd, 'D', 0, static_cast<std::uint64_t>(t.elems()));
  const void* src = upload(s, 0, t.data.data(), t.data.size());
  void* out = s.get(1, total);
  ws_ok(ws_encode_dense_dev(wdt(t.dtype), t.shape.data(), nd, src, out,
                            reinterpret_cast<ws_stream_t>(s.stream)));
  std::vector<std::uint8_t> bytes(total);
  download(s, bytes.data(), out, total);
  return bytes;
}

std::vector<std::uint8_t> encode_sparse(const SparseDelta& d, int index_width) {
  if (index_width != 4 && index_width != 8) throw PayloadFormatError("index width must be 4 or 8");
  DeviceScratch& s = scratch();
  const std::uint64_t nnz = d.indices.size();
  // the device encoder takes u32 local indices (every shard below 2^32
  // elements) and widens them to index_width on the wire
  std::vector<std::uint32_t> narrow(nnz);
  for (std::uint64_t k = 0; k < nnz; ++k) {
    if (d.indices[k] >> 32)
      throw PayloadFormatError("index " + std::to_string(d.indices[k]) +
                               " beyond the 32-bit local indices of a shard");
    narrow[k] = static_cast<std::uint32_t>(d.indices[k]);
  }
  const int nd = static_cast<int>(d.shape.size());
  const std::uint64_t total = ws_payload_bytes(wdt(d.dtype), nd, 'S', index_width, nnz);
  const auto* idx = static_cast<const std::uint32_t*>(upload(s, 0, narrow.data(), nnz * 4));
  const void* val = upload(s, 2, d.values.data(), d.values.size());
  void* out = s.get(1, total);
  ws_ok(ws_encode_sparse_dev(wdt(d.dtype), d.shape.data(), nd, index_width, idx, val, nnz, out,
                             reinterpret_cast<ws_stream_t>(s.stream)));
  std::vector<std::uint8_t> bytes(total);
  download(s, bytes.data(), out, total);
  return bytes;
}

std::size_t peek_payload_size(const std::uint8_t* data, std::size_t len) {
  DeviceScratch& s = scratch();
  // a header is at most 8 + 8 x 8 dims + 8 (nnz) bytes
  const std::size_t head = len < 96 ? len : 96;
  const void* dev = upload(s, 0, data, head);
  cuda_ok(cudaStreamSynchronize(s.stream), "sync");
  std::uint64_t total = 0;
  ws_ok(ws_peek_payload_size_dev(dev, len, &total));
  if (len > 4) host_dtype(data[4]);
  return static_cast<std::size_t>(total);
}

DecodedPayload decode_payload(const std::vector<std::uint8_t>& bytes) {
  DeviceScratch& s = scratch();
  const void* dev = upload(s, 0, bytes.data(), bytes.size());
  cuda_ok(cudaStreamSynchronize(s.stream), "sync");
  ws_payload_info info;
  ws_ok(ws_peek_payload_dev(dev, bytes.size(), &info));
  const DType dt = host_dtype(info.dtype);
  const std::vector<std::int64_t> shape(info.shape, info.shape + info.ndims);
  if (info.codec == 'D') {
    HostTensor t = HostTensor::zeros(dt, shape);
    download(s, t.data.data(), static_cast<const std::uint8_t*>(dev) + info.header_bytes,
             t.data.size());
    return DecodedPayload{std::move(t)};
  }
  SparseDelta d;
  d.dtype = dt;
  d.shape = shape;
  auto* idx = static_cast<std::uint32_t*>(s.get(1, info.nnz * 4));
  void* val = s.get(2, info.nnz * 4);
  ws_ok(ws_decode_sparse_dev(dev, &info, idx, val, reinterpret_cast<ws_stream_t>(s.stream)));
  std::vector<std::uint32_t> narrow(info.nnz);
  d.values.resize(info.nnz * 4);
  cuda_ok(cudaMemcpyAsync(narrow.data(), idx, info.nnz * 4, cudaMemcpyDeviceToHost, s.stream),
          "D2H");
  download(s, d.values.data(), val, d.values.size());
  d.indices.assign(narrow.begin(), narrow.end());
  return DecodedPayload{std::move(d)};
}

}  // namespace coserve::transfer
