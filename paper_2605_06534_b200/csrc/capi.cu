// capi.cu -- extern "C" codec entry points of include/wsync.h.
#include <cstring>
#include <string>

#include "capi_util.h"
#include "kernels.h"

using namespace wsync;

namespace wsync {

thread_local std::string g_last_error;

ws_status set_error(ws_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

ws_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return WS_OK;
  return set_error(WS_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool valid_dtype(int dt) { return dt == WS_F32 || dt == WS_I32 || dt == WS_BF16; }

ws_status check_shard(const int64_t* full, int nd, const ws_shard& d, const char* what) {
  if (nd < 1 || nd > WS_MAX_DIMS)
    return set_error(WS_INVALID_ARGUMENT, std::string(what) + ": ndims out of range");
  uint64_t n = 1;
  for (int i = 0; i < nd; ++i) {
    if (full[i] <= 0) return set_error(WS_SHAPE_MISMATCH, std::string(what) + ": non-positive dim");
    n *= (uint64_t)full[i];
  }
  if (n >= (1ull << 32))
    return set_error(WS_INVALID_ARGUMENT, std::string(what) + ": tensor of 2^32 elements or more");
  if (d.slice_dim >= 0) {
    // shard.cpp:114-121
    if (d.slice_dim >= nd)
      return set_error(WS_SHAPE_MISMATCH, std::string(what) + ": slice dim out of rank");
    if (d.start < 0 || d.end > full[d.slice_dim] || d.start >= d.end)
      return set_error(WS_SHAPE_MISMATCH, std::string(what) + ": slice out of range");
  }
  return WS_OK;
}

uint64_t shard_elems(const int64_t* full, int nd, const ws_shard& d) {
  uint64_t n = 1;
  for (int i = 0; i < nd; ++i)
    n *= (uint64_t)(d.slice_dim == i ? d.end - d.start : full[i]);
  return n;
}

}  // namespace wsync

extern "C" {

const char* ws_status_name(ws_status s) {
  switch (s) {
    case WS_OK: return "OK";
    case WS_SHAPE_MISMATCH: return "ShapeMismatch";
    case WS_PAYLOAD_FORMAT: return "PayloadFormatError";
    case WS_INDEX_OUT_OF_SHARD: return "IndexOutOfShard";
    case WS_INDIVISIBLE_SHAPE: return "IndivisibleShape";
    case WS_UNKNOWN_MODULE_KIND: return "UnknownModuleKind";
    case WS_INCOMPLETE_COVERAGE: return "IncompleteCoverage";
    case WS_RELAY_TIMEOUT: return "RelayTimeout";
    case WS_INTEGRITY: return "IntegrityError";
    case WS_KEY_FORMAT: return "KeyFormatError";
    case WS_TRANSFER_ERROR: return "TransferError";
    case WS_CUDA: return "CudaError";
    case WS_NCCL: return "NcclError";
    case WS_CAPACITY: return "Capacity";
    case WS_INVALID_ARGUMENT: return "InvalidArgument";
  }
  return "Unknown";
}

const char* ws_last_error(void) { return g_last_error.c_str(); }

int ws_abi_version(void) { return 1; }

namespace {
// [ticket @0][look-back status words @256: one per tile, the smallest tile
// being the reslice tile of 1024 records][K1 spill scratch for the grid
// ws_diff_shards uses on n elements (4-byte records: the largest)].
size_t status_bytes(uint64_t n) {
  const uint64_t tiles = (n + kResliceTile - 1) / kResliceTile + 1;
  return ((tiles * 8 + 255) / 256) * 256;
}
uint32_t diff_blocks(uint64_t n) {
  const uint64_t t = (n + encode_tile_elems(WS_F32) - 1) / encode_tile_elems(WS_F32);
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(kMaxEncodeGrid, t));
}
}  // namespace

size_t ws_diff_workspace_bytes(uint64_t n) {
  return 256 + status_bytes(n) + encode_spill_bytes(WS_F32, diff_blocks(n));
}

namespace {
struct Workspace {
  unsigned int* ticket;
  unsigned long long* status;
  size_t status_words;
  void* spill;
};
Workspace carve(void* ws, size_t bytes, uint64_t n) {
  char* b = static_cast<char*>(ws);
  Workspace w;
  w.ticket = reinterpret_cast<unsigned int*>(b);
  w.status = reinterpret_cast<unsigned long long*>(b + 256);
  w.status_words = status_bytes(n) / 8;
  w.spill = b + 256 + status_bytes(n);
  (void)bytes;
  return w;
}
uint32_t g_epoch = 1;
uint32_t next_epoch() {
  g_epoch = (g_epoch + 1) & 0x3fffffffu;
  if (g_epoch == 0) g_epoch = 1;
  return g_epoch;
}
}  // namespace

ws_status ws_diff_shards(ws_dtype dtype, const void* prev_dev, const void* next_dev, uint64_t n,
                         uint32_t* idx_dev, void* val_dev, uint64_t cap, uint64_t* nnz_dev,
                         void* workspace_dev, size_t workspace_bytes, ws_stream_t stream) {
  if (!valid_dtype(dtype)) return set_error(WS_INVALID_ARGUMENT, "ws_diff_shards: bad dtype");
  if (n >= (1ull << 32))
    return set_error(WS_INVALID_ARGUMENT, "ws_diff_shards: shard of 2^32 elements or more");
  if (((uintptr_t)prev_dev | (uintptr_t)next_dev) & 15)
    return set_error(WS_INVALID_ARGUMENT, "ws_diff_shards: prev/next must be 16-byte aligned");
  if (workspace_bytes < ws_diff_workspace_bytes(n))
    return set_error(WS_CAPACITY, "ws_diff_shards: workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Workspace w = carve(workspace_dev, workspace_bytes, n);
  const uint32_t tile = encode_tile_elems(dtype);
  const uint32_t ntiles = (uint32_t)((n + tile - 1) / tile);
  if (ntiles == 0) return cuda_status(cudaMemsetAsync(nnz_dev, 0, 8, s), "ws_diff_shards");
  EncodeArgs a{};
  a.prev = prev_dev;
  a.next = next_dev;
  a.segs = nullptr;  // single segment carried inline
  a.seg0 = SegDev{0, n, 0, cap};
  a.tile0 = nullptr;
  a.nseg = 1;
  a.ntiles = ntiles;
  a.out_idx = idx_dev;
  a.out_val = val_dev;
  a.seg_nnz = nnz_dev;
  a.status = w.status;
  a.epoch = next_epoch();
  a.ticket = w.ticket;
  a.spill = w.spill;
  a.spill_blocks = diff_blocks(n);
  return cuda_status(launch_encode(dtype, a, s), "ws_diff_shards");
}

ws_status ws_apply_delta(ws_dtype dtype, void* target_dev, uint64_t n, const uint32_t* idx_dev,
                         const void* val_dev, uint64_t nnz, const uint64_t* nnz_dev,
                         uint32_t* err_dev, ws_stream_t stream) {
  if (!valid_dtype(dtype)) return set_error(WS_INVALID_ARGUMENT, "ws_apply_delta: bad dtype");
  if (!err_dev) return set_error(WS_INVALID_ARGUMENT, "ws_apply_delta: err_dev is required");
  return cuda_status(launch_apply(dtype, target_dev, n, idx_dev, val_dev, nnz, nnz_dev, err_dev,
                                  reinterpret_cast<cudaStream_t>(stream)),
                     "ws_apply_delta");
}

ws_status ws_reslice_delta(ws_dtype dtype, const int64_t* full_shape, int ndims, ws_shard src,
                           ws_shard dst, int allow_cross_dim, const uint32_t* idx_dev,
                           const void* val_dev, uint64_t nnz, const uint64_t* nnz_dev,
                           uint32_t* out_idx_dev, void* out_val_dev, uint64_t* out_nnz_dev,
                           uint32_t* err_dev, void* workspace_dev, size_t workspace_bytes,
                           ws_stream_t stream) {
  if (!valid_dtype(dtype)) return set_error(WS_INVALID_ARGUMENT, "ws_reslice_delta: bad dtype");
  ws_status st = check_shard(full_shape, ndims, src, "ws_reslice_delta src");
  if (st != WS_OK) return st;
  st = check_shard(full_shape, ndims, dst, "ws_reslice_delta dst");
  if (st != WS_OK) return st;
  // codec.cpp:101-102
  if (!allow_cross_dim && src.slice_dim >= 0 && dst.slice_dim >= 0 &&
      src.slice_dim != dst.slice_dim)
    return set_error(WS_SHAPE_MISMATCH, "reslice_delta: slices along different dims");
  if (!err_dev) return set_error(WS_INVALID_ARGUMENT, "ws_reslice_delta: err_dev is required");
  if (workspace_bytes < ws_diff_workspace_bytes(nnz))
    return set_error(WS_CAPACITY, "ws_reslice_delta: workspace too small");
  Workspace w = carve(workspace_dev, workspace_bytes, nnz);
  ResliceArgs a{};
  a.map = make_remap(full_shape, ndims, src, dst);
  a.src_elems = shard_elems(full_shape, ndims, src);
  a.idx = idx_dev;
  a.val = val_dev;
  a.cap_in = nnz;
  a.nnz_dev = nnz_dev;
  a.nnz = nnz;
  a.out_idx = out_idx_dev;
  a.out_val = out_val_dev;
  a.out_nnz = out_nnz_dev;
  a.err = err_dev;
  a.status = w.status;
  a.epoch = next_epoch();
  a.ticket = w.ticket;
  return cuda_status(launch_reslice(dtype, a, reinterpret_cast<cudaStream_t>(stream)),
                     "ws_reslice_delta");
}

ws_status ws_copy_overlap(ws_dtype dtype, const int64_t* full_shape, int ndims, ws_shard dst,
                          void* dst_dev, ws_shard src, const void* src_dev, int64_t* copied,
                          ws_stream_t stream) {
  if (!valid_dtype(dtype)) return set_error(WS_INVALID_ARGUMENT, "ws_copy_overlap: bad dtype");
  ws_status st = check_shard(full_shape, ndims, src, "ws_copy_overlap src");
  if (st != WS_OK) return st;
  st = check_shard(full_shape, ndims, dst, "ws_copy_overlap dst");
  if (st != WS_OK) return st;
  BoxCopyArgs a{};
  const uint64_t n = make_box_copy(dtype, full_shape, ndims, dst, src, &a);
  if (copied) *copied = (int64_t)n;
  if (n == 0) return WS_OK;
  a.dst = dst_dev;
  a.src = src_dev;
  if (((uintptr_t)dst_dev | (uintptr_t)src_dev) & 15) a.vec = 0;
  return cuda_status(launch_box_copy(dtype, a, reinterpret_cast<cudaStream_t>(stream)),
                     "ws_copy_overlap");
}

ws_status ws_extract_shard(ws_dtype dtype, const int64_t* full_shape, int ndims, ws_shard desc,
                           const void* full_dev, void* out_dev, ws_stream_t stream) {
  if (!valid_dtype(dtype)) return set_error(WS_INVALID_ARGUMENT, "ws_extract_shard: bad dtype");
  ws_status st = check_shard(full_shape, ndims, desc, "extract_shard");
  if (st != WS_OK) return st;
  ws_shard full{-1, 0, 0};
  int64_t copied = 0;
  return ws_copy_overlap(dtype, full_shape, ndims, desc, out_dev, full, full_dev, &copied, stream);
}

ws_status ws_gen_pair_bf16(uint64_t seed, const char* param_name, const int64_t* full_shape,
                           int ndims, ws_shard desc, uint64_t change_thr, uint16_t* prev_dev,
                           uint16_t* next_dev, ws_stream_t stream) {
  ws_status st = check_shard(full_shape, ndims, desc, "ws_gen_pair_bf16");
  if (st != WS_OK) return st;
  return cuda_status(launch_gen_bf16(param_key(seed, param_name), full_shape, ndims, desc,
                                     change_thr, prev_dev, next_dev,
                                     reinterpret_cast<cudaStream_t>(stream)),
                     "ws_gen_pair_bf16");
}

ws_status ws_gen_pair_bf16_dim0(uint64_t seed, const char* param_name, const int64_t* full_shape,
                                int ndims, ws_shard desc, const uint64_t* thr_dim0_dev,
                                uint16_t* prev_dev, uint16_t* next_dev, ws_stream_t stream) {
  ws_status st = check_shard(full_shape, ndims, desc, "ws_gen_pair_bf16_dim0");
  if (st != WS_OK) return st;
  if (!thr_dim0_dev) return set_error(WS_INVALID_ARGUMENT, "ws_gen_pair_bf16_dim0: null table");
  return cuda_status(launch_gen_bf16(param_key(seed, param_name), full_shape, ndims, desc, 0,
                                     prev_dev, next_dev, reinterpret_cast<cudaStream_t>(stream),
                                     thr_dim0_dev),
                     "ws_gen_pair_bf16_dim0");
}

ws_status ws_expert_thresholds(int experts, double density, double zipf_s, uint64_t perm_seed,
                               uint64_t* out) {
  if (experts <= 0 || !out || !(density >= 0.0) || !(zipf_s >= 0.0))
    return set_error(WS_INVALID_ARGUMENT, "ws_expert_thresholds: bad argument");
  expert_thresholds(experts, density, zipf_s, perm_seed, out);
  return WS_OK;
}

}  // extern "C"
