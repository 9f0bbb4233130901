// wire.cu -- the reference's wire format produced and checked on the device
// (SURVEY.md 8(f) rows 1 and 3):
//   payloads  encode_sparse / encode_dense / decode_payload / peek_payload_size
//             (codec.cpp:140-263).  F32/I32 keep "CWS1"/"CWD1"; bf16 uses
//             "CWS2"/"CWD2" with 2-byte values.
//   frames    encode_bucket_frame / decode_bucket_frame (wire.cpp:35-71):
//             [key_len u32][key][payload_len u32][payload][crc32 u32], the
//             payload split into bucket_bytes buckets (engine.cpp:136-148).
//   crc32     frame_crc32 (wire.cpp:9-13), zlib's polynomial.  zlib is not in
//             /root/reference; its published algorithm is restated: a
//             table-driven CRC per 256-byte piece and the GF(2) fold
//             crc(A|B) = crc(A) * x^(8|B|) mod P  xor  crc(B), which makes
//             every piece's contribution independent (XOR-reducible).
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "capi_util.h"
#include "kernels.h"

using namespace wsync;

namespace {

constexpr uint32_t kPoly = 0xEDB88320u;  // reflected 0x04C11DB7
constexpr uint32_t kSparseMagic1 = 0x31535743u, kDenseMagic1 = 0x31445743u;  // "CWS1" "CWD1"
constexpr uint32_t kSparseMagic2 = 0x32535743u, kDenseMagic2 = 0x32445743u;  // "CWS2" "CWD2"
constexpr uint32_t kPiece = 256;       // bytes per thread piece
constexpr uint32_t kRegionPieces = 256;  // pieces per block region (64 KiB)

// ---- GF(2) arithmetic of the reflected CRC-32 (bit 31 = x^0) ---------------
__host__ __device__ inline uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

struct CrcTables {
  uint32_t x2n[32];              // x^(2^k) mod P
  uint32_t piece_pow[kRegionPieces];  // x^(8 * 256 * m) mod P
};

CrcTables make_tables() {
  CrcTables t;
  uint32_t p = 1u << 30;  // x^1
  for (int k = 0; k < 32; ++k) {
    t.x2n[k] = p;
    p = multmodp(p, p);
  }
  // x^(8*256) = x^(2^11)
  t.piece_pow[0] = 1u << 31;
  for (uint32_t m = 1; m < kRegionPieces; ++m) t.piece_pow[m] = multmodp(t.piece_pow[m - 1], t.x2n[11]);
  return t;
}

__device__ inline uint32_t x8nmodp(const uint32_t* x2n, uint64_t n) {  // x^(8n) mod P
  uint32_t p = 1u << 31;
  unsigned k = 3;
  while (n) {
    if (n & 1) p = multmodp(x2n[k & 31], p);
    n >>= 1;
    ++k;
  }
  return p;
}

// One frame (or any byte range) whose CRC is wanted: data[0, len).
struct CrcJob {
  const uint8_t* data;
  uint64_t len;
  uint64_t region0;  // first region index of this job in the flattened list
};

// crc of bytes [p, p + n) of one job, standard (init ~0, final ~).
__device__ inline uint32_t crc_bytes(const uint32_t (*T)[256], const uint8_t* p, uint32_t n) {
  uint32_t c = 0xFFFFFFFFu;
  uint32_t i = 0;
  const uint32_t head = (uint32_t)((4 - ((uintptr_t)p & 3)) & 3);
  for (; i < head && i < n; ++i) c = T[0][(c ^ p[i]) & 0xff] ^ (c >> 8);
  for (; i + 4 <= n; i += 4) {  // slicing-by-4 over aligned words
    c ^= *reinterpret_cast<const uint32_t*>(p + i);
    c = T[3][c & 0xff] ^ T[2][(c >> 8) & 0xff] ^ T[1][(c >> 16) & 0xff] ^ T[0][c >> 24];
  }
  for (; i < n; ++i) c = T[0][(c ^ p[i]) & 0xff] ^ (c >> 8);
  return ~c;
}

__global__ void __launch_bounds__(256) crc_kernel(const CrcJob* jobs, int njobs,
                                                 uint64_t nregions, CrcTables tab,
                                                 uint32_t* acc) {
  __shared__ uint32_t T[4][256];
  __shared__ uint32_t red[8];
  __shared__ uint32_t s_tail_pow;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = (uint32_t)i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
    T[0][i] = c;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = T[0][i];
    for (int k = 1; k < 4; ++k) {
      c = (c >> 8) ^ T[0][c & 0xff];
      T[k][i] = c;
    }
  }
  __syncthreads();
  for (uint64_t r = blockIdx.x; r < nregions; r += gridDim.x) {
    int lo = 0, hi = njobs;  // job of region r: jobs[lo].region0 <= r < jobs[lo+1].region0
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (jobs[mid].region0 <= r) lo = mid; else hi = mid;
    }
    const CrcJob J = jobs[lo];
    const uint64_t rb = (r - J.region0) * (uint64_t)kPiece * kRegionPieces;  // region start
    const uint64_t rlen = J.len - rb < (uint64_t)kPiece * kRegionPieces
                              ? J.len - rb : (uint64_t)kPiece * kRegionPieces;
    const uint32_t npieces = (uint32_t)((rlen + kPiece - 1) / kPiece);
    const uint32_t last_len = (uint32_t)(rlen - (uint64_t)(npieces - 1) * kPiece);
    // x^(8 * last_len): the shift every earlier piece gets from the last one
    if (threadIdx.x == 0) s_tail_pow = x8nmodp(tab.x2n, last_len);
    __syncthreads();
    uint32_t contrib = 0;
    const uint32_t p = threadIdx.x;
    if (p < npieces) {
      const uint32_t n = p + 1 == npieces ? last_len : kPiece;
      const uint32_t c = crc_bytes(T, J.data + rb + (uint64_t)p * kPiece, n);
      // x^(8 * bytes of the region after this piece)
      uint32_t pw;
      if (p + 1 == npieces) pw = 1u << 31;
      else pw = multmodp(tab.piece_pow[npieces - 2 - p], s_tail_pow);
      contrib = multmodp(pw, c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) contrib ^= __shfl_xor_sync(0xffffffffu, contrib, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = contrib;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t rc = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) rc ^= red[w];
      // the region's place in its job: x^(8 * bytes after the region)
      const uint64_t after = J.len - rb - rlen;
      atomicXor(acc + lo, after ? multmodp(x8nmodp(tab.x2n, after), rc) : rc);
    }
    __syncthreads();
  }
}

// dst[0, n) = src[0, n), any alignment: aligned 4-byte stores assembled from
// aligned 4-byte loads with funnel shifts (bytes outside [0, n) untouched).
__device__ inline void copy_bytes_block(uint8_t* dst, const uint8_t* src, uint64_t n) {
  if (n == 0) return;
  const uint64_t dhead = (4 - ((uintptr_t)dst & 3)) & 3;
  const uint64_t head = dhead < n ? dhead : n;
  if (threadIdx.x < head) dst[threadIdx.x] = src[threadIdx.x];
  const uint64_t words = (n - head) / 4;
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst + head);
  const uint8_t* s = src + head;
  const uint32_t sh = (uint32_t)((uintptr_t)s & 3);
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(s - sh);
  for (uint64_t j = threadIdx.x; j < words; j += blockDim.x) {
    if (sh == 0) {
      dw[j] = sw[j];
    } else {
      const uint32_t a = sw[j], b = sw[j + 1];
      dw[j] = __funnelshift_r(a, b, 8 * sh);
    }
  }
  const uint64_t done = head + words * 4;
  if (threadIdx.x < n - done) dst[done + threadIdx.x] = src[done + threadIdx.x];
}

// One bucket frame per block iteration: lengths, key, payload slice.
struct FrameDesc {
  uint64_t out_off;     // frame start in the output buffer
  uint64_t key_off;     // key bytes in the key blob
  uint64_t payload_off; // bucket start in the payload
  uint32_t key_len, payload_len;
};

__global__ void frame_kernel(const FrameDesc* fr, int n, const uint8_t* keys,
                             const uint8_t* payload, uint8_t* out) {
  for (int f = blockIdx.x; f < n; f += gridDim.x) {
    const FrameDesc F = fr[f];
    uint8_t* o = out + F.out_off;
    if (threadIdx.x < 4) {
      o[threadIdx.x] = (uint8_t)(F.key_len >> (8 * threadIdx.x));
      o[4 + F.key_len + threadIdx.x] = (uint8_t)(F.payload_len >> (8 * threadIdx.x));
    }
    for (uint32_t i = threadIdx.x; i < F.key_len; i += blockDim.x) o[4 + i] = keys[F.key_off + i];
    copy_bytes_block(o + 8 + F.key_len, payload + F.payload_off, F.payload_len);
  }
}

struct HeaderWords {
  uint64_t w[12];
  uint32_t n;
};
__global__ void header_kernel(uint64_t* out, HeaderWords h) {
  if (threadIdx.x < h.n) out[threadIdx.x] = h.w[threadIdx.x];
}

__global__ void widen_kernel(const uint32_t* idx, uint64_t n, uint64_t* out) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x)
    out[k] = idx[k];
}

// codec.cpp:252-259 restated on the device, plus the narrowing to u32 local
// indices (every shard here has < 2^32 elements): err bit 1 = not strictly
// ascending, bit 2 = index beyond u32.
__global__ void decode_idx_kernel(const uint8_t* blk, int iw, uint64_t nnz, uint32_t* out,
                                  uint32_t* err) {
  bool bad_order = false, bad_width = false;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t i, p = 0;
    if (iw == 4) {
      i = reinterpret_cast<const uint32_t*>(blk)[k];
      if (k) p = reinterpret_cast<const uint32_t*>(blk)[k - 1];
    } else {
      i = reinterpret_cast<const uint64_t*>(blk)[k];
      if (k) p = reinterpret_cast<const uint64_t*>(blk)[k - 1];
    }
    if (k && i <= p) bad_order = true;
    if (i > 0xFFFFFFFFull) bad_width = true;
    if (out) out[k] = (uint32_t)i;
  }
  if (bad_order) atomicOr(err, 1u);
  if (bad_width) atomicOr(err, 2u);
}

bool magic_for(int dtype, bool sparse, uint32_t* magic) {
  if (dtype == WS_BF16) *magic = sparse ? kSparseMagic2 : kDenseMagic2;
  else if (dtype == WS_F32 || dtype == WS_I32) *magic = sparse ? kSparseMagic1 : kDenseMagic1;
  else return false;
  return true;
}

// encode_header (codec.cpp:145-154) into little-endian 8-byte words.
HeaderWords make_header(uint32_t magic, int dtype, const int64_t* shape, int nd, int iw,
                        bool with_nnz, uint64_t nnz) {
  HeaderWords h{};
  uint8_t b[8];
  std::memcpy(b, &magic, 4);
  b[4] = (uint8_t)dtype;
  b[5] = (uint8_t)nd;
  b[6] = (uint8_t)iw;
  b[7] = 0;
  std::memcpy(&h.w[0], b, 8);
  for (int d = 0; d < nd; ++d) std::memcpy(&h.w[1 + d], &shape[d], 8);
  h.n = 1 + nd;
  if (with_nnz) h.w[h.n++] = nnz;
  return h;
}

int grid_for(uint64_t work, int threads) {
  const uint64_t want = (work + threads - 1) / threads;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sm_count() * 8));
}

ws_status wire_cuda(cudaError_t e, const char* what) { return cuda_status(e, what); }


// Stream-ordered scratch from this library's own memory pool per device,
// which keeps freed memory cached. Through the default pool, with its release
// threshold of 0, every synchronisation handed the memory back to the driver,
// so each call paid a full allocation (~4 ms per decode on the relay path).
// The process's default pool is left untouched.
}  // namespace

namespace wsync {
std::mutex g_scratch_mu;
cudaMemPool_t g_scratch_pools[64] = {};

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  std::mutex& mu = g_scratch_mu;
  cudaMemPool_t* pools = g_scratch_pools;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev], &props);
      if (e != cudaSuccess) {
        pools[dev] = nullptr;
        return e;
      }
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}
}  // namespace wsync

namespace {

}  // namespace

namespace wsync {
// Hands the cached scratch of `dev` back to the driver (after the work that
// used it has completed).
void scratch_trim(int dev) {
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  if (dev >= 0 && dev < 64 && g_scratch_pools[dev]) cudaMemPoolTrimTo(g_scratch_pools[dev], 0);
}
}  // namespace wsync

extern "C" {

uint64_t ws_payload_bytes(ws_dtype dtype, int ndims, char codec, int index_width, uint64_t count) {
  const uint64_t hdr = 8 + 8 * (uint64_t)ndims;
  const uint64_t esz = dtype == WS_BF16 ? 2 : 4;
  if (codec == 'S') return hdr + 8 + count * ((uint64_t)index_width + esz);
  return hdr + count * esz;
}

ws_status ws_encode_sparse_dev(ws_dtype dtype, const int64_t* shape, int ndims, int index_width,
                               const uint32_t* idx_dev, const void* val_dev, uint64_t nnz,
                               void* out_dev, ws_stream_t stream) {
  uint32_t magic;
  if (!magic_for(dtype, true, &magic)) return set_error(WS_INVALID_ARGUMENT, "bad dtype");
  if (index_width != 4 && index_width != 8)
    return set_error(WS_PAYLOAD_FORMAT, "index width must be 4 or 8");
  if (ndims < 0 || ndims > 8) return set_error(WS_INVALID_ARGUMENT, "ndims");
  if ((uintptr_t)out_dev & 7) return set_error(WS_INVALID_ARGUMENT, "payload must be 8-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const HeaderWords h = make_header(magic, dtype, shape, ndims, index_width, true, nnz);
  uint8_t* out = static_cast<uint8_t*>(out_dev);
  header_kernel<<<1, 32, 0, s>>>(reinterpret_cast<uint64_t*>(out), h);
  uint8_t* ib = out + 8 * h.n;
  if (nnz) {
    if (index_width == 4) {
      cudaError_t e = cudaMemcpyAsync(ib, idx_dev, nnz * 4, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return wire_cuda(e, "encode_sparse idx");
    } else {
      widen_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(idx_dev, nnz, reinterpret_cast<uint64_t*>(ib));
    }
    cudaError_t e = cudaMemcpyAsync(ib + nnz * (uint64_t)index_width, val_dev,
                                    nnz * (dtype == WS_BF16 ? 2 : 4), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return wire_cuda(e, "encode_sparse val");
  }
  return wire_cuda(cudaGetLastError(), "ws_encode_sparse_dev");
}

ws_status ws_encode_dense_dev(ws_dtype dtype, const int64_t* shape, int ndims, const void* data_dev,
                              void* out_dev, ws_stream_t stream) {
  uint32_t magic;
  if (!magic_for(dtype, false, &magic)) return set_error(WS_INVALID_ARGUMENT, "bad dtype");
  if (ndims < 0 || ndims > 8) return set_error(WS_INVALID_ARGUMENT, "ndims");
  if ((uintptr_t)out_dev & 7) return set_error(WS_INVALID_ARGUMENT, "payload must be 8-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const HeaderWords h = make_header(magic, dtype, shape, ndims, 0, false, 0);
  uint8_t* out = static_cast<uint8_t*>(out_dev);
  header_kernel<<<1, 32, 0, s>>>(reinterpret_cast<uint64_t*>(out), h);
  uint64_t n = 1;
  for (int d = 0; d < ndims; ++d) n *= (uint64_t)shape[d];
  if (n) {
    cudaError_t e = cudaMemcpyAsync(out + 8 * h.n, data_dev, n * (dtype == WS_BF16 ? 2 : 4),
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return wire_cuda(e, "encode_dense");
  }
  return wire_cuda(cudaGetLastError(), "ws_encode_dense_dev");
}

// decode_header + the size checks of decode_payload / peek_payload_size
// (codec.cpp:196-263), reading the header from device memory.
// exact: the payload is `len` bytes (decode_payload's size checks); else
// `len` bytes of it are present and only the header must fit (peek).
static ws_status peek_impl(const void* payload_dev, uint64_t len, ws_payload_info* info,
                           bool exact) {
  if (!info) return set_error(WS_INVALID_ARGUMENT, "null info");
  std::memset(info, 0, sizeof(*info));
  uint8_t h[88] = {0};
  const uint64_t hn = len < sizeof(h) ? len : sizeof(h);
  if (hn) {
    cudaError_t e = cudaMemcpy(h, payload_dev, hn, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return wire_cuda(e, "peek header");
  }
  auto need = [&](uint64_t upto, const char* what) -> ws_status {
    if (upto > len) return set_error(WS_PAYLOAD_FORMAT, std::string("payload truncated reading ") + what);
    return WS_OK;
  };
  ws_status st = need(4, "magic");
  if (st != WS_OK) return st;
  uint32_t magic;
  std::memcpy(&magic, h, 4);
  const bool s1 = magic == kSparseMagic1 || magic == kSparseMagic2;
  const bool d1 = magic == kDenseMagic1 || magic == kDenseMagic2;
  if (!s1 && !d1) return set_error(WS_PAYLOAD_FORMAT, "bad payload magic");
  if ((st = need(5, "dtype")) != WS_OK) return st;
  const int dt = h[4];
  const bool v2 = magic == kSparseMagic2 || magic == kDenseMagic2;
  if (v2 ? dt != WS_BF16 : dt > 1) return set_error(WS_PAYLOAD_FORMAT, "bad dtype " + std::to_string(dt));
  if ((st = need(6, "ndims")) != WS_OK) return st;
  const int nd = h[5];
  if ((st = need(7, "index width")) != WS_OK) return st;
  const int iw = h[6];
  if ((st = need(8, "pad")) != WS_OK) return st;
  if (nd > 8) return set_error(WS_PAYLOAD_FORMAT, "ndims beyond 8");
  uint64_t elems = 1;
  for (int d = 0; d < nd; ++d) {
    if ((st = need(8 + 8 * (uint64_t)d + 8, "dim")) != WS_OK) return st;
    int64_t v;
    std::memcpy(&v, h + 8 + 8 * d, 8);
    if (v <= 0) return set_error(WS_PAYLOAD_FORMAT, "non-positive dim");
    info->shape[d] = v;
    // a dense payload carries every element; any payload stays below 2^62
    // bytes -- so the product cannot overflow below
    if ((uint64_t)v > ((exact && d1) ? len : (1ull << 62)) / elems)
      return set_error(WS_PAYLOAD_FORMAT, "payload size mismatch: dims exceed the payload");
    elems *= (uint64_t)v;
  }
  uint64_t pos = 8 + 8 * (uint64_t)nd;
  const uint64_t esz = dt == WS_BF16 ? 2 : 4;
  info->dtype = dt;
  info->ndims = nd;
  info->header_bytes = pos;
  if (d1) {
    info->codec = 'D';
    info->index_width = 0;
    info->total_bytes = pos + elems * esz;
    if (exact && info->total_bytes != len)
      return set_error(WS_PAYLOAD_FORMAT, "dense payload size mismatch: header implies " +
                                              std::to_string(info->total_bytes) + ", got " +
                                              std::to_string(len));
    return WS_OK;
  }
  if (iw != 4 && iw != 8) return set_error(WS_PAYLOAD_FORMAT, "sparse index width");
  if ((st = need(pos + 8, "nnz")) != WS_OK) return st;
  uint64_t nnz;
  std::memcpy(&nnz, h + pos, 8);
  pos += 8;
  info->codec = 'S';
  info->index_width = iw;
  info->nnz = nnz;
  info->header_bytes = pos;
  const uint64_t room = exact ? (len >= pos ? len - pos : 0) : (1ull << 62);
  if (nnz > room / ((uint64_t)iw + esz))  // no wrap in the product
    return set_error(WS_PAYLOAD_FORMAT, "sparse payload size mismatch: nnz " +
                                            std::to_string(nnz) + " exceeds the payload");
  info->total_bytes = pos + nnz * ((uint64_t)iw + esz);
  if (exact && info->total_bytes != len)
    return set_error(WS_PAYLOAD_FORMAT, "sparse payload size mismatch: header implies " +
                                            std::to_string(info->total_bytes) + ", got " +
                                            std::to_string(len));
  return WS_OK;
}

ws_status ws_peek_payload_dev(const void* payload_dev, uint64_t len, ws_payload_info* info) {
  return peek_impl(payload_dev, len, info, true);
}

ws_status ws_peek_payload_size_dev(const void* payload_dev, uint64_t len, uint64_t* total) {
  if (!total) return set_error(WS_INVALID_ARGUMENT, "null total");
  ws_payload_info info;
  const ws_status st = peek_impl(payload_dev, len, &info, false);
  if (st == WS_OK) *total = info.total_bytes;
  return st;
}

ws_status ws_decode_sparse_dev(const void* payload_dev, const ws_payload_info* info,
                               uint32_t* idx_dev, void* val_dev, ws_stream_t stream) {
  if (!info || info->codec != 'S') return set_error(WS_INVALID_ARGUMENT, "not a sparse payload");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint8_t* p = static_cast<const uint8_t*>(payload_dev);
  if ((uintptr_t)p & 7) return set_error(WS_INVALID_ARGUMENT, "payload must be 8-byte aligned");
  uint32_t* d_err = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&d_err), 4, s);
  if (e != cudaSuccess) return wire_cuda(e, "decode");
  cudaMemsetAsync(d_err, 0, 4, s);
  if (info->nnz)
    decode_idx_kernel<<<grid_for(info->nnz, 256), 256, 0, s>>>(p + info->header_bytes,
                                                              info->index_width, info->nnz,
                                                              idx_dev, d_err);
  const uint64_t esz = info->dtype == WS_BF16 ? 2 : 4;
  if (info->nnz && val_dev)
    cudaMemcpyAsync(val_dev, p + info->header_bytes + info->nnz * (uint64_t)info->index_width,
                    info->nnz * esz, cudaMemcpyDeviceToDevice, s);
  uint32_t err = 0;
  cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d_err, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return wire_cuda(e, "decode");
  if (err & 1) return set_error(WS_PAYLOAD_FORMAT, "indices not strictly ascending");
  if (err & 2) return set_error(WS_CAPACITY, "sparse index beyond 2^32");
  return WS_OK;
}

ws_status ws_crc32_dev(const void* const* data_dev, const uint64_t* len, int n, uint32_t* crc_out,
                       ws_stream_t stream) {
  if (n < 0 || (n && (!data_dev || !len || !crc_out)))
    return set_error(WS_INVALID_ARGUMENT, "ws_crc32_dev: bad arguments");
  if (n == 0) return WS_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  static const CrcTables tab = make_tables();
  std::vector<CrcJob> jobs(n);
  uint64_t regions = 0;
  const uint64_t rbytes = (uint64_t)kPiece * kRegionPieces;
  for (int k = 0; k < n; ++k) {
    jobs[k] = CrcJob{static_cast<const uint8_t*>(data_dev[k]), len[k], regions};
    regions += (len[k] + rbytes - 1) / rbytes;
  }
  CrcJob* d_jobs = nullptr;
  uint32_t* d_acc = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&d_jobs), n * sizeof(CrcJob), s);
  if (e == cudaSuccess) e = scratch_alloc(reinterpret_cast<void**>(&d_acc), n * 4, s);
  if (e != cudaSuccess) return wire_cuda(e, "crc alloc");
  cudaMemcpyAsync(d_jobs, jobs.data(), n * sizeof(CrcJob), cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(d_acc, 0, n * 4, s);
  if (regions)
    crc_kernel<<<(int)std::min<uint64_t>(regions, (uint64_t)sm_count() * 8), kRegionPieces, 0, s>>>(
        d_jobs, n, regions, tab, d_acc);
  cudaMemcpyAsync(crc_out, d_acc, n * 4, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d_jobs, s);
  cudaFreeAsync(d_acc, s);
  e = cudaStreamSynchronize(s);
  return wire_cuda(e == cudaSuccess ? cudaGetLastError() : e, "ws_crc32_dev");
}

ws_status ws_encode_bucket_frames_dev(const void* payload_dev, uint64_t payload_len,
                                      uint64_t bucket_bytes, const char* const* keys,
                                      const uint64_t* key_lens, int nbuckets, void* out_dev,
                                      uint64_t out_cap, uint64_t* frame_off, ws_stream_t stream) {
  // engine.cpp:139: at least one bucket, even for an empty payload
  const uint64_t want = payload_len ? (payload_len + bucket_bytes - 1) / bucket_bytes : 1;
  if (bucket_bytes == 0 || nbuckets != (int)want)
    return set_error(WS_INVALID_ARGUMENT, "bucket count must be max(1, ceil(len / bucket_bytes))");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  std::vector<FrameDesc> fr(nbuckets);
  std::string blob;
  uint64_t off = 0;
  for (int k = 0; k < nbuckets; ++k) {
    if (key_lens[k] > 64u * 1024u) return set_error(WS_PAYLOAD_FORMAT, "key too long");
    const uint64_t b0 = (uint64_t)k * bucket_bytes;
    const uint64_t pl = std::min<uint64_t>(bucket_bytes, payload_len - std::min(payload_len, b0));
    if (pl > (1ull << 30)) return set_error(WS_PAYLOAD_FORMAT, "payload too long");
    fr[k] = FrameDesc{off, blob.size(), b0, (uint32_t)key_lens[k], (uint32_t)pl};
    blob.append(keys[k], key_lens[k]);
    frame_off[k] = off;
    off += 12 + key_lens[k] + pl;
  }
  frame_off[nbuckets] = off;
  if (off > out_cap) return set_error(WS_CAPACITY, "frame buffer too small");
  FrameDesc* d_fr = nullptr;
  uint8_t* d_keys = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&d_fr), nbuckets * sizeof(FrameDesc), s);
  if (e == cudaSuccess)
    e = scratch_alloc(reinterpret_cast<void**>(&d_keys), std::max<size_t>(1, blob.size()), s);
  if (e != cudaSuccess) return wire_cuda(e, "frames alloc");
  cudaMemcpyAsync(d_fr, fr.data(), nbuckets * sizeof(FrameDesc), cudaMemcpyHostToDevice, s);
  if (!blob.empty()) cudaMemcpyAsync(d_keys, blob.data(), blob.size(), cudaMemcpyHostToDevice, s);
  uint8_t* out = static_cast<uint8_t*>(out_dev);
  frame_kernel<<<std::min(nbuckets, sm_count() * 4), 256, 0, s>>>(
      d_fr, nbuckets, d_keys, static_cast<const uint8_t*>(payload_dev), out);
  // the CRC of every frame covers all its preceding bytes (wire.cpp:45)
  std::vector<const void*> ptr(nbuckets);
  std::vector<uint64_t> len(nbuckets);
  std::vector<uint32_t> crc(nbuckets);
  for (int k = 0; k < nbuckets; ++k) {
    ptr[k] = out + fr[k].out_off;
    len[k] = 8 + (uint64_t)fr[k].key_len + fr[k].payload_len;
  }
  e = cudaStreamSynchronize(s);  // the host blob/desc vectors outlive the copies
  cudaFreeAsync(d_fr, s);
  cudaFreeAsync(d_keys, s);
  if (e != cudaSuccess) return wire_cuda(e, "frames");
  ws_status st = ws_crc32_dev(ptr.data(), len.data(), nbuckets, crc.data(), stream);
  if (st != WS_OK) return st;
  for (int k = 0; k < nbuckets; ++k) {
    e = cudaMemcpyAsync(out + fr[k].out_off + len[k], &crc[k], 4, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return wire_cuda(e, "frame crc");
  }
  return wire_cuda(cudaStreamSynchronize(s), "ws_encode_bucket_frames_dev");
}

ws_status ws_bucket_key(uint64_t step, const char* param, int tp_rank, int tp_size, int pp_stage,
                        ws_shard desc, char codec, int index_width, uint32_t seq, char* out,
                        uint64_t cap, uint64_t* out_len) {
  // key.cpp:47-69 (BucketKey::encode) with key.cpp:8-20's escaping
  if (!param || !out_len) return set_error(WS_INVALID_ARGUMENT, "ws_bucket_key: null argument");
  std::string k = "w|s" + std::to_string(step) + "|p";
  for (const char* c = param; *c; ++c) {
    if (*c == '%') k += "%25";
    else if (*c == '|') k += "%7C";
    else k += *c;
  }
  k += "|t" + std::to_string(tp_rank) + "." + std::to_string(tp_size);
  k += "|g" + std::to_string(pp_stage) + "|d";
  if (desc.slice_dim < 0) k += "F";
  else k += std::to_string(desc.slice_dim) + ":" + std::to_string(desc.start) + ":" +
            std::to_string(desc.end);
  k += "|c";
  k += codec;
  k += std::to_string(index_width) + "|q" + std::to_string(seq);
  *out_len = k.size();
  if (k.size() > cap) return set_error(WS_CAPACITY, "key buffer too small");
  std::memcpy(out, k.data(), k.size());
  return WS_OK;
}

}  // extern "C"
