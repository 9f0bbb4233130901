// kernels_codec.cu -- K1 encode, K4 apply, reslice, box copy, generator.
//
// K1 (encode) replaces the reference's diff_shards + density check +
// encode_sparse packing (codec.cpp:34-63, engine.cpp:118-127,
// codec.cpp:164-183).  One pass over prev/next: 128-bit streaming loads, a
// per-vector change mask (bit compare for bf16/i32, value compare for f32),
// popc per thread, a block scan of four packed 16-bit lane counts, and a
// decoupled look-back across the tiles of each segment, then the records
// are written at their final ascending position.  Segments are independent
// look-back chains so every segment's records start at its own base.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace wsync {

namespace {

constexpr int kThreads = kEncodeThreads;
constexpr int kWarps = kThreads / 32;
constexpr int kVPT = kEncodeVPT;

__device__ __forceinline__ int find_segment(const uint32_t* tile0, int nseg, uint32_t t) {
  int lo = 0, hi = nseg;  // tile0[lo] <= t < tile0[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(tile0 + mid) <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// Block-wide exclusive scan of a packed u64 (4 x 16-bit lanes).  Returns the
// thread's exclusive value; *total receives the block sum.  Uses s_warp[kWarps+1].
__device__ __forceinline__ unsigned long long block_scan_packed(unsigned long long x,
                                                                unsigned long long* s_warp,
                                                                unsigned long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(kFullMask, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < kWarps ? s_warp[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFullMask, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kWarps) s_warp[lane] = wi - w;
    if (lane == kWarps - 1) s_warp[kWarps] = wi;
  }
  __syncthreads();
  *total = s_warp[kWarps];
  return inc - x + s_warp[warp];
}

// One block owns one super-tile (kEncodeSubTiles sub-tiles of kThreads x
// kVPT 16-byte vectors) at a time; records are ordered by element, i.e. by
// chunk c = (sub-tile g, vector slot v, warp w) and then lane/element.
//   phase 1 (warp-local, no block barrier): each warp streams its chunks with
//     128-bit loads, builds the change masks, ranks records with a shuffle
//     scan of popc(mask) and stages them in its own shared-memory slice;
//   phase 2: one block scan over the 256 chunk counts gives every chunk's
//     super-tile-local offset, and warp 0 resolves the super-tile's offset in
//     its segment with the decoupled look-back (one per 256 KB of input);
//   phase 3: each warp flushes its staged records with coalesced stores.
// A warp whose chunks overflow its staging slice re-derives the overflow
// records from global memory (warp-local slow path).
template <int DT>
__device__ __noinline__ void encode_overflow(const EncodeArgs& a, const SegDev& sg, uint64_t e0,
                                             uint32_t cnt, uint64_t prefix, const uint32_t* s_cnt,
                                             const uint32_t* s_off, uint32_t wstart_lane) {
  using Tr = Traits<DT>;
  using T = typename Tr::T;
  constexpr int VE = Tr::kVE;
  constexpr uint32_t SUB = kThreads * kVPT * VE;
  constexpr uint32_t WCAP = kStageCap / kWarps;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const T* prevT = reinterpret_cast<const T*>(a.prev);
  const T* nextT = reinterpret_cast<const T*>(a.next);
  T* out_val = reinterpret_cast<T*>(a.out_val);
  for (int c = 0; c < kEncodeSubTiles * kVPT; ++c) {
    const uint32_t ccnt = s_cnt[c * kWarps + w];
    const uint32_t start = __shfl_sync(kFullMask, wstart_lane, c);
    if (start + ccnt <= WCAP || ccnt == 0) continue;  // fully staged
    const int g = c / kVPT, v = c % kVPT;
    const uint32_t off = g * SUB + (uint32_t)(v * kThreads + w * 32 + lane) * VE;
    uint32_t m = 0;
    T ta[VE], tb[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      const bool in = off + e < cnt;
      ta[e] = in ? prevT[sg.base + e0 + off + e] : T(0);
      tb[e] = in ? nextT[sg.base + e0 + off + e] : T(0);
      if (in && Tr::changed(ta[e], tb[e])) m |= 1u << e;
    }
    uint32_t incl = __popc(m);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFullMask, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t k = incl - __popc(m);
    const uint64_t goff = prefix + s_off[c * kWarps + w];
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      if (m & (1u << e)) {
        const uint64_t pos = goff + k;
        if (start + k >= WCAP && pos < sg.cap) {
          a.out_idx[sg.rec + pos] = (uint32_t)(e0 + off + e);
          out_val[sg.rec + pos] = Tr::delta(ta[e], tb[e]);
        }
        ++k;
      }
    }
  }
}

template <int DT>
__global__ void __launch_bounds__(kThreads, 4) encode_kernel(EncodeArgs a) {
  using Tr = Traits<DT>;
  using T = typename Tr::T;
  constexpr int VE = Tr::kVE;
  constexpr uint32_t SUB = kThreads * kVPT * VE;
  constexpr uint32_t SUPER = SUB * kEncodeSubTiles;
  constexpr int NCH = kEncodeSubTiles * kVPT;  // chunks per warp per super-tile (32)
  constexpr uint32_t WCAP = kStageCap / kWarps;
  static_assert(NCH == 32, "one lane per chunk in the flush");
  static_assert(NCH * kWarps == kThreads, "one thread per chunk in the block scan");

  __shared__ unsigned long long s_warp[kWarps + 1];
  __shared__ uint32_t s_tile[2];
  __shared__ uint32_t s_prefix;
  __shared__ uint32_t s_cnt[NCH * kWarps];   // chunk counts, index c * kWarps + w
  __shared__ uint32_t s_off[NCH * kWarps];   // chunk offsets within the super-tile
  __shared__ uint32_t s_idx[kStageCap];      // warp w stages at [w * WCAP, (w + 1) * WCAP)
  __shared__ T s_val[kStageCap];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile[0] = atomicAdd(a.ticket, 1u);
  __syncthreads();
  if (blockIdx.x == 0 && a.segs) {  // empty segments have no tile
    for (int s = tid; s < a.nseg; s += kThreads)
      if (a.segs[s].n == 0) a.seg_nnz[s] = 0;
  }
  const uint4* prev4 = reinterpret_cast<const uint4*>(a.prev);
  const uint4* next4 = reinterpret_cast<const uint4*>(a.next);
  const T* prevT = reinterpret_cast<const T*>(a.prev);
  const T* nextT = reinterpret_cast<const T*>(a.next);
  T* out_val = reinterpret_cast<T*>(a.out_val);
  uint32_t* w_idx = s_idx + w * WCAP;
  T* w_val = s_val + w * WCAP;

  for (int it = 0;; ++it) {
    const uint32_t t = s_tile[it & 1];
    if (t >= a.ntiles) break;
    if (tid == 0) s_tile[(it + 1) & 1] = atomicAdd(a.ticket, 1u);

    const int s = a.tile0 ? find_segment(a.tile0, a.nseg, t) : 0;
    const SegDev sg = a.segs ? a.segs[s] : a.seg0;
    const uint32_t lt = a.tile0 ? t - __ldg(a.tile0 + s) : t;
    const uint64_t e0 = (uint64_t)lt * SUPER;
    const uint64_t rem_n = sg.n - e0;
    const uint32_t cnt = rem_n < SUPER ? (uint32_t)rem_n : SUPER;
    const bool last_tile = (a.tile0 ? __ldg(a.tile0 + s + 1) : a.ntiles) == t + 1;
    const uint64_t vbase = (sg.base + e0) / VE;

    // ---- phase 1: warp-local streaming, ranking and staging
    uint32_t running = 0;  // records staged by this warp so far (warp-uniform)
#pragma unroll 1
    for (int g = 0; g < kEncodeSubTiles; ++g) {
      const uint32_t g0 = g * SUB;
      uint4 pa[kVPT], pb[kVPT];
#pragma unroll
      for (int v = 0; v < kVPT; ++v) {
        const uint32_t off = g0 + (uint32_t)(v * kThreads + tid) * VE;
        if (off + VE <= cnt) {
          pa[v] = ld_stream(prev4 + vbase + off / VE);
          pb[v] = ld_stream(next4 + vbase + off / VE);
        } else {
          pa[v] = make_uint4(0, 0, 0, 0);
          pb[v] = make_uint4(0, 0, 0, 0);
          if (off < cnt) {  // ragged tail
            T ta[VE], tb[VE];
#pragma unroll
            for (int e = 0; e < VE; ++e) {
              ta[e] = off + e < cnt ? prevT[sg.base + e0 + off + e] : T(0);
              tb[e] = off + e < cnt ? nextT[sg.base + e0 + off + e] : T(0);
            }
            memcpy(&pa[v], ta, 16);
            memcpy(&pb[v], tb, 16);
          }
        }
      }
#pragma unroll
      for (int v = 0; v < kVPT; ++v) {
        const uint32_t m = change_mask<DT>(pa[v], pb[v]);
        uint32_t incl = __popc(m);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFullMask, incl, o);
          if (lane >= o) incl += y;
        }
        const uint32_t tot = __shfl_sync(kFullMask, incl, 31);
        if (lane == 0) s_cnt[(g * kVPT + v) * kWarps + w] = tot;
        if (m) {
          uint32_t k = running + incl - __popc(m);
          const uint32_t off = g0 + (uint32_t)(v * kThreads + tid) * VE;
#pragma unroll
          for (int e = 0; e < VE; ++e) {
            if (m & (1u << e)) {
              if (k < WCAP) {
                w_idx[k] = off + e;
                w_val[k] = Tr::delta(Tr::get(pa[v], e), Tr::get(pb[v], e));
              }
              ++k;
            }
          }
        }
        running += tot;
      }
    }
    __syncthreads();

    // ---- phase 2: chunk offsets (block scan) + look-back for the super-tile
    unsigned long long total;
    const uint32_t my_cnt = s_cnt[tid];
    s_off[tid] = (uint32_t)block_scan_packed(my_cnt, s_warp, &total);
    const uint32_t tile_count = (uint32_t)total;
    if (w == 0) {
      uint32_t prefix = 0;
      if (lt == 0 || (a.debug & 1)) {
        if (tid == 0) st_relaxed_u64(a.status + t, make_status(a.epoch, kFlagPrefix, tile_count));
      } else {
        if (tid == 0) st_relaxed_u64(a.status + t, make_status(a.epoch, kFlagAggregate, tile_count));
        prefix = warp_lookback(a.status, t, (int64_t)t - lt, a.epoch);
        if (tid == 0)
          st_relaxed_u64(a.status + t, make_status(a.epoch, kFlagPrefix, prefix + tile_count));
      }
      if (tid == 0) {
        s_prefix = prefix;
        if (last_tile) a.seg_nnz[s] = (uint64_t)prefix + tile_count;
      }
    }
    __syncthreads();
    const uint64_t prefix = s_prefix;

    // ---- phase 3: flush this warp's staged records (lane c owns chunk c)
    const uint32_t ccnt = s_cnt[lane * kWarps + w];
    uint32_t wincl = ccnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFullMask, wincl, o);
      if (lane >= o) wincl += y;
    }
    const uint32_t wstart = wincl - ccnt;  // chunk's first slot in the warp's staging
    const uint32_t staged = min(running, WCAP);
    if (!(a.debug & 2)) {
      for (uint32_t k0 = 0; k0 < staged; k0 += 32) {
        const uint32_t k = k0 + lane;
        // owner chunk of staged record k: the largest c with start(c) <= k
        // (starts are non-decreasing; an empty chunk shares its successor's)
        int c = 0;
#pragma unroll
        for (int b = 16; b > 0; b >>= 1)
          if (__shfl_sync(kFullMask, wstart, c + b) <= k) c += b;
        const uint32_t cstart = __shfl_sync(kFullMask, wstart, c);
        if (k < staged) {
          const uint64_t pos = prefix + s_off[c * kWarps + w] + (k - cstart);
          if (pos < sg.cap) {
            a.out_idx[sg.rec + pos] = (uint32_t)(e0 + w_idx[k]);
            out_val[sg.rec + pos] = w_val[k];
          }
        }
      }
    }
    if (running > WCAP && !(a.debug & 2))
      encode_overflow<DT>(a, sg, e0, cnt, prefix, s_cnt, s_off, wstart);
    __syncthreads();  // staging, s_cnt and s_prefix are reused by the next super-tile
  }
}

// ---- apply (codec.cpp:65-92) ---------------------------------------------------

__global__ void validate_kernel(const uint32_t* idx, uint64_t nnz, const uint64_t* nnz_dev,
                                uint64_t n, uint32_t* err) {
  const uint64_t cnt = nnz_dev ? *nnz_dev : nnz;
  bool bad = false;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < cnt;
       k += (uint64_t)gridDim.x * blockDim.x)
    bad |= (uint64_t)__ldg(idx + k) >= n;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, WS_ERRBIT_INDEX_OUT_OF_SHARD);
}

template <int DT>
__global__ void apply_kernel(typename Traits<DT>::T* target, const uint32_t* idx,
                             const typename Traits<DT>::T* val, uint64_t nnz,
                             const uint64_t* nnz_dev, const uint32_t* err) {
  if (*err & WS_ERRBIT_INDEX_OUT_OF_SHARD) return;  // no partial writes
  const uint64_t cnt = nnz_dev ? *nnz_dev : nnz;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < cnt;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = __ldg(idx + k);
    target[i] = Traits<DT>::add(target[i], __ldg(val + k));
  }
}

// ---- reslice (codec.cpp:94-138): order-preserving filter + re-index ----------

__global__ void validate_src_kernel(const uint32_t* idx, uint64_t nnz, const uint64_t* nnz_dev,
                                    uint64_t src_elems, uint32_t* err) {
  const uint64_t cnt = nnz_dev ? *nnz_dev : nnz;
  bool bad = false;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < cnt;
       k += (uint64_t)gridDim.x * blockDim.x)
    bad |= (uint64_t)__ldg(idx + k) >= src_elems;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, WS_ERRBIT_INDEX_OUT_OF_SHARD);
}

template <int DT>
__global__ void __launch_bounds__(kThreads) reslice_kernel(ResliceArgs a) {
  using T = typename Traits<DT>::T;
  constexpr int R = 4;  // records per thread per tile
  __shared__ unsigned long long s_warp[kWarps + 1];
  __shared__ uint32_t s_tile[2];
  __shared__ uint32_t s_prefix;
  if (*a.err & WS_ERRBIT_INDEX_OUT_OF_SHARD) return;
  const int tid = threadIdx.x;
  const uint64_t cnt = a.nnz_dev ? *a.nnz_dev : a.nnz;
  const uint32_t ntiles = (uint32_t)((cnt + kResliceTile - 1) / kResliceTile);
  if (tid == 0) s_tile[0] = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const T* val = reinterpret_cast<const T*>(a.val);
  T* out_val = reinterpret_cast<T*>(a.out_val);
  for (int it = 0;; ++it) {
    const uint32_t t = s_tile[it & 1];
    if (t >= ntiles) break;
    if (tid == 0) s_tile[(it + 1) & 1] = atomicAdd(a.ticket, 1u);
    unsigned long long di[R];
    unsigned long long packed = 0;
#pragma unroll
    for (int v = 0; v < R; ++v) {
      const uint64_t k = (uint64_t)t * kResliceTile + v * kThreads + tid;
      di[v] = k < cnt ? remap_index(a.map, __ldg(a.idx + k)) : ~0ull;
      packed |= (unsigned long long)(di[v] != ~0ull) << (16 * v);
    }
    unsigned long long total;
    const unsigned long long excl = block_scan_packed(packed, s_warp, &total);
    uint32_t vstart[R], tile_count = 0;
#pragma unroll
    for (int v = 0; v < R; ++v) {
      vstart[v] = tile_count;
      tile_count += (uint32_t)(total >> (16 * v)) & 0xffffu;
    }
    if ((tid >> 5) == 0) {
      uint32_t prefix = 0;
      if (t == 0) {
        if (tid == 0) st_relaxed_u64(a.status + t, make_status(a.epoch, kFlagPrefix, tile_count));
      } else {
        if (tid == 0) st_relaxed_u64(a.status + t, make_status(a.epoch, kFlagAggregate, tile_count));
        prefix = warp_lookback(a.status, t, 0, a.epoch);
        if (tid == 0)
          st_relaxed_u64(a.status + t, make_status(a.epoch, kFlagPrefix, prefix + tile_count));
      }
      if (tid == 0) {
        s_prefix = prefix;
        if (t + 1 == ntiles) *a.out_nnz = (uint64_t)prefix + tile_count;
      }
    }
    __syncthreads();
    const uint32_t prefix = s_prefix;
#pragma unroll
    for (int v = 0; v < R; ++v) {
      if (di[v] == ~0ull) continue;
      const uint64_t k = (uint64_t)t * kResliceTile + v * kThreads + tid;
      const uint64_t pos = (uint64_t)prefix + vstart[v] + ((excl >> (16 * v)) & 0xffffu);
      a.out_idx[pos] = (uint32_t)di[v];
      out_val[pos] = __ldg(val + k);
    }
  }
}

// ---- dense box copy (shard.cpp:136-170 generalised) -------------------------

template <typename T>
__global__ void box_copy_kernel(BoxCopyArgs a) {
  // blockIdx.y (and z) walk rows; x walks the contiguous run.
  for (uint64_t r = blockIdx.y + (uint64_t)blockIdx.z * gridDim.y; r < a.rows;
       r += (uint64_t)gridDim.y * gridDim.z) {
    uint64_t so = a.src_base, dso = a.dst_base, rem = r;
    for (int d = a.nd_outer - 1; d >= 0; --d) {
      const uint64_t c = rem % a.outer_ext[d];
      rem /= a.outer_ext[d];
      so += c * a.src_stride[d];
      dso += c * a.dst_stride[d];
    }
    if (a.vec) {
      constexpr int VE = 16 / sizeof(T);
      const uint4* s4 = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(a.src) + so);
      uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<T*>(a.dst) + dso);
      const uint64_t nv = a.run / VE;
      for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nv;
           j += (uint64_t)gridDim.x * blockDim.x)
        d4[j] = ld_stream(s4 + j);
    } else {
      const T* s = reinterpret_cast<const T*>(a.src) + so;
      T* d = reinterpret_cast<T*>(a.dst) + dso;
      for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < a.run;
           j += (uint64_t)gridDim.x * blockDim.x)
        d[j] = s[j];
    }
  }
}

// ---- synthetic generator ------------------------------------------------------

__global__ void gen_kernel(uint64_t key, Box box, uint32_t full_ext_nd, uint64_t full_strides0,
                           uint64_t full_strides1, uint64_t full_strides2, uint64_t full_strides3,
                           uint64_t n, uint64_t change_thr, uint16_t* prev, uint16_t* next) {
  const uint64_t fs[4] = {full_strides0, full_strides1, full_strides2, full_strides3};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t rem = i, g = 0;
    for (int d = (int)full_ext_nd - 1; d >= 0; --d) {
      const uint64_t c = rem % box.ext[d] + box.lo[d];
      rem /= box.ext[d];
      g += c * fs[d];
    }
    uint16_t p, q;
    gen_elem_bf16(key, g, change_thr, p, q);
    prev[i] = p;
    if (next) next[i] = q;
  }
}

template <typename K>
int occupancy_grid(K kernel, int threads) {
  static int cached = 0;
  if (!cached) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
    cached = std::max(1, per_sm) * sm_count();
  }
  return cached;
}

}  // namespace

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_encode(int dtype, const EncodeArgs& a, cudaStream_t s, int* grid_out) {
  int grid = 0;
  switch (dtype) {
    case WS_BF16: grid = occupancy_grid(encode_kernel<WS_BF16>, kThreads); break;
    case WS_I32: grid = occupancy_grid(encode_kernel<WS_I32>, kThreads); break;
    case WS_F32: grid = occupancy_grid(encode_kernel<WS_F32>, kThreads); break;
    default: return cudaErrorInvalidValue;
  }
  grid = (int)std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)grid, std::max(a.ntiles, 1u)));
  if (const char* g = getenv("WSYNC_ENCODE_GRID")) grid = std::max(1, atoi(g));
  EncodeArgs a2 = a;
  if (const char* d = getenv("WSYNC_ENCODE_DEBUG")) a2.debug = (uint32_t)atoi(d);
  if (grid_out) *grid_out = grid;
  cudaError_t e = cudaMemsetAsync(a.ticket, 0, sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  switch (dtype) {
    case WS_BF16: encode_kernel<WS_BF16><<<grid, kThreads, 0, s>>>(a2); break;
    case WS_I32: encode_kernel<WS_I32><<<grid, kThreads, 0, s>>>(a2); break;
    default: encode_kernel<WS_F32><<<grid, kThreads, 0, s>>>(a2); break;
  }
  return cudaGetLastError();
}

static int stream_grid(uint64_t work, int threads) {
  const uint64_t want = (work + threads - 1) / threads;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sm_count() * 8));
}

cudaError_t launch_apply(int dtype, void* target, uint64_t n, const uint32_t* idx,
                         const void* val, uint64_t nnz, const uint64_t* nnz_dev,
                         uint32_t* err, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(err, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const int grid = stream_grid(nnz, 256);
  validate_kernel<<<grid, 256, 0, s>>>(idx, nnz, nnz_dev, n, err);
  switch (dtype) {
    case WS_BF16:
      apply_kernel<WS_BF16><<<grid, 256, 0, s>>>((uint16_t*)target, idx, (const uint16_t*)val,
                                                  nnz, nnz_dev, err);
      break;
    case WS_I32:
      apply_kernel<WS_I32><<<grid, 256, 0, s>>>((uint32_t*)target, idx, (const uint32_t*)val,
                                                 nnz, nnz_dev, err);
      break;
    case WS_F32:
      apply_kernel<WS_F32><<<grid, 256, 0, s>>>((uint32_t*)target, idx, (const uint32_t*)val,
                                                 nnz, nnz_dev, err);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_reslice(int dtype, const ResliceArgs& a, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(a.err, 0, sizeof(uint32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.out_nnz, 0, sizeof(uint64_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.ticket, 0, sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  validate_src_kernel<<<stream_grid(a.cap_in, 256), 256, 0, s>>>(a.idx, a.nnz, a.nnz_dev,
                                                                 a.src_elems, a.err);
  const uint64_t tiles = (a.cap_in + kResliceTile - 1) / kResliceTile;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)sm_count() * 4));
  switch (dtype) {
    case WS_BF16: reslice_kernel<WS_BF16><<<grid, kThreads, 0, s>>>(a); break;
    case WS_I32: reslice_kernel<WS_I32><<<grid, kThreads, 0, s>>>(a); break;
    case WS_F32: reslice_kernel<WS_F32><<<grid, kThreads, 0, s>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_box_copy(int dtype, const BoxCopyArgs& a, cudaStream_t s) {
  if (a.rows == 0 || a.run == 0) return cudaSuccess;
  const uint64_t per_row = a.vec ? a.run / (16 / dtype_size(dtype)) : a.run;
  const unsigned gx = (unsigned)std::min<uint64_t>((per_row + 255) / 256, 65535);
  const uint64_t rows = a.rows;
  const unsigned gy = (unsigned)std::min<uint64_t>(rows, 65535);
  const unsigned gz = (unsigned)std::min<uint64_t>((rows + gy - 1) / gy, 64);
  dim3 grid(std::max(1u, gx), gy, gz);
  if (dtype == WS_BF16)
    box_copy_kernel<uint16_t><<<grid, 256, 0, s>>>(a);
  else
    box_copy_kernel<uint32_t><<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

Box shard_box(const int64_t* full, int nd, const ws_shard& d) {
  Box b{};
  b.nd = nd;
  for (int i = 0; i < nd; ++i) {
    b.lo[i] = 0;
    b.ext[i] = (uint32_t)full[i];
  }
  if (d.slice_dim >= 0) {
    b.lo[d.slice_dim] = (uint32_t)d.start;
    b.ext[d.slice_dim] = (uint32_t)(d.end - d.start);
  }
  return b;
}

Remap make_remap(const int64_t* full, int nd, const ws_shard& src, const ws_shard& dst) {
  const Box S = shard_box(full, nd, src), D = shard_box(full, nd, dst);
  Remap m{};
  m.nd = nd;
  for (int i = 0; i < nd; ++i) {
    m.src_ext[i] = S.ext[i];
    m.dst_ext[i] = D.ext[i];
    m.shift[i] = (int64_t)S.lo[i] - (int64_t)D.lo[i];
  }
  return m;
}

uint64_t make_box_copy(int dtype, const int64_t* full, int nd, const ws_shard& dst,
                       const ws_shard& src, BoxCopyArgs* out) {
  const Box S = shard_box(full, nd, src), D = shard_box(full, nd, dst);
  int64_t lo[WS_MAX_DIMS] = {0, 0, 0, 0}, ext[WS_MAX_DIMS] = {1, 1, 1, 1};
  uint64_t count = 1;
  for (int d = 0; d < nd; ++d) {
    lo[d] = std::max<int64_t>(S.lo[d], D.lo[d]);
    const int64_t hi = std::min<int64_t>((int64_t)S.lo[d] + S.ext[d], (int64_t)D.lo[d] + D.ext[d]);
    ext[d] = hi - lo[d];
    if (ext[d] <= 0) return 0;
    count *= (uint64_t)ext[d];
  }
  // Row-major strides of both boxes.
  uint64_t ss[WS_MAX_DIMS], ds[WS_MAX_DIMS];
  uint64_t a = 1, b = 1;
  for (int d = nd - 1; d >= 0; --d) {
    ss[d] = a;
    ds[d] = b;
    a *= S.ext[d];
    b *= D.ext[d];
  }
  // Merge trailing dims that are whole in the overlap, the source and the
  // destination into one contiguous run.
  int k = nd - 1;
  uint64_t run = (uint64_t)ext[k];
  while (k > 0 && (uint64_t)ext[k] == S.ext[k] && (uint64_t)ext[k] == D.ext[k]) {
    --k;
    run *= (uint64_t)ext[k];
  }
  BoxCopyArgs r{};
  r.run = run;
  r.nd_outer = k;
  r.rows = 1;
  r.src_base = 0;
  r.dst_base = 0;
  for (int d = 0; d < nd; ++d) {
    r.src_base += (uint64_t)(lo[d] - S.lo[d]) * ss[d];
    r.dst_base += (uint64_t)(lo[d] - D.lo[d]) * ds[d];
  }
  for (int d = 0; d < k; ++d) {
    r.outer_ext[d] = (uint32_t)ext[d];
    r.src_stride[d] = ss[d];
    r.dst_stride[d] = ds[d];
    r.rows *= (uint64_t)ext[d];
  }
  const uint64_t ve = elems_per_vec(dtype);
  bool vec = run % ve == 0 && r.src_base % ve == 0 && r.dst_base % ve == 0;
  for (int d = 0; d < k; ++d) vec = vec && ss[d] % ve == 0 && ds[d] % ve == 0;
  r.vec = vec ? 1 : 0;
  *out = r;
  return count;
}

uint64_t param_key(uint64_t seed, const char* name) {
  uint64_t h = 0xcbf29ce484222325ull;  // fnv1a64 (rng.hpp:80-87)
  for (const unsigned char* p = (const unsigned char*)name; *p; ++p) {
    h ^= *p;
    h *= 0x100000001b3ull;
  }
  uint64_t x = seed ^ h;  // splitmix64 (rng.hpp:73-78)
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

cudaError_t launch_gen_bf16(uint64_t key, const int64_t* full, int nd, const ws_shard& desc,
                            uint64_t change_thr, uint16_t* prev, uint16_t* next,
                            cudaStream_t s) {
  const Box b = shard_box(full, nd, desc);
  uint64_t n = 1, fs[4] = {0, 0, 0, 0}, st = 1;
  for (int d = 0; d < nd; ++d) n *= b.ext[d];
  for (int d = nd - 1; d >= 0; --d) {
    fs[d] = st;
    st *= (uint64_t)full[d];
  }
  if (n == 0) return cudaSuccess;
  gen_kernel<<<stream_grid(n, 256), 256, 0, s>>>(key, b, (uint32_t)nd, fs[0], fs[1], fs[2], fs[3],
                                                 n, change_thr, prev, next);
  return cudaGetLastError();
}

}  // namespace wsync
