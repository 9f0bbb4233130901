// kernels_codec.cu -- K1 encode, K4 apply, reslice, box copy, generator.
//
// K1 (encode) replaces the reference's diff_shards + density check +
// encode_sparse packing (codec.cpp:34-63, engine.cpp:118-127,
// codec.cpp:164-183): one pass over prev/next that writes every change as an
// (ascending local index, delta) record at its final position in its
// segment's stream, via a decoupled look-back prefix sum over super-tiles
// (segments are independent look-back chains).  The design and the
// measurements behind it are in DESIGN.md §4.
#include <algorithm>
#include <atomic>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>

#include "kernels.h"

namespace wsync {

namespace {

constexpr int kThreads = kEncodeThreads;
constexpr int kWarps = kThreads / 32;

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

// K1 as a warp-specialised pipeline (one persistent block per SM):
//   warp 16      producer: claims super-tiles in order (one ticket each) and
//                streams their sub-tiles of prev and next into a kRing-deep
//                shared-memory ring with 1-D bulk copies (cp.async.bulk)
//                completing on per-stage mbarriers;
//   warps 0-15   consumers: per 16-byte vector the change mask (SWAR bit
//                compare for bf16, lane compare for i32, value compare for
//                f32); every change is appended to the thread's private
//                shared-memory slots and marked in the super-tile's change
//                bitmap -- no warp-level communication per vector.  Each
//                stage is released as soon as it is read, so HBM streams
//                continuously;
//   warps 17..   resolvers (one per staging buffer): popcount-scan the
//                bitmap (the ascending rank of every change inside its
//                super-tile) and place the super-tile in its segment's
//                stream: one atomic reservation (the engine: super-tiles in
//                any order, records ascending inside each) or the decoupled
//                look-back (ws_diff_shards: one ascending stream);
//   each consumer warp writes its staged records of super-tile i to
//   base + rank after staging super-tile i + NB - 1, applying them in place
//   to a serving shard on this GPU when the engine asks for the fused apply;
//   SA (streamed apply): the producer also streams the serving sub-tile, and
//   consumers store serve + (next - prev) per changed vector at staging.
// A thread with more than SLOTS changes in one super-tile re-derives the
// rest from global memory at write-out; the bitmap still gives their ranks.
constexpr int kStagedBar = 2;  // named barriers 2.. : "super-tile staged in buffer b"

struct StageMeta {
  SegDev sg;
  uint32_t t, s, lt, nsub, cnt, last;
  uint32_t count_only;  // segment predicted dense: count, stage nothing
  uint32_t sa;          // streamed apply: the serving sub-tile is in the third ring
};

#ifndef WS_ENC_SLOTS
#define WS_ENC_SLOTS 6
#endif
#ifndef WS_ENC_PREFETCH
#define WS_ENC_PREFETCH 1
#endif
#ifndef WS_ENC_EVICT
#define WS_ENC_EVICT 0  // (measured: no gain) prev/next streamed evict-first, prefetched serving words evict-last
#endif

template <int DT, bool SA = false>
struct EncCfg {
  using T = typename Traits<DT>::T;
  static constexpr int VE = Traits<DT>::kVE;                          // elements per vector
  static constexpr int NCW = kEncConsumers / 32;                      // consumer warps
  static constexpr uint32_t VPT = kStageBytes / 16 / kEncConsumers;   // vectors per thread per stage
  static constexpr uint32_t SUB = kStageBytes / sizeof(T);            // elements per sub-tile
  static constexpr uint32_t SUPER = SUB * kEncodeSubTiles;
  // staged changes per thread per super-tile (SA: fewer, to fit the third ring)
  static constexpr int K = SA ? 4 : WS_ENC_SLOTS;
  static constexpr uint32_t SPW = SUPER / NCW;                        // spill capacity per warp (all its elements)
  using SpillRec = typename std::conditional<sizeof(T) == 2, uint32_t, uint2>::type;  // li | val
  static constexpr uint32_t WORDS = SUPER / 32;                       // change-bitmap words
  static constexpr int NB = kEncBuffers;                              // staging buffers
  // bf16: the serving word a fused record updates is fetched (cp.async) into
  // shared memory when the record is staged
  // (SA: streamed tiles need no prefetch; the other fused tiles read the
  // word at the flush -- the engine runs SA only when most tiles stream)
  static constexpr bool PRE = WS_ENC_PREFETCH && DT == WS_BF16 && !SA;
  // streamed apply: three arrays per stage (prev, next, serving)
  static constexpr int RING = kRing;
  static constexpr size_t kRingBytes = (SA ? 3 : 2) * RING * (size_t)kStageBytes;
  // per buffer: bitmap u32[WORDS] | [serving words u32[K][threads]] | val T[K][threads] |
  //             word prefix u16[WORDS] | idx u16[K][threads]
  static constexpr size_t kBufBytes =
      WORDS * 6 + (size_t)K * kEncConsumers * (sizeof(T) + 2 + (PRE ? 4 : 0));
  static constexpr size_t kSmem = kRingBytes + NB * kBufBytes +
                                  (RING + NB) * sizeof(StageMeta) + NB * 8 +
                                  (2 * RING + 2 * NB) * 8 + NB * NCW * 4 + NB * 4 + 4 + 32;
  static_assert(VPT >= 1 && VPT * 16 * kEncConsumers == kStageBytes, "stage split");
  static_assert(SUPER <= 65536, "u16 in-tile index");
  static_assert(WORDS % 128 == 0, "bitmap words per resolver lane in 16-byte loads");
  static_assert(kBufBytes % 16 == 0, "buffer alignment");
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
};

// Resolver step for one staged super-tile (one warp): word prefix of the
// change bitmap, the super-tile's count, and its place in its segment.
template <int DT>
__device__ __forceinline__ void resolve_tile(const EncodeArgs& a, const StageMeta& ti,
                                             const uint32_t* bm, uint16_t* wpre,
                                             unsigned long long* s_prefix, uint32_t* s_tcnt) {
  using C = EncCfg<DT>;
  constexpr int PER = C::WORDS / 32;
  const int lane = threadIdx.x & 31;
  if (ti.count_only) {  // the consumers summed the count; nothing is staged
    if (lane == 0) {
      const uint32_t count = *s_tcnt;
      *s_tcnt = 0;
      if (count) atomicAdd(reinterpret_cast<unsigned long long*>(a.seg_nnz + ti.s),
                           (unsigned long long)count);
      a.tile_cnt[ti.t] = 0;
      a.tile_base[ti.t] = 0;
      *s_prefix = ~0ull;
    }
    return;
  }
  const uint4* b4 = reinterpret_cast<const uint4*>(bm + lane * PER);
  uint32_t sum = 0;
#pragma unroll
  for (int q = 0; q < PER / 4; ++q) {
    const uint4 w = b4[q];
    sum += __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFullMask, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t count = __shfl_sync(kFullMask, incl, 31);
  uint32_t run = incl - sum;  // < 2^16: at most SUPER - 32
  uint2* p2 = reinterpret_cast<uint2*>(wpre + lane * PER);
#pragma unroll
  for (int q = 0; q < PER / 4; ++q) {
    const uint4 w = b4[q];
    uint2 o;
    o.x = run;
    run += __popc(w.x);
    o.x |= run << 16;
    run += __popc(w.y);
    o.y = run;
    run += __popc(w.z);
    o.y |= run << 16;
    run += __popc(w.w);
    p2[q] = o;
  }
  if (a.unordered) {  // one atomic reserves the super-tile's place in its segment
    if (lane == 0) {
      unsigned long long base = 0;
      if (count)  // the fixup pass reserves in `fill` (seg_nnz holds the count already)
        base = atomicAdd(a.fill ? a.fill + ti.s
                                : reinterpret_cast<unsigned long long*>(a.seg_nnz + ti.s),
                         (unsigned long long)count);
      a.tile_cnt[ti.t] = count;
      a.tile_base[ti.t] = (uint32_t)base;  // <= segment size < 2^32
      *s_prefix = base;
    }
    return;
  }
  const bool head = ti.lt == 0 || (a.debug & 1);
  if (lane == 0)
    st_relaxed_u64(a.status + ti.t,
                   make_status(a.epoch, head ? kFlagPrefix : kFlagAggregate, count));
  uint32_t prefix = 0;
  if (!head) {
    prefix = warp_lookback(a.status, ti.t, (int64_t)ti.t - ti.lt, a.epoch);
    if (lane == 0)
      st_relaxed_u64(a.status + ti.t, make_status(a.epoch, kFlagPrefix, prefix + count));
  }
  if (lane == 0) {
    if (ti.last) a.seg_nnz[ti.s] = (uint64_t)prefix + count;
    *s_prefix = prefix;
  }
}

// What a consumer thread keeps (in registers) about a staged super-tile
// until it writes the records out.
struct PendingSlice {
  uint64_t base, rec, cap;
  uint32_t lt, nsub, cnt, seg;
  uint32_t mine;  // this thread's changes in the super-tile
  uint32_t sa;    // applied by the streamed apply at staging
};

// serve[dst(i)] += v for a record of a segment with a local serving shard
// (codec.cpp:80-91 applied at the moment K1 writes the record).
template <int DT>
__device__ __forceinline__ typename Traits<DT>::T* fuse_target(const FuseEntry* __restrict__ f,
                                                                typename Traits<DT>::T* serve,
                                                                uint32_t i) {
  uint64_t d;
  if (f->mode == 1) {
    if (i < f->keep_lo || i >= f->keep_hi) return nullptr;
    d = (uint64_t)((int64_t)i + f->shift);
  } else {
    d = remap_index(f->map, i);
    if (d == ~0ull) return nullptr;
  }
  return serve + f->dst_base + d;
}

#ifndef WS_FLUSH_BATCH
#define WS_FLUSH_BATCH 1
#endif

// Fused remote emission (bf16): the record (segment-local i, value v) of a
// lane with `valid`, re-indexed into route M's destination shard, stored
// (shard-local index, value) into every replica's region.
// Warp-collective: every lane calls it.
__device__ __forceinline__ void emit_remote(const RemoteMap& M, bool valid, uint32_t i,
                                            uint16_t v) {
  uint64_t d = 0;
  if (valid) {
    if (M.identity) {
      valid = i >= M.keep_lo && i < M.keep_hi;
      d = (uint64_t)((int64_t)i + M.shift);
    } else {
      d = remap_index(M.map, i);
      valid = d != ~0ull;
    }
  }
  const unsigned bal = __ballot_sync(kFullMask, valid);
  if (!bal) return;
  const int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == 0) base = atomicAdd(M.cnt, (unsigned)__popc(bal));
  base = __shfl_sync(kFullMask, base, 0);
  if (!valid) return;
  const uint64_t slot = (uint64_t)base + __popc(bal & ((1u << lane) - 1u));
  if (slot >= M.cap) return;  // cannot happen: a sparse segment fits its regions
#pragma unroll 1
  for (int r = 0; r < 8 && M.rec[r]; ++r) {  // SoA region: shard-local index | value
    reinterpret_cast<uint32_t*>(M.rec[r])[slot] = (uint32_t)d;
    reinterpret_cast<uint16_t*>(reinterpret_cast<uint32_t*>(M.rec[r]) + M.cap)[slot] = v;
  }
}

// Ascending rank of in-tile element li among the super-tile's changes.
__device__ __forceinline__ uint32_t tile_rank(const uint32_t* bm, const uint16_t* wpre, uint32_t li) {
  const uint32_t w = li >> 5;
  return wpre[w] + __popc(bm[w] & ((1u << (li & 31)) - 1u));
}

// A consumer warp writes the staged records of its threads for a resolved
// super-tile (warp-cooperative: record r of the warp is slot r - start(l)
// of the lane l owning it), then the spilled ones, then clears its bitmap
// words for the buffer's next super-tile.
template <int DT, bool REMOTE, bool SA>
__device__ __forceinline__ void flush_slice(const EncodeArgs& a, const PendingSlice& ti,
                                            uint64_t prefix, uint32_t* bm, const uint16_t* wpre,
                                            const uint16_t* sidx,
                                            const typename Traits<DT>::T* sval,
                                            const uint32_t* spre, uint32_t* ovf,
                                            const typename EncCfg<DT, SA>::SpillRec* spill,
                                            const uint32_t* s_acks) {
  using C = EncCfg<DT, SA>;
  using Tr = Traits<DT>;
  using T = typename Tr::T;
  constexpr int VE = C::VE, K = C::K;
  constexpr uint32_t VPT = C::VPT, SUB = C::SUB, SUPER = C::SUPER;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (!__any_sync(kFullMask, ti.mine != 0)) return;  // no bit of this warp is set
  const uint64_t e0 = (uint64_t)ti.lt * SUPER;
  if (!(a.debug & 2) && prefix < ti.cap) {
    T* out_val = reinterpret_cast<T*>(a.out_val);
    const FuseEntry* fz = (!ti.sa && a.fuse && a.fuse[ti.seg].mode && a.fuse_on[ti.seg])
                              ? a.fuse + ti.seg
                              : nullptr;
    // identity-mapped fused segments had their serving words fetched at staging
    const bool pre = C::PRE && fz && fz->mode == 1;
    // routes of this segment to other GPUs (bf16 engine, P2P): emitted here
    uint32_t rm0 = 0, rm1 = 0;
    if (REMOTE) {
      rm0 = a.remote.seg_first[ti.seg];
      rm1 = a.remote.seg_first[ti.seg + 1];
      if (rm1 > rm0)
        while (!ld_acquire_cta_u32(s_acks)) __nanosleep(256);
    }
    T* serve = reinterpret_cast<T*>(a.serve);
    const uint32_t mine = ti.mine < (uint32_t)K ? ti.mine : (uint32_t)K;
    uint32_t start = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFullMask, start, o);
      if (lane >= o) start += y;
    }
    const uint32_t staged = __shfl_sync(kFullMask, start, 31);
    start -= mine;
    constexpr int FB = WS_FLUSH_BATCH;
    for (uint32_t r0 = 0; r0 < staged; r0 += 32 * FB) {
      uint64_t pos[FB];
      uint32_t ii[FB], sl[FB];
      T vv[FB], old[FB];
      T* tp[FB];
#pragma unroll
      for (int j = 0; j < FB; ++j) {
        const uint32_t r = r0 + j * 32 + lane;
        int l = 0;  // owner lane: the largest l with start(l) <= r
#pragma unroll
        for (int b = 16; b > 0; b >>= 1)
          if (__shfl_sync(kFullMask, start, l + b) <= r) l += b;
        const uint32_t st = __shfl_sync(kFullMask, start, l);
        pos[j] = ~0ull;
        tp[j] = nullptr;
        if (r < staged) {
          const uint32_t slot = (r - st) * kEncConsumers + w * 32 + l;
          sl[j] = slot;
          const uint32_t li = sidx[slot];
          const uint64_t p = prefix + tile_rank(bm, wpre, li);
          if (p < ti.cap) {
            pos[j] = p;
            ii[j] = (uint32_t)(e0 + li);
            vv[j] = sval[slot];
            if (fz) tp[j] = fuse_target<DT>(fz, serve, ii[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < FB; ++j)
        if (tp[j]) {
          if (pre) {  // the half of the prefetched word holding the element
            const uint32_t wv = spre[sl[j]];
            old[j] = (T)((reinterpret_cast<uintptr_t>(tp[j]) & 2) ? (wv >> 16) : (wv & 0xffffu));
          } else {
            old[j] = *tp[j];
          }
        }
#pragma unroll
      for (int j = 0; j < FB; ++j) {
        if (pos[j] == ~0ull) continue;
        a.out_idx[ti.rec + pos[j]] = ii[j];
        out_val[ti.rec + pos[j]] = vv[j];
        if (tp[j]) *tp[j] = Tr::add(old[j], vv[j]);
      }
      if constexpr (REMOTE)
        for (uint32_t q = rm0; q < rm1; ++q)
#pragma unroll
          for (int j = 0; j < FB; ++j)
            emit_remote(a.remote.maps[q], pos[j] != ~0ull, ii[j], (uint16_t)vv[j]);
    }
    // changes past the slots: from this warp's spill region (written at
    // staging, still in L2), in any order -- the bitmap gives their ranks
    const uint32_t nov = *ovf;
    for (uint32_t r0 = 0; r0 < nov; r0 += 32) {  // warp-uniform trip count
      const uint32_t r = r0 + lane;
      bool ok = r < nov;
      uint32_t li = 0;
      T dv = 0;
      if (ok) {
        if constexpr (sizeof(T) == 2) {
          const uint32_t x = spill[r];
          li = x & 0xffffu;
          dv = (T)(x >> 16);
        } else {
          const uint2 x = spill[r];
          li = x.x;
          dv = (T)x.y;
        }
        const uint64_t pos = prefix + tile_rank(bm, wpre, li);
        ok = pos < ti.cap;
        if (ok) {
          a.out_idx[ti.rec + pos] = (uint32_t)(e0 + li);
          out_val[ti.rec + pos] = dv;
          if (fz) {
            T* p = fuse_target<DT>(fz, serve, (uint32_t)(e0 + li));
            if (p) *p = Tr::add(*p, dv);
          }
        }
      }
      if constexpr (REMOTE)
        for (uint32_t q = rm0; q < rm1; ++q)
          emit_remote(a.remote.maps[q], ok, (uint32_t)(e0 + li), (uint16_t)dv);
    }
  }
  __syncwarp();  // every lane of the warp is done reading the bitmap
  if (lane == 0) *ovf = 0;
  constexpr uint32_t LPW = 32 / VE;  // lanes sharing one bitmap word
  if ((threadIdx.x & (LPW - 1)) == 0)
    for (uint32_t g = 0; g < ti.nsub; ++g)
      for (uint32_t v = 0; v < VPT; ++v)
        bm[(g * SUB + (v * kEncConsumers + threadIdx.x) * VE) >> 5] = 0;
}

template <int DT, bool REMOTE, bool SA>
__global__ void __launch_bounds__(kEncodeBlock, 1) encode_kernel(EncodeArgs a) {
  using C = EncCfg<DT, SA>;
  constexpr int kRing = C::RING;
  using Tr = Traits<DT>;
  using T = typename Tr::T;
  constexpr int VE = C::VE, NCW = C::NCW, NB = C::NB, K = C::K;
  constexpr uint32_t VPT = C::VPT, SUB = C::SUB, SUPER = C::SUPER, WORDS = C::WORDS;
  constexpr uint32_t END = 0xffffffffu;

  extern __shared__ __align__(128) uint8_t dsm[];
  uint8_t* ring_prev = dsm;
  uint8_t* ring_next = dsm + kRing * kStageBytes;
  uint8_t* ring_serve = dsm + 2 * kRing * kStageBytes;  // SA only
  uint8_t* bufs = dsm + C::kRingBytes;  // NB x kBufBytes
  auto buf_bm = [&](int b) { return reinterpret_cast<uint32_t*>(bufs + b * C::kBufBytes); };
  auto buf_pre = [&](int b) { return buf_bm(b) + WORDS; };  // K x threads words when PRE
  auto buf_val = [&](int b) {
    return reinterpret_cast<T*>(buf_pre(b) + (C::PRE ? (size_t)K * kEncConsumers : 0));
  };
  auto buf_wpre = [&](int b) {
    return reinterpret_cast<uint16_t*>(buf_val(b) + (size_t)K * kEncConsumers);
  };
  auto buf_idx = [&](int b) { return buf_wpre(b) + WORDS; };
  StageMeta* meta = reinterpret_cast<StageMeta*>(bufs + NB * C::kBufBytes);  // [kRing]
  StageMeta* tinfo = meta + kRing;                                          // [NB]
  unsigned long long* s_prefix = reinterpret_cast<unsigned long long*>(tinfo + NB);  // [NB]
  uint64_t* full = reinterpret_cast<uint64_t*>(s_prefix + NB);              // [kRing]
  uint64_t* empty = full + kRing;                                           // [kRing]
  uint64_t* resolved = empty + kRing;                                       // [NB]
  uint32_t* s_ovf = reinterpret_cast<uint32_t*>(resolved + NB);             // [NB][NCW]
  uint32_t* s_tcnt = s_ovf + NB * NCW;                                      // [NB] count-only
  uint32_t* s_acks = s_tcnt + NB;                                           // remote acks seen
  using SpillRec = typename C::SpillRec;
  SpillRec* spill_blk = reinterpret_cast<SpillRec*>(a.spill) +
                        (size_t)blockIdx.x * NB * NCW * C::SPW;             // [NB][NCW][SPW]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.ntiles_dev && *a.ntiles_dev <= blockIdx.x) return;  // fixup pass: nothing for this block
  for (uint32_t i = tid; i < NB * WORDS; i += blockDim.x)
    buf_bm(i / WORDS)[i % WORDS] = 0;
  for (uint32_t i = tid; i < NB * NCW + NB + 1; i += blockDim.x) s_ovf[i] = 0;
  if (tid == 0) {
    for (int k = 0; k < kRing; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], NCW);
    }
    for (int b = 0; b < NB; ++b) mbar_init(&resolved[b], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const T* prevT = reinterpret_cast<const T*>(a.prev);
  const T* nextT = reinterpret_cast<const T*>(a.next);
  // streamed apply of a super-tile: its segment is fused with SA (fuse_on 2)
  // through an identity route whose keep window holds the whole super-tile,
  // and whose serving sub-tiles are 16-byte aligned; returns the serving
  // element of in-tile index 0, or null
  auto sa_dst = [&](uint32_t s, uint64_t e0, uint32_t cnt) -> T* {
    if (!SA || !a.fuse || a.fuse_on[s] != 2u) return nullptr;
    const FuseEntry* f = a.fuse + s;
    if (f->mode != 1 || e0 < f->keep_lo || e0 + cnt > f->keep_hi || (cnt % VE)) return nullptr;
    const int64_t off = (int64_t)f->dst_base + f->shift;
    if (off & (VE - 1)) return nullptr;
    return reinterpret_cast<T*>(a.serve) + off + e0;
  };

  if (warp == NCW) {
    // ---------------- producer ----------------
    if (lane == 0) {
      uint32_t ebits = (1u << kRing) - 1u;  // the first wait on each empty barrier passes
      const uint64_t pol = policy_evict_first();
      // fused remote emission: the receivers must have consumed last step's
      // records before this step's reach their regions.  Polled between
      // super-tiles (never blocking the stream); emitting warps wait on the flag.
      uint32_t pending = REMOTE ? a.remote.ack_mask : 0u;
      auto poll_acks = [&] {
        for (uint32_t m = pending; m; m &= m - 1) {
          const int q = __ffs(m) - 1;
          if (ld_acquire_sys(a.remote.ack + q) >= a.remote.epoch - 1) pending &= ~(1u << q);
        }
        if (!pending) st_release_cta_u32(s_acks, 1u);
      };
      if (!REMOTE) *s_acks = 1u;
      // waiting for a free stage keeps polling the acks: emitting consumers
      // hold their stages until the flag is up
      auto wait_empty = [&](int kk) {
        while (pending) {
          if (mbar_try_wait(&empty[kk], (ebits >> kk) & 1u)) return;
          poll_acks();
        }
        mbar_wait(&empty[kk], (ebits >> kk) & 1u);
      };
      int k = 0;
      while (true) {
        // Claimed only when the ring can take it: claiming further ahead
        // delays this super-tile's count and lengthens every look-back
        // (measured: 4.29 -> 3.46 TB/s with one-ahead claiming).
        if (pending) poll_acks();
        const uint32_t tk = atomicAdd(a.ticket, 1u);
        if (tk >= (a.ntiles_dev ? *a.ntiles_dev : a.ntiles)) {
          while (pending) poll_acks();
          wait_empty(k);
          meta[k].t = END;
          mbar_arrive(&full[k]);
          break;
        }
        const uint32_t t = a.tile_list ? __ldg(a.tile_list + tk) : tk + a.tile_offset;
        const int s = a.tile_seg ? (int)__ldg(a.tile_seg + t)
                                 : (a.tile0 ? find_segment(a.tile0, a.nseg, t) : 0);
        const SegDev sg = a.segs ? a.segs[s] : a.seg0;
        const uint32_t lt = a.tile0 ? t - __ldg(a.tile0 + s) : t;
        const uint64_t e0 = (uint64_t)lt * SUPER;
        const uint64_t rem_n = sg.n - e0;
        const uint32_t cnt = rem_n < SUPER ? (uint32_t)rem_n : SUPER;
        const uint32_t nsub = (cnt + SUB - 1) / SUB;
        const uint32_t last = (a.tile0 ? __ldg(a.tile0 + s + 1) : a.ntiles) == t + 1;
        const uint32_t count_only = a.seg_mode ? __ldg(a.seg_mode + s) : 0u;
        const T* sv = count_only ? nullptr : sa_dst((uint32_t)s, e0, cnt);
        for (uint32_t g = 0; g < nsub; ++g) {
          wait_empty(k);
          ebits ^= 1u << k;
          StageMeta& m = meta[k];
          m.sg = sg;
          m.t = t;
          m.s = (uint32_t)s;
          m.lt = lt;
          m.nsub = nsub;
          m.cnt = cnt;
          m.last = last;
          m.count_only = count_only;
          m.sa = sv != nullptr;
          const uint32_t sub_cnt = min(SUB, cnt - g * SUB);
          const uint32_t bytes = (sub_cnt / VE) * 16u;
          mbar_arrive_expect_tx(&full[k], (sv ? 3 : 2) * bytes);
          if (bytes) {
            const uint64_t el = sg.base + e0 + (uint64_t)g * SUB;
            if (WS_ENC_EVICT) {
              tma_load_1d_hint(ring_prev + k * kStageBytes, prevT + el, bytes, &full[k], pol);
              tma_load_1d_hint(ring_next + k * kStageBytes, nextT + el, bytes, &full[k], pol);
            } else {
              tma_load_1d(ring_prev + k * kStageBytes, prevT + el, bytes, &full[k]);
              tma_load_1d(ring_next + k * kStageBytes, nextT + el, bytes, &full[k]);
            }
            if (SA && sv)
              tma_load_1d(ring_serve + k * kStageBytes, sv + (uint64_t)g * SUB, bytes, &full[k]);
          }
          k = (k + 1) % kRing;
        }
      }
    }
    return;
  }

  if (warp > NCW) {
    // ---------------- resolvers: warp NCW+1+b owns staging buffer b ----------------
    const int b = warp - NCW - 1;
    while (true) {
      // blocked in hardware (no polling) until the 16 consumer warps arrive
      named_barrier(kStagedBar + b, kEncConsumers + 32);
      const StageMeta ti = tinfo[b];
      if (ti.t == END) break;
      resolve_tile<DT>(a, ti, buf_bm(b), buf_wpre(b), &s_prefix[b], s_tcnt + b);
      __syncwarp();
      if (lane == 0) mbar_arrive(&resolved[b]);
    }
    return;
  }

  // ---------------- consumers (warps 0..15) ----------------
  if (blockIdx.x == 0 && a.segs) {  // empty segments have no tile
    for (int s = tid; s < a.nseg; s += kEncConsumers)
      if (a.segs[s].n == 0) a.seg_nnz[s] = 0;
  }
  // Super-tile i is staged in buffer i % NB and written out after super-tile
  // i + NB - 1 is staged, so its placement has NB - 1 periods to complete.
  static_assert(NB == 2 || NB == 3, "one or two pending super-tiles are kept in registers");
  auto flush_tile = [&](int pb, const PendingSlice& p, uint32_t& rbits, bool drain) {
    if (C::PRE) {  // this super-tile's serving words are in (the two later groups may not be)
      if (drain) cp_async_wait<0>(); else cp_async_wait<NB - 1>();
      __syncwarp();
    }
    mbar_wait(&resolved[pb], (rbits >> pb) & 1u);
    rbits ^= 1u << pb;
    flush_slice<DT, REMOTE, SA>(a, p, s_prefix[pb], buf_bm(pb), buf_wpre(pb), buf_idx(pb), buf_val(pb),
                    buf_pre(pb), s_ovf + pb * NCW + warp,
                    spill_blk + ((size_t)pb * NCW + warp) * C::SPW, s_acks);
  };
  PendingSlice pend0{}, pend1{};  // super-tiles i-2 and i-1 of this thread
  const uint64_t pol_keep = policy_evict_last();
  uint32_t fbits = 0, rbits = 0;
  int k = 0;
  uint32_t i = 0;
  for (;; ++i) {
    const int b = (int)(i % NB);
    mbar_wait(&full[k], (fbits >> k) & 1u);
    if (meta[k].t == END) break;
    const StageMeta ti = meta[k];
    const uint64_t e0 = (uint64_t)ti.lt * SUPER;
    uint32_t* bm = buf_bm(b);
    T* sval = buf_val(b) + tid;
    uint16_t* sidx = buf_idx(b) + tid;
    uint32_t* spre = buf_pre(b) + tid;
    uint32_t mine = 0;  // this thread's changes in this super-tile
    const T* pf = nullptr;  // fused identity segment: serving element of in-tile index 0
    uint32_t pf_lo = 0, pf_n = 0;
    T* sa_out = nullptr;  // streamed apply: serving element of in-tile index 0
    if (SA && ti.sa) {
      const FuseEntry* f = a.fuse + ti.s;
      sa_out = reinterpret_cast<T*>(a.serve) + ((int64_t)f->dst_base + f->shift) + e0;
    } else if (C::PRE && a.fuse && a.fuse_on[ti.s]) {
      const FuseEntry* f = a.fuse + ti.s;
      if (f->mode == 1) {
        pf = reinterpret_cast<const T*>(a.serve) + ((int64_t)f->dst_base + f->shift) + e0;
        pf_lo = f->keep_lo > e0 ? (uint32_t)(f->keep_lo - e0) : 0u;
        pf_n = f->keep_hi > e0 + pf_lo ? (uint32_t)(f->keep_hi - e0 - pf_lo) : 0u;
      }
    }
#pragma unroll 1
    for (int g = 0; g < (int)ti.nsub; ++g) {
      const int kk = (k + g) % kRing;
      if (g > 0) mbar_wait(&full[kk], (fbits >> kk) & 1u);
      fbits ^= 1u << kk;
      const uint32_t sub_cnt = min(SUB, ti.cnt - g * SUB);
      const uint32_t nvec = sub_cnt / VE;
      const uint4* P = reinterpret_cast<const uint4*>(ring_prev + kk * kStageBytes);
      const uint4* N = reinterpret_cast<const uint4*>(ring_next + kk * kStageBytes);
      const uint4* S = reinterpret_cast<const uint4*>(ring_serve + kk * kStageBytes);
#pragma unroll
      for (uint32_t v = 0; v < VPT; ++v) {
        const uint32_t j = v * kEncConsumers + tid;
        uint4 pa, pb;
        uint32_t mv = 0;
        if (j < nvec) {
          pa = P[j];
          pb = N[j];
          if ((pa.x ^ pb.x) | (pa.y ^ pb.y) | (pa.z ^ pb.z) | (pa.w ^ pb.w) || DT == WS_F32)
            mv = change_mask<DT>(pa, pb);
        } else if (j == nvec && (sub_cnt % VE)) {  // ragged tail from global memory
          const uint64_t el = ti.sg.base + e0 + (uint64_t)g * SUB + j * VE;
          T ta[VE], tb[VE];
          for (int e = 0; e < VE; ++e) {
            const bool in = (uint32_t)e < sub_cnt % VE;
            ta[e] = in ? prevT[el + e] : T(0);
            tb[e] = in ? nextT[el + e] : T(0);
            if (in && Tr::changed(ta[e], tb[e])) mv |= 1u << e;
          }
          memcpy(&pa, ta, 16);
          memcpy(&pb, tb, 16);
        }
        if (ti.count_only) {
          mine += __popc(mv);
        } else if (mv) {
          if (SA && sa_out) {  // the whole vector: unchanged lanes add 0 (u16 wrap)
            const uint4 so = S[j];
            uint4 o;
            o.x = __vadd2(so.x, __vsub2(pb.x, pa.x));
            o.y = __vadd2(so.y, __vsub2(pb.y, pa.y));
            o.z = __vadd2(so.z, __vsub2(pb.z, pa.z));
            o.w = __vadd2(so.w, __vsub2(pb.w, pa.w));
            *reinterpret_cast<uint4*>(sa_out + g * SUB + j * VE) = o;
          }
          const uint32_t li = g * SUB + j * VE;
          atomicOr(bm + (li >> 5), mv << (li & 31));
          const T* Pe = reinterpret_cast<const T*>(P) + (size_t)j * VE;
          const T* Ne = reinterpret_cast<const T*>(N) + (size_t)j * VE;
          do {
            const int e = __ffs(mv) - 1;
            mv &= mv - 1;
            const T dv = j < nvec ? Tr::delta(Pe[e], Ne[e])
                                  : Tr::delta(Tr::get(pa, e), Tr::get(pb, e));
            if (mine >= (uint32_t)K) {  // past the slots: this warp's spill region
              const uint32_t o = atomicAdd(s_ovf + b * NCW + warp, 1u);
              SpillRec* sp = spill_blk + ((size_t)b * NCW + warp) * C::SPW + o;
              if constexpr (sizeof(T) == 2) *sp = (uint32_t)(li + e) | ((uint32_t)dv << 16);
              else *sp = make_uint2(li + e, (uint32_t)dv);
            } else {
              sidx[mine * kEncConsumers] = (uint16_t)(li + e);
              if (C::PRE && pf && li + e - pf_lo < pf_n) {
                const void* src = reinterpret_cast<const void*>(
                    reinterpret_cast<uintptr_t>(pf + li + e) & ~uintptr_t(3));
                if (WS_ENC_EVICT) cp_async4_hint(spre + mine * kEncConsumers, src, pol_keep);
                else cp_async4(spre + mine * kEncConsumers, src);
              }
              sval[mine * kEncConsumers] = dv;
            }
            ++mine;
          } while (mv);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[kk]);  // this warp is done with the stage
    }
    k = (k + ti.nsub) % kRing;
    if (ti.count_only) {  // publish the warp's count; nothing to write out later
      uint32_t w = mine;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(kFullMask, w, o);
      if (lane == 0 && w) atomicAdd(s_tcnt + b, w);
      mine = 0;
    }
    if (C::PRE) cp_async_commit();  // one group per super-tile
    if (tid == 0) tinfo[b] = ti;  // for the resolver only
    __syncwarp();
    named_arrive(kStagedBar + b, kEncConsumers + 32);
    const PendingSlice cur{ti.sg.base, ti.sg.rec, ti.sg.cap, ti.lt,  ti.nsub,
                           ti.cnt,     ti.s,      mine,      ti.sa};
    if constexpr (NB == 3) {
      if (i >= 2) flush_tile((int)((i - 2) % NB), pend0, rbits, false);  // super-tile i-2
      pend0 = pend1;
      pend1 = cur;
    } else {
      if (i >= 1) flush_tile((int)((i - 1) % NB), pend1, rbits, false);  // super-tile i-1
      pend1 = cur;
    }
  }
  // ---- drain: write out the pending super-tiles, then stop the resolvers
  if (NB == 3 && i >= 2) flush_tile((int)((i - 2) % NB), pend0, rbits, true);
  if (i >= 1) flush_tile((int)((i - 1) % NB), pend1, rbits, true);
  named_barrier(1, kEncConsumers);  // every warp is past its last use of tinfo
  if (tid == 0)
    for (int b = 0; b < NB; ++b) tinfo[b].t = END;
  __syncwarp();
  for (int b = 0; b < NB; ++b) named_arrive(kStagedBar + b, kEncConsumers + 32);
}

// ---- compaction of an unordered K1 output ---------------------------------------

// Exclusive scan of the super-tile record counts of one segment (one block;
// a segment has at most a few tens of thousands of super-tiles).
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* tile_cnt,
                                                         uint32_t ntiles, uint32_t* out_off) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t t0 = 0; t0 < ntiles; t0 += 1024) {
    const uint32_t c = t0 + tid < ntiles ? tile_cnt[t0 + tid] : 0u;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFullMask, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = s_warp[lane];
      uint32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[lane] = wi - w;
    }
    __syncthreads();
    const uint32_t carry = s_carry;
    if (t0 + tid < ntiles) out_off[t0 + tid] = carry + s_warp[warp] + inc - c;
    __syncthreads();
    if (tid == 1023) s_carry = carry + s_warp[31] + inc;
    __syncthreads();
  }
}

// One warp per super-tile: its records, ascending inside the tile, move to
// their place in the segment's ascending stream (positions >= cap dropped).
template <typename T>
__global__ void __launch_bounds__(256) compact_kernel(const uint32_t* tile_cnt,
                                                      const uint32_t* tile_base,
                                                      const uint32_t* out_off, uint32_t ntiles,
                                                      uint64_t cap, const uint32_t* in_idx,
                                                      const T* in_val, uint32_t* out_idx,
                                                      T* out_val) {
  const int lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles; t += nw) {
    const uint32_t n = tile_cnt[t];
    const uint64_t b = tile_base[t], o = out_off[t];
    for (uint32_t k = lane; k < n; k += 32)
      if (b + k < cap && o + k < cap) {
        out_idx[o + k] = in_idx[b + k];
        out_val[o + k] = in_val[b + k];
      }
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
                           uint64_t n, uint64_t change_thr, const uint64_t* thr_dim0,
                           uint16_t* prev, uint16_t* next) {
  const uint64_t fs[4] = {full_strides0, full_strides1, full_strides2, full_strides3};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t rem = i, g = 0, c0 = 0;
    for (int d = (int)full_ext_nd - 1; d >= 0; --d) {
      const uint64_t c = rem % box.ext[d] + box.lo[d];
      rem /= box.ext[d];
      g += c * fs[d];
      c0 = c;
    }
    uint16_t p, q;
    gen_elem_bf16(key, g, thr_dim0 ? thr_dim0[c0] : change_thr, p, q);
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

__global__ void fixup_plan_kernel(const uint32_t* tile0, int seg_begin, int seg_end,
                                  const uint64_t* seg_nnz, const uint64_t* seg_cap,
                                  uint32_t* seg_mode, uint32_t* tile_list, uint32_t* ntiles_dev) {
  __shared__ uint32_t s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  for (int s = seg_begin + threadIdx.x; s < seg_end; s += blockDim.x) {
    const bool dense = seg_nnz[s] > seg_cap[s];
    if (seg_mode[s] && !dense) {  // counted only, but sparse after all: list its tiles
      const uint32_t t0 = tile0[s], nt = tile0[s + 1] - t0;
      const uint32_t o = atomicAdd(&s_n, nt);
      for (uint32_t k = 0; k < nt; ++k) tile_list[o + k] = t0 + k;
    }
    seg_mode[s] = dense ? 1u : 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ntiles_dev = s_n;
}

cudaError_t launch_fixup_plan(const uint32_t* tile0, int seg_begin, int seg_end,
                              const uint64_t* seg_nnz, const uint64_t* seg_cap, uint32_t* seg_mode,
                              uint32_t* tile_list, uint32_t* ntiles_dev, cudaStream_t s) {
  fixup_plan_kernel<<<1, 256, 0, s>>>(tile0, seg_begin, seg_end, seg_nnz, seg_cap, seg_mode,
                                      tile_list, ntiles_dev);
  return cudaGetLastError();
}

size_t encode_spill_bytes(int dtype, uint32_t blocks) {
  size_t per = 0;
  switch (dtype) {
    case WS_BF16: per = sizeof(EncCfg<WS_BF16>::SpillRec) * EncCfg<WS_BF16>::SPW; break;
    case WS_I32: per = sizeof(EncCfg<WS_I32>::SpillRec) * EncCfg<WS_I32>::SPW; break;
    default: per = sizeof(EncCfg<WS_F32>::SpillRec) * EncCfg<WS_F32>::SPW; break;
  }
  return per * kEncBuffers * (kEncConsumers / 32) * blocks;
}

cudaError_t launch_encode(int dtype, const EncodeArgs& a, cudaStream_t s, int* grid_out) {
  // the shared-memory opt-in is a per-device function attribute (a process
  // may drive several GPUs: ws_group)
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_done.load() & bit)) {
    cudaFuncSetAttribute(encode_kernel<WS_BF16, false, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EncCfg<WS_BF16>::kSmem);
    cudaFuncSetAttribute(encode_kernel<WS_BF16, true, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EncCfg<WS_BF16>::kSmem);
    cudaFuncSetAttribute(encode_kernel<WS_BF16, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)EncCfg<WS_BF16, true>::kSmem);
    cudaFuncSetAttribute(encode_kernel<WS_I32, false, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EncCfg<WS_I32>::kSmem);
    cudaFuncSetAttribute(encode_kernel<WS_F32, false, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EncCfg<WS_F32>::kSmem);
    attr_done.fetch_or(bit);
  }
  // one persistent block per SM; the producer warp claims super-tiles in order
  int grid = (int)std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)sm_count(),
                                                           std::max(a.ntiles, 1u)));
  if (const char* g = ablation_env("WSYNC_ENCODE_GRID")) grid = std::max(1, atoi(g));
  if (a.max_grid) grid = std::min<int>(grid, (int)a.max_grid);
  if (!a.spill || a.spill_blocks == 0) return cudaErrorInvalidValue;
  grid = std::min<int>(grid, (int)a.spill_blocks);
  if (grid_out) *grid_out = grid;
  EncodeArgs a2 = a;
  if (const char* d = ablation_env("WSYNC_ENCODE_DEBUG")) a2.debug = (uint32_t)atoi(d);
  cudaError_t e = cudaMemsetAsync(a.ticket, 0, sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  switch (dtype) {
    case WS_BF16:
      if (a2.remote.maps)
        encode_kernel<WS_BF16, true, false>
            <<<grid, kEncodeBlock, EncCfg<WS_BF16>::kSmem, s>>>(a2);
      else if (a2.serve_stream && a2.fuse && a2.serve)
        encode_kernel<WS_BF16, false, true>
            <<<grid, kEncodeBlock, EncCfg<WS_BF16, true>::kSmem, s>>>(a2);
      else
        encode_kernel<WS_BF16, false, false>
            <<<grid, kEncodeBlock, EncCfg<WS_BF16>::kSmem, s>>>(a2);
      break;
    case WS_I32:
      encode_kernel<WS_I32, false, false><<<grid, kEncodeBlock, EncCfg<WS_I32>::kSmem, s>>>(a2);
      break;
    case WS_F32:
      encode_kernel<WS_F32, false, false><<<grid, kEncodeBlock, EncCfg<WS_F32>::kSmem, s>>>(a2);
      break;
    default: return cudaErrorInvalidValue;
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
  // count on the device and no bound given: a full grid (grid-stride loops)
  const int grid = (nnz_dev && nnz == 0) ? sm_count() * 8 : stream_grid(nnz, 256);
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
    m.div[i] = make_fastdiv(S.ext[i]);
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

void expert_thresholds(int experts, double density, double zipf_s, uint64_t perm_seed,
                       uint64_t* out) {
  // Zipf(s) weight of rank r (1-based), normalised to mean 1
  std::vector<double> w(experts);
  double sum = 0;
  for (int r = 0; r < experts; ++r) sum += (w[r] = std::pow((double)(r + 1), -zipf_s));
  // rank of every expert: a Fisher-Yates shuffle driven by splitmix64(perm_seed + k)
  std::vector<int> rank(experts);
  for (int e = 0; e < experts; ++e) rank[e] = e;
  uint64_t st = perm_seed;
  for (int i = experts - 1; i > 0; --i) {
    st += 0x9e3779b97f4a7c15ull;
    uint64_t x = st;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    x ^= x >> 31;
    std::swap(rank[i], rank[x % (uint64_t)(i + 1)]);
  }
  for (int e = 0; e < experts; ++e) {
    double d = density * w[rank[e]] * experts / sum;
    d = d < 0 ? 0 : (d > 1 ? 1 : d);
    out[e] = (uint64_t)(d * 4294967296.0);
  }
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
                            uint64_t change_thr, uint16_t* prev, uint16_t* next, cudaStream_t s,
                            const uint64_t* thr_dim0) {
  const Box b = shard_box(full, nd, desc);
  uint64_t n = 1, fs[4] = {0, 0, 0, 0}, st = 1;
  for (int d = 0; d < nd; ++d) n *= b.ext[d];
  for (int d = nd - 1; d >= 0; --d) {
    fs[d] = st;
    st *= (uint64_t)full[d];
  }
  if (n == 0) return cudaSuccess;
  gen_kernel<<<stream_grid(n, 256), 256, 0, s>>>(key, b, (uint32_t)nd, fs[0], fs[1], fs[2], fs[3],
                                                 n, change_thr, thr_dim0, prev, next);
  return cudaGetLastError();
}

cudaError_t launch_compact(int dtype, const uint32_t* tile_cnt, const uint32_t* tile_base,
                           uint32_t ntiles, uint64_t cap, const uint32_t* in_idx,
                           const void* in_val, uint32_t* out_idx, void* out_val, cudaStream_t s) {
  if (!ntiles) return cudaSuccess;
  uint32_t* off = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&off), (size_t)ntiles * 4, s);
  if (e != cudaSuccess) return e;
  tile_scan_kernel<<<1, 1024, 0, s>>>(tile_cnt, ntiles, off);
  const int grid = (int)std::min<uint64_t>((ntiles + 7) / 8, (uint64_t)sm_count() * 8);
  if (dtype == WS_BF16)
    compact_kernel<uint16_t><<<grid, 256, 0, s>>>(tile_cnt, tile_base, off, ntiles, cap, in_idx,
                                                  (const uint16_t*)in_val, out_idx,
                                                  (uint16_t*)out_val);
  else
    compact_kernel<uint32_t><<<grid, 256, 0, s>>>(tile_cnt, tile_base, off, ntiles, cap, in_idx,
                                                  (const uint32_t*)in_val, out_idx,
                                                  (uint32_t*)out_val);
  e = cudaGetLastError();
  cudaFreeAsync(off, s);
  return e;
}

}  // namespace wsync
