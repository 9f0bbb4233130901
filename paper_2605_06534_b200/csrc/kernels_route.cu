// kernels_route.cu -- K3/K4 on the serving side of the engine.
//
// After K1 every trainer segment's delta stream (or, above the density
// threshold, its dense `next` snapshot) must land in each serving shard it
// intersects.  For destinations on the same GPU this is done here without
// materialising resliced streams: a tiny single-block kernel turns the
// per-segment record counts into a work list (records in chunks for sparse
// segments, row runs for dense ones), and one persistent kernel walks it,
// re-indexing each record into the destination shard (codec.cpp:125-131,
// box-generalised) and applying it in place (codec.cpp:80-91), or copying
// the dense overlap (shard.cpp:161-168).
#include <algorithm>

#include "route.h"

namespace wsync {

namespace {

constexpr int kWlThreads = 1024;
constexpr int kCopyIlp = 4;  // dense box copies: 16-byte vectors per thread in flight

__device__ __forceinline__ bool seg_dense(const RouteSideArgs& a, int seg) {
  return !a.sparse || a.seg_nnz[seg] > a.seg_cap[seg];
}

// K1 applied entry e's records as it wrote them (the segment's only local
// route, fused this sync)
__device__ __forceinline__ bool entry_fused(const RouteSideArgs& a, const LocalEntry& e) {
  return a.fused && e.fused_ok && a.fuse_on[e.seg];
}

// sparse, not fused, and dense enough to apply by streaming (local routes)
__device__ __forceinline__ bool entry_stream(const RouteSideArgs& a, const LocalEntry& e) {
  return a.stream_apply && !entry_fused(a, e) &&
         a.seg_nnz[e.seg] * kStreamDiv > a.segs[e.seg].n;
}

// Super-tiles [*ta, *tb) of an entry's segment that can hold records for it:
// an identity route only reads its keep window.
__device__ __forceinline__ void entry_tiles(const RouteSideArgs& a, const LocalEntry& e,
                                            uint32_t* ta, uint32_t* tb) {
  const uint32_t nt = a.tile0[e.seg + 1] - a.tile0[e.seg];
  if (e.identity) {
    *ta = e.keep_lo / a.tile_elems;
    const uint32_t hi = (uint32_t)(((uint64_t)e.keep_hi + a.tile_elems - 1) / a.tile_elems);
    *tb = hi < nt ? hi : nt;
    if (*ta > *tb) *ta = *tb;
  } else {
    *ta = 0;
    *tb = nt;
  }
}

// Units of one entry: groups of kTilesPerUnit super-tiles of records
// (sparse) or row-run chunks (dense).
__device__ __forceinline__ uint64_t entry_units(const RouteSideArgs& a, const LocalEntry& e) {
  if (seg_dense(a, e.seg) || entry_stream(a, e)) {
    const uint64_t per_row = (e.box.run + kCopyChunk - 1) / kCopyChunk;
    return e.box.rows * per_row;
  }
  if (entry_fused(a, e)) return 0;  // K1 applied the sparse records as it wrote them
  if (a.k1_emitted) return 0;                  // K1 stored them into the receivers' regions
  if (a.seg_nnz[e.seg] == 0) return 0;
  uint32_t ta, tb;
  entry_tiles(a, e, &ta, &tb);
  return (tb - ta + kTilesPerUnit - 1) / kTilesPerUnit;
}

// Record range [*k0, *k1) (segment-stream positions) of the super-tile this
// warp owns in unit lu of entry E; empty when the unit has fewer tiles.
__device__ __forceinline__ void warp_tile_records(const RouteSideArgs& a, const LocalEntry& E,
                                                  uint64_t lu, int warp, uint64_t* k0,
                                                  uint64_t* k1) {
  uint32_t ta, tb;
  entry_tiles(a, E, &ta, &tb);
  const uint64_t t = ta + lu * kTilesPerUnit + (uint64_t)warp;
  *k0 = *k1 = 0;
  if (t >= tb) return;
  const uint32_t gt = a.tile0[E.seg] + (uint32_t)t;
  *k0 = a.tile_base[gt];
  *k1 = *k0 + a.tile_cnt[gt];
}

__global__ void __launch_bounds__(kWlThreads) worklist_kernel(RouteSideArgs a) {
  __shared__ uint64_t s_carry, s_sa[2];
  __shared__ uint64_t s_warp[kWlThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = s_sa[0] = s_sa[1] = 0;
  __syncthreads();
  for (int base = 0; base < a.nentries; base += kWlThreads) {
    const int e = base + tid;
    const uint64_t u = e < a.nentries ? entry_units(a, a.entries[e]) : 0;
    if (e < a.nentries && a.fused && a.entries[e].fused_ok) {
      // Next sync: fuse the apply into K1 only for segments that stayed well
      // below the dense threshold; the others skip the scattered
      // read-modify-writes of records a dense copy would overwrite anyway.
      // With K1's streamed apply (fuse_on = 2) the serving tile is read
      // sequentially, which beats the per-record RMW from 1/sa_div up to the
      // dense threshold.
      const int s = a.entries[e].seg;
      const uint64_t nz = a.seg_nnz[s], n = a.segs[s].n;
      // (only identity routes can stream the serving tile)
      const bool stream =
          a.sa_div && a.entries[e].identity && nz * a.sa_div >= n && nz <= a.seg_cap[s];
      const uint32_t on = stream ? 2u : (nz * kStreamDiv <= n ? 1u : 0u);
      a.fuse_on[s] = on;
      if (on && a.sa_elems)  // fused elements: [0] streamed, [1] per-record RMW
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sa[on == 2u ? 0 : 1]), n);
    }
    uint64_t inc = u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFullMask, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = s_warp[lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(kFullMask, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[lane] = wi - w;
    }
    __syncthreads();
    const uint64_t excl = s_carry + s_warp[warp] + inc - u;
    if (e < a.nentries) a.unit_off[e] = excl;
    __syncthreads();
    if (tid == kWlThreads - 1) s_carry = excl + u;
    __syncthreads();
  }
  if (tid == 0) {
    a.unit_off[a.nentries] = s_carry;
    // the host picks K1's instantiation for the next sync from this word
    if (a.fused && a.sa_elems) {
      reinterpret_cast<volatile uint64_t*>(a.sa_elems)[0] = s_sa[0];
      reinterpret_cast<volatile uint64_t*>(a.sa_elems)[1] = s_sa[1];
    }
  }
}

// Block-cooperative copy of one route entry into shared memory (the caller
// synchronises before use).
__device__ __forceinline__ void load_entry(LocalEntry* dst, const LocalEntry* src) {
  static_assert(sizeof(LocalEntry) % 4 == 0, "word copy");
  const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
  uint32_t* d = reinterpret_cast<uint32_t*>(dst);
  for (uint32_t w = threadIdx.x; w < sizeof(LocalEntry) / 4; w += blockDim.x) d[w] = __ldg(s + w);
}

__device__ __forceinline__ int find_entry(const uint64_t* off, int n, uint64_t u) {
  int lo = 0, hi = n;  // off[lo] <= u < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= u) lo = mid; else hi = mid;
  }
  return lo;
}

template <int DT>
__global__ void __launch_bounds__(256) local_apply_kernel(RouteSideArgs a) {
  using Tr = Traits<DT>;
  using T = typename Tr::T;
  __shared__ int s_entry;
  __shared__ uint64_t s_u0;
  __shared__ LocalEntry s_E;  // the unit's entry (read per record: kept on chip)
  int cur = -1;
  const uint64_t total = a.unit_off[a.nentries];
  T* serve = reinterpret_cast<T*>(a.serve);
  const T* val = reinterpret_cast<const T*>(a.rec_val);
  const T* next = reinterpret_cast<const T*>(a.train_next);
  for (uint64_t u = blockIdx.x; u < total; u += gridDim.x) {
    if (threadIdx.x == 0) {
      const int e = find_entry(a.unit_off, a.nentries, u);
      s_entry = e;
      s_u0 = a.unit_off[e];
    }
    __syncthreads();
    const int ei = s_entry;
    const uint64_t lu = u - s_u0;
    if (ei != cur) load_entry(&s_E, a.entries + ei), cur = ei;
    __syncthreads();
    const LocalEntry& E = s_E;
    const bool stream = !seg_dense(a, E.seg) && entry_stream(a, E);
    if (!seg_dense(a, E.seg) && !stream) {
      uint64_t k0, k1;
      warp_tile_records(a, E, lu, threadIdx.x >> 5, &k0, &k1);
      const uint64_t rec = a.seg_rec[E.seg];
      T* dst = serve + E.dst_base;
      const int lane = threadIdx.x & 31;
      if (E.identity) {
        for (uint64_t k = k0 + lane; k < k1; k += 32) {
          const uint32_t i = __ldg(a.rec_idx + rec + k);
          if (i < E.keep_lo || i >= E.keep_hi) continue;
          const uint64_t d = (uint64_t)((int64_t)i + E.shift);
          dst[d] = Tr::add(dst[d], __ldg(val + rec + k));
        }
      } else {
        for (uint64_t k = k0 + lane; k < k1; k += 32) {
          const uint64_t d = remap_index(E.map, __ldg(a.rec_idx + rec + k));
          if (d == ~0ull) continue;
          dst[d] = Tr::add(dst[d], __ldg(val + rec + k));
        }
      }
    } else {
      // dense fallback: copy one chunk of one row of the overlap
      const BoxCopyArgs& B = E.box;
      const uint64_t per_row = (B.run + kCopyChunk - 1) / kCopyChunk;
      const uint64_t row = lu / per_row, c0 = (lu % per_row) * kCopyChunk;
      const uint64_t c1 = min(B.run, c0 + kCopyChunk);
      uint64_t so = B.src_base, dso = B.dst_base, rem = row;
      for (int d = B.nd_outer - 1; d >= 0; --d) {
        const uint64_t c = rem % B.outer_ext[d];
        rem /= B.outer_ext[d];
        so += c * B.src_stride[d];
        dso += c * B.dst_stride[d];
      }
      const T* src = next + a.seg_base[E.seg] + so;
      T* dst = serve + E.dst_base + dso;
      if (stream) {  // serve += next - prev where changed (codec.cpp:80-91 over the box)
        const T* psrc = reinterpret_cast<const T*>(a.train_prev) + a.seg_base[E.seg] + so;
        if (B.vec) {
          constexpr int VE = Tr::kVE;
          const uint4* p4 = reinterpret_cast<const uint4*>(psrc + c0);
          const uint4* n4 = reinterpret_cast<const uint4*>(src + c0);
          uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
          for (uint64_t j = threadIdx.x; j < (c1 - c0) / VE; j += blockDim.x) {
            const uint4 pv = ld_stream(p4 + j), nv = ld_stream(n4 + j);
            if (!change_mask<DT>(pv, nv)) continue;
            uint4 sv = d4[j];
            T* se = reinterpret_cast<T*>(&sv);
            const T* pe = reinterpret_cast<const T*>(&pv);
            const T* ne = reinterpret_cast<const T*>(&nv);
#pragma unroll
            for (int e = 0; e < VE; ++e)
              if (Tr::changed(pe[e], ne[e])) se[e] = Tr::add(se[e], Tr::delta(pe[e], ne[e]));
            d4[j] = sv;
          }
        } else {
          for (uint64_t j = c0 + threadIdx.x; j < c1; j += blockDim.x)
            if (Tr::changed(psrc[j], src[j])) dst[j] = Tr::add(dst[j], Tr::delta(psrc[j], src[j]));
        }
      } else if (B.vec) {
        constexpr int VE = Tr::kVE;
        const uint4* s4 = reinterpret_cast<const uint4*>(src + c0);
        uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
        const uint64_t nv = (c1 - c0) / VE;
        for (uint64_t j0 = threadIdx.x; j0 < nv; j0 += (uint64_t)blockDim.x * kCopyIlp) {
          uint4 v[kCopyIlp];
#pragma unroll
          for (int q = 0; q < kCopyIlp; ++q) {
            const uint64_t j = j0 + (uint64_t)q * blockDim.x;
            if (j < nv) v[q] = ld_stream(s4 + j);
          }
#pragma unroll
          for (int q = 0; q < kCopyIlp; ++q) {
            const uint64_t j = j0 + (uint64_t)q * blockDim.x;
            if (j < nv) d4[j] = v[q];
          }
        }
      } else {
        for (uint64_t j = c0 + threadIdx.x; j < c1; j += blockDim.x) dst[j] = src[j];
      }
    }
  }
}

template <int DT>
__global__ void __launch_bounds__(256, 4) pack_kernel(PackArgs pa) {
  using Tr = Traits<DT>;
  using T = typename Tr::T;
  const RouteSideArgs& a = pa.r;
  __shared__ int s_entry;
  __shared__ uint64_t s_u0;
  __shared__ LocalEntry s_E;  // the unit's entry (read per record: kept on chip)
  int cur = -1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint64_t total = a.unit_off[a.nentries];
  const T* val = reinterpret_cast<const T*>(a.rec_val);
  const T* next = reinterpret_cast<const T*>(a.train_next);
  const P2PArgs& P = pa.p2p;
  const int W = P.world;
  if (P.on && threadIdx.x == 0) {
    // every destination must have consumed our previous step's records
    for (int c = 0; c < kMaxWorld; ++c)
      for (int r = 0; r < kMaxReplicas && P.dest_rank[c][r] >= 0; ++r)
        if (!wait_geq_sys(P.mailbox + mb_ack(W, P.round, P.dest_rank[c][r]), P.prev_epoch) ||
            (P.dense_direct &&
             !wait_geq_sys(P.mailbox + mb_ready(W, P.dest_rank[c][r]), P.epoch)))
          atomicOr(P.err, kErrBitTimeout);
  }
  __syncthreads();
  for (uint64_t u = blockIdx.x; u < total; u += gridDim.x) {
    if (threadIdx.x == 0) {
      const int e = find_entry(a.unit_off, a.nentries, u);
      s_entry = e;
      s_u0 = a.unit_off[e];
    }
    __syncthreads();
    const int ei = s_entry;  // s_entry is rewritten for the next unit after the barrier
    const uint64_t lu = u - s_u0;
    if (ei != cur) load_entry(&s_E, a.entries + ei), cur = ei;
    __syncthreads();
    const LocalEntry& E = s_E;
    const int c = E.coord;
    // P2P: this entry's own region at every replica; NCCL: the coordinate's send region
    const EntryDest* ED = P.on ? P.edest + ei : nullptr;
    const uint64_t roff = P.on ? 0 : pa.region_off[c], rcap = P.on ? ED->cap : pa.region_cap[c];
    // stores one record at `slot` of the entry's region
    auto put = [&](uint64_t slot, uint64_t idx, T v, bool set) {
      if (slot >= rcap) {
        atomicOr(pa.err, WS_ERRBIT_CAPACITY);
        return;
      }
      if (P.on) {
        // straight into every replica's receive region over NVLink: the
        // shard-local index and the value (SoA, p2p_record_bytes)
        const uint32_t li = (uint32_t)(idx - E.dst_base);
        for (int r = 0; r < kMaxReplicas && ED->rec[r]; ++r) {
          reinterpret_cast<uint32_t*>(ED->rec[r])[slot] = li;
          reinterpret_cast<T*>(reinterpret_cast<uint32_t*>(ED->rec[r]) + rcap)[slot] = v;
        }
      } else if constexpr (DT == WS_BF16) {
        const uint64_t w = (set ? kWireSet : 0ull) | (idx << 16) | (uint64_t)v;
        reinterpret_cast<uint64_t*>(pa.send)[roff + slot] = w;
      } else {
        ulonglong2 w;
        w.x = (set ? kWireSet : 0ull) | idx;
        w.y = (unsigned long long)v;
        reinterpret_cast<ulonglong2*>(pa.send)[roff + slot] = w;
      }
    };
    // emits one record per lane with `valid`, reserving slots warp-wide
    auto emit = [&](bool valid, uint64_t idx, T v, bool set) {
      const unsigned bal = __ballot_sync(kFullMask, valid);
      if (!bal) return;
      unsigned long long base = 0;
      if (lane == 0)
        base = P.on ? atomicAdd(P.ent_cnt + ei, (unsigned)__popc(bal))
                    : atomicAdd(pa.region_cnt + c, (unsigned long long)__popc(bal));
      base = __shfl_sync(kFullMask, base, 0);
      if (valid) put(base + __popc(bal & ((1u << lane) - 1u)), idx, v, set);
    };
    if (!seg_dense(a, E.seg)) {
      uint64_t k0, k1;
      warp_tile_records(a, E, lu, warp, &k0, &k1);
      if (P.debug & 2) k1 = k0;
      const uint64_t rec = a.seg_rec[E.seg];
      // kPackBatch x 32 records per pass: their loads are all in flight
      // before the first is used, and one atomic reserves all their slots
      constexpr int kPackBatch = 4;
      for (uint64_t kb = k0; kb < k1; kb += 32 * kPackBatch) {
        uint32_t ix[kPackBatch];
        T v[kPackBatch];
#pragma unroll
        for (int b = 0; b < kPackBatch; ++b) {
          const uint64_t k = kb + b * 32 + lane;
          ix[b] = k < k1 ? __ldg(a.rec_idx + rec + k) : 0u;
          v[b] = k < k1 ? __ldg(val + rec + k) : T(0);
        }
        uint64_t d[kPackBatch];
        unsigned bal[kPackBatch];
        uint32_t total = 0;
#pragma unroll
        for (int b = 0; b < kPackBatch; ++b) {
          const uint64_t k = kb + b * 32 + lane;
          bool valid = k < k1;
          if (E.identity) {
            valid = valid && ix[b] >= E.keep_lo && ix[b] < E.keep_hi;
            d[b] = (uint64_t)((int64_t)ix[b] + E.shift);
          } else {
            d[b] = valid ? remap_index(E.map, ix[b]) : ~0ull;
            valid = d[b] != ~0ull;
          }
          bal[b] = __ballot_sync(kFullMask, valid);
          total += __popc(bal[b]);
        }
        if (!total) continue;
        unsigned long long base = 0;
        if (lane == 0)
          base = P.on ? atomicAdd(P.ent_cnt + ei, total)
                      : atomicAdd(pa.region_cnt + c, (unsigned long long)total);
        base = __shfl_sync(kFullMask, base, 0);
#pragma unroll
        for (int b = 0; b < kPackBatch; ++b) {
          if ((bal[b] >> lane) & 1u) put(base + __popc(bal[b] & ((1u << lane) - 1u)),
                                         E.dst_base + d[b], v[b], false);
          base += __popc(bal[b]);
        }
      }
    } else {
      const BoxCopyArgs& B = E.box;
      const uint64_t per_row = (B.run + kCopyChunk - 1) / kCopyChunk;
      const uint64_t row = lu / per_row, c0 = (lu % per_row) * kCopyChunk;
      const uint64_t c1 = min(B.run, c0 + kCopyChunk);
      uint64_t so = B.src_base, dso = B.dst_base, rem = row;
      for (int d = B.nd_outer - 1; d >= 0; --d) {
        const uint64_t cc = rem % B.outer_ext[d];
        rem /= B.outer_ext[d];
        so += cc * B.src_stride[d];
        dso += cc * B.dst_stride[d];
      }
      const T* src = next + a.seg_base[E.seg] + so;
      if (P.on && P.dense_direct) {
        // peer stores into every replica's serving arena; the replicas share
        // dst offsets and 16-byte aligned bases, so one alignment test serves all
        const uint64_t dofs = E.dst_base + dso;
        int nrep = 0;
        while (nrep < kMaxReplicas && P.serve_dst[c][nrep]) ++nrep;
        const T* s0 = src + c0;
        const uint64_t n = c1 - c0;
        constexpr int V = 16 / sizeof(T);
        const uintptr_t sa = reinterpret_cast<uintptr_t>(s0);
        const uintptr_t da = (dofs + c0) * sizeof(T);
        uint64_t head = n, body = 0;
        if (((sa ^ da) & 15) == 0) {
          head = ((16 - (sa & 15)) & 15) / sizeof(T);
          if (head > n) head = n;
          body = (n - head) / V;
        }
        for (uint64_t j = threadIdx.x; j < head; j += blockDim.x)
          for (int r = 0; r < nrep; ++r)
            reinterpret_cast<T*>(P.serve_dst[c][r])[dofs + c0 + j] = s0[j];
        const uint4* sv = reinterpret_cast<const uint4*>(s0 + head);
        // kCopyIlp vectors per thread in flight before they are stored
        for (uint64_t j0 = threadIdx.x; j0 < body; j0 += (uint64_t)blockDim.x * kCopyIlp) {
          uint4 v[kCopyIlp];
#pragma unroll
          for (int q = 0; q < kCopyIlp; ++q) {
            const uint64_t j = j0 + (uint64_t)q * blockDim.x;
            if (j < body) v[q] = ld_stream(sv + j);
          }
          for (int r = 0; r < nrep; ++r) {
            uint4* d = reinterpret_cast<uint4*>(reinterpret_cast<T*>(P.serve_dst[c][r]) + dofs + c0 +
                                                head);
#pragma unroll
            for (int q = 0; q < kCopyIlp; ++q) {
              const uint64_t j = j0 + (uint64_t)q * blockDim.x;
              if (j < body) d[j] = v[q];
            }
          }
        }
        for (uint64_t j = head + body * V + threadIdx.x; j < n; j += blockDim.x)
          for (int r = 0; r < nrep; ++r)
            reinterpret_cast<T*>(P.serve_dst[c][r])[dofs + c0 + j] = s0[j];
        continue;
      }
      for (uint64_t jb = c0 + (uint64_t)warp * 32; jb < c1; jb += (uint64_t)nwarps * 32) {
        const uint64_t j = jb + lane;
        const bool valid = j < c1;
        emit(valid, E.dst_base + dso + j, valid ? src[j] : T(0), true);
      }
    }
  }
  if (P.on) {
    // The last block to finish publishes every entry's record count at each
    // replica (0 for a dense segment whose box went direct: records emitted
    // for it must not be applied) and then, after a system fence, this step's
    // flag, so the records are visible before the flag.
    __shared__ int s_last;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0)
      s_last = atomicAdd(P.mailbox + mb_pack_ctr(W, P.round), 1ull) == gridDim.x - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int e = threadIdx.x; e < a.nentries; e += blockDim.x) {
        const EntryDest& D = P.edest[e];
        const unsigned c0 = *reinterpret_cast<volatile unsigned*>(P.ent_cnt + e);
        const bool dense = seg_dense(a, a.entries[e].seg);
        // a dense box that went direct sends no records; one that did not
        // sent set records (count flagged)
        const uint32_t n = (P.dense_direct && dense)
                               ? 0u
                               : ((uint32_t)(c0 < D.cap ? c0 : D.cap) | (dense ? kCountSet : 0u));
        for (int r = 0; r < kMaxReplicas && D.rec[r]; ++r) st_relaxed_sys_u32(D.cnt[r], n);
      }
      __threadfence_system();
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int c = 0; c < kMaxWorld; ++c)
          for (int r = 0; r < kMaxReplicas && P.dest_rank[c][r] >= 0; ++r)
            st_release_sys(P.peer_mailbox[P.dest_rank[c][r]] + mb_flag(W, P.round, P.rank),
                           P.epoch);
        P.mailbox[mb_pack_ctr(W, P.round)] = 0;
      }
    }
  }
}

template <int DT>
__device__ __forceinline__ void decode_wire(const void* recv, uint64_t k, uint64_t* i,
                                            typename Traits<DT>::T* v, bool* set) {
  using T = typename Traits<DT>::T;
  uint64_t key;
  if constexpr (DT == WS_BF16) {
    const uint64_t w = __ldg(reinterpret_cast<const unsigned long long*>(recv) + k);
    key = (w & kWireSet) | ((w & ~kWireSet) >> 16);
    *v = (T)(w & 0xffffu);
  } else {
    const ulonglong2 w = __ldg(reinterpret_cast<const ulonglong2*>(recv) + k);
    key = w.x;
    *v = (T)w.y;
  }
  *i = key & ~kWireSet;
  *set = (key & kWireSet) != 0;
}

// Applies the records at positions pos(k) for this thread's k = k0 + j *
// stride (j < AB) of [0, total): all serving-element loads of the batch are
// issued before any store, so a thread keeps AB scattered reads in flight.
constexpr int kApplyBatch = 4;
template <int DT, typename Pos>
__device__ __forceinline__ void apply_records(const void* recv, uint64_t total, Pos pos,
                                              typename Traits<DT>::T* serve) {
  using Tr = Traits<DT>;
  using T = typename Tr::T;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k0 < total;
       k0 += stride * kApplyBatch) {
    uint64_t ix[kApplyBatch];
    T v[kApplyBatch], o[kApplyBatch];
    bool ok[kApplyBatch], st[kApplyBatch];
#pragma unroll
    for (int j = 0; j < kApplyBatch; ++j) {
      const uint64_t k = k0 + j * stride;
      ok[j] = k < total;
      if (ok[j]) decode_wire<DT>(recv, pos(k), &ix[j], &v[j], &st[j]);
    }
#pragma unroll
    for (int j = 0; j < kApplyBatch; ++j)
      if (ok[j] && !st[j]) o[j] = serve[ix[j]];
#pragma unroll
    for (int j = 0; j < kApplyBatch; ++j)
      if (ok[j]) serve[ix[j]] = st[j] ? v[j] : Tr::add(o[j], v[j]);
  }
}

template <int DT>
__global__ void apply_wire_kernel(const void* recv, uint64_t nrec, typename Traits<DT>::T* serve) {
  apply_records<DT>(recv, nrec, [](uint64_t k) { return k; }, serve);
}

// P2P receiver: every block waits (on its own HBM) for the step flags of the
// expected sources, then the grid applies the records in the receive buffer
// (one contiguous region per source); the last block acks the sources so
// they may overwrite their regions next step.
__global__ void p2p_ready_kernel(P2PArgs P) {
  const int s = threadIdx.x;
  if (s < P.world && (P.expect_mask & (1u << s))) {
    __threadfence_system();
    st_release_sys(P.peer_mailbox[s] + mb_ready(P.world, P.rank), P.epoch);
  }
}

// P2P receiver, step 1 (one block): wait (acquire) for the step flag of
// every expected source, then turn the published per-entry counts into a
// prefix of apply units (kApplyUnit records each).
constexpr uint64_t kApplyUnit = 2048;
__global__ void __launch_bounds__(1024) p2p_recv_plan_kernel(P2PArgs P) {
  __shared__ uint64_t s_warp[32];
  __shared__ uint64_t s_carry;
  const int W = P.world, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < W && (P.expect_mask & (1u << tid)))
    if (!wait_geq_sys(P.mailbox + mb_flag(W, P.round, tid), P.epoch))
      atomicOr(P.err, kErrBitTimeout);
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < P.nrecv; base += 1024) {
    const int e = base + tid;
    const uint64_t u = e < P.nrecv
        ? ((uint64_t)(ld_acquire_sys_u32(P.recv_cnt + P.rentries[e].cnt_idx) & ~kCountSet) +
           kApplyUnit - 1) / kApplyUnit
        : 0;
    uint64_t inc = u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFullMask, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const uint64_t w = s_warp[lane];
      uint64_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(kFullMask, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[lane] = wi - w;
    }
    __syncthreads();
    const uint64_t excl = s_carry + s_warp[warp] + inc - u;
    if (e < P.nrecv) P.recv_units[e] = excl;
    __syncthreads();
    if (tid == 1023) s_carry = excl + u;
    __syncthreads();
  }
  if (tid == 0) P.recv_units[P.nrecv] = s_carry;
}

// Step 2: the grid applies unit after unit (one region slice each), then the
// last block acks the sources so they may refill their regions next step.
template <int DT>
__global__ void __launch_bounds__(256, 8) apply_p2p_kernel(P2PArgs P, typename Traits<DT>::T* serve) {
  const int W = P.world;
  using Tr = Traits<DT>;
  using T = typename Tr::T;
  __shared__ const uint32_t* s_idx;
  __shared__ const T* s_val;
  __shared__ T* s_dst;
  __shared__ uint32_t s_k0, s_k1, s_set;
  const uint64_t total = (P.debug & 1) ? 0 : P.recv_units[P.nrecv];
  for (uint64_t u = blockIdx.x; u < total; u += gridDim.x) {
    if (threadIdx.x == 0) {
      const int e = find_entry(P.recv_units, P.nrecv, u);
      const RecvEntry R = P.rentries[e];
      const uint32_t c = P.recv_cnt[R.cnt_idx];
      const uint64_t n = c & ~kCountSet;
      const uint64_t lo = (u - P.recv_units[e]) * kApplyUnit;
      const uint32_t* region =
          reinterpret_cast<const uint32_t*>(static_cast<const char*>(P.recv) + R.off);
      s_idx = region;
      s_val = reinterpret_cast<const T*>(region + R.cap);
      s_dst = serve + R.dst_base;
      s_set = (c & kCountSet) ? 1u : 0u;
      s_k0 = (uint32_t)lo;
      s_k1 = (uint32_t)(n < lo + kApplyUnit ? n : lo + kApplyUnit);
    }
    __syncthreads();
    const uint32_t* idx = s_idx;
    const T* val = s_val;
    T* dst = s_dst;
    const uint32_t k0 = s_k0, k1 = s_k1;
    const bool set = s_set != 0;
    __syncthreads();
    // block-local strided apply of [k0, k1): every serving-word load of a
    // batch is issued before any store
    for (uint32_t kb = k0 + threadIdx.x; kb < k1; kb += blockDim.x * kApplyBatch) {
      uint32_t ix[kApplyBatch];
      T v[kApplyBatch], o[kApplyBatch];
      bool ok[kApplyBatch];
#pragma unroll
      for (int j = 0; j < kApplyBatch; ++j) {
        const uint32_t k = kb + j * blockDim.x;
        ok[j] = k < k1;
        if (ok[j]) {
          ix[j] = __ldg(idx + k);
          v[j] = __ldg(val + k);
        }
      }
      if (!set) {
#pragma unroll
        for (int j = 0; j < kApplyBatch; ++j)
          if (ok[j]) o[j] = dst[ix[j]];
      }
#pragma unroll
      for (int j = 0; j < kApplyBatch; ++j)
        if (ok[j]) dst[ix[j]] = set ? v[j] : Tr::add(o[j], v[j]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long prev = atomicAdd(P.mailbox + mb_apply_ctr(W, P.round), 1ull);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      for (int s = 0; s < W; ++s)
        if (P.expect_mask & (1u << s))
          st_release_sys(P.peer_mailbox[s] + mb_ack(W, P.round, P.rank), P.epoch);
      P.mailbox[mb_apply_ctr(W, P.round)] = 0;
    }
  }
}

}  // namespace

cudaError_t launch_pack(int dtype, const PackArgs& a, int grid, cudaStream_t s) {
  if (a.r.nentries == 0) return cudaSuccess;
  worklist_kernel<<<1, kWlThreads, 0, s>>>(a.r);
  switch (dtype) {
    case WS_BF16: pack_kernel<WS_BF16><<<grid, 256, 0, s>>>(a); break;
    case WS_I32: pack_kernel<WS_I32><<<grid, 256, 0, s>>>(a); break;
    case WS_F32: pack_kernel<WS_F32><<<grid, 256, 0, s>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_p2p_ready(const P2PArgs& p, cudaStream_t s) {
  p2p_ready_kernel<<<1, 32, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_apply_p2p(int dtype, const P2PArgs& p, void* serve, int grid, cudaStream_t s) {
  p2p_recv_plan_kernel<<<1, 1024, 0, s>>>(p);
  switch (dtype) {
    case WS_BF16: apply_p2p_kernel<WS_BF16><<<grid, 256, 0, s>>>(p, (uint16_t*)serve); break;
    case WS_I32: apply_p2p_kernel<WS_I32><<<grid, 256, 0, s>>>(p, (uint32_t*)serve); break;
    case WS_F32: apply_p2p_kernel<WS_F32><<<grid, 256, 0, s>>>(p, (uint32_t*)serve); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_apply_wire(int dtype, const void* recv, uint64_t nrec, void* serve,
                             cudaStream_t s) {
  if (!nrec) return cudaSuccess;
  const int grid = (int)std::min<uint64_t>((nrec + 255) / 256, 148ull * 16);
  switch (dtype) {
    case WS_BF16: apply_wire_kernel<WS_BF16><<<grid, 256, 0, s>>>(recv, nrec, (uint16_t*)serve); break;
    case WS_I32: apply_wire_kernel<WS_I32><<<grid, 256, 0, s>>>(recv, nrec, (uint32_t*)serve); break;
    case WS_F32: apply_wire_kernel<WS_F32><<<grid, 256, 0, s>>>(recv, nrec, (uint32_t*)serve); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_local_route(int dtype, const RouteSideArgs& a, int grid, cudaStream_t s) {
  if (a.nentries == 0) return cudaSuccess;
  worklist_kernel<<<1, kWlThreads, 0, s>>>(a);
  switch (dtype) {
    case WS_BF16: local_apply_kernel<WS_BF16><<<grid, 256, 0, s>>>(a); break;
    case WS_I32: local_apply_kernel<WS_I32><<<grid, 256, 0, s>>>(a); break;
    case WS_F32: local_apply_kernel<WS_F32><<<grid, 256, 0, s>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace wsync
