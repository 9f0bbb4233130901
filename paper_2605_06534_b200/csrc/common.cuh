// common.cuh -- shared device helpers of libwsync (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "wsync.h"

namespace wsync {

constexpr unsigned kFullMask = 0xffffffffu;

// ---- dtype traits ---------------------------------------------------------
// BF16 and I32 compare bit patterns and use wrap-around arithmetic (the
// reference's exact-dtype rule, codec.cpp:52-61 / :80-91); F32 compares by
// value and uses IEEE round-to-nearest add/sub (codec.cpp:44-50 / :78).
template <int DT>
struct Traits;

template <>
struct Traits<WS_BF16> {
  using T = uint16_t;
  static constexpr int kVE = 8;  // elements per 16-byte vector
  __device__ __forceinline__ static bool changed(T a, T b) { return a != b; }
  __device__ __forceinline__ static T delta(T a, T b) { return (T)(b - a); }
  __device__ __forceinline__ static T add(T t, T v) { return (T)(t + v); }
  __device__ __forceinline__ static T get(const uint4& q, int e) {
    const uint32_t w = e < 2 ? q.x : e < 4 ? q.y : e < 6 ? q.z : q.w;
    return (T)((e & 1) ? (w >> 16) : (w & 0xffffu));
  }
};

template <>
struct Traits<WS_I32> {
  using T = uint32_t;
  static constexpr int kVE = 4;
  __device__ __forceinline__ static bool changed(T a, T b) { return a != b; }
  __device__ __forceinline__ static T delta(T a, T b) { return b - a; }
  __device__ __forceinline__ static T add(T t, T v) { return t + v; }
  __device__ __forceinline__ static T get(const uint4& q, int e) {
    return e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w;
  }
};

template <>
struct Traits<WS_F32> {
  using T = uint32_t;  // carried as raw bits
  static constexpr int kVE = 4;
  __device__ __forceinline__ static bool changed(T a, T b) {
    return !(__uint_as_float(a) == __uint_as_float(b));
  }
  __device__ __forceinline__ static T delta(T a, T b) {
    return __float_as_uint(__fsub_rn(__uint_as_float(b), __uint_as_float(a)));
  }
  __device__ __forceinline__ static T add(T t, T v) {
    return __float_as_uint(__fadd_rn(__uint_as_float(t), __uint_as_float(v)));
  }
  __device__ __forceinline__ static T get(const uint4& q, int e) {
    return e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w;
  }
};

// Change mask of the VE elements of one 16-byte vector pair.
template <int DT>
__device__ __forceinline__ uint32_t change_mask(const uint4& a, const uint4& b) {
  if constexpr (DT == WS_BF16) {
    // SWAR: bit 15 / 31 of t is set iff the low / high halfword of a^b is
    // nonzero; the eight flags are then gathered into bits 0..7.
    auto nz = [](uint32_t x) { return (((x & 0x7fff7fffu) + 0x7fff7fffu) | x) & 0x80008000u; };
    const uint32_t u = (nz(a.x ^ b.x) >> 15) | (nz(a.y ^ b.y) >> 13) | (nz(a.z ^ b.z) >> 11) |
                       (nz(a.w ^ b.w) >> 9);
    return (u | (u >> 15)) & 0xffu;
  } else {
    using Tr = Traits<DT>;
    return (Tr::changed(a.x, b.x) ? 1u : 0u) | (Tr::changed(a.y, b.y) ? 2u : 0u) |
           (Tr::changed(a.z, b.z) ? 4u : 0u) | (Tr::changed(a.w, b.w) ? 8u : 0u);
  }
}

// ---- memory helpers -------------------------------------------------------
// Streaming 128-bit load: read-once data, do not pollute L1.
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- mbarrier + 1-D TMA bulk copy (cp.async.bulk) ---------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in hardware until
// the phase completes (or ~0.5 ms passes) instead of re-issuing the probe.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 500000;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Pulls the sector holding `p` into L2 without blocking the warp.
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// Global -> shared bulk copy completing on `bar` (bytes multiple of 16).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Same, marking the source lines evict-first in L2 (read-once streams must not
// push out lines a kernel comes back to).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void named_barrier(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// 4-byte asynchronous global -> shared copy (completes per thread in groups).
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async4_hint(void* smem_dst, const void* gsrc, uint64_t policy) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Non-blocking arrival on a named barrier (the waiters use named_barrier).
__device__ __forceinline__ void named_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// ---- system-scope flags (peer GPUs over NVLink) -----------------------------
__device__ __forceinline__ uint32_t ld_acquire_cta_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Spins until *p >= want; false after ~`cycles` (a dead peer must not hang us).
__device__ __forceinline__ bool wait_geq_sys(const unsigned long long* p, unsigned long long want,
                                             long long cycles = 10ll * 2000000000ll) {
  const long long t0 = clock64();
  while (ld_acquire_sys(p) < want) {
    if (clock64() - t0 > cycles) return false;
    __nanosleep(64);
  }
  return true;
}

// ---- decoupled look-back status words ---------------------------------------
// status = epoch(30b) << 34 | flag(2b) << 32 | value(32b).  A word whose epoch
// differs from the launch's epoch is "not yet written"; the epoch advances
// per launch so the status array never needs clearing.
constexpr uint32_t kFlagAggregate = 1, kFlagPrefix = 2;

__device__ __forceinline__ unsigned long long make_status(uint32_t epoch, uint32_t flag,
                                                          uint32_t value) {
  return ((unsigned long long)(epoch & 0x3fffffffu) << 34) |
         ((unsigned long long)flag << 32) | value;
}

// Exclusive prefix of `tile` within its chain [first_tile, tile): executed by
// one full warp.  Every tile of the chain publishes its aggregate before
// looking back, and the chain head publishes an inclusive prefix, so the walk
// terminates.  Each lane inspects 4 predecessors, so one L2 round trip covers
// a window of 128 tiles (the walk's throughput bound is window / latency).
__device__ __forceinline__ uint32_t warp_lookback(const unsigned long long* status,
                                                  int64_t tile, int64_t first_tile,
                                                  uint32_t epoch) {
  constexpr int J = 4;
  const int lane = threadIdx.x & 31;
  const unsigned long long want = (unsigned long long)(epoch & 0x3fffffffu);
  uint32_t excl = 0;
  int64_t pos = tile - 1;
  while (true) {
    uint32_t flag[J], val[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int64_t my = pos - (int64_t)(lane * J + j);
      flag[j] = 0;
      val[j] = 0;
      if (my >= first_tile) {
        unsigned long long st = ld_relaxed_u64(status + my);
        while ((st >> 34) != want) {
          __nanosleep(32);
          st = ld_relaxed_u64(status + my);
        }
        flag[j] = (uint32_t)(st >> 32) & 3u;
        val[j] = (uint32_t)st;
      }
    }
    int jp = J;  // nearest predecessor of this lane holding an inclusive prefix
#pragma unroll
    for (int j = J - 1; j >= 0; --j)
      if (flag[j] == kFlagPrefix) jp = j;
    const unsigned pmask = __ballot_sync(kFullMask, jp < J);
    const int stop = pmask ? __ffs(pmask) - 1 : 32;
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (lane < stop || (lane == stop && j <= jp)) c += val[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFullMask, c, o);
    excl += c;
    if (pmask) break;
    pos -= 32 * J;
  }
  return excl;
}

// ---- geometry: shard boxes -------------------------------------------------
struct Box {
  int32_t nd;
  uint32_t lo[WS_MAX_DIMS];
  uint32_t ext[WS_MAX_DIMS];
};

// Unsigned 32-bit division by a run-time constant as a multiply-high and
// shifts (round-up method): q = (t + ((n - t) >> 1)) >> (l - 1), t =
// mulhi(m, n), l = ceil(log2 d), m = 2^32 (2^l - d) / d + 1; exact for every
// 32-bit n.  The reslice's per-record coordinate split would otherwise pay
// two hardware-less integer divisions per dimension.
struct FastDiv {
  uint32_t d, m, l;  // l == 0: d == 1
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d <= 1) return f;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.l = l;
  f.m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  return f;
}
__device__ __forceinline__ uint32_t fastdiv(const FastDiv& f, uint32_t n) {
  if (f.l == 0) return n;
  const uint32_t t = __umulhi(f.m, n);
  return (t + ((n - t) >> 1)) >> (f.l - 1);
}

// Source-local flat index -> destination-local flat index, or ~0ull when the
// element lies outside the destination box (codec.cpp:125-131 generalised).
struct Remap {
  int32_t nd;
  uint32_t src_ext[WS_MAX_DIMS];
  int64_t shift[WS_MAX_DIMS];   // src.lo - dst.lo
  uint32_t dst_ext[WS_MAX_DIMS];
  FastDiv div[WS_MAX_DIMS];     // by src_ext[d]
};

__device__ __forceinline__ unsigned long long remap_index(const Remap& m, uint32_t i) {
  uint32_t c[WS_MAX_DIMS];
  uint32_t rem = i;
#pragma unroll
  for (int d = WS_MAX_DIMS - 1; d >= 0; --d) {
    if (d < m.nd) {
      const uint32_t q = fastdiv(m.div[d], rem);
      c[d] = rem - q * m.src_ext[d];
      rem = q;
    }
  }
  unsigned long long di = 0;
#pragma unroll
  for (int d = 0; d < WS_MAX_DIMS; ++d) {
    if (d < m.nd) {
      const int64_t g = (int64_t)c[d] + m.shift[d];
      if (g < 0 || g >= (int64_t)m.dst_ext[d]) return ~0ull;
      di = di * m.dst_ext[d] + (unsigned long long)g;
    }
  }
  return di;
}

// ---- synthetic generator (oracle/wsync_oracle.c gen_elem) ------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ void gen_elem_bf16(uint64_t key, uint64_t g, uint64_t change_thr,
                                              uint16_t& p, uint16_t& n) {
  const uint64_t r0 = splitmix64(key + (2 * g) * 0x9e3779b97f4a7c15ull);
  const uint64_t r1 = splitmix64(key + (2 * g + 1) * 0x9e3779b97f4a7c15ull);
  const int32_t s = (int32_t)(r0 & 0xffff) + (int32_t)((r0 >> 16) & 0xffff) +
                    (int32_t)((r0 >> 32) & 0xffff) + (int32_t)(r0 >> 48) - 131070;
  const float v = __fmul_rn((float)s, 5.2858e-7f);
  uint32_t u = __float_as_uint(v);
  u += 0x7fffu + ((u >> 16) & 1u);
  const uint16_t pb = (uint16_t)(u >> 16);
  uint16_t nb = pb;
  if ((r1 >> 32) < change_thr) {
    const uint16_t m = (uint16_t)(1 + (r1 & 0xf));
    nb = ((r1 >> 4) & 1) ? (uint16_t)(pb - m) : (uint16_t)(pb + m);
  }
  p = pb;
  n = nb;
}

}  // namespace wsync

// ---- ablation switches --------------------------------------------------------
// The measurements DESIGN.md quotes turned individual mechanisms off through
// environment variables.  They are read only by the ablation build (make
// ABLATIONS=1 -> lib/libwsync_ablate.so, loaded with WSYNC_LIB); the
// product library always runs the measured-best configuration.
#include <cstdlib>
namespace wsync {
inline const char* ablation_env(const char* name) {
#ifdef WSYNC_ABLATIONS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}
}  // namespace wsync
