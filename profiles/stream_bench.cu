// stream_bench.cu -- B200 read-streaming microbenchmark (design evidence for
// K1): plain 128-bit LDG streaming vs a 1-D TMA (cp.async.bulk) ring, over two
// 4 GiB arrays (prev/next-like), reporting GB/s of bytes read.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int U>
__global__ void ldg_kernel(const uint4* a, const uint4* b, size_t nvec, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < nvec; base += stride) {
    uint4 x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = base + (size_t)u * blockDim.x;
      if (i < nvec) { x[u] = ldnc(a + i); y[u] = ldnc(b + i); } else { x[u] = y[u] = make_uint4(0,0,0,0); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= x[u].x ^ x[u].w ^ y[u].y ^ y[u].z;
  }
  if (acc == 0x12345678u) *sink = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void marrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" :: "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

// chunk = bytes per array per stage; ring stages; consumers = 8 warps
__global__ void tma_kernel(const uint8_t* a, const uint8_t* b, size_t bytes, uint32_t chunk, int ring,
                           unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + 2 * (size_t)ring * chunk);
  uint64_t* empty = full + ring;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = blockDim.x / 32 - 1;
  if (tid == 0) { for (int k = 0; k < ring; ++k) { minit(&full[k], 1); minit(&empty[k], nw); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const size_t nchunks = bytes / chunk;
  if (warp == nw) {
    if (lane == 0) {
      uint32_t eb = (1u << ring) - 1; int k = 0;
      for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        mwait(&empty[k], (eb >> k) & 1); eb ^= 1u << k;
        mexpect(&full[k], 2 * chunk);
        tma(sm + (size_t)k * chunk, a + c * chunk, chunk, &full[k]);
        tma(sm + (size_t)(ring + k) * chunk, b + c * chunk, chunk, &full[k]);
        k = (k + 1) % ring;
      }
    }
    return;
  }
  unsigned acc = 0; uint32_t fb = 0; int k = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    mwait(&full[k], (fb >> k) & 1); fb ^= 1u << k;
    const uint4* p = (const uint4*)(sm + (size_t)k * chunk);
    const uint4* q = (const uint4*)(sm + (size_t)(ring + k) * chunk);
    for (uint32_t j = tid; j < chunk / 16; j += nw * 32) { uint4 x = p[j], y = q[j]; acc ^= x.x ^ y.w; }
    __syncwarp();
    if (lane == 0) marrive(&empty[k]);
    k = (k + 1) % ring;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char** argv) {
  const size_t bytes = (size_t)4 << 30;
  uint8_t *a, *b; unsigned* sink;
  CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(a, 1, bytes)); CK(cudaMemset(b, 2, bytes));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto fn, const char* name) {
    for (int i = 0; i < 2; ++i) fn();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); for (int i = 0; i < 5; ++i) fn(); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-40s %8.1f GB/s\n", name, 2.0 * bytes / ms / 1e6);
  };
  char nm[128];
  for (int bps : {2, 4, 8}) for (int thr : {256, 512}) {
    snprintf(nm, sizeof nm, "ldg U=4 blocks/SM=%d thr=%d", bps, thr);
    timeit([&] { ldg_kernel<4><<<sms * bps, thr>>>((const uint4*)a, (const uint4*)b, bytes / 16, sink); }, nm);
  }
  for (int bps : {2, 4}) {
    snprintf(nm, sizeof nm, "ldg U=8 blocks/SM=%d thr=256", bps);
    timeit([&] { ldg_kernel<8><<<sms * bps, 256>>>((const uint4*)a, (const uint4*)b, bytes / 16, sink); }, nm);
  }
  CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  for (uint32_t chunk : {4096u, 8192u, 16384u, 32768u}) for (int ring : {2, 3, 4, 6, 8, 12}) {
    size_t smem = 2 * (size_t)ring * chunk + 2 * ring * 8;
    if (smem > 220 * 1024) continue;
    for (int bps : {1, 2}) {
      if (smem * bps > 225 * 1024) continue;
      snprintf(nm, sizeof nm, "tma chunk=%uK ring=%d blocks/SM=%d", chunk / 1024, ring, bps);
      timeit([&] { tma_kernel<<<sms * bps, 288, smem>>>(a, b, bytes, chunk, ring, sink); }, nm);
    }
  }
  return 0;
}
