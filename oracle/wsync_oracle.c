/*
 * wsync_oracle.c -- CPU restatement of the reference weight-sync data plane.
 *
 * TEST INFRASTRUCTURE ONLY (see wsync_oracle.h).  Plain scalar C, one
 * function per reference function, citations are to
 * /root/reference/proj/src/transfer/<file>:<line>.
 */
#include "wsync_oracle.h"

#include <string.h>

#define WSO_MAX_DIMS 8

int wso_dtype_size(int dtype) { return dtype == WSO_BF16 ? 2 : 4; }

/* ---- diff: codec.cpp:34-63 ------------------------------------------------ */
int wso_diff_shards(int dtype, const void* prev, const void* next, uint64_t n,
                    uint64_t* out_idx, void* out_val, uint64_t* out_nnz) {
  uint64_t k = 0;
  if (dtype == WSO_F32) {
    /* codec.cpp:44-50: skip when a == b (value compare), store b - a. */
    const float* a = (const float*)prev;
    const float* b = (const float*)next;
    float* v = (float*)out_val;
    for (uint64_t i = 0; i < n; ++i) {
      if (a[i] == b[i]) continue;
      out_idx[k] = i;
      v[k] = b[i] - a[i];
      ++k;
    }
  } else if (dtype == WSO_I32) {
    /* codec.cpp:52-61: skip when equal, store the u32 wrap-around b - a. */
    const uint32_t* a = (const uint32_t*)prev;
    const uint32_t* b = (const uint32_t*)next;
    uint32_t* v = (uint32_t*)out_val;
    for (uint64_t i = 0; i < n; ++i) {
      if (a[i] == b[i]) continue;
      out_idx[k] = i;
      v[k] = b[i] - a[i];
      ++k;
    }
  } else if (dtype == WSO_BF16) {
    /* Extension: the I32 rule on 16-bit words (bit-pattern compare). */
    const uint16_t* a = (const uint16_t*)prev;
    const uint16_t* b = (const uint16_t*)next;
    uint16_t* v = (uint16_t*)out_val;
    for (uint64_t i = 0; i < n; ++i) {
      if (a[i] == b[i]) continue;
      out_idx[k] = i;
      v[k] = (uint16_t)(b[i] - a[i]);
      ++k;
    }
  } else {
    return WSO_INVALID_ARGUMENT;
  }
  *out_nnz = k;
  return WSO_OK;
}

/* ---- apply: codec.cpp:65-92 ----------------------------------------------- */
int wso_apply_delta(int dtype, void* target, uint64_t n, const uint64_t* idx,
                    const void* val, uint64_t nnz) {
  for (uint64_t k = 0; k < nnz; ++k) {
    const uint64_t i = idx[k];
    if (i >= n) return WSO_INDEX_OUT_OF_SHARD; /* codec.cpp:74-77 */
    if (dtype == WSO_F32) {
      ((float*)target)[i] += ((const float*)val)[k]; /* codec.cpp:78 */
    } else if (dtype == WSO_I32) {
      uint32_t* t = (uint32_t*)target; /* codec.cpp:88-89 */
      t[i] = t[i] + ((const uint32_t*)val)[k];
    } else if (dtype == WSO_BF16) {
      uint16_t* t = (uint16_t*)target;
      t[i] = (uint16_t)(t[i] + ((const uint16_t*)val)[k]);
    } else {
      return WSO_INVALID_ARGUMENT;
    }
  }
  return WSO_OK;
}

/* ---- geometry helpers (shard.cpp:146-151 shard_shape) --------------------- */
typedef struct {
  int nd;
  int64_t lo[WSO_MAX_DIMS];
  int64_t ext[WSO_MAX_DIMS];
} box_t;

static box_t shard_box(const int64_t* full, int nd, int dim, int64_t s,
                       int64_t e) {
  box_t b;
  b.nd = nd;
  for (int i = 0; i < nd; ++i) {
    b.lo[i] = 0;
    b.ext[i] = full[i];
  }
  if (dim >= 0) {
    b.lo[dim] = s;
    b.ext[dim] = e - s;
  }
  return b;
}

static uint64_t box_elems(const box_t* b) {
  uint64_t n = 1;
  for (int i = 0; i < b->nd; ++i) n *= (uint64_t)b->ext[i];
  return n;
}

/* ---- reslice: codec.cpp:94-138 -------------------------------------------- */
int wso_reslice_delta(int dtype, const int64_t* full_shape, int ndims,
                      int src_dim, int64_t src_start, int64_t src_end,
                      int dst_dim, int64_t dst_start, int64_t dst_end,
                      int allow_cross_dim, const uint64_t* idx, const void* val,
                      uint64_t nnz, uint64_t* out_idx, void* out_val,
                      uint64_t* out_nnz) {
  if (ndims < 1 || ndims > WSO_MAX_DIMS) return WSO_INVALID_ARGUMENT;
  /* codec.cpp:101-102: both sliced, different dims -> ShapeMismatch. */
  if (src_dim >= 0 && dst_dim >= 0 && src_dim != dst_dim && !allow_cross_dim)
    return WSO_SHAPE_MISMATCH;
  const box_t S = shard_box(full_shape, ndims, src_dim, src_start, src_end);
  const box_t D = shard_box(full_shape, ndims, dst_dim, dst_start, dst_end);
  const uint64_t src_elems = box_elems(&S);
  const int esz = wso_dtype_size(dtype);
  const uint8_t* vin = (const uint8_t*)val;
  uint8_t* vout = (uint8_t*)out_val;
  uint64_t k_out = 0;
  for (uint64_t k = 0; k < nnz; ++k) {
    const uint64_t i = idx[k];
    if (i >= src_elems) return WSO_INDEX_OUT_OF_SHARD; /* codec.cpp:121-124 */
    /* Unravel i in the source shard's shape, shift to global coordinates,
     * keep iff inside the destination box, ravel in the destination shape.
     * For same-dim slices this is codec.cpp:125-131's outer/row/inner math. */
    int64_t g[WSO_MAX_DIMS];
    uint64_t rem = i;
    for (int d = ndims - 1; d >= 0; --d) {
      g[d] = (int64_t)(rem % (uint64_t)S.ext[d]) + S.lo[d];
      rem /= (uint64_t)S.ext[d];
    }
    int keep = 1;
    for (int d = 0; d < ndims; ++d)
      if (g[d] < D.lo[d] || g[d] >= D.lo[d] + D.ext[d]) keep = 0;
    if (!keep) continue; /* codec.cpp:129 */
    uint64_t di = 0;
    for (int d = 0; d < ndims; ++d)
      di = di * (uint64_t)D.ext[d] + (uint64_t)(g[d] - D.lo[d]);
    out_idx[k_out] = di;
    memcpy(vout + k_out * esz, vin + k * esz, (size_t)esz);
    ++k_out;
  }
  *out_nnz = k_out;
  return WSO_OK;
}

/* ---- extract_shard: shard.cpp:111-134 ------------------------------------- */
int wso_extract_shard(int dtype, const int64_t* full_shape, int ndims, int dim,
                      int64_t start, int64_t end, const void* full, void* out) {
  const int esz = wso_dtype_size(dtype);
  if (dim < 0) { /* shard.cpp:112: full descriptor copies everything */
    uint64_t n = 1;
    for (int i = 0; i < ndims; ++i) n *= (uint64_t)full_shape[i];
    memcpy(out, full, n * (uint64_t)esz);
    return WSO_OK;
  }
  if (dim >= ndims) return WSO_SHAPE_MISMATCH; /* shard.cpp:114-116 */
  if (start < 0 || end > full_shape[dim] || start >= end)
    return WSO_SHAPE_MISMATCH; /* shard.cpp:117-121 */
  int64_t outer = 1, inner = 1;
  for (int i = 0; i < ndims; ++i) {
    if (i < dim) outer *= full_shape[i];
    if (i > dim) inner *= full_shape[i];
  }
  const int64_t ext = full_shape[dim], rows = end - start;
  const size_t run = (size_t)(rows * inner) * (size_t)esz;
  for (int64_t o = 0; o < outer; ++o)
    memcpy((uint8_t*)out + (size_t)(o * rows * inner) * esz,
           (const uint8_t*)full + (size_t)((o * ext + start) * inner) * esz, run);
  return WSO_OK;
}

/* ---- copy_overlap: shard.cpp:136-170, generalised to boxes ---------------- */
int64_t wso_copy_overlap_box(int dtype, const int64_t* full_shape, int ndims,
                             int dst_dim, int64_t dst_start, int64_t dst_end,
                             void* dst, int src_dim, int64_t src_start,
                             int64_t src_end, const void* src) {
  if (ndims < 1 || ndims > WSO_MAX_DIMS) return -WSO_INVALID_ARGUMENT;
  const box_t S = shard_box(full_shape, ndims, src_dim, src_start, src_end);
  const box_t D = shard_box(full_shape, ndims, dst_dim, dst_start, dst_end);
  int64_t lo[WSO_MAX_DIMS], hi[WSO_MAX_DIMS];
  uint64_t count = 1;
  for (int d = 0; d < ndims; ++d) {
    lo[d] = S.lo[d] > D.lo[d] ? S.lo[d] : D.lo[d];
    const int64_t sh = S.lo[d] + S.ext[d], dh = D.lo[d] + D.ext[d];
    hi[d] = sh < dh ? sh : dh;
    if (lo[d] >= hi[d]) return 0; /* shard.cpp:149 */
    count *= (uint64_t)(hi[d] - lo[d]);
  }
  const int esz = wso_dtype_size(dtype);
  int64_t g[WSO_MAX_DIMS];
  for (int d = 0; d < ndims; ++d) g[d] = lo[d];
  for (uint64_t c = 0; c < count; ++c) {
    uint64_t si = 0, di = 0;
    for (int d = 0; d < ndims; ++d) {
      si = si * (uint64_t)S.ext[d] + (uint64_t)(g[d] - S.lo[d]);
      di = di * (uint64_t)D.ext[d] + (uint64_t)(g[d] - D.lo[d]);
    }
    memcpy((uint8_t*)dst + di * esz, (const uint8_t*)src + si * esz, (size_t)esz);
    for (int d = ndims - 1; d >= 0; --d) { /* row-major odometer */
      if (++g[d] < hi[d]) break;
      g[d] = lo[d];
    }
  }
  return (int64_t)count;
}

/* ---- density rule: engine.cpp:121 (sparse iff density <= threshold) ------- */
int wso_is_sparse(uint64_t nnz, uint64_t n, double threshold) {
  const double d = n == 0 ? 0.0 : (double)nnz / (double)n; /* codec.hpp:28-31 */
  return d <= threshold;
}

/* ---- synthetic generator (rng.hpp:73-87 splitmix64/fnv1a64) --------------- */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

static uint64_t fnv1a64(const char* s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001b3ULL;
  }
  return h;
}

uint64_t wso_param_key(uint64_t seed, const char* name) {
  return splitmix64(seed ^ fnv1a64(name)); /* rng.hpp:98 stream seeding */
}

static uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* Element g: r0 -> prev ~ N(0, 0.02) (Irwin-Hall of four u16 lanes, rounded to
 * bf16 RNE); r1 -> Bernoulli(density) change by +-[1,16] ulp-steps (u16 wrap),
 * so every chosen element differs bitwise from prev. */
static void gen_elem(uint64_t key, uint64_t g, uint64_t change_thr,
                     uint16_t* p, uint16_t* n) {
  const uint64_t r0 = splitmix64(key + (2 * g) * 0x9e3779b97f4a7c15ULL);
  const uint64_t r1 = splitmix64(key + (2 * g + 1) * 0x9e3779b97f4a7c15ULL);
  const int32_t s = (int32_t)(r0 & 0xFFFF) + (int32_t)((r0 >> 16) & 0xFFFF) +
                    (int32_t)((r0 >> 32) & 0xFFFF) + (int32_t)(r0 >> 48) - 131070;
  const float v = (float)s * 5.2858e-7f;
  const uint16_t pb = f32_to_bf16_rne(v);
  uint16_t nb = pb;
  if ((r1 >> 32) < change_thr) {
    const uint16_t m = (uint16_t)(1 + (r1 & 0xF));
    nb = ((r1 >> 4) & 1) ? (uint16_t)(pb - m) : (uint16_t)(pb + m);
  }
  *p = pb;
  *n = nb;
}

void wso_gen_pair_bf16(uint64_t key, const int64_t* full_shape, int ndims,
                       int dim, int64_t start, int64_t end, uint64_t change_thr,
                       uint16_t* prev, uint16_t* next) {
  const box_t S = shard_box(full_shape, ndims, dim, start, end);
  const uint64_t n = box_elems(&S);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t rem = i, g = 0, mul = 1;
    for (int d = ndims - 1; d >= 0; --d) {
      const uint64_t c = rem % (uint64_t)S.ext[d] + (uint64_t)S.lo[d];
      rem /= (uint64_t)S.ext[d];
      g += c * mul;
      mul *= (uint64_t)full_shape[d];
    }
    gen_elem(key, g, change_thr, &prev[i], &next[i]);
  }
}

void wso_gen_pair_bf16_dim0(uint64_t key, const int64_t* full_shape, int ndims,
                            int dim, int64_t start, int64_t end,
                            const uint64_t* thr_dim0, uint16_t* prev, uint16_t* next) {
  const box_t S = shard_box(full_shape, ndims, dim, start, end);
  const uint64_t n = box_elems(&S);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t rem = i, g = 0, mul = 1, c0 = 0;
    for (int d = ndims - 1; d >= 0; --d) {
      const uint64_t c = rem % (uint64_t)S.ext[d] + (uint64_t)S.lo[d];
      rem /= (uint64_t)S.ext[d];
      g += c * mul;
      mul *= (uint64_t)full_shape[d];
      c0 = c;
    }
    gen_elem(key, g, thr_dim0[c0], &prev[i], &next[i]);
  }
}

/* ---- sparse payload: codec.cpp:145-183 ------------------------------------ */
uint64_t wso_sparse_payload_size(int dtype, int ndims, int index_width,
                                 uint64_t nnz) {
  /* header (codec.cpp:145-154) + nnz u64 + indices + values */
  return 8 + 8 * (uint64_t)ndims + 8 +
         nnz * ((uint64_t)index_width + (uint64_t)wso_dtype_size(dtype));
}

static void put_bytes(uint8_t* out, uint64_t* pos, const void* p, size_t n) {
  memcpy(out + *pos, p, n);
  *pos += n;
}

int wso_encode_sparse(int dtype, const int64_t* shape, int ndims,
                      int index_width, const uint64_t* idx, const void* val,
                      uint64_t nnz, uint8_t* out, uint64_t* out_len) {
  if (index_width != 4 && index_width != 8) return WSO_PAYLOAD_FORMAT;
  const uint32_t magic = dtype == WSO_BF16 ? 0x32535743u  /* "CWS2" */
                                           : 0x31535743u; /* "CWS1" */
  uint64_t pos = 0;
  const uint8_t dt = (uint8_t)dtype, nd = (uint8_t)ndims,
                iw = (uint8_t)index_width, pad = 0;
  put_bytes(out, &pos, &magic, 4);
  put_bytes(out, &pos, &dt, 1);
  put_bytes(out, &pos, &nd, 1);
  put_bytes(out, &pos, &iw, 1);
  put_bytes(out, &pos, &pad, 1);
  for (int i = 0; i < ndims; ++i) put_bytes(out, &pos, &shape[i], 8);
  put_bytes(out, &pos, &nnz, 8);
  for (uint64_t k = 0; k < nnz; ++k) {
    if (index_width == 4) {
      if (idx[k] > 0xFFFFFFFFull) return WSO_PAYLOAD_FORMAT; /* codec.cpp:174-175 */
      const uint32_t i32 = (uint32_t)idx[k];
      put_bytes(out, &pos, &i32, 4);
    } else {
      put_bytes(out, &pos, &idx[k], 8);
    }
  }
  put_bytes(out, &pos, val, (size_t)(nnz * (uint64_t)wso_dtype_size(dtype)));
  *out_len = pos;
  return WSO_OK;
}
