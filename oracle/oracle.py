"""ctypes front-end to the parity checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module; the product package (``paper_2605_06534_b200``) never does.

Two checkers are exposed, both as numpy-in / numpy-out functions:

* ``Restatement`` -- oracle/_build/liboracle.so, the C restatement in
  wsync_oracle.c (F32/I32/BF16, cross-dim extension, synthetic generator).
* ``Reference``   -- oracle/_ref/libref_capi.so, the UNMODIFIED reference
  transfer engine (/root/reference/proj/src/transfer) behind ref_capi.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
F32, I32, BF16 = 0, 1, 2
NP_DTYPE = {F32: np.float32, I32: np.int32, BF16: np.uint16}
ESZ = {F32: 4, I32: 4, BF16: 2}

STATUS = {0: "OK", 1: "ShapeMismatch", 2: "PayloadFormatError", 3: "IndexOutOfShard",
          4: "IndivisibleShape", 5: "UnknownModuleKind", 6: "IncompleteCoverage",
          7: "RelayTimeout", 8: "IntegrityError", 10: "TransferError", 22: "Capacity",
          23: "InvalidArgument", 99: "Exception"}

_p = np.ctypeslib.ndpointer
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)


def build():
    """Compile the restatement (and the reference wrapper when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _shape(shape):
    return (C.c_int64 * max(1, len(shape)))(*shape)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS.get(code, str(code))


class Restatement:
    """The C restatement (wsync_oracle.c)."""

    def __init__(self, path=None):
        path = path or os.path.join(HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.wso_diff_shards.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                                      C.c_void_p, C.c_void_p, _u64p]
        L.wso_apply_delta.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p,
                                      C.c_void_p, C.c_uint64]
        L.wso_reslice_delta.argtypes = [C.c_int, _i64p, C.c_int, C.c_int, C.c_int64,
                                        C.c_int64, C.c_int, C.c_int64, C.c_int64, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                        C.c_void_p, _u64p]
        L.wso_extract_shard.argtypes = [C.c_int, _i64p, C.c_int, C.c_int, C.c_int64,
                                        C.c_int64, C.c_void_p, C.c_void_p]
        L.wso_copy_overlap_box.argtypes = [C.c_int, _i64p, C.c_int, C.c_int, C.c_int64,
                                           C.c_int64, C.c_void_p, C.c_int, C.c_int64,
                                           C.c_int64, C.c_void_p]
        L.wso_copy_overlap_box.restype = C.c_int64
        L.wso_is_sparse.argtypes = [C.c_uint64, C.c_uint64, C.c_double]
        L.wso_param_key.argtypes = [C.c_uint64, C.c_char_p]
        L.wso_param_key.restype = C.c_uint64
        L.wso_gen_pair_bf16_dim0.argtypes = [C.c_uint64, _i64p, C.c_int, C.c_int, C.c_int64,
                                             C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.wso_gen_pair_bf16.argtypes = [C.c_uint64, _i64p, C.c_int, C.c_int, C.c_int64,
                                        C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p]
        L.wso_sparse_payload_size.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64]
        L.wso_sparse_payload_size.restype = C.c_uint64
        L.wso_encode_sparse.argtypes = [C.c_int, _i64p, C.c_int, C.c_int, C.c_void_p,
                                        C.c_void_p, C.c_uint64, C.c_void_p, _u64p]

    def diff_shards(self, dtype, prev, next_):
        prev = np.ascontiguousarray(prev, NP_DTYPE[dtype]).ravel()
        next_ = np.ascontiguousarray(next_, NP_DTYPE[dtype]).ravel()
        if prev.shape != next_.shape:
            raise OracleError(1, "diff_shards shape mismatch")
        idx = np.empty(prev.size, np.uint64)
        val = np.empty(prev.size, NP_DTYPE[dtype])
        nnz = C.c_uint64()
        rc = self.lib.wso_diff_shards(dtype, _ptr(prev), _ptr(next_), prev.size,
                                      _ptr(idx), _ptr(val), C.byref(nnz))
        if rc:
            raise OracleError(rc)
        return idx[:nnz.value].copy(), val[:nnz.value].copy()

    def apply_delta(self, dtype, target, idx, val):
        """In-place on a copy; returns (result, status)."""
        t = np.ascontiguousarray(target, NP_DTYPE[dtype]).ravel().copy()
        idx = np.ascontiguousarray(idx, np.uint64)
        val = np.ascontiguousarray(val, NP_DTYPE[dtype])
        rc = self.lib.wso_apply_delta(dtype, _ptr(t), t.size, _ptr(idx), _ptr(val), idx.size)
        return t, rc

    def reslice_delta(self, dtype, full_shape, src, dst, idx, val, allow_cross_dim=True):
        """src/dst are (slice_dim, start, end) with slice_dim < 0 for full."""
        idx = np.ascontiguousarray(idx, np.uint64)
        val = np.ascontiguousarray(val, NP_DTYPE[dtype])
        oi = np.empty(max(1, idx.size), np.uint64)
        ov = np.empty(max(1, idx.size), NP_DTYPE[dtype])
        n = C.c_uint64()
        rc = self.lib.wso_reslice_delta(dtype, _shape(full_shape), len(full_shape),
                                        src[0], src[1], src[2], dst[0], dst[1], dst[2],
                                        int(allow_cross_dim), _ptr(idx), _ptr(val), idx.size,
                                        _ptr(oi), _ptr(ov), C.byref(n))
        if rc:
            raise OracleError(rc)
        return oi[:n.value].copy(), ov[:n.value].copy()

    def extract_shard(self, dtype, full, full_shape, desc):
        out = np.empty(shard_elems(full_shape, desc), NP_DTYPE[dtype])
        full = np.ascontiguousarray(full, NP_DTYPE[dtype])
        rc = self.lib.wso_extract_shard(dtype, _shape(full_shape), len(full_shape), desc[0],
                                        desc[1], desc[2], _ptr(full), _ptr(out))
        if rc:
            raise OracleError(rc)
        return out

    def copy_overlap_box(self, dtype, full_shape, dst_desc, dst, src_desc, src):
        dst = np.ascontiguousarray(dst, NP_DTYPE[dtype]).copy()
        src = np.ascontiguousarray(src, NP_DTYPE[dtype])
        n = self.lib.wso_copy_overlap_box(dtype, _shape(full_shape), len(full_shape),
                                          dst_desc[0], dst_desc[1], dst_desc[2], _ptr(dst),
                                          src_desc[0], src_desc[1], src_desc[2], _ptr(src))
        if n < 0:
            raise OracleError(-n)
        return dst, n

    def is_sparse(self, nnz, n, threshold):
        return bool(self.lib.wso_is_sparse(nnz, n, threshold))

    def param_key(self, seed, name):
        return self.lib.wso_param_key(seed, name.encode())

    def gen_pair_bf16(self, seed, name, full_shape, desc, density, thr_dim0=None):
        n = shard_elems(full_shape, desc)
        prev = np.empty(n, np.uint16)
        nxt = np.empty(n, np.uint16)
        if thr_dim0 is not None:
            tab = np.ascontiguousarray(thr_dim0, np.uint64)
            self.lib.wso_gen_pair_bf16_dim0(self.param_key(seed, name), _shape(full_shape),
                                            len(full_shape), desc[0], desc[1], desc[2],
                                            _ptr(tab), _ptr(prev), _ptr(nxt))
            return prev, nxt
        self.lib.wso_gen_pair_bf16(self.param_key(seed, name), _shape(full_shape),
                                   len(full_shape), desc[0], desc[1], desc[2],
                                   change_threshold(density), _ptr(prev), _ptr(nxt))
        return prev, nxt

    def encode_sparse(self, dtype, shape, idx, val, index_width=4):
        idx = np.ascontiguousarray(idx, np.uint64)
        val = np.ascontiguousarray(val, NP_DTYPE[dtype])
        size = self.lib.wso_sparse_payload_size(dtype, len(shape), index_width, idx.size)
        out = np.empty(size, np.uint8)
        n = C.c_uint64()
        rc = self.lib.wso_encode_sparse(dtype, _shape(shape), len(shape), index_width,
                                        _ptr(idx), _ptr(val), idx.size, _ptr(out), C.byref(n))
        if rc:
            raise OracleError(rc)
        return out[:n.value].tobytes()


def expert_thresholds(experts, density, zipf_s, perm_seed=0):
    """Config 4's per-expert change thresholds (Zipf(s) over
    the experts, normalised to mean density), restated in plain Python:
    weights r^-s of ranks 1..E, ranks assigned by a Fisher-Yates shuffle
    driven by splitmix64(perm_seed + k * golden) (the rng.hpp:73-78 mixer)."""
    M = (1 << 64) - 1
    w = [float(r + 1) ** (-zipf_s) for r in range(experts)]
    total = sum(w)
    rank = list(range(experts))
    st = perm_seed & M
    for i in range(experts - 1, 0, -1):
        st = (st + 0x9E3779B97F4A7C15) & M
        x = st
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        x ^= x >> 31
        j = x % (i + 1)
        rank[i], rank[j] = rank[j], rank[i]
    out = []
    for e in range(experts):
        d = min(max(density * w[rank[e]] * experts / total, 0.0), 1.0)
        out.append(int(d * 4294967296.0))
    return out


def change_threshold(density):
    """Bernoulli threshold on the top 32 bits of a draw: floor(d * 2^32), clamped."""
    return int(min(max(density, 0.0), 1.0) * 4294967296.0)


def shard_shape(full_shape, desc):
    s = list(full_shape)
    if desc[0] >= 0:
        s[desc[0]] = desc[2] - desc[1]
    return s


def shard_elems(full_shape, desc):
    return int(np.prod(shard_shape(full_shape, desc), dtype=np.int64))


class RefParam(C.Structure):
    _fields_ = [("name", C.c_char_p), ("kind", C.c_int), ("ndims", C.c_int),
                ("shape", C.c_int64 * 4), ("layer", C.c_int)]


def ref_params(manifest):
    """manifest: list of (name, kind, shape, layer) -> ctypes array (keeps names alive)."""
    arr = (RefParam * len(manifest))()
    keep = []
    for i, (name, kind, shape, layer) in enumerate(manifest):
        b = name.encode()
        keep.append(b)
        arr[i].name = b
        arr[i].kind = kind
        arr[i].ndims = len(shape)
        for k, d in enumerate(shape):
            arr[i].shape[k] = d
        arr[i].layer = layer
    return arr, keep


class Reference:
    """The compiled, unmodified reference (oracle/_ref/libref_capi.so)."""

    def __init__(self, path=None):
        path = path or os.path.join(HERE, "_ref", "libref_capi.so")
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_diff_shards.argtypes = [C.c_int, _i64p, C.c_int, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, _u64p]
        L.ref_apply_delta.argtypes = [C.c_int, _i64p, C.c_int, C.c_void_p, _i64p, C.c_int,
                                      C.c_void_p, C.c_void_p, C.c_uint64]
        L.ref_reslice_delta.argtypes = [C.c_int, _i64p, C.c_int, C.c_int, C.c_int64,
                                        C.c_int64, C.c_int, C.c_int64, C.c_int64, _i64p,
                                        C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                                        C.c_void_p, C.c_void_p, _u64p, _i64p]
        L.ref_extract_shard.argtypes = [C.c_int, _i64p, C.c_int, C.c_int, C.c_int64,
                                        C.c_int64, C.c_void_p, C.c_void_p]
        L.ref_copy_overlap.argtypes = [C.c_int, _i64p, C.c_int, C.c_void_p, C.c_int64,
                                       _i64p, C.c_void_p, C.c_int64, C.c_int]
        L.ref_copy_overlap.restype = C.c_int64
        L.ref_encode_sparse.argtypes = [C.c_int, _i64p, C.c_int, C.c_void_p, C.c_void_p,
                                        C.c_uint64, C.c_int, C.c_void_p, C.c_uint64, _u64p]
        L.ref_encode_dense.argtypes = [C.c_int, _i64p, C.c_int, C.c_void_p, C.c_void_p,
                                       C.c_uint64, _u64p]
        L.ref_decode_payload.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int),
                                         C.POINTER(C.c_int), _i64p, _u64p, C.c_void_p,
                                         C.c_void_p]
        L.ref_bucket_key.argtypes = [C.c_uint64, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_int64, C.c_int64, C.c_char, C.c_int, C.c_uint32,
                                     C.c_char_p, C.c_uint64, _u64p]
        L.ref_encode_bucket_frame.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                              C.c_void_p, C.c_uint64, _u64p]
        L.ref_memrelay_create.restype = C.c_void_p
        L.ref_memrelay_destroy.argtypes = [C.c_void_p]
        L.ref_memrelay_size.argtypes = [C.c_void_p]
        L.ref_memrelay_size.restype = C.c_uint64
        L.ref_memrelay_list.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_uint64]
        L.ref_memrelay_list.restype = C.c_uint64
        L.ref_memrelay_get.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, C.c_void_p, C.c_uint64]
        L.ref_memrelay_get.restype = C.c_int64
        L.ref_frame_crc32.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_frame_crc32.restype = C.c_uint32
        L.ref_peek_payload_size.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_peek_payload_size.restype = C.c_int64
        L.ref_plan.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.c_int, _i64p, C.POINTER(C.c_int), _i64p,
                               C.POINTER(C.c_int), C.c_int]
        L.ref_state_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64]
        L.ref_state_create.restype = C.c_void_p
        L.ref_state_create_toy.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                           C.c_uint64]
        L.ref_state_create_toy.restype = C.c_void_p
        L.ref_state_destroy.argtypes = [C.c_void_p]
        L.ref_state_nparams.argtypes = [C.c_void_p]
        L.ref_state_param.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), _i64p, C.POINTER(C.c_int)]
        L.ref_state_param.restype = C.c_char_p
        L.ref_state_weights.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_state_weights.restype = C.c_void_p
        L.ref_state_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double,
                                    C.c_uint64, C.c_int, C.POINTER(C.c_double)]
        L.ref_state_prepare.argtypes = [C.c_void_p]
        L.ref_state_prepare.restype = C.c_int
        L.ref_state_model_bytes.argtypes = [C.c_void_p]
        L.ref_state_model_bytes.restype = C.c_double
        L.ref_state_serve.argtypes = [C.c_void_p, C.c_int, C.c_int, _u64p]
        L.ref_state_serve.restype = C.c_void_p
        L.ref_state_ncodecs.argtypes = [C.c_void_p]
        L.ref_state_codec.argtypes = [C.c_void_p, C.c_int, _i64p]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode(errors="replace"))

    def diff_shards(self, dtype, shape, prev, next_):
        prev = np.ascontiguousarray(prev, NP_DTYPE[dtype])
        next_ = np.ascontiguousarray(next_, NP_DTYPE[dtype])
        n = int(np.prod(shape))
        idx = np.empty(max(1, n), np.uint64)
        val = np.empty(max(1, n), NP_DTYPE[dtype])
        nnz = C.c_uint64()
        self._check(self.lib.ref_diff_shards(dtype, _shape(shape), len(shape), _ptr(prev),
                                             _ptr(next_), _ptr(idx), _ptr(val), C.byref(nnz)))
        return idx[:nnz.value].copy(), val[:nnz.value].copy()

    def apply_delta(self, dtype, shape, target, delta_shape, idx, val):
        """Returns (updated target, status) -- partial on IndexOutOfShard like the ref."""
        t = np.ascontiguousarray(target, NP_DTYPE[dtype]).copy()
        idx = np.ascontiguousarray(idx, np.uint64)
        val = np.ascontiguousarray(val, NP_DTYPE[dtype])
        rc = self.lib.ref_apply_delta(dtype, _shape(shape), len(shape), _ptr(t),
                                      _shape(delta_shape), len(delta_shape), _ptr(idx),
                                      _ptr(val), idx.size)
        return t, rc

    def reslice_delta(self, dtype, full_shape, src, dst, delta_shape, idx, val):
        idx = np.ascontiguousarray(idx, np.uint64)
        val = np.ascontiguousarray(val, NP_DTYPE[dtype])
        oi = np.empty(max(1, idx.size), np.uint64)
        ov = np.empty(max(1, idx.size), NP_DTYPE[dtype])
        n = C.c_uint64()
        osh = (C.c_int64 * 8)()
        self._check(self.lib.ref_reslice_delta(
            dtype, _shape(full_shape), len(full_shape), src[0], src[1], src[2], dst[0],
            dst[1], dst[2], _shape(delta_shape), len(delta_shape), _ptr(idx), _ptr(val),
            idx.size, _ptr(oi), _ptr(ov), C.byref(n), osh))
        return oi[:n.value].copy(), ov[:n.value].copy(), list(osh[:len(full_shape)])

    def extract_shard(self, dtype, full, full_shape, desc):
        out = np.empty(shard_elems(full_shape, desc), NP_DTYPE[dtype])
        full = np.ascontiguousarray(full, NP_DTYPE[dtype])
        self._check(self.lib.ref_extract_shard(dtype, _shape(full_shape), len(full_shape),
                                               desc[0], desc[1], desc[2], _ptr(full),
                                               _ptr(out)))
        return out

    def copy_overlap(self, dtype, dst_shape, dst, dst_start, src_shape, src, src_start, dim):
        dst = np.ascontiguousarray(dst, NP_DTYPE[dtype]).copy()
        src = np.ascontiguousarray(src, NP_DTYPE[dtype])
        n = self.lib.ref_copy_overlap(dtype, _shape(dst_shape), len(dst_shape), _ptr(dst),
                                      dst_start, _shape(src_shape), _ptr(src), src_start, dim)
        if n < 0:
            raise OracleError(-n, self.lib.ref_last_error().decode(errors="replace"))
        return dst, n

    def encode_sparse(self, dtype, shape, idx, val, index_width=0):
        idx = np.ascontiguousarray(idx, np.uint64)
        val = np.ascontiguousarray(val, NP_DTYPE[dtype])
        cap = 64 + 12 * idx.size
        out = np.empty(cap, np.uint8)
        n = C.c_uint64()
        self._check(self.lib.ref_encode_sparse(dtype, _shape(shape), len(shape), _ptr(idx),
                                               _ptr(val), idx.size, index_width, _ptr(out),
                                               cap, C.byref(n)))
        return out[:n.value].tobytes()

    def encode_dense(self, dtype, shape, data):
        data = np.ascontiguousarray(data, NP_DTYPE[dtype])
        cap = 64 + 8 * len(shape) + data.nbytes
        out = np.empty(cap, np.uint8)
        n = C.c_uint64()
        self._check(self.lib.ref_encode_dense(dtype, _shape(shape), len(shape), _ptr(data),
                                              _ptr(out), cap, C.byref(n)))
        return out[:n.value].tobytes()

    def bucket_key(self, step, param, tp_rank, tp_size, pp_stage, desc, codec, iw, seq):
        """key.cpp:47-69, the reference's own BucketKey::encode."""
        raw = param.encode("utf-8", "surrogateescape") if isinstance(param, str) else param
        buf = C.create_string_buffer(8192)
        n = C.c_uint64()
        self._check(self.lib.ref_bucket_key(step, raw, tp_rank, tp_size, pp_stage, desc[0],
                                            desc[1], desc[2], codec.encode(), iw, seq, buf, 8192,
                                            C.byref(n)))
        return buf.raw[:n.value]

    def encode_bucket_frame(self, key: bytes, payload: bytes):
        """wire.cpp:35-47."""
        out = np.empty(12 + len(key) + len(payload), np.uint8)
        pl = np.frombuffer(payload, np.uint8) if payload else np.zeros(1, np.uint8)
        n = C.c_uint64()
        self._check(self.lib.ref_encode_bucket_frame(key, len(key), _ptr(pl), len(payload),
                                                     _ptr(out), out.size, C.byref(n)))
        return out[:n.value].tobytes()

    def decode_payload(self, data: bytes):
        """codec.cpp:229-263 -> (is_sparse, shape, nnz); raises OracleError."""
        arr = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        sp, nd, nnz = C.c_int(), C.c_int(), C.c_uint64()
        shape = (C.c_int64 * 16)()
        self._check(self.lib.ref_decode_payload(_ptr(arr), len(data), C.byref(sp), C.byref(nd),
                                                shape, C.byref(nnz), None, None))
        return bool(sp.value), tuple(shape[:nd.value]), nnz.value

    def memory_relay(self):
        """The reference's MemoryRelay (relay.cpp:7-59) as a ws_relay
        (ctx, put, get_any) triple of raw pointers, plus helpers."""
        return RefMemoryRelay(self.lib)

    def tcp_relay(self, flip_put=0, flip_get=0):
        """The reference's TcpRelayServer (tcp_relay.hpp) on a free localhost
        port, with a framed client for ws_relay's put_frame / get_any_frame
        (flip_*: corrupt every n-th frame in transit, to test the CRCs)."""
        return RefTcpRelay(self.lib, flip_put, flip_get)

    def frame_crc32(self, data: bytes):
        arr = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        return int(self.lib.ref_frame_crc32(_ptr(arr), len(data)))

    def plan(self, manifest, train, serve):
        """train=(tp,pp,dp), serve=(tp,pp) -> (push list, pull list) of descriptor tuples."""
        arr, keep = ref_params(manifest)
        cap = 1 << 16
        push = (C.c_int64 * (7 * cap))()
        pull = (C.c_int64 * (8 * cap))()
        npush, npull = C.c_int(), C.c_int()
        self._check(self.lib.ref_plan(arr, len(manifest), *train, *serve, push,
                                      C.byref(npush), pull, C.byref(npull), cap))
        pushes = [tuple(push[7 * i:7 * i + 7]) for i in range(npush.value)]
        pulls = [tuple(pull[8 * i:8 * i + 8]) for i in range(npull.value)]
        return pushes, pulls

    def state(self, manifest, dtype, train, serve, density, seed):
        arr, keep = ref_params(manifest)
        h = self.lib.ref_state_create(arr, len(manifest), dtype, *train, *serve, density, seed)
        if not h:
            raise OracleError(99, self.lib.ref_last_error().decode(errors="replace"))
        return RefState(self, h)

    def toy_state(self, layers, hidden, vocab, dtype, train, serve, density, seed):
        h = self.lib.ref_state_create_toy(layers, hidden, vocab, dtype, *train, *serve,
                                          density, seed)
        if not h:
            raise OracleError(99, self.lib.ref_last_error().decode(errors="replace"))
        return RefState(self, h)


REPORT_FIELDS = ("wall_s", "push_s", "pull_s", "encode_s", "apply_s", "pushed_bytes",
                 "pulled_bytes", "push_buckets", "pull_buckets", "dense_shards",
                 "sparse_shards")


class RefState:
    """A reference TrainState/ServeState pair (bench.cpp:5-43)."""

    def __init__(self, ref, h):
        self.ref, self.h, L = ref, h, ref.lib
        self.params = []
        for i in range(L.ref_state_nparams(h)):
            kind, nd, layer = C.c_int(), C.c_int(), C.c_int()
            shp = (C.c_int64 * 4)()
            name = L.ref_state_param(h, i, C.byref(kind), C.byref(nd), shp, C.byref(layer))
            self.params.append((name.decode(), kind.value, list(shp[:nd.value]), layer.value))
        self.dtype = None

    def __del__(self):
        try:
            self.ref.lib.ref_state_destroy(self.h)
        except Exception:
            pass

    def weights(self, i, which, dtype):
        n = int(np.prod(self.params[i][2]))
        p = self.ref.lib.ref_state_weights(self.h, i, which)
        buf = (C.c_uint8 * (n * ESZ[dtype])).from_address(p)
        return np.frombuffer(buf, NP_DTYPE[dtype]).copy()

    def run(self, mode_async=True, shard_aware=True, sparse=True, threshold=0.20,
            bucket_bytes=64 << 20, force_wide=False):
        rep = (C.c_double * 11)()
        self.ref._check(self.ref.lib.ref_state_run(self.h, int(mode_async), int(shard_aware),
                                                   int(sparse), threshold, bucket_bytes,
                                                   int(force_wide), rep))
        return dict(zip(REPORT_FIELDS, rep[:11]))

    def prepare(self):
        """ServeState::init ahead of the next run(), which then times
        TransferEngine::sync_step alone."""
        self.ref._check(self.ref.lib.ref_state_prepare(self.h))

    def model_bytes(self):
        return self.ref.lib.ref_state_model_bytes(self.h)

    def serve(self, rank, i, dtype):
        nb = C.c_uint64()
        p = self.ref.lib.ref_state_serve(self.h, rank, i, C.byref(nb))
        if not p:
            return None
        buf = (C.c_uint8 * nb.value).from_address(p)
        return np.frombuffer(buf, NP_DTYPE[dtype]).copy()

    def codecs(self):
        out = []
        d = (C.c_int64 * 7)()
        for k in range(self.ref.lib.ref_state_ncodecs(self.h)):
            c = self.ref.lib.ref_state_codec(self.h, k, d)
            out.append((tuple(d[:7]), chr(c)))
        return out


class RefTcpRelay:
    """The reference TCP relay server plus the framed client; `callbacks` is
    the 5-tuple (ctx, put, get_any, put_frame, get_any_frame) of raw C
    pointers for ws_engine_sync_relay (put/get_any unused: framed only)."""

    def __init__(self, lib, flip_put=0, flip_get=0):
        self.lib = lib
        for name, args, res in (
                ("ref_tcp_server_create", [], C.c_void_p),
                ("ref_tcp_server_port", [C.c_void_p], C.c_int),
                ("ref_tcp_server_buckets", [C.c_void_p], C.c_uint64),
                ("ref_tcp_server_destroy", [C.c_void_p], None),
                ("ref_tcp_client_create", [C.c_int], C.c_void_p),
                ("ref_tcp_client_destroy", [C.c_void_p], None),
                ("ref_tcp_client_get", [C.c_void_p, C.c_char_p, C.c_uint64, C.c_void_p,
                                        C.c_uint64], C.c_int64),
                ("ref_framed_client_create", [C.c_int, C.c_int, C.c_int], C.c_void_p),
                ("ref_framed_client_destroy", [C.c_void_p], None)):
            fn = getattr(lib, name)
            fn.argtypes, fn.restype = args, res
        self.server = lib.ref_tcp_server_create()
        if not self.server:
            raise OracleError(99, lib.ref_last_error().decode(errors="replace"))
        self.port = lib.ref_tcp_server_port(self.server)
        self.ctx = lib.ref_framed_client_create(self.port, flip_put, flip_get)
        self.reader = lib.ref_tcp_client_create(self.port)
        self.callbacks = (self.ctx, None, None, C.cast(lib.ref_framed_put, C.c_void_p).value,
                          C.cast(lib.ref_framed_get_any, C.c_void_p).value)

    def buckets(self):
        return int(self.lib.ref_tcp_server_buckets(self.server))

    def get(self, key: str) -> bytes:
        kb = key.encode("utf-8", "surrogateescape")
        n = self.lib.ref_tcp_client_get(self.reader, kb, len(kb), None, 0)
        if n < 0:
            raise KeyError(key)
        out = np.empty(max(1, n), np.uint8)
        self.lib.ref_tcp_client_get(self.reader, kb, len(kb), out.ctypes.data, n)
        return out[:n].tobytes()

    def close(self):
        if getattr(self, "server", None):
            self.lib.ref_framed_client_destroy(self.ctx)
            self.lib.ref_tcp_client_destroy(self.reader)
            self.lib.ref_tcp_server_destroy(self.server)
            self.server = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RefMemoryRelay:
    """The compiled reference MemoryRelay; `callbacks` are the C function
    pointers ws_engine_sync_relay calls (no Python on the data path)."""

    def __init__(self, lib):
        self.lib = lib
        self.ctx = lib.ref_memrelay_create()
        self.callbacks = (self.ctx, C.cast(lib.ref_memrelay_put, C.c_void_p).value,
                          C.cast(lib.ref_memrelay_get_any, C.c_void_p).value)

    def size(self):
        return int(self.lib.ref_memrelay_size(self.ctx))

    def keys(self, prefix=""):
        n = self.lib.ref_memrelay_list(self.ctx, prefix.encode(), None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self.lib.ref_memrelay_list(self.ctx, prefix.encode(), buf, n)
        return [k for k in buf.raw[:n].decode("utf-8", "surrogateescape").split("\n") if k]

    def get(self, key: str) -> bytes:
        kb = key.encode("utf-8", "surrogateescape")
        n = self.lib.ref_memrelay_get(self.ctx, kb, len(kb), None, 0)
        if n < 0:
            raise KeyError(key)
        out = np.empty(max(1, n), np.uint8)
        self.lib.ref_memrelay_get(self.ctx, kb, len(kb), out.ctypes.data, n)
        return out[:n].tobytes()

    def __del__(self):
        try:
            self.lib.ref_memrelay_destroy(self.ctx)
        except Exception:
            pass
