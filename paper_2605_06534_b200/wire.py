"""The reference's wire format on the device:
payloads (codec.cpp:140-263), bucket keys (key.cpp:47-69), bucket frames
with their zlib CRC-32 (wire.cpp:9-71) and the bucketisation of a shard's
payload (engine.cpp:136-148).  Every byte is produced by libwsync on the GPU;
these wrappers only allocate and marshal."""
import ctypes as C

import torch

from . import _lib
from ._lib import BF16, check, lib
from .codec import SparseDelta, _ptr, _stream

DEFAULT_BUCKET_BYTES = 64 << 20  # SyncOptions::bucket_bytes (engine.hpp:27)
_VAL = {BF16: torch.int16, _lib.I32: torch.int32, _lib.F32: torch.float32}


def payload_bytes(dtype: int, ndims: int, codec: str, index_width: int, count: int) -> int:
    return int(lib.ws_payload_bytes(dtype, ndims, codec.encode(), index_width, count))


def _shape_arr(shape):
    return (C.c_int64 * max(1, len(shape)))(*shape)


def encode_sparse(delta: SparseDelta, index_width: int = 4, device=None) -> torch.Tensor:
    """encode_sparse (codec.cpp:164-183) -> uint8 device tensor."""
    dev = device or delta.indices.device
    n = payload_bytes(delta.dtype, len(delta.shape), "S", index_width, delta.nnz())
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    idx = delta.indices.contiguous()
    val = delta.values.contiguous()
    check(lib.ws_encode_sparse_dev(delta.dtype, _shape_arr(delta.shape), len(delta.shape),
                                   index_width, _ptr(idx), _ptr(val), delta.nnz(), _ptr(out),
                                   _stream()))
    return out


def encode_dense(t: torch.Tensor, dtype: int) -> torch.Tensor:
    """encode_dense (codec.cpp:156-162) -> uint8 device tensor."""
    t = t.contiguous()
    n = payload_bytes(dtype, t.dim(), "D", 0, t.numel())
    out = torch.empty(n, dtype=torch.uint8, device=t.device)
    check(lib.ws_encode_dense_dev(dtype, _shape_arr(tuple(t.shape)), t.dim(), _ptr(t), _ptr(out),
                                  _stream()))
    return out


def peek_payload(buf: torch.Tensor) -> dict:
    """Header + size checks of decode_payload; PayloadFormatError like the
    reference."""
    info = _lib.PayloadInfo()
    check(lib.ws_peek_payload_dev(_ptr(buf), buf.numel(), C.byref(info)))
    return info.as_dict()


def decode_payload(buf: torch.Tensor):
    """decode_payload (codec.cpp:229-263): a SparseDelta, or (dtype, dense
    tensor) for a dense payload."""
    info = _lib.PayloadInfo()
    check(lib.ws_peek_payload_dev(_ptr(buf), buf.numel(), C.byref(info)))
    shape = tuple(info.shape[:info.ndims])
    if info.codec == b"D":
        body = buf[info.header_bytes:]
        return info.dtype, body.view(_VAL[info.dtype]).view(shape)
    idx = torch.empty(info.nnz, dtype=torch.int32, device=buf.device)
    val = torch.empty(info.nnz, dtype=_VAL[info.dtype], device=buf.device)
    check(lib.ws_decode_sparse_dev(_ptr(buf), C.byref(info), _ptr(idx), _ptr(val), _stream()))
    return SparseDelta(info.dtype, shape, idx, val)


def crc32(bufs) -> list:
    """frame_crc32 (wire.cpp:9-13) of each uint8 device tensor."""
    bufs = list(bufs)
    n = len(bufs)
    ptrs = (C.c_void_p * max(1, n))(*[b.data_ptr() for b in bufs])
    lens = (C.c_uint64 * max(1, n))(*[b.numel() for b in bufs])
    out = (C.c_uint32 * max(1, n))()
    check(lib.ws_crc32_dev(ptrs, lens, n, out, _stream()))
    return [int(x) for x in out[:n]]


def bucket_key(step: int, param: str, tp_rank: int, tp_size: int, pp_stage: int, desc,
               codec: str, index_width: int, seq: int) -> str:
    """BucketKey::encode (key.cpp:47-69)."""
    buf = C.create_string_buffer(4096)
    n = C.c_uint64()
    check(lib.ws_bucket_key(step, param.encode(), tp_rank, tp_size, pp_stage,
                            _lib.Shard(*desc), codec.encode(), index_width, seq, buf, 4096,
                            C.byref(n)))
    return buf.raw[:n.value].decode("utf-8", "surrogateescape")


def num_buckets(payload_len: int, bucket_bytes: int) -> int:
    """engine.cpp:139: at least one bucket even for an empty payload."""
    return max(1, -(-payload_len // bucket_bytes))


def encode_bucket_frames(payload: torch.Tensor, bucket_bytes: int, keys) -> tuple:
    """Frames of every bucket of `payload`: (uint8 device tensor, offsets)
    with frame k at [offsets[k], offsets[k+1])."""
    keys = [k.encode("utf-8", "surrogateescape") if isinstance(k, str) else bytes(k) for k in keys]
    nb = num_buckets(payload.numel(), bucket_bytes)
    if len(keys) != nb:
        raise ValueError(f"{nb} buckets need {nb} keys, got {len(keys)}")
    total = sum(12 + len(k) for k in keys) + payload.numel()
    out = torch.empty(max(1, total), dtype=torch.uint8, device=payload.device)
    karr = (C.c_char_p * nb)(*keys)
    klen = (C.c_uint64 * nb)(*[len(k) for k in keys])
    off = (C.c_uint64 * (nb + 1))()
    check(lib.ws_encode_bucket_frames_dev(_ptr(payload), payload.numel(), bucket_bytes, karr, klen,
                                          nb, _ptr(out), out.numel(), off, _stream()))
    return out[:total], [int(x) for x in off]
