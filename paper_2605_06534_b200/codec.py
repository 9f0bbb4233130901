"""The reference's codec API (proj/include/coserve/transfer/codec.hpp,
shard.hpp) on CUDA tensors, backed by libwsync's sm_100a kernels.

Names, argument meaning and error behaviour follow the reference:

* ``diff_shards(prev, next)``           codec.hpp:37  / codec.cpp:34-63
* ``apply_delta(target, delta)``        codec.hpp:41  / codec.cpp:65-92
* ``reslice_delta(delta, src, dst, full_shape)``  codec.hpp:46-48 / codec.cpp:94-138
* ``extract_shard(full, desc)``         shard.hpp:57  / shard.cpp:111-134
* ``copy_overlap(...)``                 shard.hpp:62-63 / shard.cpp:136-170

Shard descriptors are ``(slice_dim, start, end)`` tuples with ``slice_dim < 0``
for the full tensor (ShardDescriptor, shard.hpp:32-45).  Tensors are CUDA
tensors of dtype bfloat16 (the extension: 16-bit words, bit-pattern compare,
wrap-around delta), int32 or float32 (the reference's DType, tensor.hpp:26).
bf16 delta values are raw u16 words carried in an int16 tensor.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (BF16, F32, I32, IndexOutOfShard, ShapeMismatch, check, lib,
                   raise_device_error, shape_array, shard)

_DT = {torch.bfloat16: BF16, torch.int32: I32, torch.float32: F32}
_VAL_DTYPE = {BF16: torch.int16, I32: torch.int32, F32: torch.float32}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise _lib.InvalidArgument(f"unsupported dtype {t.dtype}") from None


def _stream(device=None):
    """The current stream of `device` (default: the current device).  Calls on
    tensors of another GPU run under torch.cuda.device(tensor.device), so the
    library launches there."""
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() else C.c_void_p(0)


@dataclass
class SparseDelta:
    """codec.hpp:16-32: ascending unique local flat indices (u32 carried as
    int32) and raw values of the dtype width."""
    dtype: int
    shape: tuple
    indices: torch.Tensor
    values: torch.Tensor

    def elems(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    def nnz(self) -> int:
        return int(self.indices.numel())

    def density(self) -> float:  # codec.hpp:28-31
        n = self.elems()
        return 0.0 if n == 0 else self.nnz() / n


def shard_shape(full_shape, desc):
    """shard.cpp:81-86."""
    s = list(full_shape)
    if desc[0] >= 0:
        s[desc[0]] = desc[2] - desc[1]
    return tuple(s)


def _workspace(n, device):
    return torch.empty(int(lib.ws_diff_workspace_bytes(n)), dtype=torch.uint8, device=device)


def diff_shards(prev: torch.Tensor, next_: torch.Tensor, cap: int | None = None) -> SparseDelta:
    """Every position whose value changed, ascending (K1 on one shard)."""
    with torch.cuda.device(prev.device):
        if prev.dtype != next_.dtype or tuple(prev.shape) != tuple(next_.shape):
            raise ShapeMismatch(f"diff_shards: {list(prev.shape)} vs {list(next_.shape)}")
        dt = dtype_code(prev)
        prev = prev.contiguous()
        next_ = next_.contiguous()
        n = prev.numel()
        cap = n if cap is None else cap
        dev = prev.device
        idx = torch.empty(max(1, cap), dtype=torch.int32, device=dev)
        val = torch.empty(max(1, cap), dtype=_VAL_DTYPE[dt], device=dev)
        nnz = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = _workspace(n, dev)
        check(lib.ws_diff_shards(dt, _ptr(prev), _ptr(next_), n, _ptr(idx), _ptr(val), cap,
                                 _ptr(nnz), _ptr(ws), ws.numel(), _stream()))
        k = int(nnz.item())
        k = min(k, cap)
        return SparseDelta(dt, tuple(prev.shape), idx[:k], val[:k])


def apply_delta(target: torch.Tensor, delta: SparseDelta) -> None:
    """In place ``target += delta``; validates every index before writing."""
    with torch.cuda.device(target.device):
        dt = dtype_code(target)
        if dt != delta.dtype or tuple(target.shape) != tuple(delta.shape):
            raise ShapeMismatch(f"apply_delta: target {list(target.shape)} vs delta "
                                f"{list(delta.shape)}")
        if not target.is_contiguous():
            raise _lib.InvalidArgument("apply_delta: target must be contiguous")
        err = torch.zeros(1, dtype=torch.int32, device=target.device)
        check(lib.ws_apply_delta(dt, _ptr(target), target.numel(), _ptr(delta.indices),
                                 _ptr(delta.values), delta.nnz(), None, _ptr(err), _stream()))
        raise_device_error(int(err.item()), "apply_delta")


def reslice_delta(delta: SparseDelta, src, dst, full_shape, allow_cross_dim: bool = True
                  ) -> SparseDelta:
    """Re-express a delta local to ``src`` as one local to ``dst``."""
    with torch.cuda.device(delta.indices.device):
        full_shape = tuple(int(d) for d in full_shape)
        if tuple(delta.shape) != shard_shape(full_shape, src):
            raise ShapeMismatch(f"reslice_delta: delta {list(delta.shape)} does not match source "
                                f"shard {list(shard_shape(full_shape, src))}")
        nnz = delta.nnz()
        dev = delta.indices.device
        out_idx = torch.empty(max(1, nnz), dtype=torch.int32, device=dev)
        out_val = torch.empty(max(1, nnz), dtype=delta.values.dtype, device=dev)
        out_n = torch.zeros(1, dtype=torch.int64, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        ws = _workspace(nnz, dev)
        check(lib.ws_reslice_delta(delta.dtype, shape_array(full_shape), len(full_shape),
                                   shard(src), shard(dst), int(allow_cross_dim),
                                   _ptr(delta.indices), _ptr(delta.values), nnz, None,
                                   _ptr(out_idx), _ptr(out_val), _ptr(out_n), _ptr(err), _ptr(ws),
                                   ws.numel(), _stream()))
        bits = int(err.item())
        if bits:
            raise IndexOutOfShard("reslice_delta: delta index outside the source shard")
        k = int(out_n.item())
        return SparseDelta(delta.dtype, shard_shape(full_shape, dst), out_idx[:k], out_val[:k])


def extract_shard(full: torch.Tensor, desc) -> torch.Tensor:
    """Copy of the descriptor's slice of ``full``."""
    with torch.cuda.device(full.device):
        dt = dtype_code(full)
        full = full.contiguous()
        out = torch.empty(shard_shape(full.shape, desc), dtype=full.dtype, device=full.device)
        check(lib.ws_extract_shard(dt, shape_array(full.shape), full.dim(), shard(desc), _ptr(full),
                                   _ptr(out), _stream()))
        return out


def copy_overlap(dst: torch.Tensor, dst_desc, src: torch.Tensor, src_desc, full_shape) -> int:
    """Copy the overlap of shard ``src`` into shard ``dst`` (both of one tensor
    of ``full_shape``); returns the copied element count."""
    with torch.cuda.device(dst.device):
        dt = dtype_code(dst)
        if src.dtype != dst.dtype:
            raise ShapeMismatch("copy_overlap dtype mismatch")
        full_shape = tuple(int(d) for d in full_shape)
        if tuple(dst.shape) != shard_shape(full_shape, dst_desc) or \
                tuple(src.shape) != shard_shape(full_shape, src_desc):
            raise ShapeMismatch("copy_overlap: shard shape mismatch")
        copied = C.c_int64()
        check(lib.ws_copy_overlap(dt, shape_array(full_shape), len(full_shape), shard(dst_desc),
                                  _ptr(dst), shard(src_desc), _ptr(src.contiguous()),
                                  C.byref(copied), _stream()))
        return copied.value


def expert_thresholds(experts: int, density: float, zipf_s: float, perm_seed: int = 0):
    """Per-expert change thresholds (floor(density_e * 2^32)) of config 4."""
    out = (C.c_uint64 * experts)()
    check(lib.ws_expert_thresholds(experts, density, zipf_s, perm_seed, out))
    return [int(x) for x in out]


def gen_pair_bf16(seed: int, name: str, full_shape, desc, density: float, device="cuda",
                  thr_dim0=None):
    """Synthetic bf16 pair for one shard (device generator); thr_dim0: optional
    per-dim-0-index thresholds (expert_thresholds) replacing `density`."""
    with torch.cuda.device(torch.device(device)):
        shp = shard_shape(full_shape, desc)
        prev = torch.empty(shp, dtype=torch.bfloat16, device=device)
        nxt = torch.empty(shp, dtype=torch.bfloat16, device=device)
        if thr_dim0 is not None:
            tab = torch.tensor(list(thr_dim0), dtype=torch.int64, device=device)
            check(lib.ws_gen_pair_bf16_dim0(seed, name.encode(), shape_array(full_shape),
                                            len(full_shape), shard(desc), _ptr(tab), _ptr(prev),
                                            _ptr(nxt), _stream()))
            torch.cuda.current_stream(device).synchronize()
            return prev, nxt
        thr = int(min(max(density, 0.0), 1.0) * 4294967296.0)
        check(lib.ws_gen_pair_bf16(seed, name.encode(), shape_array(full_shape), len(full_shape),
                                   shard(desc), thr, _ptr(prev), _ptr(nxt), _stream()))
        return prev, nxt
