"""ctypes binding of libwsync.so (include/wsync.h).

The product path has no fallback: if the CUDA library is missing this module
raises on import, and every entry point of the package goes through it.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WSYNC_LIB") or os.path.join(HERE, "lib", "libwsync.so")

# ---- ws_status -> the reference's TransferError hierarchy (tensor.hpp:16-24,
# codec.hpp:9-11, shard.hpp:9-14, plan.hpp:7-9, relay.hpp:17-22, key.hpp:10-12)


class TransferError(RuntimeError):
    status = 10


class ShapeMismatch(TransferError):
    status = 1


class PayloadFormatError(TransferError):
    status = 2


class IndexOutOfShard(TransferError):
    status = 3


class IndivisibleShape(TransferError):
    status = 4


class UnknownModuleKind(TransferError):
    status = 5


class IncompleteCoverage(TransferError):
    status = 6


class RelayTimeout(TransferError):
    status = 7


class IntegrityError(TransferError):
    status = 8


class KeyFormatError(TransferError):
    status = 9


class CudaError(TransferError):
    status = 20


class NcclError(TransferError):
    status = 21


class CapacityError(TransferError):
    status = 22


class InvalidArgument(TransferError):
    status = 23


_BY_STATUS = {c.status: c for c in (TransferError, ShapeMismatch, PayloadFormatError,
                                    IndexOutOfShard, IndivisibleShape, UnknownModuleKind,
                                    IncompleteCoverage, RelayTimeout, IntegrityError,
                                    KeyFormatError, CudaError, NcclError, CapacityError,
                                    InvalidArgument)}

F32, I32, BF16 = 0, 1, 2
ERRBIT_INDEX_OUT_OF_SHARD = 0x1
MAX_DIMS = 4


class Shard(C.Structure):  # ws_shard
    _fields_ = [("slice_dim", C.c_int32), ("start", C.c_int64), ("end", C.c_int64)]


class Param(C.Structure):  # ws_param
    _fields_ = [("name", C.c_char_p), ("kind", C.c_int32), ("ndims", C.c_int32),
                ("shape", C.c_int64 * MAX_DIMS), ("layer", C.c_int32)]


class TrainLayout(C.Structure):  # ws_train_layout
    _fields_ = [("scheme", C.c_int32), ("tp", C.c_int32), ("pp", C.c_int32), ("dp", C.c_int32)]


class ServeLayout(C.Structure):  # ws_serve_layout
    _fields_ = [("tp", C.c_int32), ("pp", C.c_int32), ("replicas", C.c_int32),
                ("placement", C.c_int32)]


class PlanInfo(C.Structure):  # ws_plan_info
    _fields_ = [("num_segments", C.c_int32), ("num_serve_shards", C.c_int32),
                ("num_routes", C.c_int32), ("serve_coord", C.c_int32),
                ("train_arena_elems", C.c_uint64), ("serve_arena_elems", C.c_uint64),
                ("train_elems", C.c_uint64), ("model_elems", C.c_uint64),
                ("serve_rank", C.c_int32), ("serve_replica", C.c_int32)]


class SyncOptions(C.Structure):  # ws_sync_options
    _fields_ = [("sparse", C.c_int32), ("density_threshold", C.c_double),
                ("reverse", C.c_int32)]


class Report(C.Structure):  # ws_report
    _fields_ = [("wall_s", C.c_double), ("encode_s", C.c_double), ("route_s", C.c_double),
                ("apply_s", C.c_double), ("pushed_bytes", C.c_uint64),
                ("pulled_bytes", C.c_uint64), ("nnz", C.c_uint64),
                ("dense_shards", C.c_int32), ("sparse_shards", C.c_int32),
                ("kernel_launches", C.c_uint32), ("streamed_apply", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Timing(C.Structure):  # ws_timing
    _fields_ = [("steps", C.c_uint32), ("kernel_launches", C.c_uint32), ("wall_s", C.c_double),
                ("encode_s", C.c_double), ("route_s", C.c_double), ("apply_s", C.c_double),
                ("pack_steps", C.c_uint32), ("pack_s", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class PayloadInfo(C.Structure):  # ws_payload_info
    _fields_ = [("codec", C.c_char), ("dtype", C.c_int32), ("ndims", C.c_int32),
                ("index_width", C.c_int32), ("shape", C.c_int64 * 8), ("nnz", C.c_uint64),
                ("header_bytes", C.c_uint64), ("total_bytes", C.c_uint64)]

    def as_dict(self):
        return {"codec": self.codec.decode(), "dtype": self.dtype, "ndims": self.ndims,
                "index_width": self.index_width, "shape": tuple(self.shape[:self.ndims]),
                "nnz": self.nnz, "header_bytes": self.header_bytes,
                "total_bytes": self.total_bytes}


class Relay(C.Structure):  # ws_relay (function pointers passed as raw addresses)
    _fields_ = [("ctx", C.c_void_p), ("put", C.c_void_p), ("get_any", C.c_void_p),
                ("put_frame", C.c_void_p), ("get_any_frame", C.c_void_p)]


class RelayOptions(C.Structure):  # ws_relay_options
    _fields_ = [("bucket_bytes", C.c_uint64), ("pull_batch_bytes", C.c_uint64),
                ("push_bytes_per_s", C.c_double), ("pull_bytes_per_s", C.c_double),
                ("burst_bytes", C.c_double), ("timeout_ms", C.c_int32), ("async_", C.c_int32),
                ("force_wide_index", C.c_int32), ("staging_buffers", C.c_int32)]


class RelayReport(C.Structure):  # ws_relay_report
    _fields_ = [("wall_s", C.c_double), ("push_s", C.c_double), ("pull_s", C.c_double),
                ("encode_s", C.c_double), ("apply_s", C.c_double), ("pushed_bytes", C.c_uint64),
                ("pulled_bytes", C.c_uint64), ("push_buckets", C.c_uint64),
                ("pull_buckets", C.c_uint64), ("dense_shards", C.c_uint32),
                ("sparse_shards", C.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_vp, _u64, _i64, _i32 = C.c_void_p, C.c_uint64, C.c_int64, C.c_int32
_SIGS = {
    "ws_status_name": ([C.c_int], C.c_char_p),
    "ws_last_error": ([], C.c_char_p),
    "ws_abi_version": ([], C.c_int),
    "ws_diff_workspace_bytes": ([_u64], C.c_size_t),
    "ws_diff_shards": ([C.c_int, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp, C.c_size_t, _vp],
                       C.c_int),
    "ws_apply_delta": ([C.c_int, _vp, _u64, _vp, _vp, _u64, _vp, _vp, _vp], C.c_int),
    "ws_reslice_delta": ([C.c_int, C.POINTER(_i64), C.c_int, Shard, Shard, C.c_int, _vp, _vp,
                          _u64, _vp, _vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp], C.c_int),
    "ws_copy_overlap": ([C.c_int, C.POINTER(_i64), C.c_int, Shard, _vp, Shard, _vp,
                         C.POINTER(_i64), _vp], C.c_int),
    "ws_extract_shard": ([C.c_int, C.POINTER(_i64), C.c_int, Shard, _vp, _vp, _vp], C.c_int),
    "ws_gen_pair_bf16": ([_u64, C.c_char_p, C.POINTER(_i64), C.c_int, Shard, _u64, _vp, _vp,
                          _vp], C.c_int),
    "ws_gen_pair_bf16_dim0": ([_u64, C.c_char_p, C.POINTER(_i64), C.c_int, Shard, _vp, _vp, _vp,
                               _vp], C.c_int),
    "ws_expert_thresholds": ([C.c_int, C.c_double, C.c_double, _u64, C.POINTER(_u64)], C.c_int),
    "ws_payload_bytes": ([C.c_int, C.c_int, C.c_char, C.c_int, _u64], _u64),
    "ws_encode_sparse_dev": ([C.c_int, C.POINTER(_i64), C.c_int, C.c_int, _vp, _vp, _u64, _vp,
                              _vp], C.c_int),
    "ws_encode_dense_dev": ([C.c_int, C.POINTER(_i64), C.c_int, _vp, _vp, _vp], C.c_int),
    "ws_peek_payload_dev": ([_vp, _u64, C.POINTER(PayloadInfo)], C.c_int),
    "ws_peek_payload_size_dev": ([_vp, _u64, C.POINTER(_u64)], C.c_int),
    "ws_decode_sparse_dev": ([_vp, C.POINTER(PayloadInfo), _vp, _vp, _vp], C.c_int),
    "ws_crc32_dev": ([C.POINTER(_vp), C.POINTER(_u64), C.c_int, C.POINTER(C.c_uint32), _vp],
                     C.c_int),
    "ws_encode_bucket_frames_dev": ([_vp, _u64, _u64, C.POINTER(C.c_char_p), C.POINTER(_u64),
                                     C.c_int, _vp, _u64, C.POINTER(_u64), _vp], C.c_int),
    "ws_bucket_key": ([_u64, C.c_char_p, C.c_int, C.c_int, C.c_int, Shard, C.c_char, C.c_int,
                       C.c_uint32, C.c_char_p, _u64, C.POINTER(_u64)], C.c_int),
    "ws_plan_check_exchange": ([_vp, C.c_int], C.c_int),
    "ws_plan_exchange_rounds": ([_vp, C.POINTER(C.c_int32)], C.c_int),
    "ws_plan_segment_key_fields": ([_vp, C.c_int, C.POINTER(_i32), C.POINTER(_i32),
                                    C.POINTER(_i32)], C.c_int),
    "ws_engine_sync_relay": ([_vp, _u64, C.POINTER(SyncOptions), C.POINTER(RelayOptions),
                              C.POINTER(Relay), C.POINTER(RelayReport)], C.c_int),
    "ws_engine_payload": ([_vp, C.c_int, C.c_int, _vp, C.POINTER(PayloadInfo), _vp], C.c_int),
    "ws_plan_create": ([C.POINTER(Param), C.c_int, C.c_int, C.POINTER(TrainLayout),
                        C.POINTER(ServeLayout), C.c_int, C.c_int, C.POINTER(_vp)], C.c_int),
    "ws_plan_destroy": ([_vp], None),
    "ws_plan_get_info": ([_vp, C.POINTER(PlanInfo)], C.c_int),
    "ws_plan_segment": ([_vp, C.c_int, C.POINTER(_i32), C.POINTER(Shard), C.POINTER(_u64),
                         C.POINTER(_u64)], C.c_int),
    "ws_plan_serve_shard": ([_vp, C.c_int, C.POINTER(_i32), C.POINTER(Shard), C.POINTER(_u64),
                             C.POINTER(_u64)], C.c_int),
    "ws_plan_route": ([_vp, C.c_int, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32),
                       C.POINTER(_u64)], C.c_int),
    "ws_plan_exchange_caps": ([_vp, C.POINTER(_u64), C.POINTER(_u64)], C.c_int),
    "ws_nccl_unique_id": ([C.POINTER(C.c_uint8)], C.c_int),
    "ws_engine_create": ([_vp, C.c_int, C.POINTER(C.c_uint8), C.POINTER(_vp)], C.c_int),
    "ws_engine_destroy": ([_vp], None),
    "ws_engine_bind": ([_vp, _vp, _vp, _vp], C.c_int),
    "ws_engine_generate": ([_vp, _u64, C.c_double, _vp], C.c_int),
    "ws_engine_generate_skewed": ([_vp, _u64, C.c_double, C.c_double, _u64, _vp], C.c_int),
    "ws_engine_sync_step": ([_vp, C.POINTER(SyncOptions), _vp, C.POINTER(Report)], C.c_int),
    "ws_engine_sync_step_host": ([_vp, _vp, C.POINTER(SyncOptions), _vp, C.POINTER(_u64),
                                  C.POINTER(Report)], C.c_int),
    "ws_engine_timing": ([_vp, C.c_int, C.POINTER(Timing)], C.c_int),
    "ws_engine_exchange_bytes": ([_vp, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)],
                                 C.c_int),
    "ws_engine_release_staging": ([_vp], C.c_int),
    "ws_plan_serve_shard_coord": ([_vp, C.c_int, C.POINTER(_i32)], C.c_int),
    "ws_engine_segment_counts": ([_vp, C.POINTER(_u64), C.c_char_p], C.c_int),
    "ws_group_create": ([C.c_int, C.POINTER(_vp)], C.c_int),
    "ws_group_destroy": ([_vp], None),
    "ws_engine_create_grouped": ([_vp, C.c_int, _vp, C.POINTER(_vp)], C.c_int),
    "ws_group_connect": ([_vp], C.c_int),
    "ws_group_sync_step": ([_vp, C.POINTER(SyncOptions), _vp, _vp], C.c_int),
    "ws_engine_segment_delta": ([_vp, C.c_int, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_u64),
                                 C.c_char_p], C.c_int),
    "ws_engine_segment_stream": ([_vp, C.c_int, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_u64),
                                  C.POINTER(_u64)], C.c_int),
}

SYMBOLS = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libwsync.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; "
            f"g.build()'` -- there is no CPU fallback for the sync path")
    # torch first: libwsync needs libnccl.so.2 / libcudart, which torch already mapped.
    import torch  # noqa: F401
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def check(status):
    """Raise the reference-named exception for a non-OK ws_status."""
    if status:
        msg = lib.ws_last_error().decode(errors="replace")
        raise _BY_STATUS.get(status, TransferError)(msg)


def raise_device_error(bits, what):
    if bits & ERRBIT_INDEX_OUT_OF_SHARD:
        raise IndexOutOfShard(f"{what}: delta index outside the shard")
    if bits:
        raise TransferError(f"{what}: device error bits {bits:#x}")


def shape_array(shape):
    return (C.c_int64 * max(1, len(shape)))(*shape)


def shard(desc):
    """(slice_dim, start, end) -> ws_shard; slice_dim < 0 means full."""
    d, s, e = desc
    return Shard(d, s if d >= 0 else 0, e if d >= 0 else 0)
