"""The weight-sync engine (TransferEngine::sync_step, engine.hpp:70-92) on one
GPU of a box, backed by libwsync.

One process per GPU.  ``Plan`` is the static part (plan_pushes / plan_pulls,
plan.cpp:8-121, extended with FSDP and cross-dim routes); ``TransferEngine``
owns this rank's device arenas (torch tensors: trainer ``prev``/``next``
snapshots and the resident serving shards) and runs one sync per call.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import BF16, F32, I32, check, lib
from .codec import SparseDelta, _ptr, shard_shape
from .manifest import ParamMeta

TORCH_DTYPE = {BF16: torch.bfloat16, I32: torch.int32, F32: torch.float32}
VAL_DTYPE = {BF16: torch.int16, I32: torch.int32, F32: torch.float32}


@dataclass
class TrainConfig:
    """Trainer layout: ``scheme="tp"`` is the reference's TrainConfig{tp,pp,dp}
    (plan.hpp:11-15); ``scheme="fsdp"`` splits every parameter along dim 0
    over all ranks."""
    scheme: str = "fsdp"
    tp: int = 1
    pp: int = 1
    dp: int = 1

    def c(self):
        return _lib.TrainLayout(1 if self.scheme == "fsdp" else 0, self.tp, self.pp, self.dp)


@dataclass
class ServeConfig:
    """ServeConfig{tp,pp} (plan.hpp:17-21) x ``replicas``; ``placement``
    "rank" hosts serving rank g on GPU g, "overlap" assigns serving ranks to
    GPUs for the fewest NVLink bytes (ws_placement)."""
    tp: int = 1
    pp: int = 1
    replicas: int = 1
    placement: str = "rank"

    def c(self):
        codes = {"rank": 0, "overlap": 1}
        if self.placement not in codes:
            raise ValueError(f"unknown placement {self.placement!r}")
        return _lib.ServeLayout(self.tp, self.pp, self.replicas, codes[self.placement])


class Plan:
    def __init__(self, manifest, dtype, train: TrainConfig, serve: ServeConfig, world=1, rank=0):
        self.manifest = [p if isinstance(p, ParamMeta) else ParamMeta(*p) for p in manifest]
        self.dtype = dtype
        self.world, self.rank = world, rank
        arr = (_lib.Param * len(self.manifest))()
        self._names = []
        for i, p in enumerate(self.manifest):
            b = p.name.encode()
            self._names.append(b)
            arr[i].name = b
            arr[i].kind = p.kind
            arr[i].ndims = len(p.shape)
            for k, d in enumerate(p.shape):
                arr[i].shape[k] = d
            arr[i].layer = p.layer
        h = C.c_void_p()
        check(lib.ws_plan_create(arr, len(self.manifest), dtype, C.byref(train.c()),
                                 C.byref(serve.c()), world, rank, C.byref(h)))
        self.h = h
        info = _lib.PlanInfo()
        check(lib.ws_plan_get_info(h, C.byref(info)))
        self.info = info
        self.segments = []
        for i in range(info.num_segments):
            p, d, off, n = C.c_int32(), _lib.Shard(), C.c_uint64(), C.c_uint64()
            check(lib.ws_plan_segment(h, i, C.byref(p), C.byref(d), C.byref(off), C.byref(n)))
            self.segments.append((p.value, (d.slice_dim, d.start, d.end), off.value, n.value))
        self.serve_shards = []
        for i in range(info.num_serve_shards):
            p, d, off, n = C.c_int32(), _lib.Shard(), C.c_uint64(), C.c_uint64()
            check(lib.ws_plan_serve_shard(h, i, C.byref(p), C.byref(d), C.byref(off),
                                          C.byref(n)))
            self.serve_shards.append((p.value, (d.slice_dim, d.start, d.end), off.value, n.value))
        # serving coordinate of every serving shard (all coordinates on a
        # one-GPU plan of a multi-rank layout)
        self.serve_coords = []
        for i in range(info.num_serve_shards):
            c = C.c_int32()
            check(lib.ws_plan_serve_shard_coord(h, i, C.byref(c)))
            self.serve_coords.append(c.value)
        self.routes = []
        for i in range(info.num_routes):
            s, c, r, ov = C.c_int32(), C.c_int32(), C.c_int32(), C.c_uint64()
            check(lib.ws_plan_route(h, i, C.byref(s), C.byref(c), C.byref(r), C.byref(ov)))
            self.routes.append((s.value, c.value, r.value, ov.value))

    def segment_key_fields(self, i):
        """(tp_rank, tp_size, pp_stage) of segment i's ShardDescriptor."""
        r, n, g = C.c_int32(), C.c_int32(), C.c_int32()
        check(lib.ws_plan_segment_key_fields(self.h, i, C.byref(r), C.byref(n), C.byref(g)))
        return r.value, n.value, g.value

    def __del__(self):
        try:
            lib.ws_plan_destroy(self.h)
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib.ws_nccl_unique_id(buf))
    return bytes(buf)


class TransferEngine:
    """One rank's engine.  Arenas are torch CUDA tensors owned here."""

    def __init__(self, plan: Plan, device=None, unique_id: bytes | None = None, group=None):
        self.h = None
        self.plan = plan
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else device)
        td = TORCH_DTYPE[plan.dtype]
        info = plan.info
        with torch.cuda.device(self.device):
            self.arena = [torch.zeros(max(1, info.train_arena_elems), dtype=td,
                                      device=self.device) for _ in range(2)]
            self.serve = torch.zeros(max(1, info.serve_arena_elems), dtype=td, device=self.device)
        uid = None
        if unique_id is not None:
            uid = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        if group is not None:
            check(lib.ws_engine_create_grouped(plan.h, self.device.index, group.h, C.byref(h)))
        else:
            check(lib.ws_engine_create(plan.h, self.device.index, uid, C.byref(h)))
        self.h = h
        check(lib.ws_engine_bind(h, self.arena[0].data_ptr(), self.arena[1].data_ptr(),
                                 self.serve.data_ptr()))

    def close(self):
        if self.h is not None:
            lib.ws_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- data access -------------------------------------------------------
    def segment_view(self, i, which=0):
        """Trainer shard i in arena ``which`` (0 = prev, 1 = next), shaped."""
        p, desc, off, n = self.plan.segments[i]
        shp = shard_shape(self.plan.manifest[p].shape, desc)
        return self.arena[which][off:off + n].view(shp)

    def serve_view(self, i):
        p, desc, off, n = self.plan.serve_shards[i]
        shp = shard_shape(self.plan.manifest[p].shape, desc)
        return self.serve[off:off + n].view(shp)

    # ---- sync ----------------------------------------------------------------
    def generate(self, seed=1, density=0.01, expert_zipf=None, perm_seed=0):
        """Synthetic prev/next in the trainer arenas and prev in the serving
        arena; expert_zipf=s skews the density of EXPERT tensors per expert
        (expert_thresholds)."""
        with torch.cuda.device(self.device):
            if expert_zipf is None:
                check(lib.ws_engine_generate(self.h, seed, density, _stream()))
            else:
                check(lib.ws_engine_generate_skewed(self.h, seed, density, float(expert_zipf),
                                                    perm_seed, _stream()))

    def sync_step(self, sparse=True, density_threshold=0.20, reverse=False, report=True,
                  stream=None):
        o = _lib.SyncOptions(int(sparse), density_threshold, int(reverse))
        rep = _lib.Report() if report else None
        with torch.cuda.device(self.device):
            check(lib.ws_engine_sync_step(self.h, C.byref(o), _stream(stream),
                                          C.byref(rep) if rep is not None else None))
        return rep.as_dict() if rep is not None else None

    def sync_step_host(self, next_host: torch.Tensor, sparse=True, density_threshold=0.20,
                       reverse=False, report=True, stream=None):
        """Reads the new snapshot from host memory (pinned for full speed)."""
        if next_host.device.type != "cpu" or next_host.numel() < self.plan.info.train_arena_elems:
            raise _lib.InvalidArgument("sync_step_host: host snapshot of the trainer arena needed")
        o = _lib.SyncOptions(int(sparse), density_threshold, int(reverse))
        rep = _lib.Report() if report else None
        nnz = (C.c_uint64 * max(1, len(self.plan.segments)))()
        with torch.cuda.device(self.device):
            check(lib.ws_engine_sync_step_host(self.h, next_host.data_ptr(), C.byref(o),
                                               _stream(stream), nnz,
                                               C.byref(rep) if rep is not None else None))
        return (rep.as_dict() if rep is not None else None), list(nnz)

    def timing(self, reset=True):
        """Per-stage device-time totals of the syncs since the last reset."""
        t = _lib.Timing()
        with torch.cuda.device(self.device):
            check(lib.ws_engine_timing(self.h, int(reset), C.byref(t)))
        return t.as_dict()

    def exchange_bytes(self):
        """NVLink bytes of the last sync on this rank: wire records sent (one
        copy per replica), dense boxes sent, wire records received --
        ws_engine_exchange_bytes."""
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        with torch.cuda.device(self.device):
            check(lib.ws_engine_exchange_bytes(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return {"sent_record_bytes": a.value, "sent_dense_bytes": b.value,
                "recv_record_bytes": c.value}

    def segment_payload(self, i, force_wide_index=False):
        """Segment i's payload from the last sync in the reference wire format
        (what engine.cpp:116-128 puts on the relay): (uint8 device tensor, info)."""
        info = _lib.PayloadInfo()
        with torch.cuda.device(self.device):
            check(lib.ws_engine_payload(self.h, i, int(force_wide_index), None, C.byref(info),
                                        _stream()))
            out = torch.empty(max(8, info.total_bytes), dtype=torch.uint8, device=self.device)
            check(lib.ws_engine_payload(self.h, i, int(force_wide_index), _ptr(out),
                                        C.byref(info), _stream()))
        return out[:info.total_bytes], info.as_dict()

    def sync_relay(self, relay, step=1, sparse=True, density_threshold=0.20, reverse=False,
                   bucket_bytes=64 << 20, mode="async", push_bytes_per_s=0.0,
                   pull_bytes_per_s=0.0, burst_bytes=0.0, timeout_ms=10000,
                   force_wide_index=False, staging_buffers=2):
        """TransferEngine::sync_step across clusters (engine.cpp:66-254): this
        GPU pushes its trainer shards through `relay` -- a (ctx, put, get_any)
        triple of C pointers implementing ws_relay -- and pulls every shard
        routed to its serving coordinate, from any rank; mode "async" or
        "batch" (SyncMode).  With world > 1 every rank calls it for the same
        step on a relay the ranks share."""
        o = _lib.SyncOptions(int(sparse), density_threshold, int(reverse))
        ro = _lib.RelayOptions(bucket_bytes, 256 << 20, push_bytes_per_s, pull_bytes_per_s,
                               burst_bytes, timeout_ms, int(mode == "async"),
                               int(force_wide_index), staging_buffers)
        rl = _lib.Relay(*relay)
        rep = _lib.RelayReport()
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            check(lib.ws_engine_sync_relay(self.h, step, C.byref(o), C.byref(ro), C.byref(rl),
                                           C.byref(rep)))
        return rep.as_dict()

    def release_staging(self):
        """Frees sync_relay's staging and cached decode scratch
        (ws_engine_release_staging)."""
        with torch.cuda.device(self.device):
            check(lib.ws_engine_release_staging(self.h))

    def segment_frames(self, i, step, bucket_bytes=None, force_wide_index=False):
        """The relay frames of segment i for `step` (engine.cpp:136-148 +
        wire.cpp:35-47): (uint8 device tensor, keys, frame offsets)."""
        from . import wire
        bucket_bytes = bucket_bytes or wire.DEFAULT_BUCKET_BYTES
        payload, info = self.segment_payload(i, force_wide_index)
        p, desc, off, n = self.plan.segments[i]
        r, size, stage = self.plan.segment_key_fields(i)
        name = self.plan.manifest[p].name
        nb = wire.num_buckets(info["total_bytes"], bucket_bytes)
        keys = [wire.bucket_key(step, name, r, size, stage, desc, info["codec"],
                                info["index_width"], q) for q in range(nb)]
        with torch.cuda.device(self.device):
            frames, offs = wire.encode_bucket_frames(payload, bucket_bytes, keys)
        return frames, keys, offs

    def segment_delta(self, i) -> tuple:
        """(SparseDelta of segment i from the last sync, codec 'S'/'D')."""
        idx, val, nnz, codec = C.c_void_p(), C.c_void_p(), C.c_uint64(), C.create_string_buffer(1)
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            check(lib.ws_engine_segment_delta(self.h, i, C.byref(idx), C.byref(val),
                                              C.byref(nnz), codec))
        p, desc, off, n = self.plan.segments[i]
        shp = shard_shape(self.plan.manifest[p].shape, desc)
        c = codec.raw[:1].decode()
        k = nnz.value if c == "S" else 0
        return SparseDelta(self.plan.dtype, shp, _wrap(idx.value, k, torch.int32, self.device),
                           _wrap(val.value, k, VAL_DTYPE[self.plan.dtype], self.device)), c, nnz.value


    def segment_stream(self, i):
        """Segment i's records as K1 wrote them in the last sync (one run per
        super-tile, runs in reservation order, ascending inside each):
        (idx int32 tensor, val tensor, super-tile elements) --
        ws_engine_segment_stream."""
        idx, val, n, te = C.c_void_p(), C.c_void_p(), C.c_uint64(), C.c_uint64()
        with torch.cuda.device(self.device):
            check(lib.ws_engine_segment_stream(self.h, i, C.byref(idx), C.byref(val), C.byref(n),
                                               C.byref(te)))
        k = n.value
        return (_wrap(idx.value, k, torch.int32, self.device),
                _wrap(val.value, k, VAL_DTYPE[self.plan.dtype], self.device), te.value)


class EngineGroup:
    """Every rank of a multi-GPU layout as an engine of THIS process on one
    GPU (ws_group, include/wsync.h): the ranks share mailboxes, receive
    regions and serving arenas as plain device pointers, and one group sync
    runs all ranks' kernels -- K1, the local route, the NVLink pack
    (pack_kernel) and the receive-side apply (apply_p2p_kernel) -- phase by
    phase on one stream.  It is the multi-GPU data path of any layout
    (TrainConfig{tp,pp,dp} -> ServeConfig{tp,pp} x replicas, FSDP, EP) on a
    single device, which is how the parity tests run it on one B200."""

    def __init__(self, manifest, dtype, train: TrainConfig, serve: ServeConfig, world: int,
                 device=None):
        """device: one GPU for every rank, or a list with one GPU per rank
        (the ranks then sync concurrently, each on its GPU, peer memory over
        NVLink)."""
        self.world = world
        devices = list(device) if isinstance(device, (list, tuple)) else [device] * world
        self.plans = [Plan(manifest, dtype, train, serve, world=world, rank=r)
                      for r in range(world)]
        h = C.c_void_p()
        check(lib.ws_group_create(world, C.byref(h)))
        self.h = h
        self.engines = []
        try:
            for plan, dev in zip(self.plans, devices):
                self.engines.append(TransferEngine(plan, dev, group=self))
            with torch.cuda.device(self.engines[0].device):
                check(lib.ws_group_connect(h))
        except Exception:
            self.close()
            raise

    def generate(self, seed=1, density=0.01, expert_zipf=None, perm_seed=0):
        for e in self.engines:
            e.generate(seed=seed, density=density, expert_zipf=expert_zipf, perm_seed=perm_seed)

    def sync_step(self, sparse=True, density_threshold=0.20, reverse=False, report=True,
                  stream=None):
        """One sync of every rank (ws_group_sync_step); per-rank reports."""
        o = _lib.SyncOptions(int(sparse), density_threshold, int(reverse))
        reps = (_lib.Report * self.world)() if report else None
        with torch.cuda.device(self.engines[0].device):
            check(lib.ws_group_sync_step(self.h, C.byref(o), _stream(stream), reps))
        return [r.as_dict() for r in reps] if report else None

    def close(self):
        for e in getattr(self, "engines", []):
            e.close()
        if getattr(self, "h", None) is not None:
            lib.ws_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class _CudaArray:
    def __init__(self, ptr, n, typestr, device):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


def _wrap(ptr, n, dtype, device):
    """Zero-copy torch view of engine-owned device memory (copied for safety)."""
    if n == 0 or not ptr:
        return torch.empty(0, dtype=dtype, device=device)
    typestr = {torch.int32: "<i4", torch.int16: "<i2", torch.float32: "<f4"}[dtype]
    return torch.as_tensor(_CudaArray(ptr, n, typestr, device), device=device).clone()
