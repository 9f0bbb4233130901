"""The GPU-aware relay path: ws_engine_sync_relay runs
TransferEngine::sync_step's pusher and puller (engine.cpp:66-254) with the
encode/decode/reslice/apply on the GPU, through the reference's own
MemoryRelay (relay.cpp, compiled in oracle/_ref).  Checked: the serving
weights equal the synthetic `next` bit for bit; the relay holds exactly the
keys the reference pusher would put, each bucket byte-equal to the
reference encoding of the oracle delta (or dense snapshot); Batch and Async
agree; TokenBucket pacing holds the push rate; Async overlaps (mode
ordering)."""
import struct

import numpy as np
import pytest
import torch

from oracle.oracle import BF16

pytestmark = pytest.mark.gpu


def _engine(layers=2, hidden=64, vocab=256):
    import paper_2605_06534_b200 as ws
    plan = ws.Plan(ws.toy_transformer_manifest(layers=layers, hidden=hidden, vocab=vocab), ws.BF16,
                   ws.TrainConfig("fsdp"), ws.ServeConfig(1, 1, 1))
    return ws, plan, ws.TransferEngine(plan, device=0)


def _bits(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16).ravel()


def _expected_payload(restatement, ws, meta, desc, n, seed, density):
    prev, nxt = restatement.gen_pair_bf16(seed, meta.name, meta.shape, desc, density)
    wi, wv = restatement.diff_shards(BF16, prev, nxt)
    shp = ws.shard_shape(meta.shape, desc)
    if restatement.is_sparse(wi.size, n, 0.20):
        return restatement.encode_sparse(BF16, shp, wi.astype(np.uint64), wv, 4), "S", 4, nxt
    body = b"CWD2" + bytes([BF16, len(shp), 0, 0]) + b"".join(struct.pack("<q", d) for d in shp)
    return body + nxt.tobytes(), "D", 0, nxt


@pytest.mark.parametrize("mode,density", [("async", 0.01), ("batch", 0.01), ("async", 0.4)])
def test_sync_through_reference_memory_relay(restatement, reference, mode, density):
    ws, plan, eng = _engine()
    eng.generate(seed=4, density=density)
    relay = reference.memory_relay()
    bucket = 512
    rep = eng.sync_relay(relay.callbacks, step=9, mode=mode, bucket_bytes=bucket)
    want_keys = set()
    for i, (p, desc, off, n) in enumerate(plan.segments):
        meta = plan.manifest[p]
        payload, codec, iw, nxt = _expected_payload(restatement, ws, meta, desc, n, 4, density)
        r, size, stage = plan.segment_key_fields(i)
        for q in range(ws.wire.num_buckets(len(payload), bucket)):
            k = reference.bucket_key(9, meta.name, r, size, stage, desc, codec, iw, q).decode()
            want_keys.add(k)
            assert relay.get(k) == payload[q * bucket:(q + 1) * bucket], k
        assert _bits(eng.serve_view(i)).tobytes() == nxt.tobytes(), meta.name
    assert set(relay.keys("w|s9|")) == want_keys
    assert rep["push_buckets"] == rep["pull_buckets"] == len(want_keys)
    assert rep["pushed_bytes"] == rep["pulled_bytes"]


def test_reverse_sync_through_relay_restores_prev(restatement, reference):
    ws, plan, eng = _engine()
    eng.generate(seed=2, density=0.02)
    r1, r2 = reference.memory_relay(), reference.memory_relay()  # alive across the calls
    eng.sync_relay(r1.callbacks, step=1)
    eng.sync_relay(r2.callbacks, step=2, reverse=True)
    for i in range(len(plan.segments)):
        assert _bits(eng.serve_view(i)).tobytes() == _bits(eng.segment_view(i, 0)).tobytes()


def test_pacing_and_mode_ordering(reference):
    """TokenBucket (relay.cpp:69-84) holds each direction at its rate; Async
    (pullers ingest as buckets land) beats Batch (pull after push) when both
    directions are paced -- the ordering of the reference's modes."""
    ws, plan, eng = _engine(layers=4, hidden=256, vocab=1024)
    eng.generate(seed=1, density=0.01)
    rate = 10e6
    times = {}
    for mode in ("batch", "async"):
        relay = reference.memory_relay()
        rep = eng.sync_relay(relay.callbacks, step=5, mode=mode,
                             bucket_bytes=16384, push_bytes_per_s=rate, pull_bytes_per_s=rate,
                             burst_bytes=16384, reverse=(mode == "async"))
        assert rep["push_s"] >= 0.8 * (rep["pushed_bytes"] - 16384) / rate
        times[mode] = rep["wall_s"]
    assert times["async"] < times["batch"]


def test_missing_buckets_time_out(reference):
    """A puller that never sees its keys fails with RelayTimeout, as
    MemoryRelay::get_any does (relay.cpp:29-45)."""
    import ctypes as C

    import paper_2605_06534_b200 as ws
    _, plan, eng = _engine()
    eng.generate(seed=1, density=0.01)
    relay = reference.memory_relay()
    drop = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_char_p, C.c_uint64, C.c_void_p, C.c_uint64)(
        lambda *a: 0)
    cb = (relay.ctx, C.cast(drop, C.c_void_p).value, relay.callbacks[2])
    with pytest.raises(ws.RelayTimeout):
        eng.sync_relay(cb, step=1, timeout_ms=200)


@pytest.mark.parametrize("mode,density", [("async", 0.01), ("batch", 0.4)])
def test_gpu_frames_through_reference_tcp_relay(restatement, reference, mode, density):
    """SURVEY §8(f) rank 3 on a real transport: every bucket travels as the
    reference's frame (wire.cpp:35-47) built and CRC-32'd on the GPU, written
    after the PUT op byte to the reference's own TcpRelayServer, which checks
    the CRC and stores the bucket; the puller gets frames back over GET_ANY
    and checks key and CRC on the GPU.  The stored buckets equal the
    reference encoding of the oracle delta; serving == next."""
    ws, plan, eng = _engine()
    eng.generate(seed=4, density=density)
    tcp = reference.tcp_relay()
    bucket = 512
    rep = eng.sync_relay(tcp.callbacks, step=3, mode=mode, bucket_bytes=bucket)
    nb = 0
    for i, (p, desc, off, n) in enumerate(plan.segments):
        meta = plan.manifest[p]
        payload, codec, iw, nxt = _expected_payload(restatement, ws, meta, desc, n, 4, density)
        r, size, stage = plan.segment_key_fields(i)
        for q in range(ws.wire.num_buckets(len(payload), bucket)):
            k = reference.bucket_key(3, meta.name, r, size, stage, desc, codec, iw, q).decode()
            assert tcp.get(k) == payload[q * bucket:(q + 1) * bucket], k
            nb += 1
        assert _bits(eng.serve_view(i)).tobytes() == nxt.tobytes(), meta.name
    assert tcp.buckets() == nb == rep["push_buckets"] == rep["pull_buckets"]
    tcp.close()


@pytest.mark.parametrize("flip", ["put", "get"])
def test_corrupted_frames_raise_integrity_error(reference, flip):
    """A bit flipped in transit: on PUT the reference server's CRC check
    rejects the GPU-built frame (status 3); on GET the engine's GPU CRC check
    catches it.  Either way the sync fails with IntegrityError
    (relay.hpp:20-22)."""
    ws, plan, eng = _engine()
    eng.generate(seed=5, density=0.01)
    tcp = reference.tcp_relay(flip_put=5 if flip == "put" else 0,
                              flip_get=5 if flip == "get" else 0)
    with pytest.raises(ws.IntegrityError):
        eng.sync_relay(tcp.callbacks, step=1, bucket_bytes=512, timeout_ms=2000)
    tcp.close()
