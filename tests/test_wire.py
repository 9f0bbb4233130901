"""The reference wire format produced on the device (SURVEY.md 8(f) rows 1 and
3): payloads vs the compiled reference's encode_sparse / encode_dense /
decode_payload (codec.cpp:140-263) and the bf16 restatement (CWS2), bucket
keys vs key.cpp, bucket frames and their CRC-32 vs wire.cpp -- pinned by the
reference's golden frame (transfer_wire_test.cpp:14-30) and zlib."""
import random
import struct
import zlib

import numpy as np
import pytest
import torch

from oracle.oracle import BF16, F32, I32

GOLDEN_KEY = "w|s7|pk|t0.1|g0|dF|cD0|q0"
GOLDEN_FRAME = bytes([
    0x19, 0x00, 0x00, 0x00, 0x77, 0x7C, 0x73, 0x37, 0x7C, 0x70, 0x6B,
    0x7C, 0x74, 0x30, 0x2E, 0x31, 0x7C, 0x67, 0x30, 0x7C, 0x64, 0x46,
    0x7C, 0x63, 0x44, 0x30, 0x7C, 0x71, 0x30, 0x04, 0x00, 0x00, 0x00,
    0xDE, 0xAD, 0xBE, 0xEF, 0x0C, 0x62, 0x41, 0xF9])  # transfer_wire_test.cpp:16-20


# ---- host side (no GPU) -------------------------------------------------------

def test_golden_frame_pins_reference_and_zlib(reference):
    """The oracle for row 3 is zlib's CRC-32: the reference's frame_crc32 and
    Python's zlib agree on the reference's golden frame."""
    assert reference.encode_bucket_frame(GOLDEN_KEY.encode(), bytes([0xDE, 0xAD, 0xBE, 0xEF])) \
        == GOLDEN_FRAME
    assert reference.frame_crc32(GOLDEN_FRAME[:-4]) == 0xF941620C == zlib.crc32(GOLDEN_FRAME[:-4])


def test_bucket_keys_match_reference(reference):
    """key.cpp:47-69 incl. escaping of hostile names (transfer_test.cpp:147-190)."""
    import paper_2605_06534_b200 as ws
    assert ws.wire.bucket_key(7, "k", 0, 1, 0, (-1, 0, 0), "D", 0, 0) == GOLDEN_KEY
    rng = random.Random(7)
    alphabet = "abc|%.:wSD123"
    for _ in range(300):
        name = "".join(rng.choice(alphabet) for _ in range(rng.randint(1, 24)))
        tp_rank = rng.randint(0, 7)
        desc = (rng.randint(0, 2), s := rng.randint(0, 1000), s + rng.randint(1, 1000)) \
            if rng.random() < 0.7 else (-1, 0, 0)
        codec, iw = ("S", rng.choice((4, 8))) if rng.random() < 0.5 else ("D", 0)
        args = (rng.randint(0, 1 << 20), name, tp_rank, tp_rank + rng.randint(1, 8),
                rng.randint(0, 3), desc, codec, iw, rng.randint(0, 1 << 16))
        assert ws.wire.bucket_key(*args).encode() == reference.bucket_key(*args)


def test_payload_sizes():
    import paper_2605_06534_b200 as ws
    assert ws.wire.payload_bytes(F32, 2, "D", 0, 24) == 8 + 16 + 96      # codec.cpp:156-162
    assert ws.wire.payload_bytes(I32, 2, "S", 4, 2) == 8 + 16 + 8 + 16   # :164-183
    assert ws.wire.payload_bytes(BF16, 1, "S", 8, 3) == 8 + 8 + 8 + 30
    assert ws.wire.num_buckets(0, 64) == 1 and ws.wire.num_buckets(129, 64) == 3


# ---- device (GPU) ---------------------------------------------------------------

def _dev(b: bytes):
    return torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda() if b else \
        torch.empty(0, dtype=torch.uint8, device="cuda")


@pytest.mark.gpu
def test_crc32_matches_zlib():
    import paper_2605_06534_b200 as ws
    rng = np.random.default_rng(5)
    base = rng.integers(0, 256, (1 << 21) + 64, dtype=np.uint8)
    dbase = torch.from_numpy(base).cuda()
    cases = [(0, 0), (0, 1), (1, 3), (3, 5), (0, 255), (1, 256), (2, 257), (3, 4095),
             (0, 65536), (5, 65537), (7, 1 << 20), (1, (1 << 21) + 13)]
    got = ws.wire.crc32([dbase[o:o + n] for o, n in cases])
    assert got == [zlib.crc32(base[o:o + n].tobytes()) for o, n in cases]
    assert ws.wire.crc32([_dev(GOLDEN_FRAME[:-4])]) == [0xF941620C]


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [F32, I32])
@pytest.mark.parametrize("iw", [4, 8])
def test_sparse_payload_matches_reference(reference, dt, iw):
    import paper_2605_06534_b200 as ws
    rng = np.random.default_rng(dt * 10 + iw)
    shape = (37, 11)
    idx = np.sort(rng.choice(37 * 11, 40, replace=False)).astype(np.uint64)
    val = rng.integers(-1000, 1000, 40).astype(np.int32)
    if dt == F32:
        val = val.astype(np.float32) / 7
    want = reference.encode_sparse(dt, shape, idx, val, iw)
    d = ws.SparseDelta(dt, shape, torch.from_numpy(idx.astype(np.int32)).cuda(),
                       torch.from_numpy(val).cuda())
    got = ws.wire.encode_sparse(d, iw)
    assert bytes(got.cpu().numpy()) == want
    back = ws.wire.decode_payload(got)
    assert back.indices.cpu().numpy().view(np.uint32).tolist() == idx.tolist()
    assert back.values.cpu().numpy().tobytes() == val.tobytes()
    assert ws.wire.peek_payload(got)["total_bytes"] == len(want)


@pytest.mark.gpu
def test_bf16_payload_matches_restatement(restatement):
    import paper_2605_06534_b200 as ws
    rng = np.random.default_rng(3)
    idx = np.sort(rng.choice(4096, 100, replace=False)).astype(np.uint64)
    val = rng.integers(0, 1 << 16, 100).astype(np.uint16)
    want = restatement.encode_sparse(BF16, (64, 64), idx, val, 4)
    d = ws.SparseDelta(BF16, (64, 64), torch.from_numpy(idx.astype(np.int32)).cuda(),
                       torch.from_numpy(val.view(np.int16)).cuda())
    got = ws.wire.encode_sparse(d, 4)
    assert bytes(got.cpu().numpy()) == want and want[:4] == b"CWS2"
    t = torch.from_numpy(val.view(np.int16).reshape(10, 10)).cuda().view(torch.bfloat16)
    dense = ws.wire.encode_dense(t, BF16)
    hdr = b"CWD2" + bytes([BF16, 2, 0, 0]) + struct.pack("<qq", 10, 10)
    assert bytes(dense.cpu().numpy()) == hdr + val.tobytes()
    dt, back = ws.wire.decode_payload(dense)
    assert dt == BF16 and back.cpu().numpy().view(np.uint16).tobytes() == val.tobytes()


@pytest.mark.gpu
def test_dense_payload_and_rejections_match_reference(reference):
    """codec.cpp:196-263 and transfer_test.cpp:272-295: the device decoder
    rejects exactly what the reference rejects."""
    import paper_2605_06534_b200 as ws
    from oracle.oracle import OracleError
    t = np.arange(16, dtype=np.int32).reshape(4, 4)
    dense = reference.encode_dense(I32, (4, 4), t)
    got = ws.wire.encode_dense(torch.from_numpy(t).cuda(), I32)
    assert bytes(got.cpu().numpy()) == dense
    t2 = t.copy().ravel()
    t2[1] += 1
    t2[7] += 1
    sp = bytearray(reference.encode_sparse(I32, (4, 4), np.array([1, 7], np.uint64),
                                           np.array([1, 1], np.int32), 4))
    sp[32:36], sp[36:40] = sp[36:40], sp[32:36]
    bad_magic = bytearray(dense)
    bad_magic[0] ^= 0xFF
    cases = [bytes(bad_magic), dense[:-3], dense + b"\0", bytes(sp),
             dense[:2], b"CWS1" + bytes([7, 0, 4, 0])]
    for c in cases:
        with pytest.raises(OracleError) as e:
            reference.decode_payload(c)
        assert e.value.kind == "PayloadFormatError"
        buf = torch.empty(len(c) + 8, dtype=torch.uint8, device="cuda")[:len(c)]
        buf.copy_(_dev(c)) if c else None
        with pytest.raises(ws.PayloadFormatError):
            ws.wire.decode_payload(buf)


@pytest.mark.gpu
@pytest.mark.parametrize("plen,bucket", [(0, 64), (1, 64), (64, 64), (1000, 64), (4097, 1000)])
def test_bucket_frames_match_reference(reference, plen, bucket):
    import paper_2605_06534_b200 as ws
    rng = np.random.default_rng(plen)
    payload = rng.integers(0, 256, plen, dtype=np.uint8).tobytes()
    nb = ws.wire.num_buckets(plen, bucket)
    keys = [ws.wire.bucket_key(3, "layers.0|w%", 1, 2, 0, (0, 0, 8), "S", 4, q) for q in range(nb)]
    frames, offs = ws.wire.encode_bucket_frames(_dev(payload), bucket, keys)
    host = bytes(frames.cpu().numpy())
    want = b"".join(reference.encode_bucket_frame(k.encode(), payload[q * bucket:(q + 1) * bucket])
                    for q, k in enumerate(keys))
    assert host == want and offs[-1] == len(want)


@pytest.mark.gpu
@pytest.mark.parametrize("density", [0.01, 0.4])
def test_engine_segment_frames(restatement, reference, density):
    """What the pusher would put on the relay for every segment of a sync
    (engine.cpp:116-148): payload == the restatement's encode of the oracle
    delta (or the dense snapshot), keys == key.cpp, frames == wire.cpp."""
    import paper_2605_06534_b200 as ws
    plan = ws.Plan(ws.toy_transformer_manifest(layers=2, hidden=64, vocab=256), ws.BF16,
                   ws.TrainConfig("fsdp"), ws.ServeConfig(1, 1, 1))
    eng = ws.TransferEngine(plan, device=0)
    eng.generate(seed=9, density=density)
    eng.sync_step(sparse=True, density_threshold=0.20)
    for i, (p, desc, off, n) in enumerate(plan.segments):
        meta = plan.manifest[p]
        prev, nxt = restatement.gen_pair_bf16(9, meta.name, meta.shape, desc, density)
        wi, wv = restatement.diff_shards(BF16, prev, nxt)
        shp = ws.shard_shape(meta.shape, desc)
        if restatement.is_sparse(wi.size, n, 0.20):
            want = restatement.encode_sparse(BF16, shp, wi.astype(np.uint64), wv, 4)
            codec, iw = "S", 4
        else:
            want = b"CWD2" + bytes([BF16, len(shp), 0, 0]) + \
                b"".join(struct.pack("<q", d) for d in shp) + nxt.tobytes()
            codec, iw = "D", 0
        payload, info = eng.segment_payload(i)
        assert bytes(payload.cpu().numpy()) == want, meta.name
        frames, keys, offs = eng.segment_frames(i, step=5, bucket_bytes=256)
        r, size, stage = plan.segment_key_fields(i)
        wframes = b""
        for q in range(ws.wire.num_buckets(len(want), 256)):
            k = reference.bucket_key(5, meta.name, r, size, stage, desc, codec, iw, q)
            assert keys[q].encode() == k
            wframes += reference.encode_bucket_frame(k, want[q * 256:(q + 1) * 256])
        assert bytes(frames.cpu().numpy()) == wframes, meta.name
