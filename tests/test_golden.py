"""Parity against committed golden vectors of the compiled reference
(tests/golden/reference_vectors.npz, written by tests/golden/make_golden.py
from the unmodified reference's own functions), so the pin holds on hosts
where neither /root/reference nor oracle/_ref exists (the GPU boxes).

CPU: the fixture equals what the reference computes now (when it is
compiled here), and the C restatement reproduces it.  GPU: the CUDA path
(diff, apply, reslice, wire payloads, keys, frames, CRC, whole syncs through
the engine's exchange) reproduces it byte for byte."""
import os

import numpy as np
import pytest
import torch

from oracle.oracle import BF16, F32, I32

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                      "reference_vectors.npz")


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(GOLDEN))


def _cases(g, prefix):
    return sorted({k[len(prefix):].split("/")[0] for k in g if k.startswith(prefix)})


def _desc(a):
    return tuple(int(x) for x in a)


# ---------------------------------------------------------------- CPU --------

def test_golden_is_what_the_reference_computes(golden, reference):
    """Regenerates every vector with the compiled reference and compares."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "make_golden", os.path.join(os.path.dirname(GOLDEN), "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    fresh = mg.generate(reference)
    assert sorted(fresh) == sorted(golden)
    for k, v in fresh.items():
        assert np.asarray(v).tobytes() == golden[k].tobytes(), k


def test_restatement_reproduces_golden(golden, restatement):
    for dt in (F32, I32):
        for k in _cases(golden, f"diff/{dt}/"):
            p = f"diff/{dt}/{k}/"
            idx, val = restatement.diff_shards(dt, golden[p + "prev"], golden[p + "next"])
            assert idx.astype(np.uint64).tobytes() == golden[p + "idx"].tobytes(), p
            assert val.tobytes() == golden[p + "val"].tobytes(), p
            got, rc = restatement.apply_delta(dt, golden[p + "target"], golden[p + "idx"],
                                              golden[p + "val"])
            assert rc == 0 and got.tobytes() == golden[p + "applied"].tobytes(), p
        p = f"wire/{dt}/"
        for iw in (4, 8):
            pay = restatement.encode_sparse(dt, list(golden[p + "shape"]), golden[p + "idx"],
                                            golden[p + "val"], iw)
            assert bytes(pay) == golden[p + f"sparse{iw}"].tobytes(), (p, iw)
    for k in _cases(golden, "bf16/"):
        p = f"bf16/{k}/"
        idx, val = restatement.diff_shards(BF16, golden[p + "prev"], golden[p + "next"])
        assert idx.astype(np.uint64).tobytes() == golden[p + "idx"].tobytes(), p
        assert val.view(np.uint16).tobytes() == golden[p + "val"].tobytes(), p
        got, rc = restatement.apply_delta(BF16, golden[p + "target"], golden[p + "idx"],
                                          golden[p + "val"])
        assert rc == 0 and got.view(np.uint16).tobytes() == golden[p + "applied"].tobytes(), p
    for k in _cases(golden, "reslice/"):
        p = f"reslice/{k}/"
        oi, ov = restatement.reslice_delta(I32, list(golden[p + "full"]), _desc(golden[p + "src"]),
                                           _desc(golden[p + "dst"]), golden[p + "idx"],
                                           golden[p + "val"], allow_cross_dim=False)
        assert oi.astype(np.uint64).tobytes() == golden[p + "out_idx"].tobytes(), p
        assert ov.tobytes() == golden[p + "out_val"].tobytes(), p


# ---------------------------------------------------------------- GPU --------

def _dev(a, dt):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.view(torch.float32 if dt == F32 else torch.int32).cuda()


@pytest.mark.gpu
def test_cuda_codec_reproduces_golden(golden):
    import paper_2605_06534_b200 as ws
    for dt in (F32, I32):
        for k in _cases(golden, f"diff/{dt}/"):
            p = f"diff/{dt}/{k}/"
            shape = tuple(int(x) for x in golden[p + "shape"])
            d = ws.diff_shards(_dev(golden[p + "prev"], dt).view(shape),
                               _dev(golden[p + "next"], dt).view(shape))
            idx = d.indices.cpu().numpy().view(np.uint32).astype(np.uint64)
            assert idx.tobytes() == golden[p + "idx"].tobytes(), p
            assert d.values.cpu().numpy().tobytes() == golden[p + "val"].tobytes(), p
            tgt = _dev(golden[p + "target"], dt).view(shape)
            ws.apply_delta(tgt, d)
            assert tgt.cpu().numpy().tobytes() == golden[p + "applied"].tobytes(), p
    for k in _cases(golden, "bf16/"):
        p = f"bf16/{k}/"
        prev = torch.from_numpy(golden[p + "prev"].view(np.int16).copy()).cuda().view(torch.bfloat16)
        nxt = torch.from_numpy(golden[p + "next"].view(np.int16).copy()).cuda().view(torch.bfloat16)
        d = ws.diff_shards(prev, nxt)
        idx = d.indices.cpu().numpy().view(np.uint32).astype(np.uint64)
        assert idx.tobytes() == golden[p + "idx"].tobytes(), p
        assert d.values.cpu().numpy().view(np.uint16).tobytes() == golden[p + "val"].tobytes(), p
        tgt = torch.from_numpy(golden[p + "target"].view(np.int16).copy()).cuda().view(
            torch.bfloat16)
        ws.apply_delta(tgt, d)
        assert tgt.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() == \
            golden[p + "applied"].tobytes(), p
    for k in _cases(golden, "reslice/"):
        p = f"reslice/{k}/"
        full = tuple(int(x) for x in golden[p + "full"])
        src, dst = _desc(golden[p + "src"]), _desc(golden[p + "dst"])
        sshape = ws.shard_shape(full, src)
        idx = torch.from_numpy(golden[p + "idx"].astype(np.int64)).to(torch.int32).cuda()
        delta = ws.SparseDelta(I32, sshape, idx, _dev(golden[p + "val"], I32))
        out = ws.reslice_delta(delta, src, dst, full, allow_cross_dim=False)
        got = out.indices.cpu().numpy().view(np.uint32).astype(np.uint64)
        assert got.tobytes() == golden[p + "out_idx"].tobytes(), p
        assert out.values.cpu().numpy().tobytes() == golden[p + "out_val"].tobytes(), p
        assert tuple(out.shape) == tuple(int(x) for x in golden[p + "out_shape"]), p


@pytest.mark.gpu
def test_cuda_wire_reproduces_golden(golden):
    import paper_2605_06534_b200 as ws
    for dt in (F32, I32):
        p = f"wire/{dt}/"
        shape = tuple(int(x) for x in golden[p + "shape"])
        idx = torch.from_numpy(golden[p + "idx"].astype(np.int64)).to(torch.int32).cuda()
        delta = ws.SparseDelta(dt, shape, idx, _dev(golden[p + "val"], dt))
        for iw in (4, 8):
            pay = ws.wire.encode_sparse(delta, iw)
            assert pay.cpu().numpy().tobytes() == golden[p + f"sparse{iw}"].tobytes(), (p, iw)
            back = ws.wire.decode_payload(pay)
            assert torch.equal(back.indices, idx) and torch.equal(back.values, delta.values)
        dense = ws.wire.encode_dense(_dev(golden[p + "next"], dt).view(shape), dt)
        assert dense.cpu().numpy().tobytes() == golden[p + "dense"].tobytes(), p
    for k in _cases(golden, "key/"):
        p = f"key/{k}/"
        ints = [int(x) for x in golden[p + "ints"]]
        key = ws.wire.bucket_key(int(golden[p + "step"][0]), golden[p + "param"].tobytes().decode(),
                                 ints[0], ints[1], ints[2], tuple(ints[3:6]),
                                 golden[p + "codec"].tobytes().decode(), ints[6], ints[7])
        assert key.encode("utf-8", "surrogateescape") == golden[p + "key"].tobytes(), p
        payload = torch.from_numpy(golden[p + "payload"].copy()).cuda()
        assert ws.wire.crc32([payload]) == [int(golden[p + "crc"][0])], p
        frames, off = ws.wire.encode_bucket_frames(payload, max(1, payload.numel()), [key])
        assert frames.cpu().numpy().tobytes() == golden[p + "frame"].tobytes(), p


@pytest.mark.gpu
@pytest.mark.parametrize("placement", ["rank", "overlap"])
def test_engine_sync_reproduces_golden(golden, placement):
    """The reference's TransferEngine::sync_step result on a toy model,
    reproduced by a process-local group on one GPU: every rank's K1, local
    route, NVLink-protocol pack and receive-side apply; each replica equals
    the reference's serving rank of its coordinate."""
    import paper_2605_06534_b200 as ws
    layouts = sorted({k.split("/")[1] for k in golden if k.startswith("sync/")})
    assert layouts
    for name in layouts:
        p = f"sync/{name}/"
        train = tuple(int(x) for x in golden[p + "train"])
        serve = tuple(int(x) for x in golden[p + "serve"])
        manifest = []
        for s in golden[p + "params"]:
            n, kind, shape, layer = str(s).split("|")
            manifest.append(ws.ParamMeta(n, int(kind), tuple(int(x) for x in shape.split("x")),
                                         int(layer)))
        world = train[0] * train[1] * train[2]
        coords = serve[0] * serve[1]
        g = ws.EngineGroup(manifest, ws.I32, ws.TrainConfig("tp", *train),
                           ws.ServeConfig(serve[0], serve[1], world // coords, placement), world,
                           device=0)
        full = {i: (_dev(golden[p + f"prev/{i}"], I32).view(m.shape),
                    _dev(golden[p + f"next/{i}"], I32).view(m.shape))
                for i, m in enumerate(manifest)}
        for eng in g.engines:
            for s, (q, desc, off, n) in enumerate(eng.plan.segments):
                eng.segment_view(s, 0).copy_(ws.extract_shard(full[q][0], desc))
                eng.segment_view(s, 1).copy_(ws.extract_shard(full[q][1], desc))
            for s, (q, desc, off, n) in enumerate(eng.plan.serve_shards):
                eng.serve_view(s).copy_(ws.extract_shard(full[q][0], desc))
        reps = g.sync_step()
        want = [int(x) for x in golden[p + "report"]]
        assert sum(r["dense_shards"] for r in reps) == want[0], name
        assert sum(r["sparse_shards"] for r in reps) == want[1], name
        assert sum(r["pushed_bytes"] for r in reps) == want[2], name
        for eng in g.engines:
            c = eng.plan.info.serve_coord
            for s, (q, desc, off, n) in enumerate(eng.plan.serve_shards):
                got = eng.serve_view(s).reshape(-1).cpu().numpy()
                assert got.tobytes() == golden[p + f"serve/{c}/{q}"].tobytes(), (name, c, q)
        g.close()
