"""GPU parity of one whole sync (encode -> route -> apply) on one GPU.

bf16: against the C restatement on the synthetic pair (segment delta streams
and patched serving weights, bit for bit).  F32/I32: against the compiled,
unmodified reference engine (TransferEngine::sync_step over MemoryRelay) run
on the same weights -- serving weights and per-shard codecs must agree."""
import numpy as np
import pytest
import torch

from oracle.oracle import BF16, F32, I32

pytestmark = pytest.mark.gpu


def bits(t):
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16).ravel()
    return t.numpy().ravel()


def _engine(manifest, dtype=None, train=None, serve=None):
    import paper_2605_06534_b200 as ws
    plan = ws.Plan(manifest, ws.BF16 if dtype is None else dtype,
                   train or ws.TrainConfig("fsdp"), serve or ws.ServeConfig(1, 1, 1))
    return ws, plan, ws.TransferEngine(plan, device=0)


@pytest.mark.parametrize("density", [0.0, 0.01, 0.15])
def test_bf16_sync_matches_oracle(restatement, density):
    import paper_2605_06534_b200 as ws
    _, plan, eng = _engine(ws.toy_transformer_manifest(layers=3, hidden=64, vocab=384))
    eng.generate(seed=5, density=density)
    rep = eng.sync_step(sparse=True, density_threshold=0.20)
    total, dense = 0, 0
    for i, (p, desc, off, n) in enumerate(plan.segments):
        meta = plan.manifest[p]
        prev, nxt = restatement.gen_pair_bf16(5, meta.name, meta.shape, desc, density)
        assert bits(eng.segment_view(i, 0)).tobytes() == prev.tobytes()
        want_i, want_v = restatement.diff_shards(BF16, prev, nxt)
        delta, codec, nnz = eng.segment_delta(i)
        assert nnz == want_i.size
        # engine.cpp:121: small shards can exceed the threshold at 15% density
        assert codec == ("S" if restatement.is_sparse(nnz, n, 0.20) else "D")
        if codec == "S":
            assert delta.indices.cpu().numpy().view(np.uint32).tolist() == want_i.tolist()
            assert delta.values.cpu().numpy().view(np.uint16).tobytes() == want_v.tobytes()
        else:
            dense += 1
        assert bits(eng.serve_view(i)).tobytes() == nxt.tobytes(), meta.name
        total += want_i.size
    assert rep["nnz"] == total and rep["dense_shards"] == dense
    # reverse sync restores the previous version exactly
    eng.sync_step(sparse=True, density_threshold=0.20, reverse=True)
    for i, (p, desc, off, n) in enumerate(plan.segments):
        assert bits(eng.serve_view(i)).tobytes() == bits(eng.segment_view(i, 0)).tobytes()


def test_bf16_dense_fallback_and_sparse_off(restatement):
    import paper_2605_06534_b200 as ws
    ws_, plan, eng = _engine(ws.toy_transformer_manifest(layers=2, hidden=32, vocab=64))
    eng.generate(seed=9, density=0.45)  # engine.cpp:121 threshold 0.20 -> all dense
    rep = eng.sync_step(sparse=True, density_threshold=0.20)
    assert rep["sparse_shards"] == 0 and rep["dense_shards"] == len(plan.segments)
    for i in range(len(plan.segments)):
        assert eng.segment_delta(i)[1] == "D"
        assert bits(eng.serve_view(i)).tobytes() == bits(eng.segment_view(i, 1)).tobytes()
    eng.sync_step(sparse=False, reverse=True)
    for i in range(len(plan.segments)):
        assert bits(eng.serve_view(i)).tobytes() == bits(eng.segment_view(i, 0)).tobytes()


def test_threshold_is_inclusive():
    """Exactly threshold*n changes stay sparse, one more goes dense (engine.cpp:121)."""
    import paper_2605_06534_b200 as ws
    K = ws.ModuleKind
    _, plan, eng = _engine([ws.ParamMeta("w", K.NORM, (1000,), 0),
                            ws.ParamMeta("v", K.NORM, (1000,), 0)])
    a0, a1 = eng.segment_view(0, 0), eng.segment_view(1, 0)
    a0.zero_(), a1.zero_()
    eng.segment_view(0, 1).zero_()
    eng.segment_view(1, 1).zero_()
    eng.segment_view(0, 1).view(torch.int16)[:200] = 1
    eng.segment_view(1, 1).view(torch.int16)[:201] = 1
    rep = eng.sync_step(sparse=True, density_threshold=0.20)
    assert eng.segment_delta(0)[1] == "S" and eng.segment_delta(1)[1] == "D"
    assert rep["sparse_shards"] == 1 and rep["dense_shards"] == 1


def test_qwen_subset_bf16(restatement):
    import paper_2605_06534_b200 as ws
    m = ws.MODELS["qwen2.5-0.5b"](layer_subset=[0, 23])
    _, plan, eng = _engine(m)
    eng.generate(seed=1, density=0.01)
    rep = eng.sync_step()
    assert rep["dense_shards"] == 0
    for i, (p, desc, off, n) in enumerate(plan.segments):
        meta = plan.manifest[p]
        prev, nxt = restatement.gen_pair_bf16(1, meta.name, meta.shape, desc, 0.01)
        assert bits(eng.serve_view(i)).tobytes() == nxt.tobytes(), meta.name


def test_sync_step_host_e2e(restatement):
    """The new snapshot comes from pinned host memory (the e2e path)."""
    import paper_2605_06534_b200 as ws
    _, plan, eng = _engine(ws.toy_transformer_manifest(layers=2, hidden=64, vocab=128))
    eng.generate(seed=3, density=0.02)
    host = eng.arena[1].cpu().pin_memory()
    eng.arena[1].zero_()
    rep, nnz = eng.sync_step_host(host)
    for i, (p, desc, off, n) in enumerate(plan.segments):
        meta = plan.manifest[p]
        prev, nxt = restatement.gen_pair_bf16(3, meta.name, meta.shape, desc, 0.02)
        assert nnz[i] == int((prev != nxt).sum())
        assert bits(eng.serve_view(i)).tobytes() == nxt.tobytes()


def _load_reference_state(eng, plan, st, dtype):
    """Upload the reference's prev/next into our trainer arenas and its prev
    slices into our serving arena (ServeState::init, engine.cpp:34-49)."""
    import paper_2605_06534_b200 as ws
    td = {I32: torch.int32, F32: torch.float32}[dtype]
    full = {}
    for i in range(len(plan.manifest)):
        full[i] = (torch.from_numpy(st.weights(i, 0, dtype)).cuda(),
                   torch.from_numpy(st.weights(i, 1, dtype)).cuda())
    for s, (p, desc, off, n) in enumerate(plan.segments):
        shp = plan.manifest[p].shape
        eng.segment_view(s, 0).copy_(ws.extract_shard(full[p][0].view(shp).to(td), desc))
        eng.segment_view(s, 1).copy_(ws.extract_shard(full[p][1].view(shp).to(td), desc))
    for s, (p, desc, off, n) in enumerate(plan.serve_shards):
        shp = plan.manifest[p].shape
        eng.serve_view(s).copy_(ws.extract_shard(full[p][0].view(shp).to(td), desc))


@pytest.mark.parametrize("dtype", [I32, F32])
@pytest.mark.parametrize("density,sparse", [(0.05, True), (0.45, True), (0.05, False)])
def test_matches_reference_engine(reference, dtype, density, sparse):
    """Same weights through the reference's sync_step and ours (TP1 -> TP1)."""
    import paper_2605_06534_b200 as ws
    st = reference.toy_state(3, 64, 128, dtype, (1, 1, 1), (1, 1), density, 42)
    ref_rep = st.run(mode_async=True, shard_aware=True, sparse=sparse, threshold=0.20,
                     bucket_bytes=8192)
    plan = ws.Plan([ws.ParamMeta(n, k, tuple(s), l) for (n, k, s, l) in st.params], dtype,
                   ws.TrainConfig("tp", 1, 1, 1), ws.ServeConfig(1, 1, 1))
    eng = ws.TransferEngine(plan, device=0)
    _load_reference_state(eng, plan, st, dtype)
    rep = eng.sync_step(sparse=sparse, density_threshold=0.20)
    assert rep["dense_shards"] == ref_rep["dense_shards"]
    assert rep["sparse_shards"] == ref_rep["sparse_shards"]
    assert rep["pushed_bytes"] == ref_rep["pushed_bytes"]  # transfer_cases.hpp:187-199
    codecs = {d[0]: c for d, c in st.codecs()}
    for s, (p, desc, off, n) in enumerate(plan.segments):
        assert eng.segment_delta(s)[1] == codecs[p]
    for s, (p, desc, off, n) in enumerate(plan.serve_shards):
        want = st.serve(0, p, dtype)
        assert bits(eng.serve_view(s)).tobytes() == want.tobytes(), plan.manifest[p].name


def _check_segment_on_device(eng, i, reverse=False):
    """Size-independent properties of segment i's delta stream, checked with
    plain torch ops: ascending unique indices, exactly the changed positions,
    values = next - prev (u16 wrap; the snapshots swap roles when reverse)."""
    a, b = (1, 0) if reverse else (0, 1)
    prev = eng.segment_view(i, a).reshape(-1).view(torch.int16).to(torch.int32) & 0xFFFF
    nxt = eng.segment_view(i, b).reshape(-1).view(torch.int16).to(torch.int32) & 0xFFFF
    changed = torch.nonzero(prev != nxt).flatten()
    delta, codec, nnz = eng.segment_delta(i)
    assert nnz == changed.numel()
    if codec != "S":
        return 0
    idx = delta.indices.to(torch.int64) & 0xFFFFFFFF
    assert torch.equal(idx, changed)
    want = (nxt[changed] - prev[changed]) & 0xFFFF
    assert torch.equal(delta.values.to(torch.int32) & 0xFFFF, want)
    return nnz


def _check_stream_as_written(eng, i):
    """Segment i's records exactly as K1 left them in the engine (before any
    compaction; what the local route and the NVLink pack read): every
    super-tile's records are one contiguous run, strictly ascending inside
    it, and the stream sorted is the compacted ascending stream, values
    attached (codec.cpp:48-49 order restored)."""
    idx, val, tile_elems = eng.segment_stream(i)
    delta, codec, nnz = eng.segment_delta(i)
    if codec != "S":
        assert idx.numel() == 0
        return
    assert idx.numel() == nnz
    if nnz == 0:
        return
    ii = idx.to(torch.int64) & 0xFFFFFFFF
    tile = ii // tile_elems
    starts = torch.cat([torch.zeros(1, dtype=torch.int64, device=ii.device),
                        torch.nonzero(tile[1:] != tile[:-1]).flatten() + 1])
    run_tiles = tile[starts]
    assert run_tiles.unique().numel() == run_tiles.numel(), i  # one run per super-tile
    same = tile[1:] == tile[:-1]
    assert bool((ii[1:][same] > ii[:-1][same]).all()), i
    order = torch.argsort(ii)
    assert torch.equal(ii[order], delta.indices.to(torch.int64) & 0xFFFFFFFF), i
    assert torch.equal(val[order].view(torch.int16), delta.values.view(torch.int16)), i


@pytest.mark.parametrize("density", [0.01, 0.05, 0.15])
def test_k1_stream_as_written(density):
    """The engine's unordered record stream itself (ws_engine_segment_stream),
    both K1 instantiations: the first sync runs the per-record one, later
    syncs the streamed-apply one (4 staging slots per thread, so 5% and 15%
    push many records through the spill path)."""
    import paper_2605_06534_b200 as ws
    _, plan, eng = _engine(ws.MODELS["qwen2.5-0.5b"]([0, 1, 23]))
    eng.generate(seed=5, density=density)
    variants = []
    for k in range(3):
        rep = eng.sync_step(reverse=bool(k % 2))
        variants.append(rep["streamed_apply"])
        for i in range(len(plan.segments)):
            _check_stream_as_written(eng, i)
            _check_segment_on_device(eng, i, reverse=bool(k % 2))
    assert variants[0] == 0 and variants[-1] == 1, variants


@pytest.mark.parametrize("model,density", [("qwen2.5-0.5b", 0.01), ("qwen2.5-0.5b", 0.1)])
def test_full_model_bf16(restatement, model, density):
    """A whole model through the engine (many super-tiles per block, so warp
    drift and the look-back are exercised), checked on the device, plus two
    segments against the C oracle bit for bit."""
    import paper_2605_06534_b200 as ws
    _, plan, eng = _engine(ws.MODELS[model]())
    eng.generate(seed=11, density=density)
    rep = eng.sync_step()
    torch.cuda.synchronize()
    total = 0
    for i in range(len(plan.segments)):
        total += _check_segment_on_device(eng, i)
        assert torch.equal(eng.serve_view(i).view(torch.int16), eng.segment_view(i, 1).view(torch.int16))
    assert rep["nnz"] >= total
    # the largest segment (the embedding) and a bias, bit for bit vs the oracle
    sizes = [n for (_, _, _, n) in plan.segments]
    for i in (sizes.index(max(sizes)), sizes.index(min(sizes))):
        p, desc, off, n = plan.segments[i]
        meta = plan.manifest[p]
        pv, nx = restatement.gen_pair_bf16(11, meta.name, meta.shape, desc, density)
        wi, wv = restatement.diff_shards(BF16, pv, nx)
        delta, codec, nnz = eng.segment_delta(i)
        assert codec == "S" and nnz == wi.size
        assert delta.indices.cpu().numpy().view(np.uint32).tolist() == wi.tolist()
        assert delta.values.cpu().numpy().view(np.uint16).tobytes() == wv.tobytes()
    # the reverse sync restores prev everywhere
    eng.sync_step(reverse=True)
    for i in range(len(plan.segments)):
        assert torch.equal(eng.serve_view(i).view(torch.int16), eng.segment_view(i, 0).view(torch.int16))


def test_single_shard_many_tiles():
    """ws_diff_shards on a 300M-element shard: device-checked properties."""
    import paper_2605_06534_b200 as ws
    n = 300_000_000 + 5  # ragged tail
    prev, nxt = ws.gen_pair_bf16(4, "big", (n,), (-1, 0, 0), 0.02)
    d = ws.diff_shards(prev, nxt)
    p = prev.view(torch.int16).to(torch.int32) & 0xFFFF
    q = nxt.view(torch.int16).to(torch.int32) & 0xFFFF
    changed = torch.nonzero(p != q).flatten()
    assert torch.equal(d.indices.to(torch.int64) & 0xFFFFFFFF, changed)
    assert torch.equal(d.values.to(torch.int32) & 0xFFFF, (q[changed] - p[changed]) & 0xFFFF)


@pytest.mark.parametrize("first", [0.45, 0.0])
def test_predicted_dense_segments_fixup(restatement, first):
    """Segments dense in one sync are only counted in the next; when they come
    out sparse after all, the device-side fixup pass produces their records
    (and sparse segments predicted sparse that come out dense still fall back)."""
    import paper_2605_06534_b200 as ws
    _, plan, eng = _engine(ws.toy_transformer_manifest(layers=3, hidden=64, vocab=384))
    second = 0.01 if first > 0.2 else 0.45
    eng.generate(seed=3, density=first)
    eng.sync_step(sparse=True, density_threshold=0.20)
    for density in (second, first, second):
        eng.generate(seed=11, density=density)
        rep = eng.sync_step(sparse=True, density_threshold=0.20)
        total = 0
        for i, (p, desc, off, n) in enumerate(plan.segments):
            meta = plan.manifest[p]
            prev, nxt = restatement.gen_pair_bf16(11, meta.name, meta.shape, desc, density)
            want_i, want_v = restatement.diff_shards(BF16, prev, nxt)
            delta, codec, nnz = eng.segment_delta(i)
            assert nnz == want_i.size, meta.name
            assert codec == ("S" if restatement.is_sparse(nnz, n, 0.20) else "D")
            if codec == "S":
                assert delta.indices.cpu().numpy().view(np.uint32).tolist() == want_i.tolist()
                assert delta.values.cpu().numpy().view(np.uint16).tobytes() == want_v.tobytes()
            assert bits(eng.serve_view(i)).tobytes() == nxt.tobytes(), meta.name
            total += want_i.size
        assert rep["nnz"] == total


@pytest.mark.parametrize("density", [0.006, 0.012, 0.03, 0.15])
def test_streamed_apply_adds_delta(density):
    """K1's streamed apply (fuse_on = 2): from the second sync
    on, fused segments denser than 1/sa_div get serve + (next - prev) stored
    per changed 16-byte vector.  The serving shards are perturbed first, so
    overwriting with `next` (or touching unchanged lanes) would fail: the
    result must be the reference's in-place add (codec.cpp:80-91), or `next`
    for segments that went dense."""
    import paper_2605_06534_b200 as ws
    _, plan, eng = _engine(ws.MODELS["qwen2.5-0.5b"]([0, 1]))
    eng.generate(seed=7, density=density)
    eng.sync_step()
    eng.sync_step(reverse=True)  # fuse_on now reflects this density
    gen = torch.Generator(device="cuda").manual_seed(1)
    before = []
    for i in range(len(plan.segments)):
        v = eng.serve_view(i).view(torch.int16)
        flip = torch.randint(0, 2, v.shape, device=v.device, generator=gen, dtype=torch.int16)
        v.bitwise_xor_(flip * 0x0101)
        before.append(v.to(torch.int32) & 0xFFFF)
    rep = eng.sync_step()
    torch.cuda.synchronize()
    assert rep["streamed_apply"] == 1, rep
    dense = 0
    for i in range(len(plan.segments)):
        p = eng.segment_view(i, 0).view(torch.int16).to(torch.int32) & 0xFFFF
        q = eng.segment_view(i, 1).view(torch.int16).to(torch.int32) & 0xFFFF
        got = eng.serve_view(i).view(torch.int16).to(torch.int32) & 0xFFFF
        if eng.segment_delta(i)[1] == "D":
            dense += 1
            assert torch.equal(got, q), i
        else:
            assert torch.equal(got, (before[i] + q - p) & 0xFFFF), i
    assert rep["dense_shards"] == dense


def test_qwen3_8b_whole_model_bench_config(restatement):
    """The configuration the headline number comes from (bench.py, BASELINE
    config 2 at N = 1): the whole Qwen3-8B (8.19 G elements, 399 segments),
    FSDP1 -> TP1, 1% density, four alternating syncs.  From the second sync
    on K1 runs its streamed-apply instantiation (the first sync's density,
    1% >= 1/250, selects it) -- the one the bench times.  After the first
    and the last sync every segment's record stream (as K1 wrote it and
    compacted) and every serving shard is checked on the device; the largest segment (the
    622 M-element embedding) and the smallest against the C oracle."""
    import paper_2605_06534_b200 as ws
    _, plan, eng = _engine(ws.MODELS["qwen3-8b"]())
    assert plan.info.model_elems == 8_190_735_360
    eng.generate(seed=1, density=0.01)
    sizes = [n for (_, _, _, n) in plan.segments]
    variants = []
    for k in range(4):
        rev = bool(k % 2)
        rep = eng.sync_step(reverse=rev)
        variants.append(rep["streamed_apply"])
        assert rep["dense_shards"] == 0
        if k not in (0, 3):
            continue
        torch.cuda.synchronize()
        total = 0
        for i in range(len(plan.segments)):
            total += _check_segment_on_device(eng, i, reverse=rev)
            _check_stream_as_written(eng, i)
            want = eng.segment_view(i, 0 if rev else 1).view(torch.int16)
            assert torch.equal(eng.serve_view(i).view(torch.int16), want), i
        assert rep["nnz"] == total
        for i in (sizes.index(max(sizes)), sizes.index(min(sizes))):
            p, desc, off, n = plan.segments[i]
            meta = plan.manifest[p]
            pv, nx = restatement.gen_pair_bf16(1, meta.name, meta.shape, desc, 0.01)
            wi, wv = restatement.diff_shards(BF16, nx, pv) if rev else \
                restatement.diff_shards(BF16, pv, nx)
            delta, codec, nnz = eng.segment_delta(i)
            assert codec == "S" and nnz == wi.size
            assert np.array_equal(delta.indices.cpu().numpy().view(np.uint32), wi)
            assert delta.values.cpu().numpy().view(np.uint16).tobytes() == wv.tobytes()
    assert variants[1:] == [1, 1, 1], variants
