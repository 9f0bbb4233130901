"""The multi-GPU data path on one GPU: every rank of a layout as an engine of
one process (ws_group, include/wsync.h).

A group sync runs the same kernels as the one-process-per-GPU deployment --
K1, the local route, pack_kernel (records and dense boxes stored into the
peers' receive regions / serving arenas) and apply_p2p_kernel (the
receiver's scatter) -- with the peers' memory shared as plain pointers, so
the whole exchange protocol (ready flags, per-round epochs, acks, published
counts) and every layout of the reference are checked here on one B200:

* bf16: every rank's serving shards equal the generator's `next` (then
  `prev` after a reverse sync) for FSDP-N -> TP2 x N/2 (BASELINE config 2's
  layout), TP8 -> TP4 x 2 (config 3), expert-sharded TP -> EP (config 4),
  replica fan-out, dense fallback, sparse=False;
* I32 / F32: the reference's own layouts, TrainConfig{tp,pp,dp} ->
  ServeConfig{tp,pp} (transfer_cases.hpp:19-35's space), against the
  compiled reference engine's serving weights (TransferEngine::sync_step,
  engine.cpp:66-254) -- every replica must equal the reference's serving
  rank of its coordinate.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import F32, I32

pytestmark = pytest.mark.gpu


def _serve_equals_gen(ws, group, seed, density, which, tabs=None):
    bad = []
    for q, eng in enumerate(group.engines):
        plan = eng.plan
        for i, (p, desc, off, n) in enumerate(plan.serve_shards):
            meta = plan.manifest[p]
            pv, nx = ws.gen_pair_bf16(seed, meta.name, meta.shape, desc, density,
                                      device=eng.device, thr_dim0=(tabs or {}).get(p))
            want = (nx if which == "next" else pv).view(torch.int16)
            if not torch.equal(eng.serve_view(i).view(torch.int16), want):
                bad.append((q, meta.name))
    return bad


def _layouts(ws):
    return {
        # BASELINE config 2's layout (FSDP8 -> TP2 x 4) and its smaller worlds
        "fsdp2-tp2": (ws.TrainConfig("fsdp"), ws.ServeConfig(2, 1, 1), 2),
        "fsdp4-tp2x2": (ws.TrainConfig("fsdp"), ws.ServeConfig(2, 1, 2), 4),
        "fsdp8-tp2x4": (ws.TrainConfig("fsdp"), ws.ServeConfig(2, 1, 4), 8),
        # replica fan-out (every record to 4 serving ranks)
        "fsdp4-tp1x4": (ws.TrainConfig("fsdp"), ws.ServeConfig(1, 1, 4), 4),
        # the reference's TrainConfig{tp,pp,dp} -> ServeConfig{tp,pp} x replicas
        "tp2pp2-tp1pp2x2": (ws.TrainConfig("tp", 2, 2, 1), ws.ServeConfig(1, 2, 2), 4),
        "tp2dp2-tp2x2": (ws.TrainConfig("tp", 2, 1, 2), ws.ServeConfig(2, 1, 2), 4),
        "tp1pp2dp2-tp2pp2": (ws.TrainConfig("tp", 1, 2, 2), ws.ServeConfig(2, 2, 1), 4),
        "tp2pp2dp2-tp4pp2": (ws.TrainConfig("tp", 2, 2, 2), ws.ServeConfig(4, 2, 1), 8),
        # BASELINE config 3's layout (TP8 -> TP4 x 2)
        "tp8-tp4x2": (ws.TrainConfig("tp", 8, 1, 1), ws.ServeConfig(4, 1, 2), 8),
        # serving ranks placed for the fewest NVLink bytes (WS_PLACE_OVERLAP)
        "fsdp4-tp2x2-overlap": (ws.TrainConfig("fsdp"), ws.ServeConfig(2, 1, 2, "overlap"), 4),
        "fsdp8-tp2x4-overlap": (ws.TrainConfig("fsdp"), ws.ServeConfig(2, 1, 4, "overlap"), 8),
        "tp8-tp4x2-overlap": (ws.TrainConfig("tp", 8, 1, 1), ws.ServeConfig(4, 1, 2, "overlap"),
                              8),
        "tp2pp2dp2-tp4pp2-overlap": (ws.TrainConfig("tp", 2, 2, 2),
                                     ws.ServeConfig(4, 2, 1, "overlap"), 8),
    }


@pytest.mark.parametrize("layout", ["fsdp2-tp2", "fsdp4-tp2x2", "fsdp8-tp2x4", "fsdp4-tp1x4",
                                    "tp2pp2-tp1pp2x2", "tp2dp2-tp2x2", "tp1pp2dp2-tp2pp2",
                                    "tp2pp2dp2-tp4pp2", "tp8-tp4x2", "fsdp4-tp2x2-overlap",
                                    "fsdp8-tp2x4-overlap", "tp8-tp4x2-overlap",
                                    "tp2pp2dp2-tp4pp2-overlap"])
def test_group_bf16_layouts(layout):
    """bf16 sparse sync (1%), reverse sync, dense fallback (45%), sparse=False
    on the toy transformer (4 layers, so PP=2 has two stages)."""
    import paper_2605_06534_b200 as ws
    train, serve, world = _layouts(ws)[layout]
    manifest = ws.toy_transformer_manifest(layers=4, hidden=64, vocab=512)
    g = ws.EngineGroup(manifest, ws.BF16, train, serve, world, device=0)
    g.generate(seed=3, density=0.01)
    reps = g.sync_step()
    assert _serve_equals_gen(ws, g, 3, 0.01, "next") == []
    assert sum(r["sparse_shards"] for r in reps) > 0
    g.sync_step(reverse=True)
    assert _serve_equals_gen(ws, g, 3, 0.01, "prev") == []
    g.generate(seed=4, density=0.45)  # engine.cpp:121: (nearly) every shard dense
    reps = g.sync_step()
    assert sum(r["dense_shards"] for r in reps) > 4 * sum(r["sparse_shards"] for r in reps)
    assert _serve_equals_gen(ws, g, 4, 0.45, "next") == []
    g.sync_step(sparse=False, reverse=True)
    assert _serve_equals_gen(ws, g, 4, 0.45, "prev") == []
    g.close()


def test_group_config2_layout_qwen():
    """BASELINE config 2's layout, FSDP8 -> TP2 x 4, on Qwen2.5-0.5B-shaped
    weights (cross-dim FSDP -> TP routes for every RowLinear), 1% density,
    10 alternating syncs (epochs and acks through several steps): an even
    count leaves every replica at `prev`, then one more at `next`.  Serving
    ranks placed as the bench places them (overlap placement)."""
    import paper_2605_06534_b200 as ws
    g = ws.EngineGroup(ws.MODELS["qwen2.5-0.5b"](), ws.BF16, ws.TrainConfig("fsdp"),
                       ws.ServeConfig(2, 1, 4, "overlap"), 8, device=0)
    assert [e.plan.info.serve_coord for e in g.engines] == [0, 0, 0, 0, 1, 1, 1, 1]
    g.generate(seed=8, density=0.01)
    for k in range(10):
        g.sync_step(reverse=bool(k % 2), report=False)
    torch.cuda.synchronize()
    assert _serve_equals_gen(ws, g, 8, 0.01, "prev") == []
    reps = g.sync_step()
    assert _serve_equals_gen(ws, g, 8, 0.01, "next") == []
    assert all(r["dense_shards"] == 0 for r in reps)
    # every rank ran the exchange: pack + apply kernels on top of K1
    assert all(r["kernel_launches"] >= 6 for r in reps), reps
    g.close()


def test_group_config3_and_config4_layouts():
    """Config 3 (Qwen3-32B TP8 -> TP4 x 2, 0.5%) and config 4 (Qwen3-30B-A3B
    expert-sharded TP8 -> EP8, Zipf(1.1) per-expert densities around 1%) on
    layer subsets."""
    import paper_2605_06534_b200 as ws
    g = ws.EngineGroup(ws.MODELS["qwen3-32b"]([1, 2]), ws.BF16, ws.TrainConfig("tp", 8, 1, 1),
                       ws.ServeConfig(4, 1, 2), 8, device=0)
    g.generate(seed=5, density=0.005)
    g.sync_step()
    assert _serve_equals_gen(ws, g, 5, 0.005, "next") == []
    g.sync_step(reverse=True)
    assert _serve_equals_gen(ws, g, 5, 0.005, "prev") == []
    g.close()
    manifest = ws.MODELS["qwen3-30b-a3b"]([1, 2])
    g = ws.EngineGroup(manifest, ws.BF16, ws.TrainConfig("tp", 8, 1, 1), ws.ServeConfig(8, 1, 1),
                       8, device=0)
    g.generate(seed=5, density=0.01, expert_zipf=1.1, perm_seed=11)
    tabs = {i: ws.expert_thresholds(m.shape[0], 0.01, 1.1, 11)
            for i, m in enumerate(manifest) if m.kind == ws.ModuleKind.EXPERT}
    g.sync_step()
    assert _serve_equals_gen(ws, g, 5, 0.01, "next", tabs) == []
    g.close()


def test_group_threshold_raise_resizes_regions():
    """Receive regions are sized for density_threshold (0.20 by default,
    engine.hpp:27), so a sync with a higher threshold whose shards stay
    sparse at ~30% must grow them first (collectively) and still be exact."""
    import paper_2605_06534_b200 as ws
    manifest = ws.toy_transformer_manifest(layers=2, hidden=64, vocab=256)
    g = ws.EngineGroup(manifest, ws.BF16, ws.TrainConfig("fsdp"), ws.ServeConfig(2, 1, 2), 4,
                       device=0)
    g.generate(seed=6, density=0.3)
    reps = g.sync_step(density_threshold=0.20)
    dense20 = sum(r["dense_shards"] for r in reps)
    assert dense20 > sum(r["sparse_shards"] for r in reps)
    assert _serve_equals_gen(ws, g, 6, 0.3, "next") == []
    reps = g.sync_step(density_threshold=0.45, reverse=True)
    assert sum(r["dense_shards"] for r in reps) < dense20 // 4
    assert _serve_equals_gen(ws, g, 6, 0.3, "prev") == []
    reps = g.sync_step(density_threshold=0.45)
    assert _serve_equals_gen(ws, g, 6, 0.3, "next") == []
    g.close()


def _load_reference_state(ws, eng, st, dtype):
    td = {I32: torch.int32, F32: torch.float32}[dtype]
    plan = eng.plan
    for s, (p, desc, off, n) in enumerate(plan.segments):
        shp = plan.manifest[p].shape
        for which in (0, 1):
            full = torch.from_numpy(st.weights(p, which, dtype)).to(eng.device).view(shp).to(td)
            eng.segment_view(s, which).copy_(ws.extract_shard(full, desc))
    for s, (p, desc, off, n) in enumerate(plan.serve_shards):
        full = torch.from_numpy(st.weights(p, 0, dtype)).to(eng.device)
        eng.serve_view(s).copy_(ws.extract_shard(full.view(plan.manifest[p].shape).to(td), desc))


# (train tp, pp, dp) -> (serve tp, pp): the reference's randomized layout
# space (transfer_cases.hpp:19-35: train tp in {1,2,4}, pp in {1,2}, dp 1-3,
# serve pp in {1,2}); replicas fill the world
REF_LAYOUTS = [((2, 1, 1), (2, 1)), ((2, 1, 1), (1, 1)), ((1, 2, 1), (1, 2)),
               ((2, 2, 1), (1, 2)), ((1, 1, 2), (1, 1)), ((2, 1, 2), (2, 1)),
               ((4, 1, 1), (2, 1)), ((1, 2, 3), (1, 2)), ((2, 2, 2), (4, 2)),
               ((4, 2, 1), (2, 2)), ((1, 1, 3), (1, 1))]


@pytest.mark.parametrize("train,serve", REF_LAYOUTS)
@pytest.mark.parametrize("dtype", [I32, F32])
@pytest.mark.parametrize("placement", ["rank", "overlap"])
def test_group_matches_reference_engine(reference, dtype, train, serve, placement):
    """Same weights through the reference's sync_step (MemoryRelay, Async,
    shard-aware, sparse, 0.20) and through the group; 5% density so most
    shards are sparse and the small ones go dense."""
    import paper_2605_06534_b200 as ws
    world = train[0] * train[1] * train[2]
    coords = serve[0] * serve[1]
    if world % coords:
        pytest.skip("serving coordinates must divide the world")
    st = reference.toy_state(4, 64, 128, dtype, train, serve, 0.05, 42)
    ref_rep = st.run(mode_async=True, shard_aware=True, sparse=True, threshold=0.20,
                     bucket_bytes=8192)
    manifest = [ws.ParamMeta(n, k, tuple(s), l) for (n, k, s, l) in st.params]
    g = ws.EngineGroup(manifest, dtype, ws.TrainConfig("tp", *train),
                       ws.ServeConfig(serve[0], serve[1], world // coords, placement), world,
                       device=0)
    for eng in g.engines:
        _load_reference_state(ws, eng, st, dtype)
    reps = g.sync_step()
    assert sum(r["dense_shards"] for r in reps) == ref_rep["dense_shards"]
    assert sum(r["sparse_shards"] for r in reps) == ref_rep["sparse_shards"]
    assert sum(r["pushed_bytes"] for r in reps) == ref_rep["pushed_bytes"]
    bad = []
    for q, eng in enumerate(g.engines):
        coord = eng.plan.info.serve_coord
        for s, (p, desc, off, n) in enumerate(eng.plan.serve_shards):
            want = st.serve(coord, p, dtype)
            got = eng.serve_view(s).reshape(-1).cpu().numpy()
            if got.tobytes() != np.ascontiguousarray(want).tobytes():
                bad.append((q, eng.plan.manifest[p].name))
    assert bad == []
    g.close()


@pytest.mark.parametrize("placement", ["rank", "overlap"])
def test_group_one_rank_per_gpu(placement):
    """The same group with one rank per GPU of the process (peer memory over
    NVLink, every rank's sync concurrent on its GPU): FSDP-N -> TP2 x N/2 on
    the GPUs present (skipped on a one-GPU box)."""
    import paper_2605_06534_b200 as ws
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs 2+ GPUs")
    n = 4 if n >= 4 else 2
    manifest = ws.MODELS["qwen2.5-0.5b"]([0, 1, 23])
    g = ws.EngineGroup(manifest, ws.BF16, ws.TrainConfig("fsdp"),
                       ws.ServeConfig(2, 1, n // 2, placement), n, device=list(range(n)))
    g.generate(seed=2, density=0.01)
    for k in range(4):
        g.sync_step(reverse=bool(k % 2), report=False)
    assert _serve_equals_gen(ws, g, 2, 0.01, "prev") == []
    reps = g.sync_step()
    assert _serve_equals_gen(ws, g, 2, 0.01, "next") == []
    assert all(r["dense_shards"] == 0 for r in reps)
    g.close()
