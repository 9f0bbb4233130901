"""One-GPU plans of multi-rank layouts (ws_plan_create with world 1 and a
TrainConfig{tp,pp,dp} / ServeConfig{tp,pp} of several ranks): the GPU
encodes every trainer rank's shards and holds every serving coordinate, all
routes local -- TransferEngine::sync_step's whole layout (engine.cpp:66-254)
on one device.  Checked against the compiled reference engine on the
reference's own randomized layout space (transfer_cases.hpp:19-35), I32 and
F32, and bf16 against the generator."""
import numpy as np
import pytest
import torch

from oracle.oracle import F32, I32

pytestmark = pytest.mark.gpu

LAYOUTS = [((2, 1, 2), (2, 1)), ((1, 2, 3), (1, 2)), ((4, 2, 3), (2, 2)), ((2, 2, 1), (4, 1)),
           ((1, 1, 3), (2, 2)), ((4, 1, 1), (1, 2))]


@pytest.mark.parametrize("train,serve", LAYOUTS)
@pytest.mark.parametrize("dtype", [I32, F32])
@pytest.mark.parametrize("density", [0.05, 0.45])
def test_one_gpu_layout_matches_reference_engine(reference, dtype, train, serve, density):
    import paper_2605_06534_b200 as ws
    st = reference.toy_state(4, 64, 128, dtype, train, serve, density, 7)
    ref_rep = st.run(mode_async=True, shard_aware=True, sparse=True, threshold=0.20,
                     bucket_bytes=8192)
    manifest = [ws.ParamMeta(n, k, tuple(s), l) for (n, k, s, l) in st.params]
    plan = ws.Plan(manifest, dtype, ws.TrainConfig("tp", *train),
                   ws.ServeConfig(serve[0], serve[1], 1), world=1, rank=0)
    assert plan.info.serve_coord == -1 and set(plan.serve_coords) == set(range(serve[0] * serve[1]))
    eng = ws.TransferEngine(plan, device=0)
    td = {I32: torch.int32, F32: torch.float32}[dtype]
    for s, (p, desc, off, n) in enumerate(plan.segments):
        shp = plan.manifest[p].shape
        for which in (0, 1):
            full = torch.from_numpy(st.weights(p, which, dtype)).cuda().view(shp).to(td)
            eng.segment_view(s, which).copy_(ws.extract_shard(full, desc))
    for s, (p, desc, off, n) in enumerate(plan.serve_shards):
        full = torch.from_numpy(st.weights(p, 0, dtype)).cuda().view(plan.manifest[p].shape)
        eng.serve_view(s).copy_(ws.extract_shard(full.to(td), desc))
    rep = eng.sync_step(sparse=True, density_threshold=0.20)
    assert rep["dense_shards"] == ref_rep["dense_shards"]
    assert rep["sparse_shards"] == ref_rep["sparse_shards"]
    assert rep["pushed_bytes"] == ref_rep["pushed_bytes"]
    for s, (p, desc, off, n) in enumerate(plan.serve_shards):
        want = st.serve(plan.serve_coords[s], p, dtype)
        got = eng.serve_view(s).reshape(-1).cpu().numpy()
        assert got.tobytes() == np.ascontiguousarray(want).tobytes(), (plan.manifest[p].name,
                                                                        plan.serve_coords[s])


def test_one_gpu_layout_bf16_qwen():
    """bf16 Qwen2.5-0.5B layers, trainer TP2 x PP2 x DP2 -> serving TP4 x PP2
    on one GPU: several local routes per segment (a TP2 shard feeds two TP4
    coordinates), so only single-route segments are fused into K1."""
    import paper_2605_06534_b200 as ws
    m = ws.MODELS["qwen2.5-0.5b"]([0, 1, 2, 23])
    plan = ws.Plan(m, ws.BF16, ws.TrainConfig("tp", 2, 2, 2), ws.ServeConfig(4, 2, 1),
                   world=1, rank=0)
    eng = ws.TransferEngine(plan, device=0)
    eng.generate(seed=4, density=0.01)
    for k in range(3):
        eng.sync_step(reverse=bool(k % 2))
    for i, (p, desc, off, n) in enumerate(plan.serve_shards):
        meta = plan.manifest[p]
        pv, nx = ws.gen_pair_bf16(4, meta.name, meta.shape, desc, 0.01, device=eng.device)
        assert torch.equal(eng.serve_view(i).view(torch.int16), nx.view(torch.int16)), meta.name
