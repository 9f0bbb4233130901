"""The N>1 host logic on CPU: two gloo ranks (world_size 2), no GPU.

* Every rank's static exchange sizes agree with its peers' (what rank r may
  send to coordinate c is what each receiver holding c expects from r).
* A whole distributed sync is simulated with the C restatement over the
  engine's own plan: each rank diffs its trainer shards (FSDP dim-0 slices),
  reslices every route's records into the destination serving shard --
  including RowLinear cross-dim routes -- ships them to the ranks holding
  that coordinate over gloo, and applies them.  Every serving shard must then
  equal the generator's `next` values.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        q.put((rank, _run(rank, world)))
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put((rank, "ERROR " + repr(e) + traceback.format_exc()))


def _run(rank, world):
    import paper_2605_06534_b200 as ws
    from oracle.oracle import BF16, Restatement
    orc = Restatement()
    manifest = ws.toy_transformer_manifest(layers=2, hidden=32, vocab=64)
    serve = ws.ServeConfig(2, 1, world // 2)
    plan = ws.Plan(manifest, ws.BF16, ws.TrainConfig("fsdp"), serve, world=world, rank=rank)

    # 1. exchange capacities agree across ranks
    s_cap = (C.c_uint64 * 2)()
    r_cap = (C.c_uint64 * world)()
    ws._lib.check(ws._lib.lib.ws_plan_exchange_caps(plan.h, s_cap, r_cap))
    caps = [None] * world
    dist.all_gather_object(caps, (plan.info.serve_coord, list(s_cap), list(r_cap)))
    for g, (coord_g, _, recv_g) in enumerate(caps):
        for r, (_, send_r, _) in enumerate(caps):
            if r != g:
                assert recv_g[r] == send_r[coord_g], (g, r)

    # 2. distributed sync through the plan's routes, computed with the oracle
    seed, density = 5, 0.05
    coord_plans = {c: ws.Plan(manifest, ws.BF16, ws.TrainConfig("fsdp"), serve, world=world,
                              rank=c) for c in range(2)}
    outbox = []  # (coord, param, dst desc, idx, val)
    for (seg, coord, nrep, ov) in plan.routes:
        p, src, off, n = plan.segments[seg]
        meta = plan.manifest[p]
        prev, nxt = orc.gen_pair_bf16(seed, meta.name, meta.shape, src, density)
        idx, val = orc.diff_shards(BF16, prev, nxt)
        dst = next(d for (pp, d, o, nn) in coord_plans[coord].serve_shards if pp == p)
        ri, rv = orc.reslice_delta(BF16, meta.shape, src, dst, idx, val, allow_cross_dim=True)
        outbox.append((coord, p, dst, ri.tolist(), rv.tolist()))
    inboxes = [None] * world
    dist.all_gather_object(inboxes, outbox)
    my_coord = plan.info.serve_coord
    bad = 0
    for (p, dst, off, n) in plan.serve_shards:
        meta = plan.manifest[p]
        tgt, want = orc.gen_pair_bf16(seed, meta.name, meta.shape, dst, density)
        for box in inboxes:
            for (coord, pp, d, ri, rv) in box:
                if coord == my_coord and pp == p:
                    tgt, rc = orc.apply_delta(BF16, tgt, np.array(ri, np.uint64),
                                              np.array(rv, np.uint16))
                    assert rc == 0
        bad += int(tgt.tobytes() != want.tobytes())
    return {"coord": my_coord, "bad": bad, "shards": len(plan.serve_shards)}


@pytest.mark.parametrize("world", [2])
def test_two_ranks_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(results[r], str), results[r]
        assert results[r]["bad"] == 0 and results[r]["shards"] > 0, results[r]
