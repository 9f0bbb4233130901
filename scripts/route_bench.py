#!/usr/bin/env python
"""The route stage (pack -> NVLink stores -> receive-side scatter) measured in
ONE process: an EngineGroup with one rank per GPU (peer memory over NVLink),
the deployment's kernels, so ncu -- which profiles one process -- can read
the NVLink counters of pack_kernel.

    python scripts/route_bench.py --gpus 2 [--steps 10 --model qwen3-8b --density 0.01]

Prints one JSON line: per-rank stage times (CUDA events), the bytes each rank
stored into its peers (ws_engine_exchange_bytes) and the NVLink rate over the
pack kernel's window.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_06534_b200 as ws  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--model", default="qwen3-8b")
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--serve-tp", type=int, default=2)
    ap.add_argument("--dense", action="store_true", help="sparse=False syncs (dense box copies)")
    ap.add_argument("--placement", default="overlap", choices=["rank", "overlap"])
    args = ap.parse_args()
    n = args.gpus
    tp = min(args.serve_tp, n)
    g = ws.EngineGroup(ws.MODELS[args.model](), ws.BF16, ws.TrainConfig("fsdp"),
                       ws.ServeConfig(tp, 1, n // tp, args.placement), n,
                       device=list(range(n)))
    g.generate(seed=1, density=args.density)
    rev = False
    for _ in range(args.warmup):
        g.sync_step(sparse=not args.dense, reverse=rev, report=False)
        rev = not rev
    for e in g.engines:
        e.timing(reset=True)
    for _ in range(args.steps):
        g.sync_step(sparse=not args.dense, reverse=rev, report=False)
        rev = not rev
    ranks = []
    for e in g.engines:
        t = e.timing(reset=True)
        xb = e.exchange_bytes()
        k = max(1, t["steps"])
        pack = t["pack_s"] / t["pack_steps"] if t["pack_steps"] else None
        sent = xb["sent_record_bytes"] + xb["sent_dense_bytes"]
        ranks.append({"device": e.device.index, "encode_ms": t["encode_s"] / k * 1e3,
                      "route_ms": t["route_s"] / k * 1e3,
                      "pack_ms": pack * 1e3 if pack else None, **xb,
                      "nvlink_gbs_over_pack": sent / pack / 1e9 if pack else None})
    ok = True
    for q, e in enumerate(g.engines):  # serving == the direction of the last sync
        for i, (p, desc, off, nn) in enumerate(e.plan.serve_shards):
            meta = e.plan.manifest[p]
            pv, nx = ws.gen_pair_bf16(1, meta.name, meta.shape, desc, args.density,
                                      device=e.device)
            want = nx if rev else pv
            ok &= bool(torch.equal(e.serve_view(i).view(torch.int16), want.view(torch.int16)))
    print(json.dumps({"gpus": n, "model": args.model, "density": args.density, "dense": args.dense,
                      "placement": args.placement,
                      "layout": f"FSDP{n} -> TP{tp} x {n // tp}", "steps": args.steps,
                      "verified": ok, "ranks": ranks}), flush=True)
    g.close()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
