"""BASELINE config 5: change-density sweep on Qwen3-8B shapes, sparse deltas
(with the 0.20 dense fallback) vs always-dense transfer, at N GPUs.

    python scripts/density_sweep.py [--model qwen3-8b] [--steps 5]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/density_sweep.py

One JSON line per density (rank 0): device ms per sync and dense-equivalent
GB/s for both modes, and the crossover the engine's threshold implies.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2605_06534_b200 as ws  # noqa: E402

DENSITIES = [1e-4, 1e-3, 1e-2, 5e-2, 0.1, 0.2, 0.3, 0.5]


def timed(eng, steps, **kw):
    rev = False
    for _ in range(2):
        eng.sync_step(reverse=rev, report=False, **kw)
        rev = not rev
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.timing(reset=True)
    if dist.is_initialized():
        dist.barrier()
        # every GPU's start event follows the same collective (bench.py)
        dist.all_reduce(torch.zeros(1, device="cuda"))
    s.record()
    for _ in range(steps):
        eng.sync_step(reverse=rev, report=False, **kw)
        rev = not rev
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    tm = eng.timing(reset=True)
    timed.stages = {k: round(tm[k] * 1e3 / max(1, tm["steps"]), 3)
                    for k in ("encode_s", "apply_s", "route_s") if k in tm}
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # leave serving == arena[0] (even number of syncs per phase)
    if rev:
        eng.sync_step(reverse=True, report=False, **kw)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen3-8b")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--densities", default=None, help="comma-separated subset")
    ap.add_argument("--placement", default="overlap", choices=["rank", "overlap"])
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [ws.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    tp = 1 if world == 1 else 2
    plan = ws.Plan(ws.MODELS[args.model](), ws.BF16, ws.TrainConfig("fsdp"),
                   ws.ServeConfig(tp, 1, world // tp, args.placement), world=world, rank=rank)
    eng = ws.TransferEngine(plan, device=local, unique_id=uid)
    dense_eq = 2 * plan.info.model_elems
    for d in ([float(x) for x in args.densities.split(',')] if args.densities else DENSITIES):
        eng.generate(seed=1, density=d)
        rep = eng.sync_step(reverse=False)
        eng.sync_step(reverse=True, report=False)
        ms_sparse = timed(eng, args.steps, sparse=True, density_threshold=0.20)
        stages = timed.stages
        ms_dense = timed(eng, args.steps, sparse=False)
        if rank == 0:
            print(json.dumps({
                "config": 5, "model": args.model, "n_gpus": world, "density": d,
                "placement": args.placement,
                "sparse_ms": round(ms_sparse, 3), "dense_ms": round(ms_dense, 3),
                "sparse_gbs": round(dense_eq / ms_sparse / 1e6, 1),
                "dense_gbs": round(dense_eq / ms_dense / 1e6, 1),
                "sparse_shards": rep["sparse_shards"], "dense_shards": rep["dense_shards"],
                "sparse_faster": ms_sparse < ms_dense, "sparse_stages_ms": stages}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
