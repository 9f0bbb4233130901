#!/usr/bin/env python
"""A heavy-exchange layout on the GPUs at hand: Qwen3-8B FSDP-N -> TP1 x N
replicas (every record to N - 1 peers: remote share N - 1, like BASELINE
config 2 at N = 8 with 3.15).  torchrun, one rank per GPU; aligned CUDA-event
timing as bench.py; prints one JSON line (rank 0)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2605_06534_b200 as ws  # noqa: E402


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [ws.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    density = float(os.environ.get("FANOUT_DENSITY", "0.01"))
    steps = int(os.environ.get("FANOUT_STEPS", "10"))
    plan = ws.Plan(ws.MODELS["qwen3-8b"](), ws.BF16, ws.TrainConfig("fsdp"),
                   ws.ServeConfig(1, 1, world, "overlap"), world=world, rank=rank)
    eng = ws.TransferEngine(plan, device=local, unique_id=obj[0])
    eng.generate(seed=1, density=density)
    rev = False
    for _ in range(4):
        eng.sync_step(reverse=rev, report=False)
        rev = not rev
    torch.cuda.synchronize()
    eng.timing(reset=True)
    dist.barrier()
    dist.all_reduce(torch.zeros(1, device="cuda"))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        eng.sync_step(reverse=rev, report=False)
        rev = not rev
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / steps], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tm = eng.timing(reset=True)
    if rank == 0:
        print(json.dumps({"layout": f"FSDP{world} -> TP1 x {world}", "density": density,
                          "ms_per_step": round(float(t.item()), 4),
                          "encode_ms": round(tm["encode_s"] * 1e3 / max(1, tm["steps"]), 3),
                          "route_ms": round(tm["route_s"] * 1e3 / max(1, tm["steps"]), 3),
                          "overlap_sms": os.environ.get("WSYNC_OVERLAP_SMS"),
                          "rounds": os.environ.get("WSYNC_ROUNDS")}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
