#!/usr/bin/env python
"""Where bench.py's e2e step goes at N GPUs: per step, the host wall of
ws_engine_sync_step_host and the report's device stages (wall includes the
H2D of the snapshot), beside a plain torch H2D of the same bytes.  torchrun."""
import json
import os
import sys
import time

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
    plan = ws.Plan(ws.MODELS["qwen3-8b"](), ws.BF16, ws.TrainConfig("fsdp"),
                   ws.ServeConfig(2, 1, world // 2, "overlap"), world=world, rank=rank)
    eng = ws.TransferEngine(plan, device=local, unique_id=obj[0])
    eng.generate(seed=1, density=0.01)
    host = [torch.empty(eng.arena[i].shape, dtype=eng.arena[i].dtype, pin_memory=True)
            for i in range(2)]
    for i in range(2):
        host[i].copy_(eng.arena[i])
    torch.cuda.synchronize()
    scratch = torch.empty_like(eng.arena[0])
    dist.barrier()
    t0 = time.perf_counter()
    scratch.copy_(host[0], non_blocking=True)
    torch.cuda.synchronize()
    h2d = time.perf_counter() - t0
    rev = False
    rows = []
    for k in range(5):
        dist.barrier()
        t0 = time.perf_counter()
        rep, _ = eng.sync_step_host(host[0] if rev else host[1], reverse=rev, report=True)
        torch.cuda.synchronize()
        rows.append({"host_ms": round((time.perf_counter() - t0) * 1e3, 2),
                     "dev_wall_ms": round(rep["wall_s"] * 1e3, 2),
                     "encode_ms": round(rep["encode_s"] * 1e3, 2),
                     "route_ms": round(rep["route_s"] * 1e3, 2)})
        rev = not rev
    print(json.dumps({"rank": rank, "bytes": host[0].numel() * 2,
                      "torch_h2d_ms": round(h2d * 1e3, 2), "steps": rows}), flush=True)


if __name__ == "__main__":
    main()
