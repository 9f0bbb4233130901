"""BASELINE configs 3 and 4 timed at the available GPU count (torchrun):
  3: Qwen3-32B, trainer TP-N -> serving TP-N/2 x 2 replicas, 0.5% density;
  4: Qwen3-30B-A3B, expert-sharded trainer TP-N -> EP-N serving, Zipf(1.1)
     per-expert densities around 1%.
By default, layer subsets keep the worst-case receive regions within HBM;
--full runs the whole models and needs WSYNC_MAX_THRESHOLD=0.2.
The reported figure is dense-equivalent GB/s over the synced elements.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/config_bench.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2605_06534_b200 as ws  # noqa: E402


def timed(eng, steps):
    rev = False
    for _ in range(3):
        eng.sync_step(reverse=rev, report=False)
        rev = not rev
    torch.cuda.synchronize()
    rep = eng.sync_step(reverse=rev, report=True)
    rev = not rev
    if dist.is_initialized():
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        eng.sync_step(reverse=rev, report=False)
        rev = not rev
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / steps], device="cuda", dtype=torch.float64)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), rep


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true",
                    help="whole models (set WSYNC_MAX_THRESHOLD=0.2 to bound the receive regions)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def fresh_uid():  # one NCCL communicator per engine
        if world == 1:
            return None
        obj = [ws.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]
    half = max(1, world // 2)
    cases = [
        ("config3", "qwen3-32b", None if args.full else list(range(0, 64, 4)),
         ws.TrainConfig("tp", world, 1, 1), ws.ServeConfig(half, 1, world // half), 0.005, None),
        ("config4", "qwen3-30b-a3b", None if args.full else list(range(0, 48, 4)),
         ws.TrainConfig("tp", world, 1, 1), ws.ServeConfig(world, 1, 1), 0.01, 1.1),
    ]
    for name, model, layers, train, serve, density, zipf in cases:
        manifest = ws.MODELS[model](layers)
        plan = ws.Plan(manifest, ws.BF16, train, serve, world=world, rank=rank)
        eng = ws.TransferEngine(plan, device=local, unique_id=fresh_uid())
        eng.generate(seed=2, density=density, expert_zipf=zipf, perm_seed=11)
        ms, rep = timed(eng, 10)
        elems = plan.info.model_elems
        if rank == 0:
            print(json.dumps({"config": name, "model": model,
                              "layers": "all" if layers is None else len(layers),
                              "elements": elems, "n_gpus": world, "density": density,
                              "expert_zipf": zipf, "train": train.scheme if hasattr(train, "scheme") else "tp",
                              "serve": f"tp{serve.tp}x{serve.replicas}", "ms_per_sync": round(ms, 3),
                              "dense_eq_gbs": round(2 * elems / ms / 1e6, 1),
                              "rank0_sparse_shards": rep["sparse_shards"],
                              "rank0_dense_shards": rep["dense_shards"]}), flush=True)
        del eng
        torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
