"""Debug probe: config 3 layout (TP-N -> TP-N/2 x 2) on a small manifest, P2P
mode; per wrong serving shard, how many elements equal next / prev."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import torch.distributed as dist
import paper_2605_06534_b200 as ws

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(rank % torch.cuda.device_count())
obj = [ws.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
manifest = ws.MODELS["qwen3-32b"]([0, 63]) if os.environ.get("BIG") else ws.toy_transformer_manifest(layers=2, hidden=64, vocab=256)
half = max(1, world // 2)
plan = ws.Plan(manifest, ws.BF16, ws.TrainConfig("tp", world, 1, 1), ws.ServeConfig(half, 1, world // half),
               world=world, rank=rank)
eng = ws.TransferEngine(plan, device=rank % torch.cuda.device_count(), unique_id=obj[0])
eng.generate(seed=5, density=float(os.environ.get("D", "0.01")))
rep = eng.sync_step()
out = {"rank": rank, "coord": plan.info.serve_coord, "nroutes": len(plan.routes), "rep": {k: rep[k] for k in ("nnz", "dense_shards", "sparse_shards")}, "bad": []}
for i, (p, desc, off, n) in enumerate(plan.serve_shards):
    meta = plan.manifest[p]
    pv, nx = ws.gen_pair_bf16(5, meta.name, meta.shape, desc, float(os.environ.get("D", "0.01")), device=eng.device)
    got = eng.serve_view(i).view(torch.int16).reshape(-1)
    nx = nx.view(torch.int16).reshape(-1); pv = pv.view(torch.int16).reshape(-1)
    if not torch.equal(got, nx):
        out["bad"].append((meta.name, desc, int((got == nx).sum()), int((got == pv).sum()), int((nx != pv).sum()), got.numel()))
allr = [None] * world
dist.all_gather_object(allr, out)
if rank == 0:
    for r in allr:
        print(json.dumps(r))
dist.destroy_process_group()
