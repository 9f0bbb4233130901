#!/usr/bin/env python
"""Time of the ordered stream of the largest Qwen3-8B segment (the 622 M-
element embedding, 1%): ws_engine_segment_delta's compaction of K1's
unordered per-super-tile record layout (tile-count scan + one warp per
super-tile), CUDA events around repeated calls of the same launch pair."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_06534_b200 as ws  # noqa: E402

m = [p for p in ws.MODELS["qwen3-8b"]() if p.name.endswith("embed_tokens.weight")]
plan = ws.Plan(m, ws.BF16, ws.TrainConfig("fsdp"), ws.ServeConfig(1, 1, 1))
eng = ws.TransferEngine(plan, device=0)
eng.generate(seed=1, density=0.01)
eng.sync_step()
delta, codec, nnz = eng.segment_delta(0)  # warm-up (allocates the ordered buffer)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
reps = 20
ev[0].record()
for _ in range(reps):
    eng.segment_delta(0)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / reps
print(json.dumps({"segment": m[0].name, "elements": plan.segments[0][3], "records": nnz,
                  "ms_per_ordered_stream_incl_host_sync": round(ms, 4),
                  "bytes_moved": nnz * 12}))
