"""Perf probe for K1 on one big shard (ws_diff_shards): GB/s of prev+next read."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_06534_b200 as ws  # noqa: E402
from paper_2605_06534_b200 import codec  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1 << 30
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
density = float(os.environ.get("DENSITY", "0.01"))
full = (n // 4096, 4096)
prev, nxt = ws.gen_pair_bf16(1, "probe", full, (-1, 0, 0), density)
cap = int(0.2 * n)
idx = torch.empty(cap, dtype=torch.int32, device="cuda")
val = torch.empty(cap, dtype=torch.int16, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
wsb = codec._workspace(n, "cuda")
L, P = ws._lib.lib, codec._ptr


def run():
    ws._lib.check(L.ws_diff_shards(ws.BF16, P(prev), P(nxt), prev.numel(), P(idx), P(val), cap,
                                   P(cnt), P(wsb), wsb.numel(), codec._stream()))


for _ in range(3):
    run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(iters):
    run()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / iters
nbytes = 4 * prev.numel()
print(f"n={prev.numel()} debug={os.environ.get('WSYNC_ENCODE_DEBUG', '0')} "
      f"grid={os.environ.get('WSYNC_ENCODE_GRID', 'auto')} nnz={int(cnt.item())} "
      f"ms={ms:.3f} GB/s={nbytes / ms / 1e6:.1f}")
