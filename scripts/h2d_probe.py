#!/usr/bin/env python
"""Host->device copy rate of pinned memory per GPU, each rank alone and all
ranks at once (what bounds bench.py's e2e at N > 1).  torchrun, one rank per
GPU; prints one JSON line per rank."""
import json
import os
import time

import torch
import torch.distributed as dist


def rate(dst, src, reps=3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    return reps * src.numel() * src.element_size() / (time.perf_counter() - t0) / 1e9


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    out = {"rank": rank, "world": world}
    gib = float(os.environ.get("H2D_GIB", "2"))
    nbuf = int(os.environ.get("H2D_BUFS", "1"))
    n = int(gib * (1 << 30)) // 2
    dst = torch.empty(n, dtype=torch.int16, device=dev)
    srcs = [torch.empty(n, dtype=torch.int16, pin_memory=True) for _ in range(nbuf)]
    for s in srcs:
        s.fill_(1)
    rate(dst, srcs[0], 1)
    alone = None
    for r in range(world):
        dist.barrier()
        if r == rank:
            alone = rate(dst, srcs[0])
    dist.barrier()
    t0 = time.perf_counter()
    for k in range(6):  # alternating buffers, as bench.py's e2e does
        dst.copy_(srcs[k % nbuf], non_blocking=True)
        torch.cuda.synchronize()
    together = 6 * n * 2 / (time.perf_counter() - t0) / 1e9
    dist.barrier()
    d2h = rate(srcs[0], dst, 3)
    out.update({"gib": gib, "bufs": nbuf, "h2d_alone_gbs": round(alone, 1),
                "h2d_all_ranks_gbs": round(together, 1), "d2h_gbs": round(d2h, 1)})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
