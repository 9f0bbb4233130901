"""The GPU-aware relay path timed beside the
reference: TransferEngine::sync_step through the compiled reference
MemoryRelay (oracle/_ref, unthrottled, Async), ours with the encode /
decode / reslice / apply on the GPU (ws_engine_sync_relay, bf16) and the
reference's own CPU engine (I32 weights of the same element counts -- the
reference has no bf16).  Both on Qwen2.5-0.5B TP1 -> TP1 at 1% density.

    python scripts/relay_bench.py [--model qwen2.5-0.5b] [--steps 3]

Prints one JSON line: wall seconds per sync and dense-equivalent GB/s
(2 B x elements / wall) for each side.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_06534_b200 as ws  # noqa: E402
from oracle.oracle import I32, Reference  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-0.5b")
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    ref = Reference()
    manifest = ws.MODELS[args.model]()
    elems = sum(p.numel() for p in manifest)

    plan = ws.Plan(manifest, ws.BF16, ws.TrainConfig("fsdp"), ws.ServeConfig(1, 1, 1))
    eng = ws.TransferEngine(plan, device=0)
    eng.generate(seed=1, density=args.density)
    ours, rev, reps = [], False, []
    for k in range(args.steps + 1):  # the first sync warms up
        relay = ref.memory_relay()
        rep = eng.sync_relay(relay.callbacks, step=k + 1, mode="async", reverse=rev)
        rev = not rev
        reps.append({k2: round(v, 4) if isinstance(v, float) else v for k2, v in rep.items()})
        if k:
            ours.append(rep["wall_s"])
    torch.cuda.synchronize()

    st = ref.state([p.as_tuple() for p in manifest], I32, (1, 1, 1), (1, 1), args.density, 1)
    theirs = [st.run(True, True, True, 0.20, 64 << 20)["wall_s"] for _ in range(args.steps)]

    o, t = statistics.median(ours), statistics.median(theirs)
    print(json.dumps({"path": "sync_step through MemoryRelay (Async, unthrottled)",
                      "model": args.model, "elements": elems, "density": args.density,
                      "ours": {"wall_s": round(o, 4), "dense_eq_gbs": round(2 * elems / o / 1e9, 2),
                               "dtype": "bf16", "device": torch.cuda.get_device_name(0),
                               "reports": reps},
                      "reference": {"wall_s": round(t, 4),
                                    "dense_eq_gbs": round(2 * elems / t / 1e9, 3),
                                    "dtype": "i32 (same element count)", "threads": "engine's own"},
                      "speedup": round(t / o, 1)}), flush=True)


if __name__ == "__main__":
    main()
