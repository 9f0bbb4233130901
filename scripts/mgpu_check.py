"""Multi-GPU parity check of the engine (one process per GPU, torchrun).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/mgpu_check.py

Every rank checks its own serving shards after each sync:
  * bf16 FSDP-N -> TP2 x N/2 (cross-dim routes for RowLinear): serving ==
    the generator's `next` values for that shard (regenerated on the device
    from the global element index, so no rank needs another rank's data);
    then a reverse sync restores `prev`; then the dense fallback (45%) and
    sparse=False paths;
  * I32 and F32 with the reference's own layouts (TrainConfig{N,1,1} ->
    ServeConfig{N,1}): serving == the compiled reference engine's serving
    shards (oracle/_ref, run on the same weights on the host).
  * the relay path (ws_engine_sync_relay) with one pusher and one puller
    per rank through a relay shared by the processes (a directory): serving
    == `next`, then a reverse sync through a fresh relay == `prev`.
Prints one JSON line per rank; exits non-zero on any mismatch.
"""
import ctypes as C
import hashlib
import json
import os
import shutil
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2605_06534_b200 as ws  # noqa: E402



# serving-rank placement of every layout (ws_placement); WSYNC_CHECK_PLACEMENT=rank
# checks the reference's rank order instead
PLACEMENT = os.environ.get("WSYNC_CHECK_PLACEMENT", "overlap")


def serve_cfg(tp, pp, replicas):
    return ws.ServeConfig(tp, pp, replicas, PLACEMENT)

def serve_equals_gen(eng, plan, seed, density, which, tabs=None):
    bad = []
    for i, (p, desc, off, n) in enumerate(plan.serve_shards):
        meta = plan.manifest[p]
        pv, nx = ws.gen_pair_bf16(seed, meta.name, meta.shape, desc, density, device=eng.device,
                                  thr_dim0=(tabs or {}).get(p))
        want = (nx if which == "next" else pv).view(torch.int16)
        if not torch.equal(eng.serve_view(i).view(torch.int16), want):
            bad.append(meta.name)
    return bad


class DirRelay:
    """A relay the ranks share through a directory (test infrastructure): put
    writes the bucket to a file named by the key's hash and renames it into
    place; get_any polls the candidate keys until one exists, as
    MemoryRelay::get_any waits on its condition variable (relay.cpp:29-45)."""
    PUT = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64)
    GET = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64), C.c_int,
                      C.c_int, C.POINTER(C.c_int), C.c_void_p, C.c_uint64)

    def __init__(self, path):
        self.path = path
        self._put, self._get = self.PUT(self.put), self.GET(self.get_any)
        self.callbacks = (None, C.cast(self._put, C.c_void_p).value,
                          C.cast(self._get, C.c_void_p).value)

    def _file(self, key):
        return os.path.join(self.path, hashlib.sha1(key).hexdigest())

    def put(self, ctx, key, klen, data, n):
        f = self._file(C.string_at(key, klen))
        with open(f + ".tmp", "wb") as fh:
            fh.write(C.string_at(data, n) if n else b"")
        os.rename(f + ".tmp", f)
        return 0

    def get_any(self, ctx, keys, lens, n, timeout_ms, hit, out, cap):
        files = [self._file(C.string_at(keys[i], lens[i])) for i in range(n)]
        end = time.time() + timeout_ms / 1e3
        while True:
            for i, f in enumerate(files):
                if os.path.exists(f):
                    with open(f, "rb") as fh:
                        b = fh.read()
                    hit[0] = i
                    if len(b) <= cap:
                        C.memmove(out, b, len(b))
                    return len(b)
            if time.time() > end:
                return -1
            time.sleep(0.001)


def relay_case(rank, world, uid_fn, manifest, density, seed, mode):
    """ws_engine_sync_relay on every rank at once (FSDP-N -> TP2 x N/2):
    each rank pushes its trainer shards and pulls every shard routed to its
    serving coordinate (engine.cpp:109-238, one puller per serving rank)."""
    tp = 1 if world == 1 else 2
    plan = ws.Plan(manifest, ws.BF16, ws.TrainConfig("fsdp"), serve_cfg(tp, 1, world // tp),
                   world=world, rank=rank)
    eng = ws.TransferEngine(plan, device=rank % torch.cuda.device_count(), unique_id=uid_fn())
    eng.generate(seed=seed, density=density)
    obj = [tempfile.mkdtemp(prefix="wsync_relay_") if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    bad = []
    for step, (rev, which) in enumerate(((False, "next"), (True, "prev")), start=1):
        relay = DirRelay(obj[0])
        dist.barrier()
        rep = eng.sync_relay(relay.callbacks, step=step, mode=mode, reverse=rev,
                             bucket_bytes=8 << 20, timeout_ms=60000)
        torch.cuda.synchronize()
        bad += [f"step{step}:{b}" for b in serve_equals_gen(eng, plan, seed, density, which)]
        dist.barrier()
    if rank == 0:
        shutil.rmtree(obj[0], ignore_errors=True)
    return bad, rep


def bf16_case(rank, world, uid_fn, manifest, density, seed):
    tp = 1 if world == 1 else 2
    plan = ws.Plan(manifest, ws.BF16, ws.TrainConfig("fsdp"), serve_cfg(tp, 1, world // tp),
                   world=world, rank=rank)
    eng = ws.TransferEngine(plan, device=rank % torch.cuda.device_count(), unique_id=uid_fn())
    eng.generate(seed=seed, density=density)
    rep = eng.sync_step()
    bad = serve_equals_gen(eng, plan, seed, density, "next")
    eng.sync_step(reverse=True)
    bad += serve_equals_gen(eng, plan, seed, density, "prev")
    eng.sync_step(sparse=False)
    bad += serve_equals_gen(eng, plan, seed, density, "next")
    return bad, rep


def layout_case(rank, world, uid_fn, manifest, train, serve, density, seed, zipf=None):
    """BASELINE configs 3/4 at this world size: any trainer -> serving layout,
    optionally with Zipf-skewed per-expert densities; serving == `next`, then
    a reverse sync restores `prev`."""
    plan = ws.Plan(manifest, ws.BF16, train, serve, world=world, rank=rank)
    eng = ws.TransferEngine(plan, device=rank % torch.cuda.device_count(), unique_id=uid_fn())
    eng.generate(seed=seed, density=density, expert_zipf=zipf, perm_seed=11)
    tabs = {}
    if zipf is not None:
        tabs = {i: ws.expert_thresholds(m.shape[0], density, zipf, 11)
                for i, m in enumerate(manifest) if m.kind == ws.ModuleKind.EXPERT}
    rep = eng.sync_step()
    bad = serve_equals_gen(eng, plan, seed, density, "next", tabs)
    eng.sync_step(reverse=True)
    bad += serve_equals_gen(eng, plan, seed, density, "prev", tabs)
    return bad, rep


def ref_case(rank, world, uid_fn, dtype, density, sparse):
    from oracle.oracle import Reference
    ref = Reference()
    st = ref.toy_state(3, 64, 128, dtype, (world, 1, 1), (world, 1), density, 7)
    st.run(mode_async=True, shard_aware=True, sparse=sparse, threshold=0.20, bucket_bytes=8192)
    manifest = [ws.ParamMeta(n, k, tuple(s), l) for (n, k, s, l) in st.params]
    plan = ws.Plan(manifest, dtype, ws.TrainConfig("tp", world, 1, 1), serve_cfg(world, 1, 1),
                   world=world, rank=rank)
    eng = ws.TransferEngine(plan, device=rank % torch.cuda.device_count(), unique_id=uid_fn())
    td = {ws.I32: torch.int32, ws.F32: torch.float32}[dtype]
    full = {i: (torch.from_numpy(st.weights(i, 0, dtype)).to(eng.device),
                torch.from_numpy(st.weights(i, 1, dtype)).to(eng.device))
            for i in range(len(manifest))}
    for s, (p, desc, off, n) in enumerate(plan.segments):
        shp = manifest[p].shape
        eng.segment_view(s, 0).copy_(ws.extract_shard(full[p][0].view(shp).to(td), desc))
        eng.segment_view(s, 1).copy_(ws.extract_shard(full[p][1].view(shp).to(td), desc))
    for s, (p, desc, off, n) in enumerate(plan.serve_shards):
        eng.serve_view(s).copy_(ws.extract_shard(full[p][0].view(manifest[p].shape).to(td), desc))
    eng.sync_step(sparse=sparse)
    bad = []
    for s, (p, desc, off, n) in enumerate(plan.serve_shards):
        want = st.serve(plan.info.serve_coord, p, dtype)
        got = eng.serve_view(s).reshape(-1).cpu().numpy()
        if got.tobytes() != want.tobytes():
            bad.append(manifest[p].name)
    return bad


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(rank % torch.cuda.device_count())

    def uid():
        if world == 1:
            return None
        obj = [ws.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    results = {}
    ok = True
    for name, manifest in (("toy", ws.toy_transformer_manifest(layers=3, hidden=64, vocab=256)),
                           ("qwen2.5-0.5b[0,1,23]", ws.MODELS["qwen2.5-0.5b"]([0, 1, 23]))):
        for density in (0.01, 0.45):
            bad, rep = bf16_case(rank, world, uid, manifest, density, 3)
            results[f"bf16 {name} d={density}"] = bad or "ok"
            ok &= not bad
    # many alternating syncs (the bench's pattern), P2P epochs/acks wrapping
    # through several steps: an even count must leave serving == prev
    manifest = ws.MODELS["qwen2.5-0.5b"]([0, 23])
    tp = 1 if world == 1 else 2
    plan = ws.Plan(manifest, ws.BF16, ws.TrainConfig("fsdp"), serve_cfg(tp, 1, world // tp),
                   world=world, rank=rank)
    eng = ws.TransferEngine(plan, device=rank % torch.cuda.device_count(), unique_id=uid())
    eng.generate(seed=8, density=0.02)
    for k in range(10):
        eng.sync_step(reverse=bool(k % 2), report=False, sparse=(k % 3 != 2))
    torch.cuda.synchronize()
    bad = serve_equals_gen(eng, plan, 8, 0.02, "prev")
    results["10 alternating syncs"] = bad or "ok"
    ok &= not bad
    if world > 1:
        # receive regions are sized for density_threshold 0.20 (engine.hpp:27);
        # a sync asking for more grows them on every rank first, and a 30%
        # sync that stays sparse at 0.45 must still be exact
        eng.generate(seed=9, density=0.3)
        eng.sync_step(density_threshold=0.45, report=False)
        eng.sync_step(density_threshold=0.45, reverse=True, report=False)
        eng.sync_step(density_threshold=0.45, report=False)
        torch.cuda.synchronize()
        bad = serve_equals_gen(eng, plan, 9, 0.3, "next")
        results["threshold raised to 0.45"] = bad or "ok"
        ok &= not bad
    del eng

    # BASELINE config 3 (Qwen3-32B TP8 -> TP4 x 2, 0.5%) and config 4
    # (Qwen3-30B-A3B expert-sharded, Zipf(1.1) per-expert densities around
    # 1%), on layer subsets, scaled to this world size
    half = max(1, world // 2)
    for name, manifest, train, serve, density, zipf in (
            ("config3 qwen3-32b[0,63]", ws.MODELS["qwen3-32b"]([0, 63]),
             ws.TrainConfig("tp", world, 1, 1), serve_cfg(half, 1, world // half), 0.005,
             None),
            ("config4 qwen3-30b-a3b[0,47]", ws.MODELS["qwen3-30b-a3b"]([0, 47]),
             ws.TrainConfig("tp", world, 1, 1), serve_cfg(world, 1, 1), 0.01, 1.1)):
        bad, rep = layout_case(rank, world, uid, manifest, train, serve, density, 5, zipf)
        results[name] = bad or "ok"
        results[name + " shards dense/sparse"] = (rep["dense_shards"], rep["sparse_shards"])
        ok &= not bad
    # replica fan-out: FSDP-N -> TP1 x N replicas, every record to all N
    # serving ranks (the N = 8 bench layout sends to 4 replicas)
    if world > 1:
        for density in (0.01, 0.45):
            bad, rep = layout_case(rank, world, uid, ws.MODELS["qwen2.5-0.5b"]([0, 23]),
                                   ws.TrainConfig("fsdp"), serve_cfg(1, 1, world), density, 7)
            results[f"fan-out tp1x{world} d={density}"] = bad or "ok"
            ok &= not bad
    for dtype in (ws.I32, ws.F32):
        for density, sparse in ((0.05, True), (0.45, True), (0.05, False)):
            bad = ref_case(rank, world, uid, dtype, density, sparse)
            results[f"ref dtype={dtype} d={density} sparse={sparse}"] = bad or "ok"
            ok &= not bad
    if world > 1:
        for density, mode in ((0.01, "async"), (0.45, "batch")):
            bad, rep = relay_case(rank, world, uid, ws.MODELS["qwen2.5-0.5b"]([0, 23]), density, 6,
                                  mode)
            results[f"relay {mode} d={density}"] = bad or (rep["pull_buckets"], rep["push_buckets"])
            ok &= not bad
    # rank 0 prints every rank's line (concurrent writers can interleave)
    allres = [None] * world
    dist.all_gather_object(allres, {"rank": rank, "world": world, "ok": ok, "results": results})
    if rank == 0:
        for r in allres:
            print(json.dumps(r), flush=True)
    dist.destroy_process_group()
    return 0 if all(r["ok"] for r in allres) else 1


if __name__ == "__main__":
    sys.exit(main())
