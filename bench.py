#!/usr/bin/env python
"""Benchmark: dense-equivalent weight-sync GB/s (encode+route+apply) on B200.

Workload (BASELINE.json configs[1], scaled to the GPUs given): a Qwen3-8B-
shaped bf16 model (8.19 G elements), 1% i.i.d. change density, trainer
FSDP-N shards (every parameter split along dim 0 over the N ranks) -> serving
TP2 replicas (TP1 at N=1), one rank per GPU.  A "step" is one full sync of
the whole model: K1 encode on every trainer shard, route (reslice + NVLink
exchange at N>1) and in-place apply on every serving shard.  Steps alternate
direction (prev->next, next->prev) so every step is a genuine sync and the
serving weights stay verifiable.

    python bench.py [--gpus N --steps K --warmup W]          # our arm
    python bench.py --impl reference [...]                   # the reference's CPU path

Value = 2 B x model elements / (max over ranks of device time per step).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "dense-equivalent weight-sync GB/s (encode+route+apply) at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default=None)
    ap.add_argument("--density", type=float, default=None)
    ap.add_argument("--threshold", type=float, default=0.20)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-layers", type=int, default=1,
                    help="Qwen layers per CPU thread in the reference sample")
    ap.add_argument("--placement", default="overlap", choices=["rank", "overlap"],
                    help="which serving rank each GPU hosts (ws_placement): 'overlap' keeps "
                         "the most trainer->serving elements on their own GPU")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4],
                    help="BASELINE.json config: 2 Qwen3-8B FSDP-N -> TP2 x N/2 at 1%% (default), "
                         "3 Qwen3-32B TP-N -> TP-N/2 x 2 at 0.5%%, 4 Qwen3-30B-A3B expert-sharded "
                         "TP-N -> EP-N, Zipf(1.1) per-expert densities around 1%% (3/4: N >= 2)")
    ap.add_argument("--no-verify", action="store_true",
                    help="skip the bit-exact check of every serving shard after the run")
    args = ap.parse_args()
    preset = CONFIGS[args.config]
    if args.model is None:
        args.model = preset["model"]
    if args.density is None:
        args.density = preset["density"]
    return args


# BASELINE.json configs this bench can run (config 1 is the CPU reference's
# own case; config 5 is the density sweep, scripts/density_sweep.py)
CONFIGS = {
    2: {"model": "qwen3-8b", "density": 0.01},
    3: {"model": "qwen3-32b", "density": 0.005},
    4: {"model": "qwen3-30b-a3b", "density": 0.01, "zipf": 1.1},
}


def load_manifest_module():
    """paper_2605_06534_b200/manifest.py by path: the model shapes without
    importing the package (whose __init__ maps libwsync.so) -- the reference
    arm must not load this repo's library."""
    import importlib.util
    path = os.path.join(ROOT, "paper_2605_06534_b200", "manifest.py")
    spec = importlib.util.spec_from_file_location("_wsync_manifest", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_wsync_manifest"] = mod
    spec.loader.exec_module(mod)
    return mod


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def layouts(n, config=2):
    """(trainer layout, serving tp, replicas, description) at n GPUs:
    config 2: FSDP-N -> TP2 x N/2 (TP1 at N=1); config 3: TP-N -> TP-N/2 x 2;
    config 4: expert-sharded TP-N -> EP-N (one replica)."""
    if config == 3:
        tp = max(1, n // 2)
        return ("tp", n), tp, n // tp, f"trainer TP{n} -> serving TP{tp} x {n // tp} replica(s)"
    if config == 4:
        return ("tp", n), n, 1, f"expert-sharded trainer TP{n} -> serving EP{n} (TP{n})"
    tp = 1 if n == 1 else 2
    return ("fsdp", n), tp, n // tp, f"trainer FSDP{n} -> serving TP{tp} x {n // tp} replica(s)"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons of this rank's GPU, sampled
    through NVML every ~5 ms while the timed region runs (the same counters
    nvidia-smi's clocks.sm / clocks_event_reasons.* report)."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu):
        self.gpu, self.rows, self.h, self.stop = gpu, [], None, threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[gpu]) if vis and vis.split(",")[0].isdigit() else gpu
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except AttributeError:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.rows.append((sm, r))

    def _loop(self):
        while not self.stop.is_set():
            self._sample()
            self.stop.wait(0.005)

    def __enter__(self):
        if self.h is not None:
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.h is not None:
            self.stop.set()
            self.t.join(timeout=2)
            self._sample()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({name for (_, r) in self.rows for bit, name in self.REASONS.items()
                          if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.rows),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.rows),
                "source": "nvml"}


# ---------------------------------------------------------------------------
# The reference's CPU path (oracle/_ref, the unmodified transfer engine)
# ---------------------------------------------------------------------------

def cpu_reference(args, threads=None, reps=1, warmup=0):
    """Times TransferEngine::sync_step of the compiled reference on a bounded
    sample of the same workload: one Qwen layer (no embedding) per thread, I32
    weights of identical element counts (the reference has no bf16; I32 is the
    dtype whose exact wrap rule the bf16 path mirrors), Async + shard-aware +
    sparse, threshold 0.20, MemoryRelay, unthrottled.  The
    layout is TP1 -> TP1: FSDP1 -> TP1 is the same tensor set, and the
    reference cannot express FSDP -> TP2 (no cross-dim reslice)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import I32, Reference
    mf = load_manifest_module()
    ref = Reference()
    try:  # the CPUs this process may run on (cgroup / affinity), not the host's count
        nproc = len(os.sched_getaffinity(0)) or 1
    except (AttributeError, OSError):
        nproc = os.cpu_count() or 1
    layer_elems = sum(p.numel() for p in mf.MODELS[args.model](layer_subset=[1]))
    # 3 copies (prev, next, serving) at 4 B/elem per thread, at most half the free RAM
    try:
        avail = int([l for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0]
                    .split()[1]) * 1024
    except Exception:
        avail = 32 << 30
    per = layer_elems * args.cpu_sample_layers * 4 * 3 * 1.3
    t = threads or nproc
    t = max(1, min(t, nproc, int(avail * 0.5 // per)))
    states = []

    # middle layers only (layer 0 and the last carry the embedding / lm_head)
    mid = max(1, max(p.layer for p in mf.MODELS[args.model]()) - 1)

    def make(i):
        layers = [1 + i * args.cpu_sample_layers + k for k in range(args.cpu_sample_layers)]
        layers = [1 + (l - 1) % mid for l in layers]
        m = [p.as_tuple() for p in mf.MODELS[args.model](layer_subset=layers)]
        return ref.state(m, I32, (1, 1, 1), (1, 1), args.density, args.seed + i)

    with ThreadPoolExecutor(t) as ex:
        states = list(ex.map(make, range(t)))
    elems = sum(st.model_bytes() / 4 for st in states)
    walls = []
    with ThreadPoolExecutor(t) as ex:
        for it in range(warmup + reps):
            # ServeState::init outside the timed region: the timed part is
            # TransferEngine::sync_step alone, as bench.cpp:21-43 times it
            list(ex.map(lambda st: st.prepare(), states))
            t0 = time.perf_counter()
            reps_ = list(ex.map(lambda st: st.run(True, True, True, args.threshold, 64 << 20),
                                states))
            if it >= warmup:  # untimed warm-up reps first
                walls.append(time.perf_counter() - t0)
    wall = statistics.median(walls)
    gbs = elems * 2 / wall / 1e9
    return {"value": gbs, "unit": "GB/s", "cores": t, "kind": "reference",
            "sample": f"{t} thread(s) x {args.cpu_sample_layers} {args.model} layer(s) "
                      f"({int(elems):,} elements, I32 weights, {args.density:.2%} density), "
                      f"reference TransferEngine::sync_step TP1->TP1 Async+shard-aware+sparse; "
                      f"dense-eq at 2 B/elem ({gbs * 2:.3f} GB/s at 4 B/elem)",
            "wall_s": wall, "elems": int(elems),
            "sync_wall_s_max": max(r["wall_s"] for r in reps_),
            "encode_s_sum": sum(r["encode_s"] for r in reps_),
            "host_cpus": nproc}


def run_reference_arm(args):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    # bounded: at most 3 timed reps and 1 warm-up rep of the CPU sample, so the
    # arm ends within minutes
    reps, warm = max(1, min(args.steps, 3)), min(max(args.warmup, 0), 1)
    cb = cpu_reference(args, reps=reps, warmup=warm)
    mf = load_manifest_module()
    model_elems = sum(p.numel() for p in mf.MODELS[args.model]())
    line = {"metric": METRIC, "value": round(cb["value"], 4), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": reps, "warmup": warm,
            "ms_per_step": round(cb["wall_s"] * 1e3 * (model_elems / max(cb["elems"], 1)), 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "i32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.model} {args.density:.2%} density weight sync, "
                                   f"reference CPU path (TransferEngine::sync_step timed alone) "
                                   f"on a bounded layer sample (TP1->TP1)",
                       "model": args.model, "density": args.density},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": round(cb["value"], 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2605_06534_b200 as ws
    world, rank, local = dist_env()
    n = world if world > 1 else args.gpus
    if world == 1 and args.gpus != 1:
        print(json.dumps({"error": "--gpus > 1 needs torchrun (one process per GPU)"}))
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [ws.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]

    if args.config in (3, 4) and n < 2:
        print(json.dumps({"error": f"config {args.config} ({args.model}) needs >= 2 GPUs: "
                                   "prev + next + serving copies exceed one GPU's HBM"}))
        return 2
    manifest = ws.MODELS[args.model]()
    (scheme, _), tp, replicas, layout_desc = layouts(n, args.config)
    train = ws.TrainConfig("fsdp") if scheme == "fsdp" else ws.TrainConfig("tp", n, 1, 1)
    plan = ws.Plan(manifest, ws.BF16, train, ws.ServeConfig(tp, 1, replicas, args.placement),
                   world=n, rank=rank)
    eng = ws.TransferEngine(plan, device=local, unique_id=uid)
    zipf = CONFIGS[args.config].get("zipf")
    eng.generate(seed=args.seed, density=args.density, expert_zipf=zipf, perm_seed=11)
    torch.cuda.synchronize()
    model_elems = plan.info.model_elems
    dense_eq_bytes = 2 * model_elems
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    # ---- warm-up (also sizes the record buffers) ----
    rev = False
    for _ in range(max(3, args.warmup)):
        eng.sync_step(sparse=True, density_threshold=args.threshold, reverse=rev, report=False)
        rev = not rev
    torch.cuda.synchronize()
    probe = eng.sync_step(sparse=True, density_threshold=args.threshold, reverse=rev, report=True)
    rev = not rev
    xbytes = eng.exchange_bytes() if n > 1 else None
    eng.timing(reset=True)

    # ---- timed region: K syncs, no host synchronisation inside ----
    nvl = NvlinkCounters(local) if n > 1 else None
    # no collector pause while the syncs are enqueued: at N > 1 a stalled
    # rank stalls every peer's exchange
    gc.collect()
    gc.disable()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    align = torch.zeros(1, device=dev)
    # BENCH_STEP_TRACE=1: per-step device times and host enqueue times of
    # every rank on stderr (diagnostics; the line's numbers are unchanged)
    trace = os.environ.get("BENCH_STEP_TRACE") == "1"
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] if trace else []
    host_t = []
    with ClockSampler(local) as clocks:
        # the sampler and counter reads start before the barrier, so no rank
        # enters the timed region late; at N > 1 every GPU's start event
        # follows the same collective, so the ranks' regions begin together
        # (otherwise the first sync of an early rank waits for the others)
        nvl0 = nvl.read() if nvl else None
        barrier()
        torch.cuda.synchronize()
        if world > 1:
            dist.all_reduce(align)
        start.record(stream)
        h0 = time.perf_counter()
        for k in range(args.steps):
            eng.sync_step(sparse=True, density_threshold=args.threshold, reverse=rev,
                          report=False)
            rev = not rev
            if trace:
                marks[k].record(stream)
                host_t.append(round((time.perf_counter() - h0) * 1e3, 3))
        end.record(stream)
        torch.cuda.synchronize()
    gc.enable()
    if trace:
        print(json.dumps({"rank": rank, "step_end_ms": [round(start.elapsed_time(m), 3)
                                                        for m in marks],
                          "host_enqueued_ms": host_t}), file=sys.stderr, flush=True)
    nvl1 = nvl.read() if nvl else None
    barrier()
    ms = start.elapsed_time(end) / args.steps
    tim = eng.timing(reset=True)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = dense_eq_bytes / (ms_max * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (K1 encode) ----
    enc_s = tim["encode_s"] / max(1, tim["steps"])
    route_s = tim["route_s"] / max(1, tim["steps"])
    train_elems = plan.info.train_elems
    nnz = probe["nnz"]
    # K1 reads prev+next (2 B each) and writes idx u32 + val u16 per change;
    # with the fused apply (always on in the product build) it also
    # read-modify-writes the 2-B serving element of every change routed to
    # this GPU's own serving shard (4 B).
    my_coord = plan.info.serve_coord
    local_frac = (sum(ov for (_, c, _, ov) in plan.routes if c == my_coord) /
                  max(1, train_elems))
    alg_bytes = int(4 * train_elems + 6 * nnz + 4 * nnz * local_frac)
    peak, peak_src = load_peaks()
    achieved = alg_bytes / enc_s / 1e9 if enc_s > 0 else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "encode_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("model") == args.model and tr.get("n_gpus") == n:
            traffic = tr.get("dram_bytes_per_launch")
    except Exception:
        pass

    # ---- route stage on NVLink (N > 1) ----
    route = None
    if n > 1:
        sent = xbytes["sent_record_bytes"] + xbytes["sent_dense_bytes"]
        # 6 B per record (u32 index + u16 value) per remote
        # replica -- also the wire format (SoA u32 shard-local index + u16)
        wire_b = 6
        remote_recs = xbytes["sent_record_bytes"] // wire_b
        pack_s = tim["pack_s"] / tim["pack_steps"] if tim.get("pack_steps") else None
        # the NVLink kernel's window: the pack (single-round exchange), else
        # the whole route stage (pack + receiver scatter)
        win = pack_s or route_s
        route = {"bytes_per_sync": sent, "wire_bytes_per_record": wire_b,
                 "alg_bytes_per_sync": 6 * remote_recs + xbytes["sent_dense_bytes"],
                 "recv_bytes_per_sync": xbytes["recv_record_bytes"],
                 "stage_ms": round(route_s * 1e3, 4),
                 "pack_ms": round(pack_s * 1e3, 4) if pack_s else None,
                 "window": "pack_kernel (NVLink stores)" if pack_s else "route stage",
                 "nvlink_gbs": round(sent / win / 1e9, 1) if win > 0 else None,
                 "peak_gbs": 900.0, "measured_peer_copy_gbs": 770.0,
                 "frac_of_900": round(sent / win / 1e9 / 900.0, 4) if win > 0 else None,
                 "frac_of_770": round(sent / win / 1e9 / 770.0, 4) if win > 0 else None}
        try:  # the pack kernel's NVLink counters from the committed ncu capture
            with open(os.path.join(ROOT, "profiles", "route_ncu.json")) as f:
                rn = json.load(f).get(str(n))
            if rn and args.config == 2:
                route["ncu_pack_nvltx_gbs"] = round(rn["pack_nvltx_gbs_mean"], 1)
                route["ncu_pack_frac_of_900"] = round(rn["pack_frac_of_900_mean"], 4)
                route["ncu_pack_user_gbs"] = round(rn["pack_user_gbs_mean"], 1)
                route["ncu_source"] = "profiles/" + rn["source"]
        except Exception:
            pass
        if nvl0 is not None and nvl1 is not None:
            tx = (nvl1[0] - nvl0[0]) * 1024 / args.steps
            rx = (nvl1[1] - nvl0[1]) * 1024 / args.steps
            route["nvml_tx_bytes_per_sync"] = int(tx)
            route["nvml_rx_bytes_per_sync"] = int(rx)
            if win > 0:
                route["nvml_tx_gbs_over_window"] = round(tx / win / 1e9, 1)

    # ---- end-to-end through the C-ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e, rev = run_e2e(args, eng, plan, world, local, dense_eq_bytes, barrier, rev)

    # ---- bit-exact check of every serving shard (every rank) ----
    verified = None
    if not args.no_verify:
        ok = verify_serving(ws, eng, plan, rev, args, zipf)
        v = torch.tensor([1 if ok else 0], device=dev, dtype=torch.int32)
        if world > 1:
            dist.all_reduce(v, op=dist.ReduceOp.MIN)
        verified = bool(v.item())

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference(args)
            cpu = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in cb.items()
                   if k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # the reference build is test infrastructure; report why
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": n,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_max, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u16",
            "data": "synthetic",
            "config": {"workload": f"BASELINE config {args.config}: {args.model} bf16 weight "
                                   f"sync, {args.density:.2%} "
                                   + ("Zipf(%.1f) per-expert " % zipf if zipf else "i.i.d. ")
                                   + f"change density, {layout_desc}",
                       "config": args.config, "model": args.model, "density": args.density,
                       "density_threshold": args.threshold,
                       "train": f"{scheme}{n}", "serve": f"tp{tp}x{replicas}",
                       "placement": args.placement,
                       "model_elems": model_elems,
                       "l2": "inputs larger than L2 (prev+next %.1f GB per GPU per step)"
                             % (4 * train_elems / 1e9)},
            "per_gpu_value": round(value / n, 2),
            "stages_ms": {"encode": round(enc_s * 1e3, 4),
                          "apply": round(tim["apply_s"] / max(1, tim["steps"]) * 1e3, 4),
                          "route": round(route_s * 1e3, 4)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                         "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4) if achieved else None,
                         "traffic": traffic, "kernel": "encode_kernel<bf16> (K1)",
                         "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src},
            "route": route,
            "e2e": e2e, "cpu_baseline": cpu,
            "gpu_launches": int(tim["kernel_launches"]),
            "clocks": clocks.summary(), "nnz_per_step": nnz,
            "verified": verified,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


class NvlinkCounters:
    """NVLink data throughput counters of this rank's GPU (NVML field values
    NVLINK_THROUGHPUT_DATA_TX / _RX, KiB, summed over the links): read before
    and after the timed region, they give the hardware's count of the bytes
    the exchange moved."""

    def __init__(self, gpu):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[gpu]) if vis and vis.split(",")[0].isdigit() else gpu
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.read()
        except Exception:
            self.h = None

    def read(self):
        if self.h is None:
            return None
        try:
            nv = self.nv
            vals = nv.nvmlDeviceGetFieldValues(self.h, [nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                                        nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
            out = []
            for v in vals:
                if v.nvmlReturn != 0:
                    return None
                out.append(int(v.value.ullVal))
            return out
        except Exception:
            return None


def run_e2e(args, eng, plan, world, local, dense_eq_bytes, barrier, rev):
    """Same metric through the C-ABI's host-buffer entry point: every step
    copies the new snapshot (this rank's trainer arena) from pinned host
    memory and reads the per-shard change counts back."""
    import torch
    arena_bytes = eng.arena[0].numel() * eng.arena[0].element_size()
    try:
        host = [torch.empty(eng.arena[i].shape, dtype=eng.arena[i].dtype, pin_memory=True)
                for i in range(2)]
        pinned = True
    except RuntimeError:
        host = [torch.empty(eng.arena[i].shape, dtype=eng.arena[i].dtype) for i in range(2)]
        pinned = False
    for i in range(2):
        host[i].copy_(eng.arena[i])
    steps = max(1, args.e2e_steps)
    # warm-up step in the current direction; reverse=True reads the new
    # snapshot into arena 0, reverse=False into arena 1
    eng.sync_step_host(host[0] if rev else host[1], density_threshold=args.threshold,
                       reverse=rev, report=False)
    rev = not rev
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        # reverse=True reads the new snapshot into arena 0 (the old "prev")
        eng.sync_step_host(host[0] if rev else host[1], density_threshold=args.threshold,
                           reverse=rev, report=False)
        rev = not rev
    torch.cuda.synchronize()
    barrier()
    gc.enable()
    wall = (time.perf_counter() - t0) / steps
    t = torch.tensor([wall], device=eng.device, dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    wall = float(t.item())
    del host
    return {"value": round(dense_eq_bytes / wall / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": arena_bytes, "d2h_bytes_per_step": 8 * len(plan.segments),
            "steps": steps, "ms_per_step": round(wall * 1e3, 2), "pinned": pinned,
            "path": "ws_engine_sync_step_host (C-ABI), host timer around H2D+sync+D2H"}, rev


def verify_serving(ws, eng, plan, rev, args, zipf):
    """Every serving shard of this rank, bit for bit, after the last sync:
    `next` if it ran forward, `prev` if reversed -- regenerated on the device
    from the generator (oracle/wsync_oracle.c gen_elem), so no rank needs
    another rank's data."""
    import torch
    torch.cuda.synchronize()
    which = "next" if rev else "prev"  # rev was toggled after the last sync
    tabs = {}
    if zipf is not None:
        tabs = {i: ws.expert_thresholds(m.shape[0], args.density, zipf, 11)
                for i, m in enumerate(plan.manifest) if m.kind == ws.ModuleKind.EXPERT}
    for i, (p, desc, off, n) in enumerate(plan.serve_shards):
        meta = plan.manifest[p]
        pv, nx = ws.gen_pair_bf16(args.seed, meta.name, meta.shape, desc, args.density,
                                  device=eng.device, thr_dim0=tabs.get(p))
        want = nx if which == "next" else pv
        if not torch.equal(eng.serve_view(i).view(torch.int16), want.view(torch.int16)):
            return False
        del pv, nx
    return True


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
