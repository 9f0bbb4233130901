"""Summarise the ncu captures of a round into profiles/ (run locally after
`gpurun` brought gpurun_out/ back; ncu -i works without a GPU).

    python scripts/summarize_profiles.py --round 1 --rep gpurun_out/bench_encode.ncu-rep \
        --launches gpurun_out/launches.csv --bench gpurun_out/bench_full.json

Writes profiles/r<NN>_launches.csv (the launch list: per-launch device time,
cold-cache and serialised), profiles/r<NN>_encode_ncu.txt (selected metrics of
the full K1 capture) and profiles/encode_traffic.json (DRAM bytes per K1
launch, read by bench.py's roofline `traffic`).
"""
import argparse
import csv
import re
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
           "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    vals = rows[2:]
    res = []
    for v in vals:
        d = {}
        for k, u, x in zip(hdr, units, v):
            d[k] = (x, u)
        res.append(d)
    return res


def to_si(x, u):
    try:
        f = float(x.replace(",", ""))
    except ValueError:
        return None
    return f * UNIT.get(u, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, default=1)
    ap.add_argument("--rep", default="gpurun_out/bench_encode.ncu-rep")
    ap.add_argument("--launches", default="gpurun_out/launches.csv")
    ap.add_argument("--bench", default="gpurun_out/bench_full.json")
    ap.add_argument("--model", default="qwen3-8b")
    ap.add_argument("--n-gpus", type=int, default=1)
    args = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    tag = f"r{args.round:02d}"
    if os.path.exists(args.launches):
        shutil.copy(args.launches, os.path.join(prof, f"{tag}_launches.csv"))
        # per-kernel share of the step from the launch list
        lines = [l for l in open(args.launches) if l.startswith('"')]
        rows = list(csv.reader(lines))
        hdr = rows[0]
        ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
        # the sync's kernels (libwsync's), not the setup's (torch arena
        # initialisation, the generator) or the verification's
        setup = ("gen_kernel", "vectorized_elementwise_kernel", "elementwise_kernel",
                 "reduce_kernel", "nccl")
        tot = {}
        for r in rows[1:]:
            m = re.search(r"(\w+_kernel)", r[ik])
            name = m.group(1) if m else r[ik][:40]
            if any(x in r[ik] for x in setup):
                continue
            tot[name] = tot.get(name, 0) + float(r[iv].replace(",", ""))
        s = sum(tot.values())
        with open(os.path.join(prof, f"{tag}_launch_shares.txt"), "w") as f:
            f.write("kernel (libwsync sync kernels of the captured launches), total ns, share\n")
            for k, v in sorted(tot.items(), key=lambda x: -x[1]):
                f.write(f"{k}, {v:.0f}, {v / s:.4f}\n")
    if os.path.exists(args.rep):
        ms = raw_metrics(args.rep)
        with open(os.path.join(prof, f"{tag}_encode_ncu.txt"), "w") as f:
            f.write(f"ncu --set full capture of one K1 launch ({args.rep}), selected metrics\n")
            for i, d in enumerate(ms):
                f.write(f"-- launch {i}: {d.get('Kernel Name', ('?',))[0]}\n")
                for m in METRICS:
                    if m in d:
                        f.write(f"{m:60s} {d[m][0]:>18s} {d[m][1]}\n")
        d = ms[0]
        rd = to_si(*d["dram__bytes_read.sum"])
        wr = to_si(*d["dram__bytes_write.sum"])
        dur = to_si(*d["gpu__time_duration.sum"])
        with open(os.path.join(prof, "encode_traffic.json"), "w") as f:
            json.dump({"model": args.model, "n_gpus": args.n_gpus, "round": args.round,
                       "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                       "ncu_duration_s": dur, "source": os.path.basename(args.rep)}, f, indent=1)
    if os.path.exists(args.bench):
        shutil.copy(args.bench, os.path.join(prof, f"{tag}_bench.json"))
    print("profiles written:", sorted(os.listdir(prof)))


if __name__ == "__main__":
    main()
