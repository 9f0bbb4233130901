#!/usr/bin/env python
"""Summarise an ncu CSV of the route kernels (scripts/gpu_route_ncu.sh: ncu over
scripts/route_bench.py, one process, one rank per GPU) into per-launch
NVLink / DRAM rates: prints a table and writes profiles/route_ncu.json."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = (int(d["ID"]), int(d.get("Device", 0)), d["Kernel Name"].split("(")[0])
            out.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return out


def main():
    summary = {}
    # key -> capture: the bench reads str(N) (its placement, overlap, when
    # captured); "4_rank" / "4_dense" are the rank-order and sparse=False runs
    caps = []
    for n in (2, 4, 8):
        for suffix in ("_overlap", ""):
            path = os.path.join(ROOT, "profiles", f"r02_route_ncu_n{n}{suffix}.csv")
            if os.path.exists(path):
                caps.append((str(n), path))
                break
    for key, name in (("4_rank", "r02_route_ncu_n4.csv"),
                      ("4_dense", "r02_route_ncu_dense_n4_overlap.csv")):
        path = os.path.join(ROOT, "profiles", name)
        if os.path.exists(path) and all(path != p for _, p in caps):
            caps.append((key, path))
    for n, path in caps:
        launches = []
        print(f"== N={n} ({os.path.basename(path)})")
        print(f"{'launch':>6} {'dev':>3} {'kernel':28} {'us':>8} {'nvltx MB':>9} {'user MB':>8} "
              f"{'nvltx GB/s':>10} {'of 900':>6} {'user GB/s':>9} {'dram rd MB':>10} {'dram wr MB':>10}")
        for (i, dev, name), m in sorted(load(path).items()):
            t = m["gpu__time_duration.sum"] * 1e-9
            tx, user = m["nvltx__bytes.sum"], m.get("nvltx__bytes_data_user.sum", 0.0)
            row = {"launch": i, "device": dev, "kernel": name.replace("void ", ""), "us": t * 1e6,
                   "nvltx_bytes": tx, "nvltx_user_bytes": user, "nvltx_gbs": tx / t / 1e9,
                   "frac_of_900": tx / t / 1e9 / 900, "user_gbs": user / t / 1e9,
                   "dram_read_bytes": m["dram__bytes_read.sum"],
                   "dram_write_bytes": m["dram__bytes_write.sum"]}
            launches.append(row)
            print(f"{i:>6} {dev:>3} {row['kernel'][:28]:28} {row['us']:8.1f} {tx / 1e6:9.1f} "
                  f"{user / 1e6:8.1f} {row['nvltx_gbs']:10.0f} {row['frac_of_900']:6.2f} "
                  f"{row['user_gbs']:9.0f} {row['dram_read_bytes'] / 1e6:10.0f} "
                  f"{row['dram_write_bytes'] / 1e6:10.0f}")
        packs = [r for r in launches if "pack_kernel" in r["kernel"]]
        if packs:
            best = max(packs, key=lambda r: r["nvltx_gbs"])
            mean = sum(r["nvltx_gbs"] for r in packs) / len(packs)
            print(f"pack_kernel: mean {mean:.0f} GB/s nvltx ({mean / 900:.2f} of 900), "
                  f"max {best['nvltx_gbs']:.0f}")
            summary[n] = {"pack_nvltx_gbs_mean": mean, "pack_frac_of_900_mean": mean / 900,
                               "pack_user_gbs_mean": sum(r["user_gbs"] for r in packs) / len(packs),
                               "launches": launches, "source": os.path.basename(path)}
    with open(os.path.join(ROOT, "profiles", "route_ncu.json"), "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
