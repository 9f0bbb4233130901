#!/usr/bin/env python
"""Instruction mix of every kernel in the built libwsync.so (cuobjdump -sass,
no GPU needed): the evidence that K1 streams with 1-D TMA (UBLKCP) completing
on mbarriers (SYNCS), that the fused apply prefetches with LDGSTS, and which
kernels touch peer memory with plain stores.  Writes profiles/r02_sass_summary.txt."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_06534_b200", "lib", "libwsync.so")
COLS = ["UBLKCP", "SYNCS", "LDGSTS", "LDG", "STG", "LDS", "STS", "ATOMS", "ATOMG|RED", "VOTE",
        "POPC", "SHFL", "BAR", "MEMBAR", "FENCE"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return out.stdout.splitlines() if out.returncode == 0 else names


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
    parts = re.split(r"\n\s+Function : ", sass)[1:]
    names = [p.split("\n", 1)[0].strip() for p in parts]
    pretty = demangle(names)
    lines = [f"libwsync.so SASS instruction mix (cuobjdump -sass), arch: {', '.join(arch)}",
             "counts of static instruction sites per kernel", ""]
    hdr = f"{'kernel':70}" + "".join(f"{c.split('|')[0]:>8}" for c in COLS) + f"{'total':>8}"
    lines.append(hdr)
    for name, p in sorted(zip(pretty, parts), key=lambda x: x[0]):
        ops = collections.Counter(re.findall(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", p))
        def cnt(col):
            return sum(v for k, v in ops.items() for c in col.split("|") if k.startswith(c)
                       and not (c == "LDG" and k.startswith("LDGSTS")))
        short = name.replace("(anonymous namespace)::", "").replace("wsync::", "")
        short = re.sub(r"\(.*", "", short.replace("void ", ""))
        lines.append(f"{short[:70]:70}" + "".join(f"{cnt(c):8d}" for c in COLS) +
                     f"{sum(ops.values()):8d}")
    out = "\n".join(lines) + "\n"
    with open(os.path.join(ROOT, "profiles", "r02_sass_summary.txt"), "w") as f:
        f.write(out)
    print(out)


if __name__ == "__main__":
    sys.exit(main())
