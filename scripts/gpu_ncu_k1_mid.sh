#!/bin/bash
# one ncu --set full capture (with source counters) of the kept K1 at 10% density
cd $GRAFT_REPO_ROOT
D=${D:-0.1}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_kernel --launch-skip 6 --launch-count 1 -o gpurun_out/k1_mid_$D python bench.py --density $D --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-verify > gpurun_out/ncu_k1_mid.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_k1_mid.log
