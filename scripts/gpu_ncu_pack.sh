#!/bin/bash
# one ncu --set full capture of pack_kernel in the one-process route bench (N=2)
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pack_kernel --launch-skip 6 --launch-count 1 -o gpurun_out/pack_n2 python scripts/route_bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/ncu_pack.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_pack.log
