#!/bin/bash
# ncu launch list of the N=1 bench's sync kernels (past the ~820 setup launches:
# generator and arena fills), per-launch device time, cold-cache and serialised
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 850 -c 200 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-verify > gpurun_out/ncu_launches.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_launches.log
