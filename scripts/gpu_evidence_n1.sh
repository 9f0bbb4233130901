#!/bin/bash
# N=1 evidence of the shipped build: default bench, ncu launch list of the same
# command, one ncu --set full capture of K1 (each only after its command exits 0)
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/bench_final_n1.json 2> gpurun_out/bench_final_n1.err; echo "rc=$?" >> gpurun_out/bench_final_n1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-verify > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_kernel --launch-skip 6 --launch-count 1 -o gpurun_out/k1_r02 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-verify > gpurun_out/ncu_k1.log 2>&1
echo "done" >> gpurun_out/ncu_k1.log
