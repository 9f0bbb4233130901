# ncu evidence for the N=1 bench (one ncu per call): the launch list of the
# sync kernels (per-launch durations) of the same command, after it exits 0
# without ncu.  The --set full K1 capture is scripts/gpu_ncu_k1.sh.
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"encode_kernel|worklist_kernel|local_apply_kernel|fixup_plan_kernel" -c 40 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
