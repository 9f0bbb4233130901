# Full N=1 bench line (e2e + cpu baseline) and the ncu launch list of the same command.
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.json | cut -c1-400
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"encode_kernel|fixup_plan_kernel|worklist_kernel|local_apply_kernel|pack_kernel|apply_wire_kernel|apply_p2p_kernel|p2p_ready_kernel|p2p_recv_plan_kernel" -c 40 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
