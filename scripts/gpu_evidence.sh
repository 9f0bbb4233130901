# one bench + ncu evidence run (1 GPU)
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"encode_kernel|worklist_kernel|local_apply_kernel|pack_kernel|apply_wire_kernel" -c 40 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:encode_kernel -s 4 -c 1 -o gpurun_out/bench_encode -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
./scripts/stream_bench > gpurun_out/stream_bench.txt 2>&1
cat gpurun_out/bench_full.json
