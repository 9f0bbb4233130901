# full default bench + reference arm + ncu evidence (launch list, K1 full set)
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"encode_kernel|worklist_kernel|local_apply_kernel|pack_kernel|apply_wire_kernel" -c 40 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:encode_kernel -s 4 -c 1 -o gpurun_out/bench_encode $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
cat gpurun_out/bench_full.json gpurun_out/bench_ref.json
