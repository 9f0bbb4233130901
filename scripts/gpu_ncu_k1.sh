# One ncu --set full capture of one K1 launch in the N=1 bench (after the same
# command exits 0 without ncu).
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/plain.log | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:encode_kernel -s 4 -c 1 -o gpurun_out/${TAG:-k1} -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
