# ncu --set full of K1 at a mid density (one ncu), after the same command exits 0 without it
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --density ${DENS:-0.1}"
$CMD > gpurun_out/mid_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/mid_plain.log | cut -c1-200
ncu --set full --clock-control none --import-source on -k regex:encode_kernel -s 4 -c 1 -o gpurun_out/k1_mid -f $CMD > gpurun_out/ncu_mid.log 2>&1; echo "ncu rc=$?"
