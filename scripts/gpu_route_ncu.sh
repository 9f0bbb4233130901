#!/bin/bash
# ncu NVLink / DRAM counters of the route kernels (one process, one rank per
# GPU, overlap placement): 1% sparse and sparse=False (dense boxes)
cd $GRAFT_REPO_ROOT
N=${N:-4}
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --kernel-name regex:"pack_kernel|apply_p2p_kernel" --launch-skip 8 --launch-count 12 --clock-control none --csv \
  --log-file gpurun_out/ncu_route_ov_n$N.csv python scripts/route_bench.py --gpus $N --steps 3 --warmup 2 > gpurun_out/ncu_route_ov_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_route_ov_n$N.log
timeout 900 ncu --metrics $M --kernel-name regex:"pack_kernel" --launch-skip 8 --launch-count 8 --clock-control none --csv \
  --log-file gpurun_out/ncu_route_dense_n$N.csv python scripts/route_bench.py --gpus $N --dense --steps 3 --warmup 2 > gpurun_out/ncu_route_dense_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_route_dense_n$N.log
