#!/bin/bash
# dense (sparse=False) syncs at N=4 in one process: stage times + per-kernel launch list
cd $GRAFT_REPO_ROOT
timeout 600 python scripts/route_bench.py --gpus 4 --dense --steps 10 > gpurun_out/dense_rb_n4.json 2> gpurun_out/dense_rb.err
timeout 600 python scripts/route_bench.py --gpus 4 --steps 10 > gpurun_out/sparse_rb_n4.json 2>> gpurun_out/dense_rb.err
timeout 900 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 200 --launch-count 120 --csv --log-file gpurun_out/dense_launches_n4.csv python scripts/route_bench.py --gpus 4 --dense --steps 4 --warmup 3 > gpurun_out/dense_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/dense_ncu.log
