#!/bin/bash
# 6-byte P2P records: one-GPU group parity, multi-process parity at N=2, route bench, bench, ncu route
cd $GRAFT_REPO_ROOT
N=${N:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_group_gpu.py tests/test_engine_gpu.py -q --timeout 600 > gpurun_out/w6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/w6_tests.log
timeout 900 $TR --master-port 29561 scripts/mgpu_check.py > gpurun_out/mgpu_n$N.log 2>&1; echo "mgpu rc=$?" >> gpurun_out/mgpu_n$N.log
WSYNC_EXCHANGE=nccl timeout 900 $TR --master-port 29562 scripts/mgpu_check.py > gpurun_out/mgpu_nccl_n$N.log 2>&1; echo "mgpu rc=$?" >> gpurun_out/mgpu_nccl_n$N.log
timeout 600 python scripts/route_bench.py --gpus $N --steps 10 > gpurun_out/route_n$N.json 2> gpurun_out/route_n$N.err
timeout 600 $TR --master-port 29563 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --kernel-name regex:"pack_kernel|apply_p2p_kernel" --launch-skip 8 --launch-count 8 --clock-control none --csv \
  --log-file gpurun_out/ncu_route_n$N.csv python scripts/route_bench.py --gpus $N --steps 3 --warmup 2 > gpurun_out/ncu_route_n$N.log 2>&1
