#!/bin/bash
# Multi-GPU evidence at N GPUs (N=2 or 4): multi-process parity (P2P and the
# NCCL fallback), the one-process group on N GPUs, the route stage and its ncu
# NVLink counters, bench lines for BASELINE configs 2, 3 and 4.
cd $GRAFT_REPO_ROOT
N=${N:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29571 scripts/mgpu_check.py > gpurun_out/mgpu_n$N.log 2>&1; echo "mgpu rc=$?" >> gpurun_out/mgpu_n$N.log
timeout 600 python -m pytest tests/test_group_gpu.py -q --timeout 300 -k "one_rank_per_gpu" > gpurun_out/group_md_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/group_md_n$N.log
timeout 600 python scripts/route_bench.py --gpus $N --steps 10 > gpurun_out/route_n$N.json 2> gpurun_out/route_n$N.err
timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --kernel-name regex:"pack_kernel|apply_p2p_kernel" --launch-skip 8 --launch-count 8 --clock-control none --csv \
  --log-file gpurun_out/ncu_route_n$N.csv python scripts/route_bench.py --gpus $N --steps 3 --warmup 2 > gpurun_out/ncu_route_n$N.log 2>&1
timeout 600 $TR --master-port 29572 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
timeout 900 $TR --master-port 29573 bench.py --gpus $N --config 3 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_c3_n$N.json 2> gpurun_out/bench_c3_n$N.err
timeout 900 $TR --master-port 29574 bench.py --gpus $N --config 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_c4_n$N.json 2> gpurun_out/bench_c4_n$N.err
timeout 600 $TR --master-port 29575 bench.py --impl reference --gpus $N --steps 2 --warmup 1 > gpurun_out/bench_ref_n$N.json 2> gpurun_out/bench_ref_n$N.err
