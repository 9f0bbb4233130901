#!/bin/bash
# route stage after the pack changes: parity, one-process route bench, ncu NVLink counters (N=2)
cd $GRAFT_REPO_ROOT
N=${N:-2}
timeout 900 python -m pytest tests/test_group_gpu.py tests/test_engine_gpu.py tests/test_codec_gpu.py tests/test_collapsed_gpu.py -q --timeout 600 > gpurun_out/pack_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pack_tests.log
timeout 600 python scripts/route_bench.py --gpus $N --steps 10 > gpurun_out/route_n$N.json 2> gpurun_out/route_n$N.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus $N --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --kernel-name regex:"pack_kernel|apply_p2p_kernel" --launch-skip 8 --launch-count 8 --clock-control none --csv \
  --log-file gpurun_out/ncu_route_n$N.csv python scripts/route_bench.py --gpus $N --steps 3 --warmup 2 > gpurun_out/ncu_route_n$N.log 2>&1
