#!/bin/bash
# route stage only: one-process route bench + ncu route counters (N=2)
cd $GRAFT_REPO_ROOT
N=${N:-2}
timeout 600 python -m pytest tests/test_group_gpu.py -q --timeout 600 -k "fsdp8 or config2 or matches_reference" > gpurun_out/rt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rt_tests.log
timeout 600 python scripts/route_bench.py --gpus $N --steps 10 > gpurun_out/route_n$N.json 2> gpurun_out/route_n$N.err
timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --kernel-name regex:"pack_kernel|apply_p2p_kernel" --launch-skip 8 --launch-count 8 --clock-control none --csv \
  --log-file gpurun_out/ncu_route_n$N.csv python scripts/route_bench.py --gpus $N --steps 3 --warmup 2 > gpurun_out/ncu_route_n$N.log 2>&1
