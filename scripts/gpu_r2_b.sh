#!/bin/bash
# round 2: group tests, whole-Qwen3-8B parity, bench N=1 (verified)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_group_gpu.py -q --timeout 300 > gpurun_out/group.log 2>&1
echo "group rc=$?" >> gpurun_out/group.log
timeout 600 python -m pytest tests/test_engine_gpu.py -q --timeout 500 -k "qwen3_8b or streamed" > gpurun_out/q8b.log 2>&1
echo "q8b rc=$?" >> gpurun_out/q8b.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "bench rc=$?" >> gpurun_out/bench1.err
