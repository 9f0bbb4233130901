#!/bin/bash
# round 2: group (one-GPU multi-rank) tests + the existing GPU suite
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_group_gpu.py -x -q --timeout 300 > gpurun_out/group.log 2>&1
echo "group rc=$?" >> gpurun_out/group.log
timeout 900 python -m pytest tests -q -m gpu --timeout 300 --deselect tests/test_group_gpu.py > gpurun_out/gpu_all.log 2>&1
echo "all rc=$?" >> gpurun_out/gpu_all.log
