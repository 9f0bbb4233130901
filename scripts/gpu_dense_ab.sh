#!/bin/bash
# dense-path copies: parity + sweep at the dense densities
cd $GRAFT_REPO_ROOT
N=${N:-4}
timeout 900 python -m pytest tests/test_group_gpu.py tests/test_engine_gpu.py -q --timeout 600 > gpurun_out/dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dense_tests.log
if [ "$N" = "1" ]; then
  timeout 900 python scripts/density_sweep.py --steps 6 --densities 0.01,0.5 > gpurun_out/dsweep_n$N.jsonl 2>> gpurun_out/dsweep.err
else
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 scripts/density_sweep.py --steps 6 --densities 0.01,0.5 > gpurun_out/dsweep_n$N.jsonl 2>> gpurun_out/dsweep.err
fi
