#!/bin/bash
# BASELINE config 5: density sweep (sparse vs always-dense) at N GPUs
cd $GRAFT_REPO_ROOT
N=${N:-1}
if [ "$N" = "1" ]; then
  timeout 1500 python scripts/density_sweep.py --steps 6 > gpurun_out/sweep_n$N.jsonl 2> gpurun_out/sweep_n$N.err
else
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29601 scripts/density_sweep.py --steps 6 > gpurun_out/sweep_n$N.jsonl 2> gpurun_out/sweep_n$N.err
fi
echo "rc=$?" >> gpurun_out/sweep_n$N.err
