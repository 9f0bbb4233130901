#!/bin/bash
# pinned host->device rates at N GPUs (what bounds bench.py's e2e)
cd $GRAFT_REPO_ROOT
N=${N:-4}
free -g > gpurun_out/free.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for cfg in "2 1" "4 2" "8 2"; do set -- $cfg
  H2D_GIB=$1 H2D_BUFS=$2 timeout 600 $TR --master-port 29601 scripts/h2d_probe.py >> gpurun_out/h2d_n$N.jsonl 2>> gpurun_out/h2d.err
done
