#!/bin/bash
cd $GRAFT_REPO_ROOT
N=${N:-4}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29602 scripts/e2e_probe.py > gpurun_out/e2e_probe_n$N.jsonl 2> gpurun_out/e2e_probe.err
