#!/bin/bash
# same-box A/B of BASELINE config 4 at N=4: the build of ca6c3ba (_oldtree) vs this one
cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for k in 1 2; do
  (cd _oldtree && timeout 900 $TR --master-port 2958$k bench.py --gpus 4 --config 4 --steps 10 --warmup 3 --no-e2e --no-verify >> ../gpurun_out/c4_old.jsonl 2>>../gpurun_out/c4_ab.err)
  timeout 900 $TR --master-port 2959$k bench.py --gpus 4 --config 4 --steps 10 --warmup 3 --no-e2e --no-verify >> gpurun_out/c4_new.jsonl 2>>gpurun_out/c4_ab.err
done
