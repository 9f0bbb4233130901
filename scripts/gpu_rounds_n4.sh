#!/bin/bash
# N=4 exchange-round count and streamed-apply A/B on one box
cd $GRAFT_REPO_ROOT
N=4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
ABL=$PWD/paper_2605_06534_b200/lib/libwsync_ablate.so
for R in 3 2 4 1 3; do
  WSYNC_ROUNDS=$R timeout 600 $TR --master-port 2953$R bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-verify >> gpurun_out/rounds_n4.jsonl 2>> gpurun_out/rounds_n4.err
done
WSYNC_LIB=$ABL WSYNC_SA_DIV=250 timeout 600 $TR --master-port 29541 bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-verify >> gpurun_out/rounds_n4_sa.jsonl 2>> gpurun_out/rounds_n4.err
