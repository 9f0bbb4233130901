#!/bin/bash
# exchange rounds per BASELINE config (WSYNC_ROUNDS override), alternating, at N GPUs
cd $GRAFT_REPO_ROOT
N=${N:-4}; CFG=${CFG:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for k in 1 2; do for R in ${RS:-1 3}; do
  echo -n "{\"config\": $CFG, \"rounds\": $R, \"line\": " >> gpurun_out/rcfg_n$N.jsonl
  WSYNC_ROUNDS=$R timeout 900 $TR --master-port 2965$k bench.py --gpus $N --config $CFG --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-verify 2>/dev/null | grep '^{' | tr -d '\n' >> gpurun_out/rcfg_n$N.jsonl
  echo "}" >> gpurun_out/rcfg_n$N.jsonl
done; done
