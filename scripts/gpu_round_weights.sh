#!/bin/bash
# N-GPU sync time vs unequal exchange-round sizes (WSYNC_ROUND_WEIGHTS, ablation build)
cd $GRAFT_REPO_ROOT
N=${N:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for k in 1 2; do for W in "1,1,1" "1.2,1.2,0.6" "1.5,1,0.5" "1,1,0.5" "0.8,1.1,1.1"; do
  echo -n "{\"weights\": \"$W\", \"line\": " >> gpurun_out/rw_n$N.jsonl
  WSYNC_ROUND_WEIGHTS=$W WSYNC_LIB=paper_2605_06534_b200/lib/libwsync_ablate.so timeout 300 $TR --master-port 2962$k bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-verify 2>/dev/null | grep '^{' | tr -d '\n' >> gpurun_out/rw_n$N.jsonl
  echo "}" >> gpurun_out/rw_n$N.jsonl
done; done
