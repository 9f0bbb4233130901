#!/bin/bash
# N-GPU sync time vs exchange rounds (WSYNC_ROUNDS) and the SMs left to the
# exchange kernels while K1 runs (WSYNC_OVERLAP_SMS, ablation build)
cd $GRAFT_REPO_ROOT
N=${N:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for R in ${RS:-2 3 4}; do for S in ${SS:-20 28 40 56}; do
  echo -n "{\"rounds\": $R, \"overlap_sms\": $S, \"line\": " >> gpurun_out/ovl_n$N.jsonl
  WSYNC_ROUNDS=$R WSYNC_OVERLAP_SMS=$S WSYNC_LIB=paper_2605_06534_b200/lib/libwsync_ablate.so timeout 300 $TR --master-port 29583 bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-verify 2>/dev/null | grep '^{' | tr -d '\n' >> gpurun_out/ovl_n$N.jsonl
  echo "}" >> gpurun_out/ovl_n$N.jsonl
done; done
