#!/bin/bash
# heavy-exchange layout (FSDP-N -> TP1 x N): exchange SMs beside K1 and rounds (ablation build)
cd $GRAFT_REPO_ROOT
N=${N:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
L=paper_2605_06534_b200/lib/libwsync_ablate.so
for R in 1 3 4; do for S in 28 40 56 74; do
  [ $R = 1 ] && [ $S != 28 ] && continue
  WSYNC_ROUNDS=$R WSYNC_OVERLAP_SMS=$S WSYNC_LIB=$L timeout 600 $TR --master-port 29701 scripts/fanout_bench.py 2>> gpurun_out/fanout.err | grep '^{' >> gpurun_out/fanout_n$N.jsonl
done; done
