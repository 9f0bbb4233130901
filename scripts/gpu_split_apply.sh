#!/bin/bash
# receive-side applies on their own stream (default) vs behind the packs
# (WSYNC_SPLIT_APPLY=0, ablation build): same-box A/B at N GPUs + parity + timeline
cd $GRAFT_REPO_ROOT
N=${N:-4}
O=gpurun_out/split_n$N; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
L=paper_2605_06534_b200/lib/libwsync_ablate.so
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q --timeout 800 -k "p2p and not rank" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for k in 1 2 3; do for sp in 0 1; do
  echo -n "{\"split\": $sp, \"line\": " >> $O/ab.jsonl
  WSYNC_SPLIT_APPLY=$sp WSYNC_LIB=$L timeout 300 $TR --master-port 29591 bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' | tr -d '\n' >> $O/ab.jsonl
  echo "}" >> $O/ab.jsonl
done; done
WSYNC_LIB=$L WSYNC_TIMELINE=1 timeout 300 $TR --master-port 29592 bench.py --gpus $N --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-verify > /dev/null 2> $O/timeline.err
timeout 600 $TR --master-port 29593 bench.py --gpus $N --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
