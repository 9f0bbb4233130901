#!/bin/bash
# run-to-run spread of the N-GPU bench (outlier hunt): K identical runs, with
# per-rank per-step traces (BENCH_STEP_TRACE=1) on stderr
cd $GRAFT_REPO_ROOT
N=${N:-4}; K=${K:-10}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for k in $(seq 1 $K); do
  BENCH_STEP_TRACE=1 timeout 300 $TR --master-port $((29630 + k)) bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-verify 2> gpurun_out/repeat_trace_$k.err | grep '^{' >> gpurun_out/repeat_n$N.jsonl
done
