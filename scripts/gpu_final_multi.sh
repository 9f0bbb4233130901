#!/bin/bash
# final multi-GPU evidence at N GPUs: bench lines (config 2 twice, configs 3
# and 4), the reference arm, the config-5 density sweep, multi-process parity
cd $GRAFT_REPO_ROOT
N=${N:-4}
O=gpurun_out/final_n$N; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for k in 1 2; do
  timeout 600 $TR --master-port 2964$k bench.py --gpus $N --steps 20 --warmup 5 2>> $O/err.log | grep '^{' >> $O/bench.jsonl
done
timeout 900 $TR --master-port 29643 bench.py --gpus $N --config 3 --steps 10 --warmup 3 --no-e2e 2>> $O/err.log | grep '^{' > $O/bench_c3.json
timeout 900 $TR --master-port 29644 bench.py --gpus $N --config 4 --steps 10 --warmup 3 --no-e2e 2>> $O/err.log | grep '^{' > $O/bench_c4.json
timeout 600 $TR --master-port 29645 bench.py --impl reference --gpus $N --steps 2 --warmup 1 2>> $O/err.log | grep '^{' > $O/bench_ref.json
timeout 900 $TR --master-port 29646 scripts/density_sweep.py --steps 6 2>> $O/err.log | grep '^{' > $O/sweep.jsonl
timeout 900 $TR --master-port 29647 scripts/mgpu_check.py > $O/mgpu.log 2>&1; echo "mgpu rc=$?" >> $O/mgpu.log
