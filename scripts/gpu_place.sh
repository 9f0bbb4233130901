#!/bin/bash
# Serving-rank placement (ws_placement) at N GPUs: parity (group tests incl.
# one rank per GPU, multi-process P2P/NCCL/rank-order), route stage and bench
# A/B rank vs overlap placement, configs 3/4, density sweep.
cd $GRAFT_REPO_ROOT
N=${N:-4}
O=gpurun_out/place_n$N; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_multigpu_gpu.py -q --timeout 900 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for pl in rank overlap; do
  timeout 600 python scripts/route_bench.py --gpus $N --steps 10 --placement $pl > $O/route_$pl.json 2>> $O/err.log
  timeout 600 python scripts/route_bench.py --gpus $N --steps 10 --dense --placement $pl > $O/route_dense_$pl.json 2>> $O/err.log
done
for pl in rank overlap rank overlap; do
  timeout 600 $TR --master-port 29572 bench.py --gpus $N --steps 20 --warmup 5 --placement $pl >> $O/bench_ab.jsonl 2>> $O/err.log
done
timeout 900 $TR --master-port 29573 bench.py --gpus $N --config 3 --steps 10 --warmup 3 --no-e2e > $O/bench_c3.json 2>> $O/err.log
timeout 900 $TR --master-port 29574 bench.py --gpus $N --config 4 --steps 10 --warmup 3 --no-e2e > $O/bench_c4.json 2>> $O/err.log
timeout 900 $TR --master-port 29575 scripts/density_sweep.py --steps 6 > $O/sweep.jsonl 2>> $O/err.log
