#!/bin/bash
# local route on a side stream beside the exchange (syncs without rounds):
# lib/libwsync_base.so (before) vs lib/libwsync.so, N GPUs, same box:
# config-5 sparse/dense at 1% and 50% and the default bench; then parity
cd $GRAFT_REPO_ROOT
N=${N:-4}
O=gpurun_out/side_n$N; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for k in 1 2; do for v in base new; do
  if [ $v = base ]; then L=paper_2605_06534_b200/lib/libwsync_base.so; else L=paper_2605_06534_b200/lib/libwsync.so; fi
  WSYNC_LIB=$L timeout 900 $TR --master-port 2975$k scripts/density_sweep.py --steps 6 --densities 0.01,0.5 2>/dev/null | grep '^{' | sed "s/^{/{\"v\": \"$v\", /" >> $O/sweep.jsonl
  echo -n "{\"v\": \"$v\", \"line\": " >> $O/bench.jsonl
  WSYNC_LIB=$L timeout 300 $TR --master-port 2976$k bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' | tr -d '\n' >> $O/bench.jsonl
  echo "}" >> $O/bench.jsonl
done; done
timeout 1200 python -m pytest tests/test_multigpu_gpu.py tests/test_group_gpu.py -q --timeout 900 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
