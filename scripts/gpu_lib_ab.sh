#!/bin/bash
# same-box A/B of two builds at N GPUs: lib/libwsync_base.so vs lib/libwsync.so,
# alternating bench runs (torchrun for N > 1), then the group parity tests
cd $GRAFT_REPO_ROOT
N=${N:-4}
O=gpurun_out/libab_n$N; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for k in 1 2 3; do for v in base new; do
  if [ $v = base ]; then L=paper_2605_06534_b200/lib/libwsync_base.so; else L=paper_2605_06534_b200/lib/libwsync.so; fi
  echo -n "{\"v\": \"$v\", \"line\": " >> $O/ab.jsonl
  WSYNC_LIB=$L timeout 300 $TR --master-port 2960$k bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline ${EXTRA} 2>/dev/null | grep '^{' | tr -d '\n' >> $O/ab.jsonl
  echo "}" >> $O/ab.jsonl
done; done
timeout 900 python -m pytest tests/test_group_gpu.py -q --timeout 800 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
