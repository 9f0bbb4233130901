#!/bin/bash
# plan-derived exchange rounds: parity (groups, multi-process) + bench configs 2/3/4
cd $GRAFT_REPO_ROOT
N=${N:-4}
O=gpurun_out/rchk_n$N; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_multigpu_gpu.py tests/test_golden.py -q --timeout 900 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for c in 2 3 4; do
  timeout 900 $TR --master-port 2966$c bench.py --gpus $N --config $c --steps 10 --warmup 3 --no-e2e 2>> $O/err.log | grep '^{' > $O/bench_c$c.json
done
