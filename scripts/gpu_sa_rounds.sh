#!/bin/bash
# streamed apply under overlapped exchange rounds (WSYNC_SA_DIV=250 forces it on; ablation build)
cd $GRAFT_REPO_ROOT
N=${N:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
L=paper_2605_06534_b200/lib/libwsync_ablate.so
for k in 1 2; do for c in 2 3; do for sa in off on; do
  echo -n "{\"config\": $c, \"sa\": \"$sa\", \"line\": " >> gpurun_out/sarounds_n$N.jsonl
  if [ $sa = on ]; then E="WSYNC_SA_DIV=250"; else E=""; fi
  env $E WSYNC_LIB=$L timeout 900 $TR --master-port 2967$k bench.py --gpus $N --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' | tr -d '\n' >> gpurun_out/sarounds_n$N.jsonl
  echo "}" >> gpurun_out/sarounds_n$N.jsonl
done; done; done
