#!/bin/bash
# Stage timeline of N-GPU syncs (ablation build, WSYNC_TIMELINE=1): ms from the
# sync's start to the end of every K1 round, pack, receive-side apply, local route
cd $GRAFT_REPO_ROOT
N=${N:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
WSYNC_LIB=paper_2605_06534_b200/lib/libwsync_ablate.so WSYNC_TIMELINE=1 timeout 600 $TR --master-port 29581 bench.py --gpus $N --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-verify > gpurun_out/timeline_n$N.json 2> gpurun_out/timeline_n$N.err
for R in 1 2 4; do
WSYNC_ROUNDS=$R WSYNC_LIB=paper_2605_06534_b200/lib/libwsync_ablate.so WSYNC_TIMELINE=1 timeout 600 $TR --master-port 29582 bench.py --gpus $N --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-verify > gpurun_out/timeline_n${N}_r$R.json 2> gpurun_out/timeline_n${N}_r$R.err
done
