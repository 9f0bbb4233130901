#!/bin/bash
# K1-emitted remote records (ablation build, WSYNC_FUSED_REMOTE=1) vs the pack
# kernel: parity + same-box A/B at N GPUs.  r02_fused_remote_sa_ab_n2.jsonl was
# taken with an encode_kernel<bf16, REMOTE, SA> instantiation that was not kept;
# the shipped ablation build emits without the streamed apply.
cd $GRAFT_REPO_ROOT
N=${N:-2}
O=gpurun_out/fr_n$N; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
L=paper_2605_06534_b200/lib/libwsync_ablate.so
WSYNC_FUSED_REMOTE=1 WSYNC_LIB=$L timeout 900 $TR --master-port 29731 scripts/mgpu_check.py > $O/mgpu.log 2>&1; echo "rc=$?" >> $O/mgpu.log
for k in 1 2 3; do for fr in 0 1; do
  echo -n "{\"fused_remote\": $fr, \"line\": " >> $O/ab.jsonl
  WSYNC_FUSED_REMOTE=$fr WSYNC_LIB=$L timeout 300 $TR --master-port 2974$k bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline ${EXTRA} 2>/dev/null | grep '^{' | tr -d '\n' >> $O/ab.jsonl
  echo "}" >> $O/ab.jsonl
done; done
