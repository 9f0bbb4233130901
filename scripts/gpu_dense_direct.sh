# N=4: multi-GPU parity in p2p (direct dense), p2p with dense records, nccl;
# then the density sweep with the direct dense path.
N=${N:-4}
for MODE in p2p p2prec nccl; do
  if [ $MODE = p2prec ]; then export WSYNC_EXCHANGE=p2p WSYNC_DENSE_DIRECT=0; else export WSYNC_EXCHANGE=$MODE WSYNC_DENSE_DIRECT=1; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 scripts/mgpu_check.py > gpurun_out/mgpu_check_$MODE.log 2>&1; echo "mgpu $MODE rc=$?"
  grep -o '"rank": [0-9], "world": [0-9], "ok": [a-z]*' gpurun_out/mgpu_check_$MODE.log; grep -iE "error|Traceback" gpurun_out/mgpu_check_$MODE.log | head -5
done
export WSYNC_EXCHANGE=p2p WSYNC_DENSE_DIRECT=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29515 scripts/density_sweep.py --steps 6 > gpurun_out/sweep_n${N}_direct.jsonl 2> gpurun_out/sweep_n${N}_direct.err; echo "sweep rc=$?"
cat gpurun_out/sweep_n${N}_direct.jsonl
tail -3 gpurun_out/sweep_n${N}_direct.err
