N=${N:-2}
for MODE in p2p nccl; do
  export WSYNC_EXCHANGE=$MODE
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 scripts/mgpu_check.py > gpurun_out/mgpu_check_$MODE.log 2>&1; echo "mgpu $MODE rc=$?"
  grep -o '"rank": [0-9], "world": [0-9], "ok": [a-z]*' gpurun_out/mgpu_check_$MODE.log; grep -iE "error|Traceback" gpurun_out/mgpu_check_$MODE.log | head -5
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 20 --warmup 3 --no-e2e > gpurun_out/bench_n${N}_$MODE.json 2> gpurun_out/bench_n${N}_$MODE.err; echo "bench $MODE rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench_n${N}_$MODE.json').read().strip().splitlines()[-1]);print('$MODE', d['value'], d['ms_per_step'], d['stages_ms'])"
  tail -3 gpurun_out/bench_n${N}_$MODE.err | grep -v OMP
done
