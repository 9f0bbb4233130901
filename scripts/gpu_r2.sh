run() { env $1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2.json 2> gpurun_out/r2.err
  echo "$1 rc=$? $(grep '^{' gpurun_out/r2.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d.get('stages_ms'))")"; }
run "WSYNC_ROUNDS=1" 29711
run "WSYNC_ROUNDS=3 WSYNC_SA_DIV=250" 29712
run "WSYNC_ROUNDS=3 WSYNC_SA_DIV=0" 29713
run "WSYNC_ROUNDS=2 WSYNC_SA_DIV=250" 29714
run "WSYNC_ROUNDS=1" 29715
