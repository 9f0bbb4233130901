run() { env $1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fr2.json 2> gpurun_out/fr2.err
  echo "$1 rc=$? $(grep '^{' gpurun_out/fr2.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d.get('stages_ms'))")"; }
run "WSYNC_FUSED_REMOTE=0" 29771
run "WSYNC_FUSED_REMOTE=1" 29772
run "WSYNC_FUSED_REMOTE=0" 29773
run "WSYNC_FUSED_REMOTE=1" 29774
