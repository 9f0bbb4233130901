for d in 250 0 250; do
  WSYNC_SA_DIV=$d timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29690 + (d > 0))) bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sa4_$d.json 2> gpurun_out/sa4_$d.err
  echo "div=$d rc=$? $(grep '^{' gpurun_out/sa4_$d.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d.get('stages_ms'))")"
done
