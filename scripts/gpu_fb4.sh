for v in fb1 fb2 fb1 fb2; do
  WSYNC_LIB=$PWD/paper_2605_06534_b200/lib/libwsync_$v.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29790 + ${#v})) bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fb4.json 2> gpurun_out/fb4.err
  echo "$v $(grep '^{' gpurun_out/fb4.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d.get('stages_ms'))")"
done
