# bench at N=1,2,4 on one box (torchrun for N>1)
NG=$(nvidia-smi -L | wc -l)
for n in 1 2 4; do
  [ $n -gt $NG ] && continue
  if [ $n = 1 ]; then timeout 400 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n)) bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; fi
  echo "n=$n rc=$? $(grep '^{' gpurun_out/bench_n$n.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['clocks'],d.get('stages_ms'))")"
done
