NG=$(nvidia-smi -L | wc -l)
N=$NG bash scripts/gpu_dense_direct.sh 2>&1 | grep -E "rc=|\"ok\"" | head -16
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29595 bench.py --gpus $NG --steps 20 --warmup 3 --no-e2e > gpurun_out/rounds_bench.json 2> gpurun_out/rounds_bench.err; echo "bench rc=$?"
tail -1 gpurun_out/rounds_bench.json | cut -c1-300
