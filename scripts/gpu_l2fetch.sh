b1() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/l2.json 2>gpurun_out/l2.err; echo "N1 $1: $(grep '^{' gpurun_out/l2.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['ms_per_step'],d['stages_ms'])")"; }
b4() { env $1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/l2.json 2>gpurun_out/l2.err; echo "N4 $1: $(grep '^{' gpurun_out/l2.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['ms_per_step'],d['stages_ms'])")"; }
b1 "WSYNC_SA_DIV=0"
b1 "WSYNC_SA_DIV=0 WSYNC_L2_FETCH=32"
b1 "WSYNC_L2_FETCH=0"
b1 "WSYNC_L2_FETCH=32"
b1 "WSYNC_SA_DIV=0 WSYNC_L2_FETCH=32"
b1 "WSYNC_SA_DIV=0"
b4 "WSYNC_X=0" 29741
b4 "WSYNC_L2_FETCH=32" 29742
b4 "WSYNC_X=0" 29743
b4 "WSYNC_L2_FETCH=32" 29744
