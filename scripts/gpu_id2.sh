# N=2 after restricting fuse_on=2 to identity routes: parity + bench + mid-density sweep
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 scripts/mgpu_check.py > gpurun_out/id2_check.log 2>&1; echo "check rc=$?"; grep -o '"ok": [a-z]*' gpurun_out/id2_check.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29782 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/id2.json 2> gpurun_out/id2.err
echo "bench $(grep '^{' gpurun_out/id2.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d.get('stages_ms'))")"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29783 scripts/density_sweep.py --densities 0.01,0.05,0.1,0.15 > gpurun_out/id2_sweep.jsonl 2>&1
echo "sweep $(grep '^{' gpurun_out/id2_sweep.jsonl | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['density']}:{json.loads(l)['sparse_ms']}\" for l in sys.stdin))")"
