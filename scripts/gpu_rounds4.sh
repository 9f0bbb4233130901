NG=$(nvidia-smi -L | wc -l)
for R in 1 3; do
  WSYNC_ROUNDS=$R timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2960$R bench.py --gpus $NG --steps 20 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench R=$R', d['value'], d['ms_per_step'], d['stages_ms'])"
  WSYNC_ROUNDS=$R timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2961$R scripts/density_sweep.py --steps 20 --densities 0.01 2>/dev/null | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('sweep R=$R', d['density'], d['sparse_ms'], d['sparse_stages_ms'])"
done
