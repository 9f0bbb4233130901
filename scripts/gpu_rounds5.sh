NG=$(nvidia-smi -L | wc -l)
for cfg in "WSYNC_ROUNDS=1" "WSYNC_ROUNDS=2" "WSYNC_ROUNDS=3" "WSYNC_ROUNDS=3 WSYNC_OVERLAP_SMS=40"; do
  env $cfg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus $NG --steps 20 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['ms_per_step'], d['stages_ms'])"
done
