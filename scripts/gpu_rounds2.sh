NG=$(nvidia-smi -L | wc -l)
export WSYNC_EXCHANGE=p2p
for cfg in "WSYNC_ROUNDS=4" "WSYNC_ROUNDS=3 WSYNC_OVERLAP_SMS=8" "WSYNC_ROUNDS=3 WSYNC_OVERLAP_SMS=28" "WSYNC_ROUNDS=4 WSYNC_OVERLAP_SMS=28"; do
  echo "== $cfg"
  env $cfg timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29593 scripts/density_sweep.py --steps 8 --densities 0.01,0.05 2>/dev/null | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['density'], d['sparse_ms'], d['sparse_stages_ms'])"
done
