# Fused remote emission check at the box's GPU count, each step under a hard timeout.
NG=$(nvidia-smi -L | wc -l)
export WSYNC_EXCHANGE=p2p
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29581 scripts/mgpu_check.py > gpurun_out/fr_check.log 2>&1; echo "check rc=$?"
grep -o '"rank": [0-9], "world": [0-9], "ok": [a-z]*' gpurun_out/fr_check.log
for F in 1 0; do
  echo "== WSYNC_FUSED_REMOTE=$F"
  WSYNC_FUSED_REMOTE=$F timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2958$((F+2)) scripts/density_sweep.py --steps 8 --densities 0.001,0.01,0.05 2>/dev/null | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['density'], d['sparse_ms'], d['sparse_stages_ms'])"
done
