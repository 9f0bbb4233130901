# N=4: parity in all exchange modes, then fused-remote vs pack-emitted route timing.
N=4 bash scripts/gpu_dense_direct.sh 2>&1 | grep -E "rc=|\"ok\"" | head -16
for F in 1 0; do
  echo "== WSYNC_FUSED_REMOTE=$F"
  WSYNC_FUSED_REMOTE=$F timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2957$F scripts/density_sweep.py --steps 8 --densities 0.001,0.01,0.05 2>/dev/null | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['density'], d['sparse_ms'], d['sparse_stages_ms'])"
done
