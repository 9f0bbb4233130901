# Where the N=4 route time goes: normal / no receiver scatter / no records sent.
for D in ${DS:-0 1 2 3}; do
  echo "== WSYNC_P2P_DEBUG=$D"
  WSYNC_P2P_DEBUG=$D timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954$D scripts/density_sweep.py --steps 8 --densities 0.01 2>/dev/null | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['density'], d['sparse_ms'], d['sparse_stages_ms'])"
done
