# Exchange rounds: parity (P2P, default rounds), then sync times for 1 / 2 rounds and overlap off.
NG=$(nvidia-smi -L | wc -l)
export WSYNC_EXCHANGE=p2p
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29591 scripts/mgpu_check.py > gpurun_out/rounds_check.log 2>&1; echo "check rc=$?"
grep -o '"rank": [0-9], "world": [0-9], "ok": [a-z]*' gpurun_out/rounds_check.log
grep -iE "Error" gpurun_out/rounds_check.log | head -3
for cfg in "WSYNC_ROUNDS=1" "WSYNC_ROUNDS=2" "WSYNC_ROUNDS=2 WSYNC_OVERLAP=0" "WSYNC_ROUNDS=3"; do
  echo "== $cfg"
  env $cfg timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29592 scripts/density_sweep.py --steps 8 --densities 0.001,0.01,0.05 2>/dev/null | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['density'], d['sparse_ms'], d['dense_ms'], d['sparse_stages_ms'])"
done
