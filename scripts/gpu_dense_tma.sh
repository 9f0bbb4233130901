NG=$(nvidia-smi -L | wc -l)
export WSYNC_EXCHANGE=p2p
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29631 scripts/mgpu_check.py > gpurun_out/tma_check.log 2>&1; echo "check rc=$?"
grep -o '"rank": [0-9], "world": [0-9], "ok": [a-z]*' gpurun_out/tma_check.log
for V in tma notma; do
  if [ $V = notma ]; then export WSYNC_LIB=$PWD/paper_2605_06534_b200/lib/notma/libwsync.so; fi
  timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29632 scripts/density_sweep.py --steps 6 --densities 0.01,0.3 2>/dev/null | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$V', d['density'], 'sparse', d['sparse_ms'], 'dense', d['dense_ms'])"
done
