for v in k4 k5 k4 k5; do
  WSYNC_LIB=$PWD/paper_2605_06534_b200/lib/libwsync_$v.so timeout 600 python scripts/density_sweep.py --densities 0.01,0.05,0.1,0.15 > gpurun_out/k5.jsonl 2>&1
  echo "$v $(grep '^{' gpurun_out/k5.jsonl | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['density']}:{json.loads(l)['sparse_ms']}\" for l in sys.stdin))")"
done
