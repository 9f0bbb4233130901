for v in base sb1 sb2 base sb1 sb2; do
  L=$PWD/paper_2605_06534_b200/lib/libwsync_$v.so
  WSYNC_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v3.json 2>/dev/null
  b=$(grep '^{' gpurun_out/v3.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['ms_per_step'])")
  WSYNC_LIB=$L timeout 600 python scripts/density_sweep.py --densities 0.003,0.05,0.1,0.15 > gpurun_out/v3s.jsonl 2>&1
  echo "$v 1%:$b $(grep '^{' gpurun_out/v3s.jsonl | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['density']}:{json.loads(l)['sparse_ms']}\" for l in sys.stdin))")"
done
