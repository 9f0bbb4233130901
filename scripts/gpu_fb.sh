for v in fb2 fb1 fb2 fb1; do
  L=$PWD/paper_2605_06534_b200/lib/libwsync_$v.so
  WSYNC_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fbb.json 2>/dev/null
  b=$(grep '^{' gpurun_out/fbb.json | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(d['ms_per_step'],d['roofline']['frac'],d['clocks']['reasons'])")
  WSYNC_LIB=$L timeout 600 python scripts/density_sweep.py --densities 0.0001,0.003,0.02 > gpurun_out/fb.jsonl 2>&1
  echo "$v bench:$b $(grep '^{' gpurun_out/fb.jsonl | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['density']}:{json.loads(l)['sparse_ms']}\" for l in sys.stdin))")"
done
