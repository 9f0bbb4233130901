# K1 streamed apply: parity, then bench and density sweep with it on
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q 2>&1 | tail -2
for div in ${DIVS:-200}; do
  WSYNC_SA_DIV=$div timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/sa_bench_$div.json 2> gpurun_out/sa_bench_$div.err
  echo "sa_div=$div rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/sa_bench_$div.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'])"
  WSYNC_SA_DIV=$div timeout 600 python scripts/density_sweep.py --densities ${DENS:-0.001,0.003,0.006,0.01,0.02,0.05,0.1,0.15} > gpurun_out/sa_sweep_$div.jsonl 2>&1; echo "sweep $div rc=$?"
  grep "^{" gpurun_out/sa_sweep_$div.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['density'], d['sparse_ms'])"
done
