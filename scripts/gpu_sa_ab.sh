for d in 0 250 0 250; do
  WSYNC_SA_DIV=$d timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/sa_ab_$d.json 2>/dev/null
  echo "sa_div=$d: $(python -c "import json;d=json.loads(open('gpurun_out/sa_ab_$d.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['clocks'])")"
done
