timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_codec_gpu.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'])"
for F in 1 0; do
  WSYNC_STREAM_FUSE=$F timeout 300 python scripts/density_sweep.py --steps 6 --densities 0.01,0.1,0.15,0.2 2>/dev/null | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('fuse=$F', d['density'], d['sparse_ms'], d['sparse_stages_ms'])"
done
