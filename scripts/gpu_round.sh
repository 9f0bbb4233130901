# One GPU call: GPU tests, N=1 bench + density sweep, and (when >1 GPU) the
# multi-GPU parity check in both exchange modes.
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --verify 2>&1 | tail -1 | cut -c1-900
CUDA_VISIBLE_DEVICES=0 timeout 600 python scripts/density_sweep.py --steps 6 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['density'], 'sparse_ms', d['sparse_ms'], 'dense_ms', d['dense_ms'])"
if [ $NG -gt 1 ]; then N=$NG bash scripts/gpu_dense_direct.sh 2>&1 | grep -v "^{" ; fi
