timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --verify 2>&1 | tail -1 | cut -c1-700
CUDA_VISIBLE_DEVICES=0 python scripts/density_sweep.py --steps 6 2>&1 | cut -c1-200
