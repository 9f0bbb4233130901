for d in 0 1 2; do WSYNC_ENCODE_DEBUG=$d timeout 120 python scripts/encode_probe.py 2e9 10; done
DENSITY=0.0 timeout 120 python scripts/encode_probe.py 2e9 10
DENSITY=0.1 timeout 120 python scripts/encode_probe.py 2e9 10
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --verify 2>&1 | tail -1
