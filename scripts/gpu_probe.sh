for dn in 0.01 0.1 0.0 0.3; do echo -n "d=$dn "; DENSITY=$dn timeout 120 python scripts/encode_probe.py 2e9 10; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --verify 2>&1 | tail -1
