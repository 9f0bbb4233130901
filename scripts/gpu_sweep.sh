for v in R3 R4 R5; do
  for dn in 0.01 0.1 0.0; do echo -n "$v d=$dn "; DENSITY=$dn WSYNC_LIB=paper_2605_06534_b200/lib/variants/libwsync_$v.so timeout 120 python scripts/encode_probe.py 2e9 10; done
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --verify 2>&1 | tail -1
