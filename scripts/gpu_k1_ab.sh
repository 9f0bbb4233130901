#!/bin/bash
# same-box A/B of a K1 change: lib/libwsync_prev.so (before) vs lib/libwsync.so
# (after), N=1 bench at several densities, alternating; then the K1 parity tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/k1ab; mkdir -p $O
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_codec_gpu.py tests/test_golden.py -q --timeout 800 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for k in 1 2; do for d in ${DS:-0.01 0.05 0.1}; do for v in prev new; do
  if [ $v = prev ]; then L=paper_2605_06534_b200/lib/libwsync_prev.so; else L=paper_2605_06534_b200/lib/libwsync.so; fi
  echo -n "{\"v\": \"$v\", \"d\": $d, \"line\": " >> $O/ab.jsonl
  WSYNC_LIB=$L timeout 300 python bench.py --density $d --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-verify 2>/dev/null | grep '^{' | tr -d '\n' >> $O/ab.jsonl
  echo "}" >> $O/ab.jsonl
done; done; done
