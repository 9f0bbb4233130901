# K1 configuration variants (built into paper_2605_06534_b200/lib/<name>/):
# parity tests + sparse/dense times at a few densities, N=1.
for V in base ${VARIANTS:-r5c64 r6c64 r4c32}; do
  if [ $V = base ]; then unset WSYNC_LIB; else export WSYNC_LIB=$PWD/paper_2605_06534_b200/lib/$V/libwsync.so; fi
  echo "== $V"
  timeout 600 python -m pytest tests/test_codec_gpu.py tests/test_engine_gpu.py -q -x -m gpu 2>&1 | tail -1
  timeout 600 python scripts/density_sweep.py --steps 6 --densities ${DENS:-0.0001,0.01,0.05,0.2} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['density'], 'sparse_ms', d['sparse_ms'], 'dense_ms', d['dense_ms'])"
done
