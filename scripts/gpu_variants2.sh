# K1 variants: parity (engine+codec GPU tests) + sparse times.
for V in base ${VARIANTS}; do
  if [ $V = base ]; then unset WSYNC_LIB; else export WSYNC_LIB=$PWD/paper_2605_06534_b200/lib/$V/libwsync.so; fi
  echo "== $V"
  [ -n "$NOTEST" ] || timeout 600 python -m pytest tests/test_codec_gpu.py tests/test_engine_gpu.py -q -x -m gpu 2>&1 | tail -1
  timeout 600 python scripts/density_sweep.py --steps 8 --densities ${DENS:-0.0001,0.01,0.05,0.2} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['density'], 'sparse_ms', d['sparse_ms'], d.get('sparse_stages_ms',{}))"
done
