# K1 ablation: look-back off (1), record writes off (2), both (3); per lib variant.
for V in base ${VARIANTS:-r5c64}; do
  if [ $V = base ]; then unset WSYNC_LIB; else export WSYNC_LIB=$PWD/paper_2605_06534_b200/lib/$V/libwsync.so; fi
  for D in 0 1 2 3; do
    echo "== $V debug=$D"
    WSYNC_ENCODE_DEBUG=$D timeout 600 python scripts/density_sweep.py --steps 6 --densities ${DENS:-0.0001,0.01} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['density'], 'sparse_ms', d['sparse_ms'])"
  done
done
