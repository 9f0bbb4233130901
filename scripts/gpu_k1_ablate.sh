# K1 ablation on the engine path (N=1): variants x {normal, no writes, no fused apply}.
for V in base ${VARIANTS:-r5c64 r4c32 r6c64}; do
  if [ $V = base ]; then unset WSYNC_LIB; else export WSYNC_LIB=$PWD/paper_2605_06534_b200/lib/$V/libwsync.so; fi
  for MODE in normal nowrite nofuse; do
    case $MODE in normal) E="";; nowrite) E="WSYNC_ENCODE_DEBUG=2";; nofuse) E="WSYNC_NO_FUSED_APPLY=1";; esac
    echo "== $V $MODE"
    env $E timeout 600 python scripts/density_sweep.py --steps 6 --densities ${DENS:-0.0001,0.01,0.05} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['density'], 'sparse_ms', d['sparse_ms'], d.get('sparse_stages_ms',{}))"
  done
done
