for v in st4 st2 st4 st2; do
  WSYNC_LIB=$PWD/paper_2605_06534_b200/lib/libwsync_$v.so timeout 600 python scripts/density_sweep.py --densities 0.0001,0.003,0.01,0.05,0.1,0.15 > gpurun_out/st.jsonl 2>&1
  echo "$v $(grep '^{' gpurun_out/st.jsonl | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['density']}:{json.loads(l)['sparse_ms']}\" for l in sys.stdin))")"
done
