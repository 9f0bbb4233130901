for v in A B C D E F; do
  for d in 0 1; do echo -n "$v "; WSYNC_LIB=paper_2605_06534_b200/lib/variants/libwsync_$v.so WSYNC_ENCODE_DEBUG=$d timeout 120 python scripts/encode_probe.py 2e9 10; done
  echo -n "$v "; DENSITY=0 WSYNC_LIB=paper_2605_06534_b200/lib/variants/libwsync_$v.so timeout 120 python scripts/encode_probe.py 2e9 10
done
