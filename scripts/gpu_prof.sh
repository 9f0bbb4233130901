DENSITY=0.01 python scripts/encode_probe.py 268435456 5 > gpurun_out/probe_small.log 2>&1 && \
DENSITY=0.01 ncu --set full --clock-control none --import-source on -k regex:encode_kernel -s 2 -c 1 -o gpurun_out/enc_v9 python scripts/encode_probe.py 268435456 5 > gpurun_out/ncu_enc.log 2>&1
tail -1 gpurun_out/ncu_enc.log; cat gpurun_out/probe_small.log
