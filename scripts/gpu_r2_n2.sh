#!/bin/bash
# round 2, 2 GPUs: multi-rank parity (NCCL fabric), bench N=2 with the route
# block, NVLink counters of the pack kernel (ncu on rank 0 only)
cd $GRAFT_REPO_ROOT
N=${N:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
timeout 900 $TR scripts/mgpu_check.py > gpurun_out/mgpu_n$N.log 2>&1; echo "mgpu rc=$?" >> gpurun_out/mgpu_n$N.log
timeout 600 $TR bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "rc=$?" >> gpurun_out/bench_n$N.err
ncu --query-metrics 2>/dev/null | grep -i -E "^nvl|nvlrx|nvltx" > gpurun_out/ncu_nvl_metrics.txt
cat > /tmp/rank_wrap.sh <<'EOW'
#!/bin/bash
if [ "$LOCAL_RANK" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --kernel-name regex:"pack_kernel|apply_p2p_kernel|encode_kernel|local_apply" --launch-skip 40 --launch-count 12 \
    --clock-control none --csv --log-file gpurun_out/ncu_route_n$N.csv python bench.py --gpus $N --steps 4 --warmup 3 --no-e2e --no-cpu-baseline
else
  exec python bench.py --gpus $N --steps 4 --warmup 3 --no-e2e --no-cpu-baseline
fi
EOW
chmod +x /tmp/rank_wrap.sh
N=$N timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 --no-python /tmp/rank_wrap.sh > gpurun_out/ncu_route_n$N.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_route_n$N.log
