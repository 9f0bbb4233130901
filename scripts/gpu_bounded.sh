NG=$(nvidia-smi -L | wc -l)
export WSYNC_MAX_THRESHOLD=0.2 WSYNC_EXCHANGE=p2p
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29661 scripts/mgpu_check.py > gpurun_out/bounded_check.log 2>&1; echo "check rc=$?"
grep -o '"rank": [0-9], "world": [0-9], "ok": [a-z]*' gpurun_out/bounded_check.log
grep -E "Error" gpurun_out/bounded_check.log | head -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29662 scripts/config_bench.py --full > gpurun_out/cfg_full.log 2>&1; echo "cfg rc=$?"
grep -E "^\{" gpurun_out/cfg_full.log; grep -E "Error" gpurun_out/cfg_full.log | head -3
