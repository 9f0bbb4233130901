cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for k in 1 2; do
timeout 600 $TR --master-port 2971$k scripts/fanout_bench.py 2>/dev/null | grep '^{' >> gpurun_out/fanout_default.jsonl
timeout 600 $TR --master-port 2972$k bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' >> gpurun_out/c2_default.jsonl
done
timeout 900 python -m pytest tests/test_group_gpu.py tests/test_multigpu_gpu.py -q --timeout 800 -x > gpurun_out/sms_tests.log 2>&1; echo rc=$? >> gpurun_out/sms_tests.log
