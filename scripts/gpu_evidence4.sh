# Round evidence on a 4-GPU box: tests, bench N=1/2/4 (+ reference arm),
# density sweeps N=1 and N=4, multi-GPU parity in every exchange mode.
set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/ev_bench_n1.json 2> gpurun_out/ev_bench_n1.err; echo "bench1 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_ref_n1.json 2> gpurun_out/ev_ref_n1.err; echo "ref1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/ev_bench_n$N.json 2> gpurun_out/ev_bench_n$N.err; echo "bench$N rc=$?"
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python scripts/density_sweep.py --steps 6 > gpurun_out/ev_sweep_n1.jsonl 2> gpurun_out/ev_sweep_n1.err; echo "sweep1 rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 scripts/density_sweep.py --steps 6 > gpurun_out/ev_sweep_n4.jsonl 2> gpurun_out/ev_sweep_n4.err; echo "sweep4 rc=$?"
N=4 bash scripts/gpu_dense_direct.sh > gpurun_out/ev_mgpu.log 2>&1; echo "mgpu rc=$?"
grep -E "rc=|\"ok\"" gpurun_out/ev_mgpu.log | head -20
for f in gpurun_out/ev_bench_n1.json gpurun_out/ev_bench_n2.json gpurun_out/ev_bench_n4.json gpurun_out/ev_ref_n1.json; do tail -1 $f | cut -c1-250; done
