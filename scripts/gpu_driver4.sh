python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/drv4.json 2> gpurun_out/drv4.err; echo "ours rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/drv4_ref.json 2> gpurun_out/drv4_ref.err; echo "ref rc=$?"
CUDA_VISIBLE_DEVICES=0 python scripts/density_sweep.py --steps 6 > gpurun_out/sweep_n1.jsonl 2> gpurun_out/sweep_n1.err; echo "sweep rc=$?"
cat gpurun_out/drv4.json gpurun_out/drv4_ref.json gpurun_out/sweep_n1.jsonl
