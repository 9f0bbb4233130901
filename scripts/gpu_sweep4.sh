python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 scripts/density_sweep.py --steps 6 > gpurun_out/sweep_n4.jsonl 2> gpurun_out/sweep_n4.err; echo "sweep rc=$?"
cat gpurun_out/sweep_n4.jsonl
