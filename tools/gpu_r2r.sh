python -m pytest tests/test_runtime_gpu.py -q -k non_current > gpurun_out/r2r_guard.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2r_n2.json 2> gpurun_out/r2r_n2.err
python bench.py --workload dit --steps 12 --warmup 2 --trace-dir gpurun_out/r2r_traces > gpurun_out/r2r_dit1.json 2> gpurun_out/r2r_dit1.err
