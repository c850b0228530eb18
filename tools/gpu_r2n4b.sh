#!/bin/bash
# 4-GPU refresh on the final kernels: AdaLN bench line (+ DP four-arm A/B) and the DiT workload
mkdir -p gpurun_out/r2n4b
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2n4b/bench.json 2> gpurun_out/r2n4b/bench.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 4 --workload dit --steps 16 --warmup 2 --trace-dir gpurun_out/r2n4b/traces > gpurun_out/r2n4b/dit.json 2> gpurun_out/r2n4b/dit.err
grep -c "NCCL INFO" gpurun_out/r2n4b/bench.err > gpurun_out/r2n4b/nccl_info_lines.txt
