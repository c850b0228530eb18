#!/bin/bash
# Final 4-GPU / 2-GPU refresh: AdaLN bench line (+ DP four-arm A/B) and the DiT workload.
mkdir -p gpurun_out/final4
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/final4/bench_n4.json 2> gpurun_out/final4/bench_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/final4/ref_n4.json 2> gpurun_out/final4/ref_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 4 --workload dit --steps 16 --warmup 2 --trace-dir gpurun_out/final4/dit_n4_traces > gpurun_out/final4/dit_n4.json 2> gpurun_out/final4/dit_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/final4/bench_n2.json 2> gpurun_out/final4/bench_n2.err
grep -c "NCCL INFO" gpurun_out/final4/bench_n4.err > gpurun_out/final4/nccl_info_lines.txt
tail -c 300 gpurun_out/final4/bench_n4.json
