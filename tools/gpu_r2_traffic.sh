set -x
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/_bwd_traffic_probe tools/bwd_traffic_probe.cu
for i in 1 2; do ./tools/_bwd_traffic_probe 32760 >> gpurun_out/traffic.jsonl; done
./tools/_bwd_traffic_probe 65520 >> gpurun_out/traffic.jsonl
python tools/bw_probe.py >> gpurun_out/traffic_torch.jsonl 2>&1
