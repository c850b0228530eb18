set -x
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/_bwd_traffic_probe tools/bwd_traffic_probe.cu
./tools/_bwd_traffic_probe 32760 > gpurun_out/spin.jsonl
AB_NVCC_FLAGS=-DAL_CTA_TRACE bash tools/ab_variant.sh trace paper_2605_17923_b200/csrc
AL_LIB_VARIANT=trace python tools/sm_stage_share.py 32760 > gpurun_out/share.jsonl
./tools/_sm_topology_probe > gpurun_out/topo4.jsonl
