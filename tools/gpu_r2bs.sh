#!/bin/bash
# multi-sample buckets (the sampler's B for each short S): work-stealing backward (chunk sizes)
# vs the default static partition, after the many-group stage-2 kernel
mkdir -p gpurun_out/r2bs2
for c in 16 32 64; do
  AL_BWD_STEAL=1 AL_STEAL_CHUNK=$c timeout 600 python tools/short_s_timeline.py --buckets 1560 3600 7800 14040 20280 32760 | sed "s/^{/{\"mode\": \"steal_c$c\", /" >> gpurun_out/r2bs2/steal.jsonl 2>> gpurun_out/r2bs2/steal.err
done
timeout 600 python tools/short_s_timeline.py --buckets 1560 3600 7800 14040 20280 32760 | sed "s/^{/{\"mode\": \"default\", /" >> gpurun_out/r2bs2/steal.jsonl 2>> gpurun_out/r2bs2/steal.err
