#!/bin/bash
# multi-sample buckets (the sampler's B for each short S): work-stealing backward vs default
mkdir -p gpurun_out/r2bs
for c in 8 32; do
  AL_BWD_STEAL=1 AL_STEAL_CHUNK=$c timeout 600 python tools/short_s_timeline.py --buckets 1560 3600 7800 14040 > gpurun_out/r2bs/steal_c$c.jsonl 2> gpurun_out/r2bs/steal_c$c.err
done
