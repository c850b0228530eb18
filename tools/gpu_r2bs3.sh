#!/bin/bash
# repeated, interleaved A/B: default static backward vs work stealing (chunk 32) on the sampler's
# short-length buckets; non-deterministic and deterministic flag
mkdir -p gpurun_out/r2bs3
o=gpurun_out/r2bs3/${OUT:-ab}.jsonl; : > $o
for rep in $(seq 1 ${REPS:-3}); do
  for cfg in ${CFGS:-307x1560 133x3600 49x7800}; do  # BxS tokens
    set -- ${cfg/x/ }
    for det in 0 1; do
      python tools/short_s_timeline.py --one $1 $2 $det | sed "s/^{/{\"mode\": \"default\", \"rep\": $rep, /" >> $o
      AL_BWD_STEAL=1 AL_STEAL_CHUNK=32 python tools/short_s_timeline.py --one $1 $2 $det | sed "s/^{/{\"mode\": \"steal_c32\", \"rep\": $rep, /" >> $o
    done
  done
done 2> gpurun_out/r2bs3/ab.err
