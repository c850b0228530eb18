#!/bin/bash
# many-group stage 2 threshold: AL_RED_GRP_MIN=2 / 8 vs the default 16 on few-group buckets
mkdir -p gpurun_out/r2rg
o=gpurun_out/r2rg/rg.jsonl; : > $o
for rep in 1 2; do
  for cfg in 15x14040 7x20280 2x32760 4x7800; do
    set -- ${cfg/x/ }
    for det in 0 1; do
      for m in 16 8 2; do
        AL_RED_GRP_MIN=$m python tools/short_s_timeline.py --one $1 $2 $det | sed "s/^{/{\"mode\": \"grpmin$m\", \"rep\": $rep, /" >> $o
      done
    done
  done
done 2> gpurun_out/r2rg/rg.err
