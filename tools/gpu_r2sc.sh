#!/bin/bash
# single-group / few-group launches: forced work stealing with the contiguous chunk layout
# (AL_BWD_INTERLEAVE=0) vs the interleaved layout vs the defaults (det / non-det)
mkdir -p gpurun_out/r2sc
o=gpurun_out/r2sc/sc.jsonl; : > $o
for rep in 1 2; do
  for cfg in 1x32760 1x75600 2x32760 7x20280; do
    set -- ${cfg/x/ }
    python tools/short_s_timeline.py --one $1 $2 0 | sed "s/^{/{\"mode\": \"default_dyn\", \"rep\": $rep, /" >> $o
    python tools/short_s_timeline.py --one $1 $2 1 | sed "s/^{/{\"mode\": \"default_det\", \"rep\": $rep, /" >> $o
    AL_BWD_STEAL=1 AL_BWD_INTERLEAVE=0 python tools/short_s_timeline.py --one $1 $2 1 | sed "s/^{/{\"mode\": \"steal_contig_c32\", \"rep\": $rep, /" >> $o
    AL_BWD_STEAL=1 AL_BWD_INTERLEAVE=0 AL_STEAL_CHUNK=16 python tools/short_s_timeline.py --one $1 $2 1 | sed "s/^{/{\"mode\": \"steal_contig_c16\", \"rep\": $rep, /" >> $o
    AL_BWD_STEAL=1 python tools/short_s_timeline.py --one $1 $2 1 | sed "s/^{/{\"mode\": \"steal_il\", \"rep\": $rep, /" >> $o
  done
done 2> gpurun_out/r2sc/sc.err
