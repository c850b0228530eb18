#!/bin/bash
# A/B of the PDL launch mask (AL_PDL_MASK: 1 forward, 2 backward stage 1, 4 stage 2) on the
# fwd+bwd length sweep and the back-to-back bandwidth probe.
for m in 0 4 6 1 7; do
  echo "mask=$m"
  AL_PDL_MASK=$m python tools/bw_probe.py
  AL_PDL_MASK=$m python tools/sweep_lengths.py | python3 -c "
import json,sys
print(' '.join(f\"{d['S']}:{d['gbs']}\" for d in map(json.loads, sys.stdin)))"
done
