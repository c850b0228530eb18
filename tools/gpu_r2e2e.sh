#!/bin/bash
# host-API pipeline chunk size with the resident x: e2e GB/s per chunk size (fresh processes)
mkdir -p gpurun_out/r2e2e
for mb in 8 16 32 64; do
  for rep in 1 2; do
    AL_HOST_CHUNK_MB=$mb python bench.py --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'chunk_mb': $mb, 'rep': $rep, 'e2e': d['e2e']}))" >> gpurun_out/r2e2e/chunks.jsonl
  done
done
