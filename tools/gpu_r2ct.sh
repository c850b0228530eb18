#!/bin/bash
# chunked forward tail for single-group launches (AL_FWD_DYN_GROUPS=2) vs the per-warp tail
mkdir -p gpurun_out/r2ct
o=gpurun_out/r2ct/ct.jsonl; : > $o
for rep in 1 2; do
  python tools/short_s_timeline.py 1560 3600 7800 14040 32760 75600 | sed 's/^{/{"mode": "default", /' >> $o
  AL_FWD_DYN_GROUPS=2 python tools/short_s_timeline.py 1560 3600 7800 14040 32760 75600 | sed 's/^{/{"mode": "chunk", /' >> $o
done 2> gpurun_out/r2ct/ct.err
python bench.py --steps 20 --warmup 5 > gpurun_out/r2ct/bench_default.json 2>> gpurun_out/r2ct/ct.err
AL_FWD_DYN_GROUPS=2 python bench.py --steps 20 --warmup 5 > gpurun_out/r2ct/bench_chunk.json 2>> gpurun_out/r2ct/ct.err
