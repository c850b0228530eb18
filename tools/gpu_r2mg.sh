#!/bin/bash
# multi-group vs single-group backward at the same row count (478 920 rows, D = 5120 bf16)
mkdir -p gpurun_out/r2mg
o=gpurun_out/r2mg/mg.jsonl; : > $o
for rep in 1 2; do
python tools/short_s_timeline.py --one 1 478920 0 >> $o
python tools/short_s_timeline.py --one 1 478920 1 >> $o
AL_BWD_INTERLEAVE=0 python tools/short_s_timeline.py --one 1 478920 1 >> $o
python tools/short_s_timeline.py --one 307 1560 0 >> $o
python tools/short_s_timeline.py --one 2 239460 0 >> $o
python tools/short_s_timeline.py --one 2 239460 1 >> $o
done 2> gpurun_out/r2mg/mg.err
