#!/bin/bash
# short-S device timeline: default library, then the per-CTA trace build
mkdir -p gpurun_out/r2ss
timeout 600 python tools/short_s_timeline.py 1560 3600 7800 14040 32760 > gpurun_out/r2ss/timeline.jsonl 2> gpurun_out/r2ss/timeline.err
AL_LIB_VARIANT=cta_trace timeout 600 python tools/short_s_timeline.py 1560 3600 7800 > gpurun_out/r2ss/timeline_cta.jsonl 2> gpurun_out/r2ss/timeline_cta.err
