for c in 8 64; do AL_BWD_STEAL=1 AL_STEAL_CHUNK=$c timeout 200 python tools/steal_probe.py 30 c$c >> gpurun_out/r2s3.jsonl 2>&1; done
