for c in 8 16 32; do AL_STEAL_CHUNK=$c timeout 200 python tools/steal_probe.py 30 c$c >> gpurun_out/r2t.jsonl 2>&1; done
AL_STEAL_POOL=0 timeout 200 python tools/steal_probe.py 30 nosteal >> gpurun_out/r2t.jsonl 2>&1
