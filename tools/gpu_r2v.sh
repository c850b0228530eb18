timeout 240 python -m pytest tests/test_bwd_steal_gpu.py -x -q > gpurun_out/r2v_steal.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_steal.log
for c in 8 16; do AL_STEAL_CHUNK=$c timeout 200 python tools/steal_probe.py 30 c$c >> gpurun_out/r2v.jsonl 2>&1; done
AL_STEAL_POOL=0 timeout 200 python tools/steal_probe.py 30 nosteal >> gpurun_out/r2v.jsonl 2>&1
