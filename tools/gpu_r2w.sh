timeout 240 python -m pytest tests/test_bwd_steal_gpu.py -x -q > gpurun_out/r2w_steal.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_steal.log
AL_STEAL_CHUNK=8 timeout 200 python tools/steal_probe.py 30 c8 >> gpurun_out/r2w.jsonl 2>&1
AL_STEAL_POOL=0 timeout 200 python tools/steal_probe.py 30 nosteal >> gpurun_out/r2w.jsonl 2>&1
