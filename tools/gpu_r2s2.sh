AL_BWD_STEAL=1 timeout 300 python -m pytest tests/test_bwd_steal_gpu.py -x -q > gpurun_out/r2s2_steal.log 2>&1; echo "rc=$?" >> gpurun_out/r2s2_steal.log
AL_BWD_STEAL=1 timeout 200 python tools/steal_probe.py 30 steal_il > gpurun_out/r2s2.jsonl 2>&1
AL_BWD_STEAL=1 AL_STEAL_POOL=0 timeout 200 python tools/steal_probe.py 30 steal_il_nosteal >> gpurun_out/r2s2.jsonl 2>&1
