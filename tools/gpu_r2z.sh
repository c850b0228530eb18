timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2z_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_gpu.log
AL_BWD_STEAL=1 timeout 300 python -m pytest tests/test_bwd_steal_gpu.py -x -q > gpurun_out/r2z_steal.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_steal.log
timeout 300 python tools/bwd_variants.py 30 > gpurun_out/r2z_var.jsonl 2>&1
