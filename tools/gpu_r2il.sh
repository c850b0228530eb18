timeout 600 python -m pytest tests/test_adaln_gpu.py tests/test_parity_r2_gpu.py tests/test_bwd_steal_gpu.py -x -q > gpurun_out/r2il_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2il_tests.log
timeout 300 python tools/bwd_variants.py 30 > gpurun_out/r2il_var.jsonl 2>&1
AL_BWD_INTERLEAVE=2 timeout 300 python tools/bwd_variants.py 30 > gpurun_out/r2il_var2.jsonl 2>&1
