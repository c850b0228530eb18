timeout 240 python -m pytest tests/test_bwd_steal_gpu.py -x -q > gpurun_out/r2s_steal.log 2>&1
echo "rc=$?" >> gpurun_out/r2s_steal.log
AB_LEGACY=1 timeout 300 python tools/ab_time.py 50 steal > gpurun_out/r2s_ab.jsonl 2>&1
echo "rc=$?" >> gpurun_out/r2s_ab.jsonl
