#!/bin/bash
# multi-group forward tail + many-group stage 2: tests, then the bucket sweep
mkdir -p gpurun_out/r2mg2
timeout 900 python -m pytest tests/test_multigroup_gpu.py tests/test_adaln_gpu.py tests/test_gate_residual_gpu.py tests/test_guard_bands_gpu.py -q -x -p no:cacheprovider > gpurun_out/r2mg2/pytest.log 2>&1
echo rc=$? >> gpurun_out/r2mg2/pytest.log
timeout 900 python tools/short_s_timeline.py --buckets > gpurun_out/r2mg2/buckets.jsonl 2> gpurun_out/r2mg2/buckets.err
