#!/bin/bash
# auto work stealing on multi-sample launches: full GPU suite, forced-steal suite, bucket sweep
mkdir -p gpurun_out/r2as
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2as/pytest.log 2>&1
echo rc=$? >> gpurun_out/r2as/pytest.log
AL_BWD_STEAL=1 timeout 600 python -m pytest tests/test_bwd_steal_gpu.py -q -p no:cacheprovider > gpurun_out/r2as/pytest_steal.log 2>&1
echo rc=$? >> gpurun_out/r2as/pytest_steal.log
for S in 1560 3600 7800 14040 20280 32760 46800 61200 75600; do
  for det in 0 1; do
    python tools/short_s_timeline.py --bucket1 $S $det >> gpurun_out/r2as/buckets.jsonl 2>> gpurun_out/r2as/buckets.err
  done
done
