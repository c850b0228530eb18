set -x
mkdir -p gpurun_out/gw2
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gw2/pytest.log 2>&1; echo pytest=$?
AL_BWD_STEAL=1 timeout 600 python -m pytest tests/test_bwd_steal_gpu.py tests/test_group_walk_gpu.py -x -q -p no:cacheprovider > gpurun_out/gw2/pytest_steal.log 2>&1; echo steal=$?
AL_BWD_GROUP_WALK=0 timeout 600 python -m pytest tests/test_bwd_steal_gpu.py tests/test_multigroup_gpu.py -x -q -p no:cacheprovider > gpurun_out/gw2/pytest_gw0.log 2>&1; echo gw0=$?
for S in 20280 32760; do for det in 0 1; do python tools/short_s_timeline.py --bucket1 $S $det >> gpurun_out/gw2/b.jsonl; done; done
tail -1 gpurun_out/gw2/pytest.log; tail -1 gpurun_out/gw2/pytest_steal.log; tail -1 gpurun_out/gw2/pytest_gw0.log
