set -x
mkdir -p gpurun_out/walk
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/walk/pytest_gpu2.log 2>&1; echo pytest=$?
AL_BWD_STEAL=1 timeout 600 python -m pytest tests/test_bwd_steal_gpu.py -x -q > gpurun_out/walk/pytest_steal_forced.log 2>&1; echo steal=$?
tail -1 gpurun_out/walk/pytest_gpu2.log
