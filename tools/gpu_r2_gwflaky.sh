set -x
for i in 1 2 3 4 5; do timeout 600 python -m pytest tests/test_group_walk_gpu.py -q -p no:cacheprovider 2>&1 | tail -1; done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gwflaky_full.log 2>&1; tail -3 gpurun_out/gwflaky_full.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gwflaky_full2.log 2>&1; tail -3 gpurun_out/gwflaky_full2.log
