set -x
mkdir -p gpurun_out/early2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/early2/pytest_gpu.log 2>&1; echo pytest=$?
AL_BWD_STEAL=1 timeout 600 python -m pytest tests/test_bwd_steal_gpu.py -x -q > gpurun_out/early2/pytest_steal_forced.log 2>&1; echo steal=$?
for m in 0 2; do for S in 1560 7800 14040 20280; do
AL_BWD_EARLY=$m python tools/short_s_timeline.py --bucket1 $S 1 | sed "s/^{/{\"AL_BWD_EARLY\": $m, /" >> gpurun_out/early2/buckets.jsonl
done; done
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/early2/bench.json 2> gpurun_out/early2/bench.err
tail -1 gpurun_out/early2/pytest_gpu.log
