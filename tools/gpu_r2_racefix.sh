set -x
python tools/bwd_race_stress.py 300 > gpurun_out/racefix.jsonl 2>&1
AL_BWD_EARLY=0 python tools/bwd_race_stress.py 100 >> gpurun_out/racefix.jsonl 2>&1
for i in 1 2; do timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/racefix_pytest_$i.log 2>&1; tail -1 gpurun_out/racefix_pytest_$i.log; done
AL_BWD_STEAL=1 timeout 600 python -m pytest tests/test_bwd_steal_gpu.py tests/test_group_walk_gpu.py tests/test_bwd_race_gpu.py -q -p no:cacheprovider > gpurun_out/racefix_steal.log 2>&1; tail -1 gpurun_out/racefix_steal.log
for i in 1 2; do python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/racefix_bench_$i.json 2>/dev/null; done
for S in 20280 32760; do for det in 0 1; do python tools/short_s_timeline.py --bucket1 $S $det >> gpurun_out/racefix_b.jsonl; done; done
