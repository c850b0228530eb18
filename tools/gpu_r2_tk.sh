set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/tk_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/tk_pytest.log
for i in 1 2; do python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/tk_bench_$i.json 2>/dev/null; done
python tools/bwd_race_stress.py 150 > gpurun_out/tk_race.jsonl 2>&1
