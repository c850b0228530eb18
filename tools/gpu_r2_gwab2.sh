set -x
for i in 1 2 3; do
AL_LIB_VARIANT=pre_gw python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gwab2_pre_$i.json 2>/dev/null
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gwab2_head_$i.json 2>/dev/null
done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gwab2_pytest.log 2>&1; echo pytest=$?
for S in 20280 32760; do for det in 0 1; do python tools/short_s_timeline.py --bucket1 $S $det >> gpurun_out/gwab2_b.jsonl; done; done
tail -1 gpurun_out/gwab2_pytest.log
