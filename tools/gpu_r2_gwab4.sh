set -x
for i in 1 2; do
AL_LIB_VARIANT=pre_gw python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gwab4_pre_$i.json 2>/dev/null
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gwab4_head_$i.json 2>/dev/null
for S in 20280 32760; do
AL_LIB_VARIANT=gw_common python tools/short_s_timeline.py --bucket1 $S 1 | sed 's/^{/{"lib": "gw_common", /' >> gpurun_out/gwab4_b.jsonl
python tools/short_s_timeline.py --bucket1 $S 1 | sed 's/^{/{"lib": "head", /' >> gpurun_out/gwab4_b.jsonl
python tools/short_s_timeline.py --bucket1 $S 0 | sed 's/^{/{"lib": "head", /' >> gpurun_out/gwab4_b.jsonl
done; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gwab4_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/gwab4_pytest.log
