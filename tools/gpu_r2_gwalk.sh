set -x
mkdir -p gpurun_out/gw
timeout 900 python -m pytest tests/test_group_walk_gpu.py -x -q -p no:cacheprovider > gpurun_out/gw/pytest.log 2>&1; echo pytest=$?
tail -15 gpurun_out/gw/pytest.log
for i in 1 2; do for S in 20280 32760; do for gw in 0 1 2; do
AL_BWD_GROUP_WALK=$gw python tools/short_s_timeline.py --bucket1 $S 1 | sed "s/^{/{\"gw\": $gw, /" >> gpurun_out/gw/b.jsonl
AL_BWD_GROUP_WALK=$gw python tools/short_s_timeline.py --bucket1 $S 0 | sed "s/^{/{\"gw\": $gw, /" >> gpurun_out/gw/b.jsonl
done; done; done
