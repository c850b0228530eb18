set -x
for i in 1 2; do for S in 20280 32760; do
AL_LIB_VARIANT=gw_common python tools/short_s_timeline.py --bucket1 $S 1 | sed 's/^{/{"lib": "gw_common", /' >> gpurun_out/gwab3_b.jsonl
python tools/short_s_timeline.py --bucket1 $S 1 | sed 's/^{/{"lib": "head", /' >> gpurun_out/gwab3_b.jsonl
AL_LIB_VARIANT=pre_gw python tools/short_s_timeline.py --bucket1 $S 1 | sed 's/^{/{"lib": "pre_gw", /' >> gpurun_out/gwab3_b.jsonl
done; done
