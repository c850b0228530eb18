set -x
mkdir -p gpurun_out/st0
for i in 1 2; do for S in 14040 20280 32760; do
python tools/short_s_timeline.py --bucket1 $S 1 | sed 's/^{/{"AL_BWD_STEAL": "auto", /' >> gpurun_out/st0/b.jsonl
AL_BWD_STEAL=0 python tools/short_s_timeline.py --bucket1 $S 1 | sed 's/^{/{"AL_BWD_STEAL": "0", /' >> gpurun_out/st0/b.jsonl
done; done
