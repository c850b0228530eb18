set -x
mkdir -p gpurun_out/bk
for S in 3600 7800 14040 20280; do for det in 0 1; do
python tools/short_s_timeline.py --bucket1 $S $det >> gpurun_out/bk/default.jsonl
AL_BWD_EARLY=0 python tools/short_s_timeline.py --bucket1 $S $det >> gpurun_out/bk/early0.jsonl
done; done
python tools/short_s_timeline.py --buckets 7800 14040 > gpurun_out/bk/one_process.jsonl
