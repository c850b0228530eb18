# Final HEAD: cfg1/cfg3 single-sample sweep and the sampler-batched cfg3 buckets (one process
# per bucket and mode).
set -x
mkdir -p gpurun_out/final5
python tools/sweep_lengths.py > gpurun_out/final5/lengths.jsonl 2> gpurun_out/final5/lengths.err
for S in 1560 3600 7800 14040 20280 32760 46800 61200 75600; do for det in 0 1; do
python tools/short_s_timeline.py --bucket1 $S $det >> gpurun_out/final5/buckets.jsonl 2>> gpurun_out/final5/buckets.err
done; done
