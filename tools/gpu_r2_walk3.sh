set -x
mkdir -p gpurun_out/walk3
for i in 1 2; do for t in 0 1; do
AL_BWD_TICKET=$t python tools/bwd_np_ab.py 14040 20280 32760 46800 75600 >> gpurun_out/walk3/ab.jsonl 2>> gpurun_out/walk3/ab.err
done; done
