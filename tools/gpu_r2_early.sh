set -x
for i in 1 2; do for m in 0 1 2; do
AL_BWD_EARLY=$m python tools/bwd_np_ab.py 14040 20280 32760 46800 75600 >> gpurun_out/early_ab2.jsonl 2>> gpurun_out/early_ab2.err
done; done
