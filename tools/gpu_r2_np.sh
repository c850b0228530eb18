set -x
for i in 1 2; do for m in 0 12 8; do
AL_BWD_NP=$m python tools/bwd_np_ab.py 14040 32760 75600 >> gpurun_out/np_ab.jsonl 2>> gpurun_out/np_ab.err
done; done
