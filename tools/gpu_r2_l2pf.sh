set -x
for i in 1 2; do for m in 0 1 2 4; do
AL_BWD_L2PF=$m python tools/bwd_np_ab.py 14040 32760 75600 >> gpurun_out/l2pf.jsonl 2>> gpurun_out/l2pf.err
done; done
