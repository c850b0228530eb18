set -x
for i in 1 2; do for r in 12288 0; do
AL_BWD_PIPE_ROWS=$r python tools/bwd_np_ab.py 1560 3600 7800 12000 >> gpurun_out/pipe_ab.jsonl 2>> gpurun_out/pipe_ab.err
done; done
