set -x
for i in 1 2; do for b in 0 1; do
AL_BWD_BULKDX=$b python tools/bwd_np_ab.py 14040 32760 75600 >> gpurun_out/bulkdx.jsonl 2>> gpurun_out/bulkdx.err
done; done
AL_BWD_BULKDX=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/bulkdx_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/bulkdx_pytest.log
