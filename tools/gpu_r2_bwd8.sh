set -x
for i in 1 2; do
AL_BWD8=0 python tools/bwd8_ab.py >> gpurun_out/bwd8_ab.jsonl 2>> gpurun_out/bwd8_ab.err
AL_BWD8=1 python tools/bwd8_ab.py >> gpurun_out/bwd8_ab.jsonl 2>> gpurun_out/bwd8_ab.err
done
AL_BWD8=1 timeout 600 python -m pytest tests -m gpu -x -q -k "bwd or backward or determin" > gpurun_out/bwd8_pytest.log 2>&1; echo rc=$?
tail -3 gpurun_out/bwd8_pytest.log
