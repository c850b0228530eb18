set -x
for i in 1 2; do
AL_BWD_TICKET=1 python tools/bwd_np_ab.py 32760 75600 >> gpurun_out/fake.jsonl 2>> gpurun_out/fake.err
AL_BWD_TICKET=1 AL_BWD_FAKE_TICKET=1 python tools/bwd_np_ab.py 32760 75600 >> gpurun_out/fake.jsonl 2>> gpurun_out/fake.err
AL_BWD_TICKET=1 AL_BWD_FAKE_TICKET=1 AL_BWD_EARLY=2 python tools/bwd_np_ab.py 32760 75600 >> gpurun_out/fake.jsonl 2>> gpurun_out/fake.err
done
