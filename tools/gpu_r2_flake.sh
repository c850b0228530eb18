set -x
for i in 1 2; do
AL_BWD_EARLY=0 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/flake_e0_$i.log 2>&1; tail -1 gpurun_out/flake_e0_$i.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/flake_e2_$i.log 2>&1; tail -1 gpurun_out/flake_e2_$i.log
done
