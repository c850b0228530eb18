# Flakiness / alternate-schedule check of the GPU suite on the final build.
set -x
mkdir -p gpurun_out/stab
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/stab/run$i.log 2>&1; echo run$i=$?; done
AL_BWD_TICKET=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/stab/ticket.log 2>&1; echo ticket=$?
AL_BWD_EARLY=0 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/stab/early0.log 2>&1; echo early0=$?
for f in gpurun_out/stab/*.log; do echo $f; tail -1 $f; done
