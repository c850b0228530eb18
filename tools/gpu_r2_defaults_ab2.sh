# Bench-mode A/B of the final backward defaults (interleaved walk, release after phase 1) vs the
# round-2 defaults before the pace study (ticket walk, release after the stage barrier).
set -x
for i in 1 2 3; do
AL_BWD_TICKET=1 AL_BWD_EARLY=0 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/defab2_old_$i.json 2>/dev/null
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/defab2_new_$i.json 2>/dev/null
done
