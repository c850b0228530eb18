# Bench-mode A/B of the round-2 backward defaults: old (ticket walk, slot released after the
# stage barrier) vs new (interleaved walk, early release), alternating, same box.
set -x
for i in 1 2 3; do
AL_BWD_TICKET=1 AL_BWD_EARLY=0 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/defab_old_$i.json 2>/dev/null
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/defab_new_$i.json 2>/dev/null
AL_BWD_TICKET=1 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/defab_ticketearly_$i.json 2>/dev/null
done
