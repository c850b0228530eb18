# Three-arm bench-mode A/B of the single-sample backward schedule (non-deterministic headline):
# interleaved + release after phase 1 (default), ticket + release after the barrier (old),
# ticket + release after phase 1.  Alternating, three rounds.
set -x
tag=$1
for i in 1 2 3; do
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab3_${tag}_new_$i.json 2>/dev/null
AL_BWD_TICKET=1 AL_BWD_EARLY=0 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab3_${tag}_old_$i.json 2>/dev/null
AL_BWD_TICKET=1 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab3_${tag}_tk1_$i.json 2>/dev/null
done
