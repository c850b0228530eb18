set -x
mkdir -p gpurun_out/ramp2
for i in 1 2; do for r in 1 2 4; do
AL_HOST_RAMP=$r python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ramp2/r${r}_$i.json 2>/dev/null
done; done
