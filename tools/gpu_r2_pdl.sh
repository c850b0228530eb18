set -x
mkdir -p gpurun_out/pdl
for i in 1 2; do for m in 6 7; do
AL_PDL_MASK=$m python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/pdl/m${m}_$i.json 2>/dev/null
done; done
