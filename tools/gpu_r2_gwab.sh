set -x
for i in 1 2 3; do
AL_LIB_VARIANT=pre_gw python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gwab_pre_$i.json 2>/dev/null
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gwab_head_$i.json 2>/dev/null
done
