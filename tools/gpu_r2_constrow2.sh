set -x
for i in 1 2 3; do for c in 1 0; do AL_BWD_CONST_ROW=$c python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/constrow2_bench_${c}_$i.json 2>/dev/null; done; done
