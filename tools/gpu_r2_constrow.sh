set -x
for i in 1 2; do for c in 0 1; do
AL_BWD_CONST_ROW=$c python tools/bwd_np_ab.py 14040 32760 75600 >> gpurun_out/constrow.jsonl 2>> gpurun_out/constrow.err
done; done
for c in 0 1; do AL_BWD_CONST_ROW=$c python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/constrow_bench_$c.json 2>/dev/null; done
