set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
for i in 1 2 3; do python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2a_bench_$i.json 2> gpurun_out/r2a_bench_$i.err; done
python bench.py --gpus 1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/r2a_bench_200.json 2>&1
tail -c 600 gpurun_out/r2a_bench_*.json
