# Final single-GPU numbers on the final build: smoke, reference arm, bench x2 (driver K/W),
# 200-step bench, the cfg1/cfg3 length sweep, the sampler-batched cfg3 buckets.
set -x
mkdir -p gpurun_out/final2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo smoke=$?
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final2/ref.json 2> gpurun_out/final2/ref.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.err
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final2/bench_b.json 2> /dev/null
python bench.py --gpus 1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/final2/bench_k200.json 2>/dev/null
python tools/sweep_lengths.py > gpurun_out/final2/lengths.jsonl 2> gpurun_out/final2/lengths.err
python tools/short_s_timeline.py --buckets 1560 3600 7800 14040 20280 > gpurun_out/final2/buckets.jsonl 2> gpurun_out/final2/buckets.err
