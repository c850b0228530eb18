set -x
mkdir -p gpurun_out/walk
for i in 1 2; do for t in 0 1; do
AL_BWD_TICKET=$t python tools/bwd_np_ab.py 14040 20280 32760 46800 75600 >> gpurun_out/walk/ab.jsonl 2>> gpurun_out/walk/ab.err
done; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/walk/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/walk/bench.json 2> gpurun_out/walk/bench.err
AL_BWD_TICKET=1 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/walk/bench_ticket.json 2> gpurun_out/walk/bench_ticket.err
tail -1 gpurun_out/walk/pytest_gpu.log
