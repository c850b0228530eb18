set -x
mkdir -p gpurun_out/ramp
timeout 900 python -m pytest tests -m gpu -x -q -k "host or e2e or pinned or resident or api or reference" > gpurun_out/ramp/pytest.log 2>&1; echo pytest=$?
for i in 1 2; do for r in 0 1; do
AL_HOST_RAMP=$r python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ramp/bench_r${r}_$i.json 2>/dev/null
done; done
tail -1 gpurun_out/ramp/pytest.log
