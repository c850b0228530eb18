# Round-2 re-entry confirmation on HEAD: smoke, GPU suite, N=1 bench (driver's K/W), reference arm.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c_pytest_gpu.log 2>&1; echo pytest=$?
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/c_ref.json 2> gpurun_out/c_ref.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
tail -3 gpurun_out/c_pytest_gpu.log; tail -c 400 gpurun_out/c_bench.json
