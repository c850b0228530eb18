# Final single-GPU confirmation on HEAD: smoke, GPU suite, reference arm + bench (driver K/W),
# a 200-step bench, the cfg1/cfg3 length sweep, and the PCIe ceiling of the e2e leg.
set -x
mkdir -p gpurun_out/final1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final1/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final1/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final1/ref.json 2> gpurun_out/final1/ref.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final1/bench.json 2> gpurun_out/final1/bench.err
python bench.py --gpus 1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/final1/bench_k200.json 2>/dev/null
python tools/pcie_probe.py > gpurun_out/final1/pcie.json 2>&1
python bench.py --gpus 1 --workload dit --steps 16 --warmup 2 > gpurun_out/final1/dit_n1.json 2> gpurun_out/final1/dit_n1.err
tail -2 gpurun_out/final1/pytest_gpu.log
