# HEAD confirmation: smoke, bench (driver K/W) x2, reference arm, DiT N=1.
set -x
mkdir -p gpurun_out/final3
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final3/smoke.log 2>&1; echo smoke=$?
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final3/ref.json 2> gpurun_out/final3/ref.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final3/bench.json 2> gpurun_out/final3/bench.err
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final3/bench_b.json 2> /dev/null
python bench.py --gpus 1 --workload dit --steps 16 --warmup 2 > gpurun_out/final3/dit_n1.json 2> gpurun_out/final3/dit_n1.err
