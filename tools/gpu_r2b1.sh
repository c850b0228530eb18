python bench.py --steps 20 --warmup 5 > gpurun_out/r2b1_b20.json 2> gpurun_out/r2b1_b20.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2b1_b20b.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b1_ref.json 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2b1_ncu.log 2>&1
