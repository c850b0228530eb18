# Final-build ncu: full captures (details + SASS source CSV) of the cfg2 kernels, and the launch
# list of the default bench command.
set -x
bash tools/ncu_export.sh f_bwd_dyn 'adaln_bwd_tma' 2 -- python tools/prof_r2.py
bash tools/ncu_export.sh f_bwd_det 'adaln_bwd_tma' 3 -- python tools/prof_r2.py
bash tools/ncu_export.sh f_fwd 'adaln_fwd_rows16' 2 -- python tools/prof_r2.py
bash tools/ncu_export.sh f_red 'adaln_bwd_reduce' 2 -- python tools/prof_r2.py
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f_bench_plain.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f_ncu_bench.log 2>&1
ls -la gpurun_out/
