# ncu of the final build: full captures (details + SASS source + DRAM bytes) of the cfg2 kernels
# and the launch list of the default bench command.
set -x
bash tools/ncu_export.sh g_bwd 'adaln_bwd_tma' 2 -- python tools/prof_r2.py
AL_BWD_TICKET=1 bash tools/ncu_export.sh g_bwd_ticket 'adaln_bwd_tma' 2 -- python tools/prof_r2.py
bash tools/ncu_export.sh g_fwd 'adaln_fwd_rows16' 2 -- python tools/prof_r2.py
bash tools/ncu_export.sh g_red 'adaln_bwd_reduce' 2 -- python tools/prof_r2.py
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g_ncu_bench.log 2>&1
ls -la gpurun_out/g_*
