for m in 6 7; do AL_PDL_MASK=$m python tools/bench_modes.py 20 5 >> gpurun_out/r2l_modes.jsonl 2>&1; done
for m in 6 7; do AL_PDL_MASK=$m python tools/bench_modes.py 200 10 >> gpurun_out/r2l_modes.jsonl 2>&1; done
