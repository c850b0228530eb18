nvidia-smi --query-gpu=index,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory --format=csv -lms 100 > gpurun_out/r2b_smi.csv &
SMI=$!
python tools/step_trend.py 400 0.3 > gpurun_out/r2b_trend.jsonl 2>&1
python tools/step_trend.py 400 0.0 >> gpurun_out/r2b_trend.jsonl 2>&1
kill $SMI
