#!/bin/bash
# round-2 multi-sample profiling: ncu launch lists of the sampler's buckets and full captures of
# the work-stealing backward, the many-group stage 2 and the chunked-tail forward at 307 x 1560
mkdir -p gpurun_out/r2p
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in 307x1560 133x3600 49x7800 15x14040; do
  set -- ${cfg/x/ }
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2p/launches_${cfg}.csv \
    python tools/prof_step.py --batch $1 --seq $2 --reps 2 > gpurun_out/r2p/launches_${cfg}.log 2>&1
done
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2p/launches_cfg2_det.csv \
  python tools/prof_step.py --reps 2 --det > gpurun_out/r2p/launches_cfg2_det.log 2>&1
bash tools/ncu_export.sh r2p/full_steal adaln_bwd_steal 1 -- python tools/prof_step.py --batch 307 --seq 1560 --reps 2
bash tools/ncu_export.sh r2p/full_reduce_grp adaln_bwd_reduce_grp 1 -- python tools/prof_step.py --batch 307 --seq 1560 --reps 2
bash tools/ncu_export.sh r2p/full_fwd_chunk adaln_fwd_rows16 1 -- python tools/prof_step.py --batch 307 --seq 1560 --reps 2
bash tools/ncu_export.sh r2p/full_bwd_det_lean adaln_bwd_tma 1 -- python tools/prof_step.py --reps 2 --det
ls -la gpurun_out/r2p
