#!/bin/bash
# Capture one kernel with `ncu --set full` and keep only CSV exports (details + SASS source page)
# so the results fit gpurun's copy-back limit.
#   tools/ncu_export.sh <name> <kernel-regex> <skip> -- <command...>
set -uo pipefail
name=$1; kre=$2; skip=$3; shift 4
out=gpurun_out/$name
ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c 1 -o "$out" "$@" > "$out.log" 2>&1
ncu -i "$out.ncu-rep" --page details --csv > "${out}_details.csv" 2>/dev/null
ncu -i "$out.ncu-rep" --page source --csv --print-source sass > "${out}_sass.csv" 2>/dev/null
ncu -i "$out.ncu-rep" --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum > "${out}_raw.csv" 2>/dev/null
rm -f "$out.ncu-rep"
