# A/B: tools/gpu_ab.sh <out-prefix> <variant names...> ("tree" = the in-tree build); two rounds
out=$1; shift
for r in 1 2; do for v in "$@"; do
  if [ "$v" = tree ]; then python tools/ab_time.py 50 tree >> gpurun_out/$out.jsonl 2>&1
  else AL_LIB_VARIANT=$v python tools/ab_time.py 50 $v >> gpurun_out/$out.jsonl 2>&1; fi
done; done
