#!/bin/bash
# Ring forward (variant 7) against the rows kernels over D, long and short sequences.
for dt in bf16 fp32; do
for D in 2048 3072 4096 5120 6144 8192 12288; do
  for shp in "1 32760" "4 1560"; do
    set -- $shp
    python tools/sweep.py --which fwd --dtype $dt --batch $1 --seq $2 --dim $D --variants 0,1,4 --no-ring \
      --ring7-cfgs 0:0:0,4:2:100,4:1:100,2:2:0,4:4:100 \
      | python3 -c "
import json,sys
r={}
for l in sys.stdin:
    d=json.loads(l); c=d['cfg']
    key=str(c.get('variant')) if 'V' not in c else 'r%d.%d.%d'%(c['V'],c['R'],c['smem']//1024)
    r[key]=d.get('gbs') or d.get('error','')[:40]
print(json.dumps({'dtype':'$dt','D': $D, 'B': $1, 'S': $2, 'gbs': r}))"
  done
done
done
