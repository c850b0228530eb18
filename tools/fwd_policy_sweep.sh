#!/bin/bash
# Forward rows-kernel flavours (1 packed, 4 mixed 16-bit planar, 6 two rows per warp) over D at a
# long (1 x 32760) and a short (4 x 1560) sequence, bf16 -- the data behind the auto policy.
for D in 512 768 1024 1536 2048 2560 3072 4096 5120 6144; do
  for shp in "1 32760" "4 1560"; do
    set -- $shp
    python tools/sweep.py --which fwd --dtype bf16 --batch $1 --seq $2 --dim $D --variants 1,4,6 --no-ring \
      | python3 -c "
import json,sys
r={json.loads(l)['cfg']['variant']: json.loads(l).get('gbs') for l in sys.stdin}
print(json.dumps({'D': $D, 'B': $1, 'S': $2, 'gbs': r}))"
  done
done
