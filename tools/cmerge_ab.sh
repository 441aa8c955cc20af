#!/bin/bash
# Same-session A/B: in-kernel cluster merge of attention splits (OXY_ATTN_CMERGE=16)
# vs workspace + fa_merge (0), crossed with decode-lane SM caps (OXY_LANE_SMS).
#   tools/cmerge_ab.sh [rounds]
rounds=${1:-2}
for r in $(seq "$rounds"); do
  for cm in 16 0 8; do
    for lane in 0,0 0,74; do
      for s in 1 8; do
        OXY_ATTN_CMERGE=$cm OXY_LANE_SMS=$lane python bench.py --streams $s --steps 20 --warmup 8 --no-cpu-baseline --no-extras 2>/dev/null |
          python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('cmerge=$cm lane=$lane streams=$s', round(d['frame_ms'],3), d['stage_ms'])"
      done
    done
  done
done
