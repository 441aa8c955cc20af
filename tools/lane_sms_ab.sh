#!/bin/bash
# Same-session A/B of OXY_LANE_SMS=dn,dec (per-lane SM caps of the split
# policies) on the 1-stream headline and the 8-stream frame.
#   tools/lane_sms_ab.sh "0,0 100,48 ..." [rounds]
vals=${1:-"0,0 120,0 100,0 0,100 0,74 100,48 74,74"}
rounds=${2:-2}
for r in $(seq "$rounds"); do
  for v in $vals; do
    for s in 1 8; do
      OXY_LANE_SMS=$v python bench.py --streams $s --steps 20 --warmup 8 --no-cpu-baseline --no-extras 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', 'streams=$s', round(d['frame_ms'],3), d['stage_ms'], d.get('stage_serial',{}).get('stage_ms'))"
    done
  done
done
