#!/bin/bash
# Interleaved same-session bench A/B of environment settings.
#   tools/env_ab.sh "OXY_X=0 OXY_X=1" [rounds] [streams...]   ("-" = no setting)
settings=$1
rounds=${2:-2}
shift 2 2>/dev/null
streams=${*:-1}
for r in $(seq "$rounds"); do
  for s_ in $settings; do
    for s in $streams; do
      if [ "$s_" = "-" ]; then envs=(); else envs=("$s_"); fi
      env "${envs[@]}" python bench.py --streams "$s" --steps 20 --warmup 8 --no-cpu-baseline --no-extras 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$s_ streams=$s', round(d['frame_ms'],3), d['stage_ms'])"
    done
  done
done
