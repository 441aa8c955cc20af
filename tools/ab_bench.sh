#!/bin/bash
# Interleaved same-session bench A/B of library variants (OXY_LIB_VARIANT; "" = the working build).
#   tools/ab_bench.sh "head ''" [rounds] [streams...]
variants=${1:-"head ''"}
rounds=${2:-2}
shift 2 2>/dev/null
streams=${*:-1}
for r in $(seq "$rounds"); do
  for v in $variants; do
    v=${v//\'/}
    for s in $streams; do
      OXY_LIB_VARIANT=$v python bench.py --streams "$s" --steps 20 --warmup 8 --no-cpu-baseline --no-extras 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('variant=${v:-work} streams=$s', round(d['frame_ms'],3), d['stage_ms'])"
    done
  done
done
