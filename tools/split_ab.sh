#!/bin/bash
# Interleaved A/B of per-shape chain split counts (OXY_SPLITS="n,k,s;...").
#   tools/split_ab.sh rounds "spec1" "spec2" ...   ("-" = policy defaults)
rounds=$1; shift
for r in $(seq "$rounds"); do
  for spec in "$@"; do
    if [ "$spec" = "-" ]; then e=""; else e="OXY_SPLITS=$spec"; fi
    env $e python bench.py --steps 20 --warmup 8 --no-cpu-baseline --no-extras 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$spec', round(d['frame_ms'],3), d['stage_ms'])"
  done
done
