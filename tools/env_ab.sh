#!/bin/bash
# Interleaved frame A/B of environment knobs.
#   tools/env_ab.sh rounds "K=V,K=V" "-" ...   ("-" = defaults)
rounds=$1; shift
for r in $(seq "$rounds"); do
  for spec in "$@"; do
    if [ "$spec" = "-" ]; then e=""; else e=$(echo "$spec" | tr ',' ' '); fi
    env $e python bench.py --steps 20 --warmup 8 --no-cpu-baseline --no-extras 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$spec', round(d['frame_ms'],3), d['stage_ms'])"
  done
done
