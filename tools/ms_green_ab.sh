# 8-stream frames: overlapping partitions for multi-stream overlapped frames too (A/B)
for r in 1 2; do
for spec in "-" "OXY_GREEN_MAX_STREAMS=8"; do
  if [ "$spec" = "-" ]; then e=""; else e=$(echo "$spec" | tr ',' ' '); fi
  env $e python bench.py --streams 8 --steps 10 --warmup 4 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$spec', round(d['frame_ms'],3), d['stage_ms'])"
done; done
