#!/bin/bash
# ncu --set full (with source counters) of one skinny GEMM launch inside the
# denoise chain (tools/gemm_prof.py workload, default lib).  Cold/serialised.
#   tools/ncu_gemm_denoise.sh <launch-skip> <out-name>
skip=${1:-1500}; name=${2:-gemm_denoise}
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel --launch-skip "$skip" --launch-count 1 \
    -o "gpurun_out/$name" -f python - <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images
be = Pi05Backend(Pi05Config(), num_blocks=64)
kv = be.prefill(Pi05Observation(tuple(range(100, 132)), 0, synthetic_images(3, 5)))
for _ in range(2):
    be.denoise_many([kv], 10)
PY
