#!/bin/bash
# One gpurun pass of round evidence: bench line, one-frame launch list, and
# `ncu --set full` captures of the roofline kernels (run from the repo root).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/frame_launches.csv python tools/profile_frame.py > gpurun_out/pf.log 2>&1
python tools/summarize_launches.py gpurun_out/frame_launches.csv > gpurun_out/frame_summary.txt
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 \
    -o gpurun_out/ncu_lm_head python tools/kernel_probe.py gemm 257152 2048 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_(wide_)?kernel" -s 2 -c 1 \
    -o gpurun_out/ncu_prefill_gu python tools/kernel_probe.py gemm 32768 2048 800 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn_v3 -s 2 -c 1 \
    -o gpurun_out/ncu_decode_attn python tools/kernel_probe.py decode_attention 64 1024 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:flash_tc -s 17 -c 1 \
    -o gpurun_out/ncu_flash_tc python tools/prefill_only.py > /dev/null 2>&1
ls -la gpurun_out
