#!/bin/bash
# One gpurun pass of round evidence: bench line, one-frame launch list, and
# `ncu --set full` captures of the roofline kernels (run from the repo root).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
OXY_GREEN=0 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/frame_launches.csv python tools/profile_frame.py > gpurun_out/pf.log 2>&1
python tools/summarize_launches.py gpurun_out/frame_launches.csv > gpurun_out/frame_summary.txt
full="ncu --set full --clock-control none --import-source on"
$full -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/ncu_lm_head python tools/kernel_probe.py gemm 257152 2048 6 > /dev/null 2>&1
$full -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/ncu_dn_down python tools/kernel_probe.py gemm 1024 4096 50 > /dev/null 2>&1
$full -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/ncu_dec_down python tools/kernel_probe.py gemm 2048 16384 6 > /dev/null 2>&1
$full -k regex:"gemm_(wide_)?kernel" -s 2 -c 1 -o gpurun_out/ncu_prefill_gu python tools/kernel_probe.py gemm 32768 2048 800 > /dev/null 2>&1
$full -k regex:decode_attn -s 2 -c 1 -o gpurun_out/ncu_decode_attn python tools/kernel_probe.py decode_attention 256 1024 > /dev/null 2>&1
$full -k regex:flash_tc -s 17 -c 1 -o gpurun_out/ncu_flash_tc python tools/prefill_only.py > /dev/null 2>&1
$full -k regex:vit_attn -s 27 -c 1 -o gpurun_out/ncu_vit_attn python tools/prefill_only.py > /dev/null 2>&1
ls -la gpurun_out
