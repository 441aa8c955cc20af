for shape in "3456 1152 768" "4304 1152 768" "1152 4304 768" "1152 1152 768" "2560 2048 800" "2048 2048 800"; do
  echo "== $shape default"; python tools/vit_gemm_probe.py $shape 2>&1 | tail -2
  for bn in 64 96 128 192 256; do
    echo "-- wide=2 bn=$bn"; OXY_GEMM_WIDE=2 OXY_GEMM_WIDE_BN=$bn OXY_GEMM_WIDE_SPLITS=1 python tools/vit_gemm_probe.py $shape 2>&1 | tail -2
  done
  echo "-- wide=2 auto"; OXY_GEMM_WIDE=2 python tools/vit_gemm_probe.py $shape 2>&1 | tail -2
  echo "-- smem200"; OXY_GEMM_SMEM_KB=200 python tools/vit_gemm_probe.py $shape 2>&1 | tail -2
done
