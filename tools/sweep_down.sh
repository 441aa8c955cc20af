for bn in 96 128 160 208 256; do for sp in 1 2 3 4; do
  r=$(OXY_GEMM_WIDE=2 OXY_GEMM_WIDE_BN=$bn OXY_GEMM_WIDE_SPLITS=$sp timeout 60 python tools/gemm_big_probe.py 2>&1 | grep "down.*t=800 ours")
  echo "bn=$bn sp=$sp $r"
done; done
