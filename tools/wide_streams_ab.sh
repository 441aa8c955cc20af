for w in 0 -1 2; do echo "== WIDE=$w"; OXY_GEMM_WIDE=$w timeout 300 python - <<'PY'
import sys, os; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import config_sweep as cs
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config
cfg = Pi05Config()
for r in (8, 32):
    be = Pi05Backend(cfg, num_blocks=256 + r * 8 * 14)
    cs.point("streams", be, cfg, r, 30, 5, 3, 6)
    del be
PY
done
