"""Marginal in-graph cost of each kernel group of the language-decode chain
(6 rows x 5 steps over ~800-position prefixes): decode time with OXY_DBG_SKIP
bits set (results invalid; timing only), one process per mask."""
import os, subprocess, sys
code = r'''
import os, sys, torch; sys.path.insert(0, ".")
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images
from paper_2603_14371_b200.kv_manager import BatchedState
be = Pi05Backend(Pi05Config(), num_blocks=256)
kvs = [be.prefill(Pi05Observation(tuple(range(100 + i, 132 + i)), 0, synthetic_images(3, 5 + i))) for i in range(6)]
st = BatchedState(tuple(kvs), ((),) * 6, (False,) * 6, tuple(range(6)), (1000,) * 6, (0,) * 6)
for _ in range(3): be.batched_language_decode(st, 5)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): be.batched_language_decode(st, 5)
e.record(); torch.cuda.synchronize()
print(s.elapsed_time(e) / 10)
'''
names = {0: "full", 256: "-qkv", 512: "-attention", 2048: "-o-proj+norm", 4096: "-gate/up", 8192: "-down+norm",
         16384: "-lm head", 256 + 512 + 2048 + 4096 + 8192 + 16384: "glue only"}
base = None
for m, n in names.items():
    res = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, OXY_DBG_SKIP=str(m)),
                         capture_output=True, text=True, timeout=300)
    out = res.stdout.strip().splitlines()
    if not out:
        print(n, "failed:", res.stderr.strip().splitlines()[-1:], flush=True)
        continue
    ms = float(out[-1])
    base = ms if base is None else base
    print(f"{n:14s} {ms:7.3f} ms  saves {base - ms:6.3f} ms  ({(base - ms) / 90 * 1e3:5.1f} us per layer-step)", flush=True)
