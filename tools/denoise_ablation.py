"""Marginal in-graph cost of each kernel group of the denoise chain: denoise
time with OXY_DBG_SKIP bits set (results invalid; timing only), one process per mask.
STREAMS=r: r lock-stepped streams (T = 50 r suffix tokens)."""
import os, subprocess, sys
code = r'''
import os, sys, torch; sys.path.insert(0, ".")
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images
R = int(os.environ.get("STREAMS", "1"))
be = Pi05Backend(Pi05Config(), num_blocks=64 + 16 * R)
kvs = [be.prefill(Pi05Observation(tuple(range(100 + i, 132 + i)), 0, synthetic_images(3, 5 + i))) for i in range(R)]
def dn():
    try:
        be.denoise_many(kvs, 10)
    except ValueError:  # skipped kernels leave garbage (non-finite) actions: timing only
        pass
for _ in range(3): dn()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): dn()
e.record(); torch.cuda.synchronize()
print(s.elapsed_time(e) / 10)
'''
names = {0: "full", 1 + 8 + 16 + 32: "attention only", 1 + 4 + 8 + 16 + 32: "flash_tc only", 1 + 2 + 8 + 16 + 32: "nothing but glue", 1: "-qkv", 2: "-attention", 4: "-attn merge", 8: "-o-proj+norm", 16: "-gate/up",
         32: "-down+norm", 128: "-both res-norms", 1 + 2: "-qkv -attention", 8 + 16 + 32: "-MLP & o-proj"}
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
    print(f"{n:18s} {ms:7.3f} ms  saves {base - ms:6.3f} ms  ({(base - ms) / 180 * 1e3:5.1f} us per layer-step)", flush=True)
