"""The tcgen05 flash attention (csrc/attn_tc.cu) under every key-split regime:
one split per tile .. one split for all tiles, with paged + dense key tiles in
one CTA and O rescales, re-running the oracle parity tests of
tests/test_pi05_gpu.py in a fresh process per setting (the split knob is read
at model creation).  A timeout turns a pipeline deadlock into a failure."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("splits", ["1", "3", "7", "64"])
def test_attention_splits_match_oracle(splits):
    env = dict(os.environ, OXY_ATTN_TC="1", OXY_ATTN_TC_SPLITS=splits)
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", os.path.join(ROOT, "tests", "test_pi05_gpu.py"),
           "-k", "prefill_kv or action_denoise or decode_logits or batch_invariant or graph_replay"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=240)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]


def test_tc_attention_agrees_with_mma_sync_path():
    """Full-shape prefill + denoise: tcgen05 attention vs the mma.sync kernel."""
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images\n"
        "be = Pi05Backend(Pi05Config(), num_blocks=64)\n"
        "kv = be.prefill(Pi05Observation(tuple(range(100, 132)), 0, synthetic_images(3, 5)))\n"
        "a = be.action_denoise(kv, 10).actions\n"
        "np.save(sys.argv[1], np.concatenate([a.ravel(), kv.layers[17].keys[::97].ravel()]))\n") % ROOT
    outs = []
    for tc in ("1", "0"):
        path = os.path.join("/tmp", f"attn_tc_{tc}_{os.getpid()}.npy")
        env = dict(os.environ, OXY_ATTN_TC=tc)
        res = subprocess.run([sys.executable, "-c", code, path], cwd=ROOT, env=env, capture_output=True, text=True,
                             timeout=300)
        assert res.returncode == 0, res.stderr[-3000:]
        import numpy as np
        outs.append(np.load(path))
        os.remove(path)
    import numpy as np
    rel = np.abs(outs[0] - outs[1]).max() / (np.abs(outs[1]).max() + 1e-9)
    assert rel < 3e-2, rel
