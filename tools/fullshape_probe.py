"""Measure F2 errors against the CPU oracle at the BASELINE configs[1] shape
(3 x 224^2 cameras + 32 prompt tokens, P = 800, H = 50, S = 10), and whether
batched admission is bit-identical to solo.  Prints one JSON line; the
tolerances in tests/test_pi05_full_gpu.py are set from its output."""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.pi05_ref import Pi05Ref  # noqa: E402
from paper_2603_14371_b200 import BatchedState  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-9))


def main():
    torch.set_num_threads(max(1, len(os.sched_getaffinity(0))))
    out = {}
    be = Pi05Backend(Pi05Config(), num_blocks=512)
    t0 = time.time()
    ref = Pi05Ref.from_backend(be)
    out["oracle_load_s"] = round(time.time() - t0, 1)
    obs = Pi05Observation(tuple(range(1000, 1032)), 0, synthetic_images(3, 1))
    kv = be.prefill(obs)
    t0 = time.time()
    want = ref.prefill(obs)
    out["oracle_prefill_s"] = round(time.time() - t0, 1)
    ek, ev = [], []
    for l in range(be.config.depth):
        k, v = be.read_kv(kv, l)
        ek.append(rel(k, want[l][0].numpy()))
        ev.append(rel(v, want[l][1].numpy()))
    out["kv_rel_k"] = [round(e, 6) for e in ek]
    out["kv_rel_v"] = [round(e, 6) for e in ev]
    act = be.action_denoise(kv, 10).actions
    t0 = time.time()
    ract = ref.denoise(want, 10)
    out["oracle_denoise_s"] = round(time.time() - t0, 1)
    out["action_rel"] = rel(act, ract)
    # actions from the oracle's own prefix vs from the device KV (isolates denoise error)
    dev_kvs = [tuple(torch.tensor(x, dtype=torch.float32) for x in be.read_kv(kv, l))
               for l in range(be.config.depth)]
    out["action_rel_devkv"] = rel(act, ref.denoise(dev_kvs, 10))
    res, logits = be.batched_language_decode(
        BatchedState((kv,), ((),), (False,), (0,), (5,), (0,)), 5, return_logits=True)
    toks, _, wl = ref.decode(dev_kvs, (), 5)
    cos, mx, margin = [], [], []
    for s in range(min(len(wl), logits.shape[0])):
        a, b = logits[s, 0].astype(np.float64), wl[s].astype(np.float64)
        cos.append(float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b))))
        mx.append(float(np.max(np.abs(a - b))))
        t2 = np.sort(b)[-2:]
        margin.append(float(t2[1] - t2[0]))
    out.update(logit_cos=cos, logit_maxabs=mx, top2_margin=margin, tokens=list(res.token_buffers[0]),
               oracle_tokens=list(toks))
    # batched admission vs solo (bit equality)
    obs2 = [Pi05Observation(tuple(range(1000 + i, 1032 + i)), 0, synthetic_images(3, 1 + i)) for i in range(2)]
    solo = [be.prefill(o) for o in obs2]
    both = be.prefill_many(obs2)
    out["prefill_r2_bitexact"] = [bool(a == b) for a, b in zip(solo, both)]
    a_solo = [be.action_denoise(k, 10).actions for k in solo]
    a_both = [c.actions for c in be.denoise_many(solo, 10)]
    out["denoise_r2_bitexact"] = [bool(np.array_equal(x, y)) for x, y in zip(a_solo, a_both)]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
