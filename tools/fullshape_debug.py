"""Debug probe (full shape): per-row decode logits vs the oracle, and the first
layer where a batched prefill's KV departs from the solo prefill."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.pi05_ref import Pi05Ref  # noqa: E402
from paper_2603_14371_b200 import BatchedState  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images  # noqa: E402


def obs(n_img, n_txt, seed):
    toks = tuple(1000 + (seed * 7919 + i * 104729) % 250000 for i in range(n_txt))
    return Pi05Observation(toks, 0, synthetic_images(n_img, seed) if n_img else None)


def main():
    torch.set_num_threads(16)
    be = Pi05Backend(Pi05Config(), num_blocks=2048)
    out = {}
    if "prefill" in sys.argv:
        ol = [obs(3, 32, 10 + i) for i in range(3)]
        solo = [be.prefill(o) for o in ol]
        both = be.prefill_many(ol)
        first = []
        for i in range(3):
            fl = None
            for l in range(be.config.depth):
                a, b = be.read_kv(solo[i], l), be.read_kv(both[i], l)
                if not (np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])):
                    d = np.abs(a[0] - b[0])
                    fl = (l, float(d.max()), int((d > 0).sum()), [int(x) for x in np.argwhere(d > 0)[:4, 0]])
                    break
            first.append(fl)
        out["prefill_r3_first_diff"] = first
    if "decode" in sys.argv:
        ref = Pi05Ref.from_backend(be)
        specs = [(3, 32, 3), (3, 32, 4), (2, 20, 5), (1, 40, 6), (0, 48, 7), (3, 8, 8)]
        rows, hist = [], []
        for i, (ni, nt, sd) in enumerate(specs):
            kv = be.prefill(obs(ni, nt, sd))
            toks = ()
            if i % 2:
                h = be.batched_language_decode(BatchedState((kv,), ((),), (False,), (0,), (40,), (0,)), 3)
                kv, toks = h.kv_batch[0], h.token_buffers[0]
            rows.append(kv)
            hist.append(toks)
        m = len(rows)
        res, logits = be.batched_language_decode(
            BatchedState(tuple(rows), tuple(hist), (False,) * m, tuple(range(m)), (40,) * m, (0,) * m), 5,
            return_logits=True)
        rep = []
        for r in range(m):
            dk = [tuple(torch.tensor(x, dtype=torch.float32) for x in be.read_kv(rows[r], l))
                  for l in range(be.config.depth)]
            wt, _, wl = ref.decode(dk, hist[r], 5, max_len=40)
            got = res.token_buffers[r][len(hist[r]):]
            cs = []
            for s in range(min(len(wl), len(got))):
                a, b = logits[s, r].astype(np.float64), wl[s].astype(np.float64)
                cs.append(round(float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b))), 6))
            solo, sl = be.batched_language_decode(
                BatchedState((rows[r],), (hist[r],), (False,), (0,), (40,), (0,)), 5, return_logits=True)
            rep.append(dict(row=r, seq=rows[r].seq_len, hist=list(hist[r]), got=list(got), want=list(wt), cos=cs,
                            solo_tokens=list(solo.token_buffers[0][len(hist[r]):]),
                            solo_eq=bool(np.array_equal(sl[:, 0], logits[:, r]))))
        out["decode"] = rep
    print(json.dumps(out))


if __name__ == "__main__":
    main()
