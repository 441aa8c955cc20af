"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``kvweaver`` read-only from /root/reference/pkg/src and writes
small JSON fixtures next to this file.  The fixtures travel with the repo;
nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import kvweaver as kw  # noqa: E402
from kvweaver.rng import SplitMix64  # noqa: E402


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=None, separators=(",", ":"))
    print("wrote", name)


def rng_fixture():
    out = {}
    r = SplitMix64(0)
    out["seed0_u64"] = [str(r.next_u64()) for _ in range(5)]
    r = SplitMix64(0xDEADBEEF)
    out["deadbeef_u64"] = [str(r.next_u64()) for _ in range(3)]
    r = SplitMix64(7)
    out["seed7_u64"] = [str(r.next_u64()) for _ in range(64)]
    r = SplitMix64(7)
    out["seed7_uniform"] = [r.uniform() for _ in range(64)]
    r = SplitMix64(9)
    out["seed9_below10"] = [r.below(10) for _ in range(50)]
    r = SplitMix64(11)
    out["seed11_poisson2.5"] = [r.poisson(2.5) for _ in range(50)]
    dump("rng.json", out)


def workload_fixture():
    specs = [
        dict(pattern="OnePerFrame", default_N=5, obs_len=6, num_frames=5, seed=3),
        dict(pattern="Uniform", r=3, default_N=4, obs_len=4, num_frames=4, seed=4),
        dict(pattern="Poisson", lam=1.3, default_N=7, obs_len=3, num_frames=12, seed=5),
        dict(pattern="MixedLength", short_N=3, long_N=9, p_long=0.4, obs_len=5, num_frames=8,
             seed=17),
        dict(pattern="OnePerFrame", default_N=16, obs_len=800, num_frames=2, seed=1),
    ]
    out = []
    for s in specs:
        vocab = 1024 if s["obs_len"] == 800 else 24
        arr = kw.generate_arrivals(kw.WorkloadSpec(**s), vocab)
        out.append(dict(spec=s, vocab=vocab,
                        arrivals=[[a.frame, a.n_tokens, list(a.observation.obs_tokens)]
                                  for a in arr]))
    dump("workload.json", out)


def _solo(backend, obs, max_len, k, tokens=(), kv=None):
    kv = kv or backend.prefill(kw.Observation(obs_tokens=tuple(obs), frame=0))
    b = kw.BatchedState(kv_batch=(kv,), token_buffers=(tuple(tokens),), flags=(False,),
                        request_ids=(0,), max_lens=(max_len,), created_frames=(0,))
    return backend.batched_language_decode(b, k)


def toy_fixture():
    out = {}
    # A1: default config
    b = kw.ToyBackend(kw.BackendConfig())
    obs = (11, 22, 33, 44)
    kv = b.prefill(kw.Observation(obs_tokens=obs, frame=0))
    res = _solo(b, obs, 10, 10, kv=kv)
    act = b.action_denoise(kv, 10).actions
    out["A1"] = dict(
        config=dict(), obs=list(obs), max_len=10, k=10,
        tokens=list(res.token_buffers[0]), flag=res.flags[0],
        action=act.tolist(),
        prefill_kv=[[l.keys.tolist(), l.values.tolist()] for l in kv.layers],
        final_kv=[[l.keys.tolist(), l.values.tolist()] for l in res.kv_batch[0].layers],
        recompute_logits=b.recompute_logits(list(obs) + [0]).tolist(),
        weights_head=dict(embed00=b._embed[0, :4].tolist(),
                          unembed_last=b._unembed[-1, -4:].tolist(),
                          action_head_last=b._action_head[-1, -4:].tolist()),
    )
    # A2: EOS termination KAT (tests/test_backend_toy.py:144-152)
    b = kw.ToyBackend(kw.BackendConfig(vocab=4, seed=5))
    res = _solo(b, (1,), 20, 20)
    out["A2"] = dict(config=dict(vocab=4, seed=5), obs=[1], max_len=20, k=20,
                     tokens=list(res.token_buffers[0]), flag=res.flags[0])
    # mixed termination pair (tests/test_backend_toy.py:232-249)
    res2 = _solo(b, (3, 2), 20, 20)
    out["A2b"] = dict(config=dict(vocab=4, seed=5), obs=[3, 2], max_len=20, k=20,
                      tokens=list(res2.token_buffers[0]), flag=res2.flags[0])
    # split-decode KAT (tests/test_backend_toy.py:219-230)
    b = kw.ToyBackend(kw.BackendConfig())
    res = _solo(b, (3, 1, 4, 1, 5), 12, 12)
    out["split"] = dict(config=dict(), obs=[3, 1, 4, 1, 5], max_len=12, k=12,
                        tokens=list(res.token_buffers[0]), flag=res.flags[0])
    # A3 / A4: C1 shapes, obs from WorkloadSpec(seed=1, obs_len=800)
    arr = kw.generate_arrivals(kw.WorkloadSpec(default_N=16, obs_len=800, num_frames=1, seed=1), 1024)
    obs800 = arr[0].observation.obs_tokens
    for name, nh in (("A3", 1), ("A4", 4)):
        cfg = dict(L=2, d_model=256, n_heads=nh, vocab=1024, eos_token=0, action_dim=32, H=50,
                   S=10, seed=7)
        b = kw.ToyBackend(kw.BackendConfig(**cfg))
        kv = b.prefill(kw.Observation(obs_tokens=obs800, frame=0))
        res = _solo(b, obs800, 16, 16, kv=kv)
        act = b.action_denoise(kv, 10).actions
        logits = b.recompute_logits(list(obs800) + [0])
        top2 = np.sort(logits)[-2:]
        out[name] = dict(config=cfg, obs=list(obs800), max_len=16, k=16,
                         tokens=list(res.token_buffers[0]), flag=res.flags[0],
                         action=act.tolist(), action_sum=float(act.sum()),
                         first_logits=logits.tolist(), first_margin=float(top2[1] - top2[0]),
                         kv_row0=[kv.layers[l].keys[0, :8].tolist() for l in range(2)],
                         kv_last_v_mean=kv.layers[-1].values.mean(axis=0).tolist())
    dump("toy_kat.json", out)


def sim_fixture():
    out = {}
    toy_cfg = dict(
        backend_config=dict(vocab=24, seed=6),
        workload=dict(pattern="MixedLength", obs_len=6, num_frames=10, short_N=3, long_N=9,
                      p_long=0.4, seed=17),
        k=3)
    for variant in ("Unified", "SharedNoBatch", "IsolatedSequential"):
        cfg = kw.SimConfig(variant=variant, backend_kind="Toy",
                           backend_config=kw.BackendConfig(**toy_cfg["backend_config"]),
                           workload=kw.WorkloadSpec(**toy_cfg["workload"]), k=toy_cfg["k"])
        res = kw.run_simulation(cfg)
        out[f"toy_{variant}"] = dict(
            config=toy_cfg, transcript=kw.transcript_to_json(res),
            traces=[[t.frame, t.prefill_count, t.batch_size_m, t.tokens_emitted,
                     t.actions_emitted, list(t.completed_ids), t.arrival_count] for t in res.traces])
    cost = []
    for variant in ("Unified", "SharedNoBatch", "IsolatedSequential", "IsolatedParallel"):
        for pattern, extra in (("OnePerFrame", {}), ("Poisson", dict(lam=0.9, seed=8))):
            wl = dict(pattern=pattern, default_N=12, obs_len=800, num_frames=30, **extra)
            cfg = kw.SimConfig(variant=variant, backend_kind="CostModel",
                               cost_params=kw.CostModelParams(),
                               workload=kw.WorkloadSpec(**wl), k=4)
            res = kw.run_simulation(cfg)
            rep = kw.summarize(res, cfg)
            rep_full = kw.summarize(res, cfg, include_warmup=True)
            cost.append(dict(variant=variant, workload=wl, k=4,
                             traces=[[t.frame, list(t.latency_components), t.batch_size_m,
                                      t.tokens_emitted, t.actions_emitted,
                                      list(t.completed_ids), t.deadline_met, t.total_us,
                                      t.arrival_count] for t in res.traces],
                             summary=[getattr(rep, f) for f in rep.__slots__],
                             summary_full=[getattr(rep_full, f) for f in rep_full.__slots__]))
    out["cost"] = cost
    dump("sim.json", out)


if __name__ == "__main__":
    rng_fixture()
    workload_fixture()
    toy_fixture()
    sim_fixture()
