"""Backend value objects, the latency-only cost backend, and the factory.

The backend protocol is the reference's (``kvweaver/backend.py:163-201``,
SURVEY.md §8b): ``prefill(obs) -> cache``, ``action_denoise(cache, S) ->
ActionChunk``, ``batched_language_decode(batched, k) -> BatchedState`` plus
integer-microsecond pricing.  Value objects (``Observation``, ``BackendConfig``,
``ActionChunk``, ``CostModelParams``) carry the reference's fields, defaults and
validation messages so configs and tests move over unchanged.

Backend kinds (``make_backend``):
  "Toy"        the reference toy transformer (F1) computed on the B200 by the
               CUDA extension in fp32 verification mode (``toy_b200.ToyBackend``)
  "CostModel"  latency-only model, no math (``kvweaver/backend.py:427-487``)
  "Pi05"       the pi0.5-shaped VLA (F2) in bf16 on tcgen05 (``pi05.Pi05Backend``)
There is no CPU compute path: the GPU kinds raise if the extension or the GPU
is missing.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .kv_manager import BatchedState, KvCache

__all__ = [
    "Observation", "BackendConfig", "ActionChunk", "CostModelParams",
    "PricedBackend", "CostModelBackend", "make_backend", "BACKEND_KINDS",
]

BACKEND_KINDS = ("Toy", "CostModel", "Pi05")


@dataclass(frozen=True, slots=True)
class Observation:
    """One frame's input.  ``obs_tokens`` stand in for the prefix token ids
    (``kvweaver/backend.py:56-66``); pi0.5 backends additionally accept
    ``images`` (uint8 [n_cams, 224, 224, 3]) through ``Pi05Observation``."""

    obs_tokens: tuple[int, ...]
    frame: int

    def __post_init__(self):
        object.__setattr__(self, "obs_tokens", tuple(self.obs_tokens))
        if len(self.obs_tokens) < 1:
            raise ValueError("observation needs at least one token")


@dataclass(frozen=True, slots=True)
class BackendConfig:
    """Toy model shape (``kvweaver/backend.py:69-97``)."""

    L: int = 2
    d_model: int = 32
    n_heads: int = 2
    vocab: int = 64
    eos_token: int = 0
    action_dim: int = 4
    H: int = 10
    S: int = 10
    seed: int = 7

    def __post_init__(self):
        if self.L < 1:
            raise ValueError("need at least one layer")
        if self.d_model % self.n_heads != 0:
            raise ValueError(f"d_model {self.d_model} not divisible by n_heads {self.n_heads}")
        if self.d_model % 2 != 0:
            raise ValueError("d_model must be even for sinusoidal positions")
        if self.vocab < 2:
            raise ValueError("vocab must hold at least two tokens")
        if not 0 <= self.eos_token < self.vocab:
            raise ValueError(f"eos_token {self.eos_token} outside vocab of {self.vocab}")
        if self.action_dim < 1 or self.H < 1 or self.S < 1:
            raise ValueError("action_dim, H and S must be positive")


@dataclass(frozen=True, slots=True, eq=False)
class ActionChunk:
    """[H, action_dim] float64, read-only; equality is exact."""

    actions: np.ndarray

    def __post_init__(self):
        a = np.ascontiguousarray(self.actions, dtype=np.float64)
        a.flags.writeable = False
        object.__setattr__(self, "actions", a)
        if a.ndim != 2:
            raise ValueError(f"action chunk must be 2-d, got shape {a.shape}")
        if not np.all(np.isfinite(a)):
            raise ValueError("action chunk contains non-finite values")

    @property
    def horizon(self) -> int:
        return self.actions.shape[0]

    def __eq__(self, other):
        if not isinstance(other, ActionChunk):
            return NotImplemented
        return bool(np.array_equal(self.actions, other.actions))


@dataclass(frozen=True, slots=True)
class CostModelParams:
    """Integer-us latency knobs (``kvweaver/backend.py:125-160``)."""

    c_prefill_per_token: int = 25
    c_denoise_per_step: int = 3000
    c_decode_base: int = 5900
    c_decode_per_request: int = 100
    c_contention: float = 1.6

    def __post_init__(self):
        for name in ("c_prefill_per_token", "c_denoise_per_step",
                     "c_decode_base", "c_decode_per_request"):
            v = getattr(self, name)
            if not isinstance(v, int) or v < 0:
                raise ValueError(f"{name} must be a nonnegative integer, got {v!r}")
        if self.c_contention < 1.0:
            raise ValueError(f"c_contention must be >= 1, got {self.c_contention}")

    @classmethod
    def zero(cls) -> "CostModelParams":
        return cls(0, 0, 0, 0, 1.0)


class PricedBackend:
    """Latency pricing and argument validation shared by every backend
    (``kvweaver/backend.py:163-201``).  GPU backends additionally carry a
    ``meter`` (CUDA-event stage timer); the scheduler prefers measured
    microseconds when a meter is present."""

    config: BackendConfig
    cost: CostModelParams
    backend_tag: str
    kind: str
    meter = None

    def prefill_latency_us(self, p_len: int) -> int:
        return self.cost.c_prefill_per_token * p_len

    def denoise_latency_us(self, steps: int) -> int:
        return steps * self.cost.c_denoise_per_step

    def decode_latency_us(self, steps: int, m: int) -> int:
        return steps * (self.cost.c_decode_base + self.cost.c_decode_per_request * m)

    def _check_tag(self, kv) -> None:
        if kv.backend_tag != self.backend_tag:
            raise ValueError(f"cache from backend {kv.backend_tag!r} fed to {self.backend_tag!r}")

    def _check_obs(self, obs: Observation) -> None:
        v = self.config.vocab
        for t in obs.obs_tokens:
            if not 0 <= t < v:
                raise ValueError(f"observation token {t} outside vocab of {v}")

    def _check_batch(self, batched: BatchedState, k: int) -> None:
        if k < 1:
            raise ValueError(f"decode step count must be >= 1, got {k}")
        for i in range(batched.size):
            self._check_tag(batched.kv_batch[i])
            if batched.flags[i]:
                raise ValueError(f"request {batched.request_ids[i]} is terminated, cannot decode it")


class CostModelBackend(PricedBackend):
    """Latency-only backend: caches are position counts, tokens a counter that
    skips EOS (``kvweaver/backend.py:427-487``)."""

    def __init__(self, config: BackendConfig | None = None, cost: CostModelParams | None = None):
        self.config = config or BackendConfig()
        self.cost = cost or CostModelParams()
        self.backend_tag = f"cost/L{self.config.L}-v{self.config.vocab}"
        self.kind = "CostModel"

    def _synth(self, n: int) -> int:
        v, eos = self.config.vocab, self.config.eos_token
        t = n % v
        return (t + 1) % v if t == eos else t

    def prefill(self, obs: Observation) -> KvCache:
        self._check_obs(obs)
        p = len(obs.obs_tokens)
        return KvCache((p,) * self.config.L, p, self.backend_tag)

    def action_denoise(self, kv, S: int) -> ActionChunk:
        self._check_tag(kv)
        if S < 1:
            raise ValueError(f"denoise step count must be >= 1, got {S}")
        return ActionChunk(np.zeros((self.config.H, self.config.action_dim)))

    def batched_language_decode(self, batched: BatchedState, k: int) -> BatchedState:
        self._check_batch(batched, k)
        caches, bufs, flags = [], [], []
        for kv, toks, budget in zip(batched.kv_batch, batched.token_buffers, batched.max_lens):
            buf = list(toks)
            take = min(k, budget - len(buf))
            n0 = len(buf)  # the reference draws token n from the count before the call
            buf.extend(self._synth(n0 + j) for j in range(take))
            seq = kv.seq_len + take
            caches.append(KvCache((seq,) * self.config.L, seq, self.backend_tag))
            bufs.append(tuple(buf))
            flags.append(len(buf) == budget)
        return BatchedState(tuple(caches), tuple(bufs), tuple(flags), batched.request_ids,
                            batched.max_lens, batched.created_frames)


def make_backend(kind: str, config: BackendConfig, cost: CostModelParams, **kw):
    """Factory (``kvweaver/backend.py:490-496``) extended with the GPU kinds."""
    if kind == "Toy":
        from .toy_b200 import ToyBackend
        return ToyBackend(config, cost, **kw)
    if kind == "CostModel":
        return CostModelBackend(config, cost)
    if kind == "Pi05":
        from .pi05 import Pi05Backend
        return Pi05Backend(config, cost, **kw)
    raise ValueError(f"unknown backend kind {kind!r} (use Toy, CostModel or Pi05)")
