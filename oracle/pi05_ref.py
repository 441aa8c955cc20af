"""ORACLE — test infrastructure only; never imported by the product path.

torch-CPU fp32 restatement of the pi0.5-shaped model computed by
``paper_2603_14371_b200/csrc/pi05_model.cu``.  PARITY UNPINNED by the
reference: kvweaver has no pi0.5 model (SPEC.md:13 puts real pi0.5 out of
scope; its toy is a different architecture, kvweaver/backend.py:21-33).  The
algorithm restated here is the public openpi pi0.5 structure (SURVEY.md
Appendix B) with the reference's protocol conventions: EOS as the first decode
input at position P (kvweaver/backend.py:359-362), lowest-id greedy argmax
(kvweaver/backend.py:388), per-row stop on EOS / budget (backend.py:396-397),
denoise reads the shared cache without writing it (backend.py:316-332).

Rounding mirrors the kernels: GEMM inputs and stored K/V are bf16, GEMM
accumulation and the residual stream are fp32.  Weights come from the GPU
model itself (``from_backend``) so the check isolates the math; the weight
init is checked separately against the splitmix64 counter form.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from oracle.rng_ref import counter_uniform

HD = 256
NQH = 8


def bf(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).float()


def gelu_tanh(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def rms(x, eps=1e-6):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)


def layernorm(x, w, b, eps=1e-6):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) * torch.rsqrt(var + eps) * w + b


def rope(x, pos, theta=10000.0):
    """rotate-half RoPE over the last dim (256) for [T, heads, 256]."""
    i = np.arange(128, dtype=np.float64)
    inv = torch.tensor((theta ** (-2.0 * i / HD)).astype(np.float32))
    ang = torch.tensor(pos, dtype=torch.float32)[:, None] * inv[None, :]
    s, c = torch.sin(ang)[:, None, :], torch.cos(ang)[:, None, :]
    x1, x2 = x[..., :128], x[..., 128:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1)


def attention(q, k, v, scale):
    """q [Tq, h, d], k/v [Tk, d] (MQA) or [Tk, h, d]; bidirectional; bf16 out."""
    if k.dim() == 2:
        s = torch.einsum("qhd,kd->hqk", q, k) * scale
        o = torch.einsum("hqk,kd->qhd", torch.softmax(s, -1), v)
    else:
        s = torch.einsum("qhd,khd->hqk", q, k) * scale
        o = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v)
    return bf(o)


def noise(seed: int, n: int) -> np.ndarray:
    u = counter_uniform(seed, 0, n + (n & 1))
    u1, u2 = u[0::2], u[1::2]
    r = np.sqrt(-2.0 * np.log(1.0 - u1))
    th = 6.283185307179586 * u2
    out = np.empty(len(u1) * 2)
    out[0::2] = r * np.cos(th)
    out[1::2] = r * np.sin(th)
    return out[:n].astype(np.float32)


def tensor_table(c) -> list[dict]:
    """Restatement of the weight table (names, shapes, draw offsets, bounds) of
    csrc/pi05_model.cu Model::declare; tests check it equals the device's."""
    W, We, Dv = c.width, c.expert_width, c.vit_width
    qkv, qdim = (NQH + 2) * HD, NQH * HD
    apad = (c.action_dim + 7) // 8 * 8
    mb = lambda fan: float(np.float32(math.sqrt(3.0 / fan)))
    f32 = lambda v: float(np.float32(v))  # the C++ literals are float
    rows = [("embed", c.vocab, W, "bf16", mb(W), 0.0)]
    for l in range(c.depth):
        p = f"llm.{l}."
        rows += [(p + "ln1", 1, W, "f32", f32(0.1), 0.0), (p + "wqkv", qkv, W, "bf16", mb(W), 0.0),
                 (p + "wo", W, qdim, "bf16", mb(qdim), 0.0), (p + "ln2", 1, W, "f32", f32(0.1), 0.0),
                 (p + "wgu", 2 * c.mlp, W, "bf16", mb(W), 0.0),
                 (p + "wd", W, c.mlp, "bf16", mb(c.mlp), 0.0)]
    rows += [("final_norm", 1, W, "f32", f32(0.1), 0.0), ("lm_head", c.vocab, W, "bf16", mb(W), 0.0)]
    for l in range(c.depth):
        p = f"expert.{l}."
        rows += [(p + "wqkv", qkv, We, "bf16", mb(We), 0.0),
                 (p + "wo", We, qdim, "bf16", mb(qdim), 0.0),
                 (p + "wgu", 2 * c.expert_mlp, We, "bf16", mb(We), 0.0),
                 (p + "wd", We, c.expert_mlp, "bf16", mb(c.expert_mlp), 0.0)]
    n_mod = c.depth * 6 * We + 2 * We
    rows += [("action_in", We, apad, "bf16", mb(c.action_dim), 0.0),
             ("action_in.b", 1, We, "f32", f32(0.02), 0.0),
             ("action_out", c.action_dim, We, "bf16", mb(We), 0.0),
             ("action_out.b", 1, c.action_dim, "f32", f32(0.02), 0.0),
             ("time1", We, We, "bf16", mb(We), 0.0), ("time1.b", 1, We, "f32", f32(0.02), 0.0),
             ("time2", We, We, "bf16", mb(We), 0.0), ("time2.b", 1, We, "f32", f32(0.02), 0.0),
             ("mod", n_mod, We, "bf16", float(np.float32(0.1 * np.float32(mb(We)))), 0.0),
             ("mod.b", 1, n_mod, "f32", f32(0.02), 0.0)]
    if c.vit_depth:
        rows += [("vit.patch", Dv, 640, "bf16", mb(588), 0.0), ("vit.patch.b", 1, Dv, "f32", f32(0.02), 0.0),
                 ("vit.pos", 256, Dv, "f32", f32(0.02), 0.0)]
        for l in range(c.vit_depth):
            p = f"vit.{l}."
            rows += [(p + "ln1.w", 1, Dv, "f32", f32(0.1), 1.0), (p + "ln1.b", 1, Dv, "f32", f32(0.02), 0.0),
                     (p + "wqkv", 3 * Dv, Dv, "bf16", mb(Dv), 0.0),
                     (p + "bqkv", 1, 3 * Dv, "f32", f32(0.02), 0.0),
                     (p + "wo", Dv, Dv, "bf16", mb(Dv), 0.0), (p + "bo", 1, Dv, "f32", f32(0.02), 0.0),
                     (p + "ln2.w", 1, Dv, "f32", f32(0.1), 1.0), (p + "ln2.b", 1, Dv, "f32", f32(0.02), 0.0),
                     (p + "w1", c.vit_mlp, Dv, "bf16", mb(Dv), 0.0),
                     (p + "b1", 1, c.vit_mlp, "f32", f32(0.02), 0.0),
                     (p + "w2", Dv, c.vit_mlp, "bf16", mb(c.vit_mlp), 0.0),
                     (p + "b2", 1, Dv, "f32", f32(0.02), 0.0)]
        rows += [("vit.ln.w", 1, Dv, "f32", f32(0.1), 1.0), ("vit.ln.b", 1, Dv, "f32", f32(0.02), 0.0),
                 ("vit.proj", W, Dv, "bf16", mb(Dv), 0.0), ("vit.proj.b", 1, W, "f32", f32(0.02), 0.0)]
    out, off = [], 0
    for name, r, cc, dt, bound, center in rows:
        out.append(dict(name=name, shape=(r, cc), dtype=dt, offset=off, bound=bound, center=center))
        off += r * cc
    return out


def counter_tensor(seed: int, t: dict, chunk: int = 1 << 24) -> torch.Tensor:
    """One weight tensor drawn on the CPU exactly as the device init does."""
    n = t["shape"][0] * t["shape"][1]
    out = torch.empty(n, dtype=torch.float32)
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        u = counter_uniform(seed, t["offset"] + s, m)
        v = torch.from_numpy((t["center"] + (2.0 * u - 1.0) * t["bound"]).astype(np.float32))
        out[s:s + m] = v.to(torch.bfloat16).float() if t["dtype"] == "bf16" else v
    out = out.reshape(t["shape"])
    if "zero_from" in t:          # padded input columns are zero on the device
        out[:, t["zero_from"]:] = 0.0
    return out


class Pi05Ref:
    def __init__(self, cfg, weights: dict):
        self.c = cfg
        self.w = weights

    @classmethod
    def from_backend(cls, be):
        w = {t["name"]: be.read_tensor(t).float() for t in be.tensors()}
        return cls(be.config, w)

    @classmethod
    def from_counter(cls, cfg):
        """Weights generated on the CPU (no GPU involved) from the counter form."""
        w = {}
        for t in tensor_table(cfg):
            if t["name"] == "action_in":
                t = dict(t, zero_from=cfg.action_dim)
            if t["name"] == "vit.patch":
                t = dict(t, zero_from=588)
            w[t["name"]] = counter_tensor(cfg.seed, t)
        return cls(cfg, w)

    def W(self, name):
        return self.w[name]

    def check_init(self, be, names=("embed", "llm.0.wqkv", "mod.b")):
        """Device init == splitmix64 counter form (first 4096 elements)."""
        for t in be.tensors():
            if t["name"] not in names:
                continue
            n = min(4096, t["shape"][0] * t["shape"][1])
            u = counter_uniform(self.c.seed, t["offset"], n)
            want = (t["center"] + (2.0 * u - 1.0) * t["bound"]).astype(np.float32)
            got = self.w[t["name"]].reshape(-1)[:n].numpy()
            if t["dtype"] == "bf16":
                want = torch.tensor(want).to(torch.bfloat16).float().numpy()
            np.testing.assert_array_equal(got, want)

    # ------------------------------------------------------------ vision
    def vision(self, images: np.ndarray) -> torch.Tensor:
        c = self.c
        n = images.shape[0]
        x = torch.tensor(images, dtype=torch.float32) / 127.5 - 1.0
        p = x.reshape(n, 16, 14, 16, 14, 3).permute(0, 1, 3, 2, 4, 5).reshape(n * 256, 588)
        p = bf(p)
        h = self.W("vit.pos").repeat(n, 1) + (p @ self.W("vit.patch")[:, :588].T
                                               + self.W("vit.patch.b")[0])
        Dv, nh = c.vit_width, c.vit_heads
        hd = Dv // nh
        for l in range(c.vit_depth):
            pre = f"vit.{l}."
            y = bf(layernorm(h, self.W(pre + "ln1.w")[0], self.W(pre + "ln1.b")[0]))
            qkv = bf(y @ self.W(pre + "wqkv").T + self.W(pre + "bqkv")[0])
            o = torch.empty(n * 256, Dv)
            for im in range(n):
                rows = slice(im * 256, (im + 1) * 256)
                q = qkv[rows, :Dv].reshape(256, nh, hd)
                k = qkv[rows, Dv:2 * Dv].reshape(256, nh, hd)
                v = qkv[rows, 2 * Dv:].reshape(256, nh, hd)
                o[rows] = attention(q, k, v, 1.0 / math.sqrt(hd)).reshape(256, Dv)
            h = h + (o @ self.W(pre + "wo").T + self.W(pre + "bo")[0])
            y = bf(layernorm(h, self.W(pre + "ln2.w")[0], self.W(pre + "ln2.b")[0]))
            m = bf(gelu_tanh(y @ self.W(pre + "w1").T + self.W(pre + "b1")[0]))
            h = h + (m @ self.W(pre + "w2").T + self.W(pre + "b2")[0])
        y = bf(layernorm(h, self.W("vit.ln.w")[0], self.W("vit.ln.b")[0]))
        return y @ self.W("vit.proj").T + self.W("vit.proj.b")[0]

    # ------------------------------------------------------------ prefix
    def prefill(self, obs) -> list:
        """Per-layer (K, V) [P, 256] float32 (bf16 values) of the prefix."""
        c = self.c
        parts = []
        images = getattr(obs, "images", None)
        if images is not None and len(images):
            imgs = images.cpu().numpy() if isinstance(images, torch.Tensor) else np.asarray(images)
            parts.append(self.vision(imgs))
        if obs.obs_tokens:
            parts.append(self.W("embed")[list(obs.obs_tokens)] * math.sqrt(c.width))
        x = torch.cat(parts)
        P = x.shape[0]
        pos = np.arange(P)
        kvs = []
        for l in range(c.depth):
            pre = f"llm.{l}."
            y = bf(rms(x) * (1 + self.W(pre + "ln1")[0]))
            qkv = y @ self.W(pre + "wqkv").T
            q = bf(rope(qkv[:, :NQH * HD].reshape(P, NQH, HD), pos))
            k = bf(rope(qkv[:, NQH * HD:(NQH + 1) * HD].reshape(P, 1, HD), pos)[:, 0])
            v = bf(qkv[:, (NQH + 1) * HD:])
            kvs.append((k, v))
            if l == c.depth - 1:
                break
            o = attention(q, k, v, 1.0 / 16.0).reshape(P, NQH * HD)
            x = x + o @ self.W(pre + "wo").T
            y = bf(rms(x) * (1 + self.W(pre + "ln2")[0]))
            g = y @ self.W(pre + "wgu").T
            x = x + bf(gelu_tanh(g[:, 0::2]) * g[:, 1::2]) @ self.W(pre + "wd").T
        return kvs

    # ------------------------------------------------------------ action expert
    def modulation(self, S: int) -> torch.Tensor:
        We = self.c.expert_width
        half = We // 2
        temb = np.zeros((S, We), np.float32)
        for s in range(S):
            t = 1.0 - s / S
            for i in range(half):
                frac = i / (half - 1) if half > 1 else 0.0
                period = 4e-3 * (4.0 / 4e-3) ** frac
                ang = t / period * 2.0 * math.pi
                temb[s, i] = math.sin(ang)
                temb[s, half + i] = math.cos(ang)
        tb = bf(torch.tensor(temb))
        h1 = tb @ self.W("time1").T + self.W("time1.b")[0]
        h1 = bf(h1 * torch.sigmoid(h1))
        h2 = h1 @ self.W("time2").T + self.W("time2.b")[0]
        h2 = bf(h2 * torch.sigmoid(h2))
        return h2 @ self.W("mod").T + self.W("mod.b")[0]

    def denoise(self, kvs, S: int) -> np.ndarray:
        c = self.c
        We, H, A = c.expert_width, c.H, c.action_dim
        P = kvs[0][0].shape[0]
        mod = self.modulation(S)
        a = torch.tensor(noise(c.seed ^ 0x6E6F697365, H * A).reshape(H, A))
        pos = P + np.arange(H)
        dt = -1.0 / S
        for s in range(S):
            ms = mod[s]
            X = bf(a) @ self.W("action_in")[:, :A].T + self.W("action_in.b")[0]
            for l in range(c.depth):
                pre = f"expert.{l}."
                m = ms[l * 6 * We:(l + 1) * 6 * We].reshape(6, We)
                y = bf(rms(X) * (1 + m[0]) + m[1])
                qkv = y @ self.W(pre + "wqkv").T
                q = bf(rope(qkv[:, :NQH * HD].reshape(H, NQH, HD), pos))
                k = bf(rope(qkv[:, NQH * HD:(NQH + 1) * HD].reshape(H, 1, HD), pos)[:, 0])
                v = bf(qkv[:, (NQH + 1) * HD:])
                K = torch.cat([kvs[l][0], k])
                V = torch.cat([kvs[l][1], v])
                o = attention(q, K, V, 1.0 / 16.0).reshape(H, NQH * HD)
                X = X + m[2] * (o @ self.W(pre + "wo").T)
                y = bf(rms(X) * (1 + m[3]) + m[4])
                g = y @ self.W(pre + "wgu").T
                X = X + m[5] * (bf(gelu_tanh(g[:, 0::2]) * g[:, 1::2]) @ self.W(pre + "wd").T)
            mf = ms[c.depth * 6 * We:].reshape(2, We)
            y = bf(rms(X) * (1 + mf[0]) + mf[1])
            vel = y @ self.W("action_out").T + self.W("action_out.b")[0]
            a = a + dt * vel
        return a.double().numpy()

    # ------------------------------------------------------------ language decode
    def decode(self, kvs, tokens, k, max_len=None):
        """Greedy decode of one request from a prefix/decoded cache.
        Returns (new tokens, grown kvs, per-step logits)."""
        c = self.c
        kvs = [(K.clone(), V.clone()) for K, V in kvs]
        toks = list(tokens)
        logits_all = []
        max_len = max_len if max_len is not None else len(toks) + k
        for _ in range(k):
            pos = kvs[0][0].shape[0]
            inp = toks[-1] if toks else c.eos_token
            x = self.W("embed")[[inp]] * math.sqrt(c.width)
            for l in range(c.depth):
                pre = f"llm.{l}."
                y = bf(rms(x) * (1 + self.W(pre + "ln1")[0]))
                qkv = y @ self.W(pre + "wqkv").T
                q = bf(rope(qkv[:, :NQH * HD].reshape(1, NQH, HD), [pos]))
                kk = bf(rope(qkv[:, NQH * HD:(NQH + 1) * HD].reshape(1, 1, HD), [pos])[:, 0])
                vv = bf(qkv[:, (NQH + 1) * HD:])
                K = torch.cat([kvs[l][0], kk])
                V = torch.cat([kvs[l][1], vv])
                kvs[l] = (K, V)
                o = attention(q, K, V, 1.0 / 16.0).reshape(1, NQH * HD)
                x = x + o @ self.W(pre + "wo").T
                y = bf(rms(x) * (1 + self.W(pre + "ln2")[0]))
                g = y @ self.W(pre + "wgu").T
                x = x + bf(gelu_tanh(g[:, 0::2]) * g[:, 1::2]) @ self.W(pre + "wd").T
            y = bf(rms(x) * (1 + self.W("final_norm")[0]))
            logits = (y @ self.W("lm_head").T)[0]
            logits_all.append(logits.numpy())
            tok = int(torch.argmax(logits))
            toks.append(tok)
            if tok == c.eos_token or len(toks) == max_len:
                break
        return tuple(toks[len(tokens):]), kvs, logits_all

    def decode_rows(self, kvs_rows, last_tokens, k):
        """k greedy steps for m rows at once (batched projections, per-row
        attention) — the CPU baseline's continuous-batched decode step."""
        c = self.c
        m = len(kvs_rows)
        rows = [[(K.clone(), V.clone()) for K, V in kvs] for kvs in kvs_rows]
        toks = list(last_tokens)
        out = [[] for _ in range(m)]
        for _ in range(k):
            x = self.W("embed")[toks] * math.sqrt(c.width)
            for l in range(c.depth):
                pre = f"llm.{l}."
                y = bf(rms(x) * (1 + self.W(pre + "ln1")[0]))
                qkv = y @ self.W(pre + "wqkv").T
                o = torch.empty(m, NQH * HD)
                for r in range(m):
                    pos = rows[r][l][0].shape[0]
                    q = bf(rope(qkv[r:r + 1, :NQH * HD].reshape(1, NQH, HD), [pos]))
                    kk = bf(rope(qkv[r:r + 1, NQH * HD:(NQH + 1) * HD].reshape(1, 1, HD), [pos])[:, 0])
                    vv = bf(qkv[r:r + 1, (NQH + 1) * HD:])
                    K = torch.cat([rows[r][l][0], kk])
                    V = torch.cat([rows[r][l][1], vv])
                    rows[r][l] = (K, V)
                    o[r] = attention(q, K, V, 1.0 / 16.0).reshape(NQH * HD)
                x = x + o @ self.W(pre + "wo").T
                y = bf(rms(x) * (1 + self.W(pre + "ln2")[0]))
                g = y @ self.W(pre + "wgu").T
                x = x + bf(gelu_tanh(g[:, 0::2]) * g[:, 1::2]) @ self.W(pre + "wd").T
            y = bf(rms(x) * (1 + self.W("final_norm")[0]))
            toks = [int(t) for t in torch.argmax(y @ self.W("lm_head").T, dim=1)]
            for r in range(m):
                out[r].append(toks[r])
        return out
