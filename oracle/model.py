"""Toy pre-norm decoder used by both oracle decoders (SPEC module `model`).

It stands in for the LLM "P(x | T, M)" of Alg. 2 and "P(x_batch | X_batch)" of
Alg. 1.  One call = one query token:
    x = E[tok]; per layer:  h = rmsnorm(x) g1;  q,k,v = h Wq, h Wk, h Wv;
    RoPE(q, k, pos) (rotate-half, §3.4 positions);  write k,v BEFORE attending
    (Alg. 3 "Allow attention to current node");
    o = sum_n softmax_n(q.k_n / sqrt(D)) v_n over the caller's allowed rows (§3.3);
    x += o Wo;  h2 = rmsnorm(x) g2;  x += (silu(h2 Wg) * (h2 Wu)) Wd
  logits = kappa * (rmsnorm(x) gf) W_lm;  return log_softmax(logits).
GQA: query head h reads KV head h // (Hq/Hkv).  TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .numerics import dot_rows, log_softmax, matvec, rms_norm, rope_rotate_half, silu, softmax_masked


@dataclass(frozen=True)
class ModelConfig:
    L: int = 2
    d: int = 64
    Hq: int = 4
    Hkv: int = 4
    D: int = 16
    ffn: int = 256
    V: int = 256
    rope_base: float = 10000.0
    eps: float = 1e-5
    kappa: float = 4.0  # logit scale: the convergence knob of SURVEY §8(d)

    def __post_init__(self):
        if self.Hq % self.Hkv:
            raise ValueError("Hq % Hkv != 0 (S:104)")
        if self.d != self.Hq * self.D:
            raise ValueError("d != Hq * D")


class Model:
    def __init__(self, weights: dict, cfg: ModelConfig, dtype=np.float64):
        self.cfg = cfg
        self.dtype = dtype
        cast = lambda a: np.asarray(a, dtype=dtype)
        self.emb = cast(weights["emb"])
        self.lm = cast(weights["lm"])
        self.gf = cast(weights["gf"])
        self.layers = [{k: cast(v) for k, v in lw.items()} for lw in weights["layers"]]

    def qkv(self, layer: int, x: np.ndarray, pos: int):
        """Projections + RoPE at `pos` for one token; returns (h-normed input unused), q, k, v."""
        c, lw = self.cfg, self.layers[layer]
        h = rms_norm(x, lw["g1"], c.eps)
        q = matvec(h, lw["wq"]).reshape(c.Hq, c.D)
        k = matvec(h, lw["wk"]).reshape(c.Hkv, c.D)
        v = matvec(h, lw["wv"]).reshape(c.Hkv, c.D)
        q = rope_rotate_half(q, pos, c.rope_base)
        k = rope_rotate_half(k, pos, c.rope_base)
        return q, k, v

    def attend(self, q: np.ndarray, K: np.ndarray, V: np.ndarray) -> np.ndarray:
        """q [Hq][D], K/V [n][Hkv][D] (allowed rows in sequence order) -> o [Hq][D]."""
        c = self.cfg
        g = c.Hq // c.Hkv
        scale = self.dtype(1.0 / np.sqrt(c.D))
        o = np.zeros((c.Hq, c.D), dtype=self.dtype)
        for h in range(c.Hq):
            kh = h // g
            s = dot_rows(K[:, kh, :], q[h]) * scale
            p = softmax_masked(s, np.ones(len(s), dtype=bool))
            acc = np.zeros(c.D, dtype=self.dtype)
            for n in range(len(p)):  # left to right over rows
                acc = acc + p[n] * V[n, kh, :]
            o[h] = acc
        return o

    def forward(self, token: int, pos: int, ctx) -> np.ndarray:
        """One-token forward.  `ctx(layer, k, v)` stores (k, v) for this token (write
        before read) and returns the allowed (K, V) rows [n][Hkv][D] in sequence order,
        self included.  Returns log-probabilities over the vocabulary."""
        c = self.cfg
        x = self.emb[token].copy()
        for l, lw in enumerate(self.layers):
            q, k, v = self.qkv(l, x, pos)
            K, V = ctx(l, k, v)
            o = self.attend(q, K, V)
            x = x + matvec(o.reshape(-1), lw["wo"])
            h2 = rms_norm(x, lw["g2"], c.eps)
            x = x + matvec(silu(matvec(h2, lw["wg"])) * matvec(h2, lw["wu"]), lw["wd"])
        logits = self.dtype(c.kappa) * matvec(rms_norm(x, self.gf, c.eps), self.lm)
        return log_softmax(logits)

    def forward_full_causal(self, tokens, window: int = 0) -> np.ndarray:
        """No-cache reference: recompute every position from scratch with a causal (and,
        if window > 0, sliding-window) mask; returns lp rows [T][V]."""
        c = self.cfg
        T = len(tokens)
        out = []
        for i in range(T):
            xs = [self.emb[t].copy() for t in tokens[: i + 1]]
            for l, lw in enumerate(self.layers):
                qkv = [self.qkv(l, xs[j], j) for j in range(i + 1)]
                new = []
                for j in range(i + 1):
                    lo = 0 if window <= 0 else max(0, j - window + 1)
                    K = np.stack([qkv[m][1] for m in range(lo, j + 1)])
                    V = np.stack([qkv[m][2] for m in range(lo, j + 1)])
                    o = self.attend(qkv[j][0], K, V)
                    x = xs[j] + matvec(o.reshape(-1), lw["wo"])
                    h2 = rms_norm(x, lw["g2"], c.eps)
                    x = x + matvec(silu(matvec(h2, lw["wg"])) * matvec(h2, lw["wu"]), lw["wd"])
                    new.append(x)
                xs = new
            logits = self.dtype(c.kappa) * matvec(rms_norm(xs[i], self.gf, c.eps), self.lm)
            out.append(log_softmax(logits))
        return np.stack(out)
