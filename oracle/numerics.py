"""Dense numeric primitives of the oracle (SPEC module `numkernel`).

Plain numpy, float64 by default, fixed left-to-right summation order so two calls
with identical inputs are bitwise identical ("deterministic summation
order").  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


def dot_rows(M: np.ndarray, x: np.ndarray) -> np.ndarray:
    """y[i] = sum_k M[i,k] x[k], summed left to right over k."""
    acc = np.zeros(M.shape[0], dtype=M.dtype)
    for k in range(M.shape[1]):
        acc = acc + M[:, k] * x[k]
    return acc


def matvec(x: np.ndarray, W: np.ndarray) -> np.ndarray:
    """y = x @ W for W laid out [in][out]; left-to-right over `in` (S:44 matmul)."""
    acc = np.zeros(W.shape[1], dtype=W.dtype)
    for k in range(W.shape[0]):
        acc = acc + x[k] * W[k]
    return acc


def softmax_masked(scores: np.ndarray, allow: np.ndarray) -> np.ndarray:
    """SPEC S:51-58 / PAPER §3.3: blocked positions get exactly zero weight.

    p_i = exp(s_i - max_allowed) / sum_allowed exp(s_j - max_allowed); blocked -> 0.
    An all-blocked row is an error ("signals a trie/mask construction bug").
    """
    allow = np.asarray(allow, dtype=bool)
    if not allow.any():
        raise ValueError("all-masked attention row")
    m = np.max(scores[allow])
    e = np.where(allow, np.exp(np.where(allow, scores - m, 0.0)), 0.0).astype(scores.dtype)
    total = scores.dtype.type(0)
    for v in e:  # left-to-right
        total = total + v
    return e / total


def log_softmax(x: np.ndarray) -> np.ndarray:
    """lp = x - lse, lse = m + log(sum exp(x - m)) (SURVEY §8(c) oracle model, last bullet)."""
    m = np.max(x)
    s = x.dtype.type(0)
    for v in np.exp(x - m):
        s = s + v
    return x - (m + np.log(s))


def rope_rotate_half(vec: np.ndarray, pos: int, base: float) -> np.ndarray:
    """Rotary embedding at position `pos`, rotate-half pairing (i, i + D/2).

    PAPER §3.4 requires the position of a trie node to be the one it has in
    conventional beam search; the embedding itself is a reading (R16: rotate-half,
    theta_i = base^(-2i/D), as in the HF Llama/Phi/Mistral family).  Angles in float64.
    """
    D = vec.shape[-1]
    if D % 2:
        raise ValueError("odd head dim")
    h = D // 2
    i = np.arange(h, dtype=np.float64)
    theta = base ** (-2.0 * i / D)
    ang = float(pos) * theta
    c = np.cos(ang).astype(vec.dtype)
    s = np.sin(ang).astype(vec.dtype)
    x1 = vec[..., :h]
    x2 = vec[..., h:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def rms_norm(v: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    """v_i g_i / sqrt(mean(v^2) + eps)."""
    ss = v.dtype.type(0)
    for x in v:
        ss = ss + x * x
    return v * g / np.sqrt(ss / v.shape[0] + v.dtype.type(eps))


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))
