"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no attention, no top-b, no trie
logic).  It only turns (seed, stream id, index) into numbers via SplitMix64, a
counter-based generator, so that the CPU oracle (`oracle/`) and the CUDA path
(`paper_2502_00085_b200/`) can be fed bit-identical inputs without sharing code.

Recipes:
  * weights: uniform(-1/sqrt(fan_in), +1/sqrt(fan_in)) ("uniform(-s, s) with
    s = 1/sqrt(fan_in)"); norm gains uniform(0.5, 1.5); embeddings uniform(-1, 1).
  * prompts: uniform token ids in [0, V).
  * Q/K/V for kernel-level tests and the bench: N(0, 1) (Box-Muller over two uniforms).
  * logits for beam-step tests: kappa * N(0,1).
  * beam selections (teacher forcing of the integer path): the "convergence dial"
    of SURVEY §8(d) cfg5 / SPEC S:569 -- each new rank r picks parent beam 0 with
    probability rho, else a uniform live beam; tokens uniform in [0, V).
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def u64(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    """n counter-based 64-bit words for (seed, stream), indices offset..offset+n-1."""
    base = _mix(np.array([(seed & 0xFFFFFFFFFFFFFFFF)], dtype=np.uint64) ^
                (np.array([stream & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64) * _GOLD))[0]
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(base + (idx + np.uint64(1)) * _GOLD)


def uniform01(seed: int, stream: int, n: int) -> np.ndarray:
    """float64 in [0, 1) from the top 53 bits."""
    return (u64(seed, stream, n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform(seed: int, stream: int, shape, lo: float, hi: float) -> np.ndarray:
    n = int(np.prod(shape)) if len(shape) else 1
    return (lo + (hi - lo) * uniform01(seed, stream, n)).reshape(shape)


def normal(seed: int, stream: int, shape) -> np.ndarray:
    """Standard normals via Box-Muller (two uniform streams)."""
    n = int(np.prod(shape)) if len(shape) else 1
    u1 = uniform01(seed, stream * 2 + 1, n)
    u2 = uniform01(seed, stream * 2 + 2, n)
    r = np.sqrt(-2.0 * np.log1p(-u1))  # 1-u1 in (0, 1]
    return (r * np.cos(2.0 * np.pi * u2)).reshape(shape)


def randint(seed: int, stream: int, n: int, hi: int) -> np.ndarray:
    """n integers uniform in [0, hi) (multiply-shift on the top 32 bits)."""
    hi32 = (u64(seed, stream, n) >> np.uint64(32))
    return ((hi32 * np.uint64(hi)) >> np.uint64(32)).astype(np.int64)


# ---------------------------------------------------------------------------------------
# Model configurations (shapes only; public model-card values)
# ---------------------------------------------------------------------------------------
MODEL_SHAPES = {
    # name: (L, d, Hq, Hkv, D, ffn, V, rope_base)
    "tiny": (2, 64, 4, 4, 16, 256, 256, 10000.0),          # BASELINE.json configs[0]
    "tiny_gqa": (2, 64, 4, 2, 16, 256, 256, 10000.0),
    "phi3.5-mini": (32, 3072, 32, 32, 96, 8192, 32064, 10000.0),
    "llama3.1-8b": (32, 4096, 32, 8, 128, 14336, 128256, 500000.0),
    "mistral-small-24b": (40, 5120, 32, 8, 128, 32768, 131072, 100000000.0),
}

# stream ids for weights (per layer: base + 16*layer + k)
_W_STREAMS = dict(emb=1, lm=2, gf=3)
_L_STREAMS = dict(wq=0, wk=1, wv=2, wo=3, wg=4, wu=5, wd=6, g1=7, g2=8)


def tiny_weights(seed: int, L: int, d: int, Hq: int, Hkv: int, D: int, ffn: int, V: int):
    """Random-init weights for the toy decoder (dict of float64 numpy arrays).

    Layout: projection matrices are [in][out] (x @ W).
    """
    def U(stream, shape, fan_in):
        s = 1.0 / np.sqrt(fan_in)
        return uniform(seed, stream, shape, -s, s)

    w = {
        "emb": uniform(seed, _W_STREAMS["emb"], (V, d), -1.0, 1.0),
        "lm": U(_W_STREAMS["lm"], (d, V), d),
        "gf": uniform(seed, _W_STREAMS["gf"], (d,), 0.5, 1.5),
        "layers": [],
    }
    for l in range(L):
        b = 100 + 16 * l
        w["layers"].append({
            "wq": U(b + _L_STREAMS["wq"], (d, Hq * D), d),
            "wk": U(b + _L_STREAMS["wk"], (d, Hkv * D), d),
            "wv": U(b + _L_STREAMS["wv"], (d, Hkv * D), d),
            "wo": U(b + _L_STREAMS["wo"], (Hq * D, d), Hq * D),
            "wg": U(b + _L_STREAMS["wg"], (d, ffn), d),
            "wu": U(b + _L_STREAMS["wu"], (d, ffn), d),
            "wd": U(b + _L_STREAMS["wd"], (ffn, d), ffn),
            "g1": uniform(seed, b + _L_STREAMS["g1"], (d,), 0.5, 1.5),
            "g2": uniform(seed, b + _L_STREAMS["g2"], (d,), 0.5, 1.5),
        })
    return w


def prompts(seed: int, R: int, t_max: int, V: int, lens=None):
    """[R][t_max] int32 token ids (uniform) and per-request lengths (default all t_max)."""
    toks = randint(seed, 7, R * t_max, V).reshape(R, t_max).astype(np.int32)
    if lens is None:
        lens = np.full(R, t_max, dtype=np.int32)
    return toks, np.asarray(lens, dtype=np.int32)


def selections(seed: int, steps: int, b: int, V: int, rho: float, first_live: int = 1):
    """Teacher-forced beam selections for the integer path (convergence dial).

    Returns a list of (parent_beam[int32, b_k], token[int32, b_k]) per step. Step 1 has
    first_live live beams (1 = the prompt leaf), so all parents are 0 there.  Tokens are
    (base_k + r) mod V with base_k uniform, so the b (parent, token) pairs of a step are
    distinct (as top-b candidates are); the sequence carries no arithmetic of the method.
    """
    out = []
    live = first_live
    for k in range(steps):
        u = uniform01(seed, 1000 + 3 * k, b)
        pick = randint(seed, 1001 + 3 * k, b, max(live, 1))
        par = np.where(u < rho, 0, pick).astype(np.int32)
        base = int(randint(seed, 1002 + 3 * k, 1, V)[0])
        tok = ((base + np.arange(b)) % V).astype(np.int32)  # distinct within a step
        out.append((par, tok))
        live = b
    return out


def ragged_lens(seed: int, R: int, t_max: int, t_min: int = 1) -> np.ndarray:
    return (t_min + randint(seed, 11, R, t_max - t_min + 1)).astype(np.int32)
